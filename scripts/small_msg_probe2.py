"""One 64 KiB, N = 8, 4-bit SRA allreduce with every rank on this GPU (for
ncu launch lists of the small-message path).  Development tool."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402

nbytes = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
nodes = int(sys.argv[2]) if len(sys.argv) > 2 else 8
d = nbytes // 4
rng = np.random.default_rng(5)
req = G.ReduceRequest()
req.inputs = [rng.standard_normal(d).astype(np.float32) for _ in range(nodes)]
req.segments = [G.Segment(0, d, G.CodecMode.quantize, 4, 128)]
req.op = G.ReduceOp.average
req.step_seed = 7
for _ in range(3):
    r = G.allreduce(req, nodes)
print("device us per rank", r.trace.device_time_s * 1e6 / nodes)
