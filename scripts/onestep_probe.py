"""Per-rank SRA kernel time vs message size for the one-step / two-step K1
split (run with GCX_ONESTEP_MIN_SLOTS unset and =huge).  Development tool (GPU)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402

rng = np.random.default_rng(5)
for nbytes in [1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26]:
    d = nbytes // 4
    for nodes in (2, 8):
        req = G.ReduceRequest()
        req.inputs = [rng.standard_normal(d).astype(np.float32) for _ in range(nodes)]
        req.segments = [G.Segment(0, d, G.CodecMode.quantize, 4, 128)]
        req.op = G.ReduceOp.average
        req.step_seed = 7
        G.allreduce(req, nodes)
        t = min(G.allreduce(req, nodes).trace.device_time_s for _ in range(5)) / nodes
        print(os.environ.get("GCX_ONESTEP_MIN_SLOTS", "default"), nbytes, nodes,
              f"{t * 1e6:.1f} us", flush=True)
