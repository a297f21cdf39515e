"""One N-rank SRA step of ResNet-50 fused buffer 0 on one GPU (for ncu launch lists)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402
from paper_2111_08617_b200.ddp import load_layout, resolve_codecs  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
layers = load_layout("resnet50")
codecs = resolve_codecs(layers)
fb = G.pack_fused_buffers([n for _, n, _ in layers], 64 << 20)[0]
segs = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                  codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
        for s in fb.segments]
rng = np.random.default_rng(0)
req = G.ReduceRequest()
req.inputs = [(rng.standard_normal(fb.total_elements) * 1e-3).astype(np.float32) for _ in range(N)]
req.segments = segs
req.op = G.ReduceOp.average
req.step_seed = 7
for _ in range(2):
    r = G.allreduce(req, N)
print("segments", len(segs), "elements", fb.total_elements, "device ms", r.trace.device_time_s * 1e3)
