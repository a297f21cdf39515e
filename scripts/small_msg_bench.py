"""Small-message SRA (BASELINE config 5's low end) on one GPU: per-rank kernel
time of one compressed allreduce, every rank's kernels on this B200, for
64 KiB .. 4 MiB at N = 2/4/8, 4 bits (scripts/sweep_c5.py's measurement on a
short size list).  GCX_EMUL_GRAPH=1: the step's kernels are launched as one
CUDA graph (device work only).  Development / evidence tool (GPU box)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402

rng = np.random.default_rng(5)
for nbytes in (1 << 16, 1 << 18, 1 << 20, 1 << 22):
    d = nbytes // 4
    for nodes in (2, 4, 8):
        req = G.ReduceRequest()
        req.inputs = [rng.standard_normal(d).astype(np.float32) for _ in range(nodes)]
        req.segments = [G.Segment(0, d, G.CodecMode.quantize, 4, 128)]
        req.op = G.ReduceOp.average
        req.step_seed = 7
        G.allreduce(req, nodes)
        t = min(G.allreduce(req, nodes).trace.device_time_s for _ in range(5)) / nodes
        print(f"{nbytes / 1024:8.0f} KiB N={nodes} per-rank {t * 1e6:6.1f} us", flush=True)
