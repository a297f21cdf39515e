"""Single-GPU emulation of the N-rank SRA step on the ResNet-50 layout:
collectives.allreduce runs every rank's K1 / K2 / K3 on one B200 (the
exchange is device-local).  device_time_s / N approximates one rank's kernel
time per step (NVLink transfer not included).  Development tool."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402
from paper_2111_08617_b200.ddp import load_layout, resolve_codecs  # noqa: E402


def main():
    layers = load_layout("resnet50")
    codecs = resolve_codecs(layers)
    bufs = G.pack_fused_buffers([n for _, n, _ in layers], 64 << 20)
    rng = np.random.default_rng(0)
    res = {}
    for N in (2, 4, 8):
        total = 0.0
        for b, fb in enumerate(bufs):
            segs = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                              codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
                    for s in fb.segments]
            req = G.ReduceRequest()
            req.inputs = [(rng.standard_normal(fb.total_elements) * 1e-3).astype(np.float32)
                          for _ in range(N)]
            req.segments = segs
            req.op = G.ReduceOp.average
            req.step_seed = 7
            G.allreduce(req, N)  # warm
            ts = [G.allreduce(req, N).trace.device_time_s for _ in range(3)]
            total += min(ts)
        res[N] = {"all_ranks_kernel_ms": total * 1e3, "per_rank_kernel_ms": total * 1e3 / N}
        print(N, res[N], flush=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "sra_emul.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
