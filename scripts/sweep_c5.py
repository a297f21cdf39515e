"""BASELINE config 5 on one GPU: compressed SRA allreduce of a single
quantized segment (bucket 128), message sizes 64 KiB ... 256 MiB, 1/2/4/8
bits, N = 2/4/8, every rank's kernels run on this B200 (the exchange is
device-local, so this is the compute side of the multi-GPU number).
Reports per-rank kernel time and the compressed bytes each rank would send;
writes gpurun_out/c5_sweep.json.  Development / evidence tool (GPU box)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402


def main():
    sizes = [1 << k for k in range(16, 29, 2)]  # bytes: 64 KiB .. 256 MiB
    rows = []
    rng = np.random.default_rng(5)
    for nbytes in sizes:
        d = nbytes // 4
        for nodes in (2, 4, 8):
            inputs = [rng.standard_normal(d).astype(np.float32) for _ in range(nodes)]
            for bits in (1, 2, 4, 8):
                req = G.ReduceRequest()
                req.inputs = inputs
                req.segments = [G.Segment(0, d, G.CodecMode.quantize, bits, 128)]
                req.op = G.ReduceOp.average
                req.step_seed = 7
                G.allreduce(req, nodes)  # warm
                res = [G.allreduce(req, nodes) for _ in range(3)]
                t = min(r.trace.device_time_s for r in res) / nodes
                sent = res[0].trace.device_bytes_sent / nodes
                rows.append({"bytes": nbytes, "nodes": nodes, "bits": bits,
                             "per_rank_kernel_us": t * 1e6,
                             "compressed_bytes_sent_per_rank": sent,
                             "kernel_busbw_GBps": (nbytes / t) * 2 * (nodes - 1) / nodes / 1e9})
                print(rows[-1], flush=True)
            del inputs
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "c5_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
