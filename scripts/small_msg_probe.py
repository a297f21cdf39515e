"""Where the small-message SRA floor goes: one emulated SRA step at 64 KiB,
N = 2, 4-bit/128, timed by events (device_time_s) and by the host clock.
Run plain for times, under `ncu --metrics gpu__time_duration.sum` for the
per-kernel list.  Development tool (GPU box)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_08617_b200 import _gcomm as G  # noqa: E402


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    nodes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rng = np.random.default_rng(5)
    req = G.ReduceRequest()
    req.inputs = [rng.standard_normal(d).astype(np.float32) for _ in range(nodes)]
    req.segments = [G.Segment(0, d, G.CodecMode.quantize, 4, 128)]
    req.op = G.ReduceOp.average
    req.step_seed = 7
    G.allreduce(req, nodes)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = G.allreduce(req, nodes)
        ts.append((r.trace.device_time_s * 1e6, (time.perf_counter() - t0) * 1e6))
    ts.sort()
    print("device_us", [round(a, 1) for a, _ in ts[:5]], "host_call_us", round(ts[0][1], 1))


if __name__ == "__main__":
    main()
