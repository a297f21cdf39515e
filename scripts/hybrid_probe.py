"""C1's K1 alone and the bench's two-stream K1+K3 step, eager and as a CUDA
graph, per GCX_SPAN_INLINE_MASK value (each in its own process).  The mask
selected a prefix / inline key split of the span K1 that measured slower at
every setting and was reverted; with the current build the
mask has no effect.  Development tool (GPU box):
  python scripts/hybrid_probe.py 0x0 ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    import torch
    sys.path.insert(0, ROOT)
    from paper_2111_08617_b200 import device as dev

    n, bits, bucket = 25557032, 4, 128
    sets = []
    c1 = os.environ.get("PROBE_C1") == "1"
    if c1:
        from oracle import Oracle
        orc = Oracle()
    for k in range(4):
        x = (torch.from_numpy(orc.normal_vector(n, 0x5EED + k, 1e-3)).cuda() if c1
             else torch.randn(n, device="cuda") * 1e-3)
        norms, packed = dev.alloc_compressed(n, bits, bucket)
        sets.append((x, norms, packed, torch.empty_like(x),
                     torch.full((1,), -1, dtype=torch.int64, device="cuda")))
    prefix = dev.make_prefix(n, bucket)
    s_q, s_d = torch.cuda.Stream(), torch.cuda.Stream()

    def q(k, st):
        x, norms, packed, out, bad = sets[k % 4]
        dev.quantize_prefixed(x, bits, bucket, 42 + k, prefix, norms, packed, bad, stream=st,
                              reset_bad=False)

    def alone(reps=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(4):
            q(k, s_q)
        torch.cuda.synchronize()
        e0.record(s_q)
        for k in range(reps):
            q(k, s_q)
        e1.record(s_q)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    qd = [torch.cuda.Event() for _ in range(4)]
    dd = [torch.cuda.Event() for _ in range(4)]
    used = [False] * 4

    efill = os.environ.get("PROBE_FILL") == "1"

    def pstep(k):
        slot = k % 4
        x, norms, packed, out, bad = sets[slot]
        if used[slot]:
            s_q.wait_event(dd[slot])
        if efill:
            with torch.cuda.stream(s_q):
                bad.fill_(-1)
        q(k, s_q)
        qd[slot].record(s_q)
        s_d.wait_event(qd[slot])
        dev.dequantize(norms, packed, n, bits, bucket, out, stream=s_d)
        dd[slot].record(s_d)
        used[slot] = True

    def step(reps=40):
        for k in range(8):
            pstep(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_q)
        for k in range(reps):
            pstep(k)
        s_q.wait_stream(s_d)
        e1.record(s_q)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def gstep(reps=20, fill=False):
        qd[:] = [torch.cuda.Event() for _ in range(4)]
        dd[:] = [torch.cuda.Event() for _ in range(4)]
        used[:] = [False] * 4
        for k in range(8):
            pstep(k)
        torch.cuda.synchronize()
        used[:] = [False] * 4
        qd[:] = [torch.cuda.Event() for _ in range(4)]
        dd[:] = [torch.cuda.Event() for _ in range(4)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cap = torch.cuda.current_stream()
            s_q.wait_stream(cap)
            s_d.wait_stream(cap)
            for k in range(reps):
                if fill:  # the bench's per-step non-finite sentinel reset
                    with torch.cuda.stream(s_q):
                        sets[k % 4][4].fill_(-1)
                pstep(k)
            cap.wait_stream(s_q)
            cap.wait_stream(s_d)
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps)
        return best

    a = min(alone() for _ in range(3))
    s = min(step() for _ in range(3))
    gs = gstep()
    gf = gstep(fill=True)
    qd[:] = [torch.cuda.Event() for _ in range(4)]
    dd[:] = [torch.cuda.Event() for _ in range(4)]
    used[:] = [False] * 4
    s2 = min(step() for _ in range(3))
    print(json.dumps({"mask": os.environ.get("GCX_SPAN_INLINE_MASK", "default"), "c1": c1,
                      "fill": efill,
                      "k1_alone_us": a * 1e3, "step_us": s * 1e3, "graph_step_us": gs * 1e3,
                      "graph_step_fill_us": gf * 1e3, "step_again_us": s2 * 1e3, "GBps": 4 * n / (s * 1e-3) / 1e9}),
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        for m in sys.argv[1:] or ["0x0"]:
            env = dict(os.environ, GCX_SPAN_INLINE_MASK=m)
            subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
