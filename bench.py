"""bench.py — headline benchmark of the B200 compressed-allreduce hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (BASELINE.json configs[0], the single-GPU configuration): one step =
C1, the 4-bit / bucket-128 quantize + dequantize of a 25,557,032-float
ResNet-50-sized gradient (K1 + K3).  value = uncompressed-equivalent GB/s
through the compression path, 4n / t_step.

N > 1 (configs[1], under torchrun, one rank per GPU over NCCL): one step =
the compressed SRA allreduce (average) of the ResNet-50 per-layer gradient
list through the engine's fused buffers (small layers uncompressed).
value = effective bus GB/s, (4n / t) * 2(N-1)/N (nccl-tests convention),
n = gradient elements, t = max over ranks.

Prints ONE JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("effective allreduce GB/s (uncompressed-equiv) at 1/2/4/8 B200; "
          "quantize GB/s vs HBM")
C1_N = 25_557_032
C1_BITS, C1_BUCKET, C1_SEED = 4, 128, 42
# spin-kernel length (~50 ms at 1.965 GHz) that holds a stream while Python
# enqueues a batch of event-bracketed launches
HOLD_CYCLES = 100_000_000


def compressed_bytes(n, bits, bucket):
    return (n * (bits + 1) + 7) // 8 + 4 * ((n + bucket - 1) // bucket)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle: test infrastructure, CPU only)
# ---------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_codec_sample(reps=3, threads=None):
    """The reference's own CPU codec (oracle/_ref, compiled from the reference
    sources) — or the C restatement if _ref is absent — timed on this host on
    the C1 workload: quantize + dequantize of 25,557,032 floats.  The
    reference codec is single-threaded per call, so the host's cores are used
    the way a multi-core caller would: T threads each run codec::quantize +
    codec::dequantize on one bucket-aligned 1/T slice (ctypes releases the
    GIL).  Same work as one call; the draws are keyed per slice."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import Oracle, RefOracle
    o = Oracle()
    impl, kind = (RefOracle(), "reference") if RefOracle.available() else (o, "port")
    threads = threads or host_threads()
    x = o.normal_vector(C1_N, 0x5EED, 1e-3)
    nb = (C1_N + C1_BUCKET - 1) // C1_BUCKET
    cuts = [min(C1_N, (nb * t // threads) * C1_BUCKET) for t in range(threads + 1)]
    slices = [x[cuts[t]:cuts[t + 1]] for t in range(threads)]

    def work(t):
        xs = slices[t]
        norms, packed = impl.quantize(xs, C1_BITS, C1_BUCKET, C1_SEED)
        impl.dequantize(norms, packed, xs.size, C1_BITS, C1_BUCKET)

    times = []
    with ThreadPoolExecutor(threads) as pool:
        for _ in range(reps):
            t0 = time.perf_counter()
            list(pool.map(work, range(threads)))
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": 4 * C1_N / t / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"C1 quantize+dequantize, n={C1_N}, 4b/128, {threads} threads x "
                      f"bucket-aligned 1/{threads} slices, median of {reps}",
            "cpu_model": cpu_model(), "seconds_per_step": t}


def cpu_sra_sample(nodes, n=1 << 22, reps=3):
    """The reference's own SRA allreduce (oracle/_ref: collectives::allreduce
    over SimNet, one std::thread per node) — or the C restatement if _ref is
    absent — timed on this host: one 4-bit/128 quantized segment of n floats
    per node, average, step seed 7.  -> the same effective-busbw metric."""
    from oracle import Oracle, RefOracle
    o = Oracle()
    xs = [o.normal_vector(n, o.hash_combine(0xC5, r), 1.0) for r in range(nodes)]
    segs = [(0, n, 0, C1_BITS, C1_BUCKET)]
    if RefOracle.available():
        ref, kind = RefOracle(), "reference"
        run = lambda: ref.allreduce(xs, segs, 7, True)  # noqa: E731
    else:
        kind = "port"
        run = lambda: o.sra_allreduce(xs, segs, 7, True)  # noqa: E731
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": (4 * n / t) * 2 * (nodes - 1) / nodes / 1e9, "unit": "GB/s", "cores": nodes,
            "kind": kind,
            "sample": f"SRA allreduce (SimNet, {nodes} node threads), one 4b/128 segment of "
                      f"{n} floats per node, average, median of {reps}",
            "cpu_model": cpu_model(), "seconds_per_step": t}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = max(1, args.steps)
    cb = cpu_codec_sample(reps=steps)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GB/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
            "ms_per_step": cb["seconds_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64 (codec), u8 packed",
            "data": "synthetic (keyed normal01, C1)",
            "config": {"workload": "C1: 4-bit bucket-128 quantize+dequantize of 25,557,032 "
                                   "floats (ResNet-50 size), single rank, seed 42",
                       "note": "reference CPU codec; at N>1 rank 0 runs the same bounded "
                               "codec sample (the reference allreduce is simulated-time only)"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                "cpu_model")},
            "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm, N = 1: C1 codec round trip
# ---------------------------------------------------------------------------
def run_codec(args):
    import torch

    from paper_2111_08617_b200 import device as dev

    torch.cuda.set_device(0)
    n, bits, bucket = C1_N, C1_BITS, C1_BUCKET
    from oracle import Oracle  # the input generator only (util.hpp:32-38); not timed
    orc = Oracle()
    nsets = 4  # rotating input sets: working set 4 x 221 MB > 126 MB L2
    sets = []
    for k in range(nsets):
        # set 0 is C1 exactly: 1e-3 * normal01(0x5eed, i); the others use
        # neighbouring keys of the same generator
        x = torch.from_numpy(orc.normal_vector(n, 0x5EED + k, 1e-3)).cuda()
        norms, packed = dev.alloc_compressed(n, bits, bucket)
        out = torch.empty_like(x)
        # the non-finite sentinel: K1 records the first non-finite index with
        # atomicMin and nothing clears it, so it is sticky across steps and
        # checked (dev.check_finite) after each timed section -- no per-step
        # reset kernel between two K1 launches
        bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        sets.append((x, norms, packed, out, bad))
    stream = torch.cuda.current_stream()
    # the seed-independent key prefixes T(i) of this buffer shape, built once
    # (gcx_make_prefix; a gradient buffer keeps its shape across steps)
    prefix = dev.make_prefix(n, bucket)

    def quantize(k, x, norms, packed, bad, use_prefix, st=None):
        if use_prefix:
            dev.quantize_prefixed(x, bits, bucket, C1_SEED + k, prefix, norms, packed, bad,
                                  stream=st, reset_bad=False)
        else:
            dev.quantize(x, bits, bucket, C1_SEED + k, norms, packed, bad, stream=st,
                         reset_bad=False)

    def step(k, ev=None, use_prefix=True):
        x, norms, packed, out, bad = sets[k % nsets]
        if ev:
            ev[0].record(stream)
        quantize(k, x, norms, packed, bad, use_prefix)
        if ev:
            ev[1].record(stream)
        dev.dequantize(norms, packed, n, bits, bucket, out)
        if ev:
            ev[2].record(stream)

    # the timed steps: K1 and K3 on two streams, so step k's dequantize (HBM
    # writes) overlaps step k+1's quantize (integer hashing) -- the pipelining a
    # caller gets across fused buffers.  Every step still runs both kernels
    # on its own input set; a set is reused only after its K3 finished.
    s_q, s_d = torch.cuda.Stream(), torch.cuda.Stream()
    q_done = [torch.cuda.Event() for _ in range(nsets)]
    d_done = [torch.cuda.Event() for _ in range(nsets)]
    used = [False] * nsets

    def pstep(k, seed=None):
        slot = k % nsets
        x, norms, packed, out, bad = sets[slot]
        if used[slot]:
            s_q.wait_event(d_done[slot])
        quantize(k if seed is None else seed - C1_SEED, x, norms, packed, bad, True, st=s_q)
        q_done[slot].record(s_q)
        s_d.wait_event(q_done[slot])
        dev.dequantize(norms, packed, n, bits, bucket, out, stream=s_d)
        d_done[slot].record(s_d)
        used[slot] = True

    for k in range(args.warmup):
        step(k)
        pstep(k)
    torch.cuda.synchronize()
    # Timed region: the K steps are enqueued from Python while a spin kernel
    # holds s_q, so the events bracket device work (both streams run
    # concurrently) rather than Python's ~10-20 us of launch cost per call,
    # which a training step hides behind backward compute.  Timed step j
    # uses slot j % 4; the LAST step on slot 0 runs C1 exactly (input set 0,
    # seed 42), so its outputs can be checked afterwards.
    last0 = nsets * ((args.steps - 1) // nsets)
    seeds = [(C1_SEED + 1000 * (j // nsets - last0 // nsets)) % (1 << 64)
             for j in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        time.sleep(0.25)
        torch.cuda.synchronize()
        with torch.cuda.stream(s_q):
            torch.cuda._sleep(HOLD_CYCLES)
        t0.record(s_q)
        for j in range(args.steps):
            pstep(j, seed=seeds[j])
        s_q.wait_stream(s_d)
        t1.record(s_q)
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    ms = total_ms / args.steps
    # a timed step's results against SURVEY Appendix A (the compiled
    # reference's C1 digests): packed codes, norms, dequantized output
    x0, norms0, packed0, out0, bad0 = sets[0]
    for st in sets:
        dev.check_finite(st[4])
    c1_digests = {
        "packed": orc.fnv1a64(packed0.cpu().numpy()[:(n * (bits + 1) + 7) // 8]),
        "norms": orc.fnv1a64(norms0.cpu().numpy()),
        "dequantized": orc.fnv1a64(out0.cpu().numpy())}
    want = {"packed": 0x48061E58E8EFC214, "norms": 0xA0F211F9B3554F9A,
            "dequantized": 0x475F012FF75F72F5}
    if c1_digests != want:
        raise SystemExit(f"timed C1 step differs from the reference digests: "
                         f"{ {k: hex(v) for k, v in c1_digests.items()} }")
    # the same K steps launched from Python with no hold (host launch cost
    # included), and captured once as a CUDA graph and replayed
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_q)
    for j in range(args.steps):
        pstep(j, seed=seeds[j])
    s_q.wait_stream(s_d)
    e1.record(s_q)
    torch.cuda.synchronize()
    ms_eager = e0.elapsed_time(e1) / args.steps
    q_done[:] = [torch.cuda.Event() for _ in range(nsets)]
    d_done[:] = [torch.cuda.Event() for _ in range(nsets)]
    used[:] = [False] * nsets
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        cap = torch.cuda.current_stream()
        s_q.wait_stream(cap)
        s_d.wait_stream(cap)
        for j in range(args.steps):
            pstep(j, seed=seeds[j])
        cap.wait_stream(s_q)
        cap.wait_stream(s_d)
    graph.replay()
    torch.cuda.synchronize()
    e0.record(stream)
    graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_graph = e0.elapsed_time(e1) / args.steps
    x0, norms0, packed0, out0, bad0 = sets[0]
    if orc.fnv1a64(packed0.cpu().numpy()[:(n * (bits + 1) + 7) // 8]) != want["packed"]:
        raise SystemExit("graph replay of the timed steps differs from the reference digests")
    q_done[:] = [torch.cuda.Event() for _ in range(nsets)]
    d_done[:] = [torch.cuda.Event() for _ in range(nsets)]
    used[:] = [False] * nsets
    # per-kernel times (the roofline) from the same steps run back to back.
    # The stream is held by a spin kernel while Python enqueues them, so the
    # events bracket device work, not host launch gaps.
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(HOLD_CYCLES)
    s0.record(stream)
    for k in range(args.steps):
        step(args.warmup + k, evs[k])
    s1.record(stream)
    torch.cuda.synchronize()
    ms_serial = s0.elapsed_time(s1) / args.steps
    q_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    dq_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    for s in sets:
        dev.check_finite(s[4])
    # the same K1 hashing all three finalizers per element (no prefix table)
    evi = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    torch.cuda._sleep(HOLD_CYCLES)
    for k in range(args.steps):
        step(k, evi[k], use_prefix=False)
    torch.cuda.synchronize()
    q_inline_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evi)

    # hash-only integer ceiling: variant 0 = reference 64-bit
    # form, 1 = split 32-bit form used by K1, 2 = split form 2-way ILP,
    # 5/6 = opaque-shift form (1 and 2 draws per iteration)
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    hash_ms = {}
    for variant in (0, 1, 2, 5, 6):
        dev.hash_bench(n, 42, bucket, sink, variant)
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(5):
            dev.hash_bench(n, 42, bucket, sink, variant)
        h1.record(stream)
        torch.cuda.synchronize()
        hash_ms[variant] = h0.elapsed_time(h1) / 5

    # K4 (adaptive statistics, adaptive.cpp:21-35): the per-step FP64 window
    # accumulate sum[i] += (double)g[i] over the same 25.6 M gradient
    from paper_2111_08617_b200 import _capi
    wsum = torch.zeros(n, dtype=torch.float64, device="cuda")
    nonfin = torch.zeros(1, dtype=torch.int32, device="cuda")
    for k in range(3):
        _capi.check(_capi.lib().gcx_stats_accumulate(wsum.data_ptr(), sets[k % nsets][0].data_ptr(),
                                                     n, nonfin.data_ptr(), stream.cuda_stream))
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for k in range(args.steps):
        _capi.check(_capi.lib().gcx_stats_accumulate(wsum.data_ptr(), sets[k % nsets][0].data_ptr(),
                                                     n, nonfin.data_ptr(), stream.cuda_stream))
    a1.record(stream)
    torch.cuda.synchronize()
    acc_ms = a0.elapsed_time(a1) / args.steps
    del wsum

    # the N = 8 SRA step of the ResNet-50 layer list with every rank's kernels
    # on this GPU (exchange in device memory): per-rank kernel time, the
    # compute side of the multi-GPU number (scripts/sra_emul_bench.py)
    sra8 = sra_emulation(8)
    sra8_graph = sra_emulation(8, graph=True)

    # end to end through the C-ABI with host buffers: every step copies its
    # input from pinned host memory (H2D), runs gcx_quantize + gcx_dequantize
    # and reads the result back (D2H).  Steps are double-buffered over three
    # streams (copy-in, compute, copy-out) so step k's D2H overlaps step k+1's
    # H2D on the two copy engines, as a streaming caller would run it.
    e2e_ms = e2e_codec(args, sets, n, bits, bucket)
    pcie = pcie_copy_rates(sets, n)
    peak, peak_kind = measured_peaks()
    q_bytes = 4 * n + compressed_bytes(n, bits, bucket)
    achieved = q_bytes / (q_ms * 1e-3) / 1e9
    step_bytes = 8 * n + 8 * int(prefix.numel()) + 2 * compressed_bytes(n, bits, bucket)
    cb = cpu_codec_sample(reps=3)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "round2_c1_k_span.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": 4 * n / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 in, f64 codec math, u8 packed", "data": "synthetic (C1 generator 1e-3*normal01(0x5eed+k, i), keyed)",
        "config": {"workload": "C1: 4-bit bucket-128 quantize+dequantize of 25,557,032 floats "
                               "(ResNet-50 size), single rank",
                   "convention": "value = 4n / t_step (uncompressed-equivalent bytes)",
                   "pipelining": "K1 and K3 on two streams: step k's dequantize overlaps "
                                 "step k+1's quantize",
                   "launch": "the K timed steps enqueued while a spin kernel holds the "
                             "stream (events bracket device work); ms_per_step_eager = no "
                             "hold (Python launch cost included); ms_per_step_graph = the K "
                             "steps as one CUDA graph replay (its branches ran less "
                             "concurrently than the two streams)",
                   "ms_per_step_eager": ms_eager,
                   "ms_per_step_graph": ms_graph,
                   "ms_per_step_serial": ms_serial,
                   "l2": "4 rotating input sets, working set > 126 MB L2",
                   "parity": "the last timed step on input set 0 (C1, seed 42) matches the "
                             "reference digests of SURVEY Appendix A (packed, norms, "
                             "dequantized)",
                   "quantize_ms": q_ms, "dequantize_ms": dq_ms,
                   "keys": "seed-independent key prefixes T(i) = mix64(i/B ^ mix64(i)) built "
                           "once per buffer shape (gcx_make_prefix, outside the timed region); "
                           "each step hashes mix64(seed ^ T(i)) with a fresh seed",
                   "quantize_inline_ms": q_inline_ms,
                   "sra_n8_emulated_per_rank_kernel_ms": sra8,
                   "sra_n8_emulated_per_rank_graph_ms": sra8_graph,
                   "k4_window_accumulate_ms": acc_ms,
                   "k4_window_accumulate_GBps": 20 * n / (acc_ms * 1e-3) / 1e9,
                   "k4_note": "adaptive statistics: sum[i] += (double)g[i] (read 4+8 B, write 8 B "
                              "per element), once per step inside observation windows",
                   "quantize_GBps_algorithmic": achieved,
                   # what one step must move through HBM with the prefix
                   # design: K1 reads x (4n) and the key prefixes (8 B per
                   # slot), writes the message; K3 reads it, writes 4n
                   "step_hbm_bytes": step_bytes,
                   "step_hbm_GBps": step_bytes / (ms * 1e-3) / 1e9,
                   "step_hbm_frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                   "dequantize_GBps_algorithmic": q_bytes / (dq_ms * 1e-3) / 1e9,
                   "dequantize_roofline_frac": q_bytes / (dq_ms * 1e-3) / 1e9 / peak,
                   "dequantize_kernel": "k_dspan<4,7> (K3: per-lane shuffle tables, "
                                        "coalesced 16-byte streaming stores; "
                                        "profiles/round2_c1_k_dspan.md)",
                   "hash_only_ms": {f"variant{k}": v for k, v in hash_ms.items()},
                   "hash_only_Gdraws_per_s": n / (min(hash_ms.values()) * 1e-3) / 1e9},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_span<4,7,prefix> (K1: lane-per-128-element rows staged by "
                               "2-D TMA into swizzled shared slots, fused sequential FP64 norms, "
                               "one SplitMix64 finalizer per element from the key prefixes, "
                               "register bit-packing, bulk-stored words; one launch per "
                               "gcx_quantize_prefixed)", "peak_kind": peak_kind,
                     "note": "frac counts K1's algorithmic bytes (x in, message out: 4.66 B/elem). "
                             "K1 also reads the 8-byte key prefix T(i) per element (the "
                             "seed-independent half of the reference RNG, built once per "
                             "buffer shape), so its DRAM traffic is ~12.5 B/elem (traffic, "
                             "from ncu): 320 MB per launch, 4.4-5.2 TB/s at 62-73 us -- "
                             "67-79 % of HBM on the bytes it must move.  The C1 step as a "
                             "whole moves config.step_hbm_bytes at config.step_hbm_frac of "
                             "HBM.  Hashing the prefixes inline instead costs two more "
                             "SplitMix64 finalizers per element (config.quantize_inline_ms, "
                             "config.hash_only_ms); the bit-exact contract (SURVEY Appendix B) "
                             "rules out skipping the hash.  ncu: profiles/round2_c1_k_span.md",
                     "algorithmic_bytes_per_launch": q_bytes},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                            "cpu_model")},
        "e2e": {"value": 4 * n / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
                "path": "pinned H2D -> gcx_quantize_prefixed -> gcx_dequantize -> D2H, steps double-buffered over copy-in / compute / copy-out streams",
                # the e2e roofline: the same pinned copies with no compute,
                # both directions at once (what one e2e step must move)
                "pcie_copy_GBps": pcie,
                "frac_of_copy_only": (4 * n / (e2e_ms * 1e-3) / 1e9) / pcie["bidir_per_direction"]},
        "gpu_launches": 2 * args.steps,  # k_span + k_dspan per step
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def sra_emulation(nodes, graph=False):
    """Kernel time per rank of one SRA step (ResNet-50 layer list, default
    filter, 4b/128, 64 MiB buffers, average) with all `nodes` ranks' K1 /
    fold / K3 run on this GPU; best of 3 after a warm-up.  graph: the step's
    kernels captured as a CUDA graph and launched once (GCX_EMUL_GRAPH), so
    host launch gaps between dependent kernels drop out."""
    import numpy as np
    prev = os.environ.get("GCX_EMUL_GRAPH")
    os.environ["GCX_EMUL_GRAPH"] = "1" if graph else "0"
    try:
        return _sra_emulation(nodes, np)
    finally:
        if prev is None:
            os.environ.pop("GCX_EMUL_GRAPH", None)
        else:
            os.environ["GCX_EMUL_GRAPH"] = prev


def _sra_emulation(nodes, np):

    from paper_2111_08617_b200 import _gcomm as G
    from paper_2111_08617_b200.ddp import load_layout, resolve_codecs
    layers = load_layout("resnet50")
    codecs = resolve_codecs(layers)
    total = 0.0
    rng = np.random.default_rng(0)
    for fb in G.pack_fused_buffers([n for _, n, _ in layers], 64 << 20):
        segs = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                          codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
                for s in fb.segments]
        req = G.ReduceRequest()
        req.inputs = [(rng.standard_normal(fb.total_elements) * 1e-3).astype(np.float32)
                      for _ in range(nodes)]
        req.segments = segs
        req.op = G.ReduceOp.average
        req.step_seed = 7
        G.allreduce(req, nodes)
        total += min(G.allreduce(req, nodes).trace.device_time_s for _ in range(3))
    return total * 1e3 / nodes


def pcie_copy_rates(sets, n, reps=5):
    """Pinned host<->device copy rates of one C1 gradient (4n bytes): H2D
    alone, D2H alone, and both at once on two streams (GB/s per direction),
    best of `reps`.  The ceiling of the e2e leg, which moves 4n each way per
    step."""
    import torch
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    a, b = sets[0][0], sets[1][3]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return 4 * n / best / 1e9

    def both():
        with torch.cuda.stream(s1):
            a.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(b, non_blocking=True)

    return {"h2d": timed(lambda: a.copy_(hx, non_blocking=True)),
            "d2h": timed(lambda: hy.copy_(b, non_blocking=True)),
            "bidir_per_direction": timed(both)}


def e2e_codec(args, sets, n, bits, bucket):
    import torch

    from paper_2111_08617_b200 import device as dev

    hx = [torch.empty(n, dtype=torch.float32, pin_memory=True).copy_(sets[k][0].cpu())
          for k in range(2)]
    hout = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_done = [ev(), ev()]
    x_free = [ev(), ev()]
    cmp_done = [ev(), ev()]
    out_free = [ev(), ev()]
    started = [False, False]

    prefix = dev.make_prefix(n, bucket)

    def step(k):
        slot = k % 2
        x, norms, packed, out, bad = sets[slot]
        if started[slot]:
            s_in.wait_event(x_free[slot])
        with torch.cuda.stream(s_in):
            x.copy_(hx[slot], non_blocking=True)
            in_done[slot].record(s_in)
        s_cmp.wait_event(in_done[slot])
        if started[slot]:
            s_cmp.wait_event(out_free[slot])
        dev.quantize_prefixed(x, bits, bucket, C1_SEED + k, prefix, norms, packed, bad, stream=s_cmp)
        x_free[slot].record(s_cmp)
        dev.dequantize(norms, packed, n, bits, bucket, out, stream=s_cmp)
        cmp_done[slot].record(s_cmp)
        s_out.wait_event(cmp_done[slot])
        with torch.cuda.stream(s_out):
            hout[slot].copy_(out, non_blocking=True)
            out_free[slot].record(s_out)
        started[slot] = True

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    for k in range(args.steps):
        step(args.warmup + k)
    s_in.wait_stream(s_out)
    e1.record(s_in)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.steps



def run_sra(args):
    from paper_2111_08617_b200 import sra_bench
    return sra_bench.run(args, METRIC, ClockSampler, measured_peaks, cpu_sra_sample)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus <= 1 and int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return run_codec(args)
    return run_sra(args)


if __name__ == "__main__":
    sys.exit(main())
