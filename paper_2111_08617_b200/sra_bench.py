"""bench.py's N > 1 leg: compressed SRA allreduce of the ResNet-50 per-layer
gradient list (BASELINE.json configs[1]) on N B200s, one rank per GPU.

One step = the average of all fused gradient buffers across ranks
(K1 -> NCCL all-to-all -> K2 -> NCCL all-gather -> K3 per buffer).
value = effective bus GB/s = (4n / t) * 2(N-1)/N, t = max over ranks.
Beside it: uncompressed NCCL fp32 allreduce of the same buffers (the
baseline the north star asks to beat), timed the same way.
"""
from __future__ import annotations

import json
import os
import statistics
import time


def run(args, metric, ClockSampler, measured_peaks, cpu_sra_sample):
    import torch
    import torch.distributed as dist

    from . import _gcomm as G
    from .ddp import CompressedAllreduce, load_layout, make_communicator

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = make_communicator(rank, world)
    layers = load_layout("resnet50")
    car = CompressedAllreduce(layers, comm)
    n = car.elements
    g = torch.Generator(device="cuda").manual_seed(0xC2 + rank)
    stream = torch.cuda.current_stream()

    def fill():
        for buf in car.flat:
            buf.normal_(generator=g).mul_(1e-3)

    fill()
    for k in range(args.warmup):
        car.allreduce(k)
    torch.cuda.synchronize()
    dist.barrier()

    # timed region: refill inputs (outside events) so every step reduces fresh data
    steps_ms = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            fill()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            car.allreduce(args.warmup + k)
            e1.record(stream)
            torch.cuda.synchronize()
            steps_ms.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(steps_ms) / len(steps_ms)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # baseline: uncompressed NCCL fp32 allreduce of the same buffers
    for _ in range(3):
        for buf in car.flat:
            dist.all_reduce(buf)
    torch.cuda.synchronize()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(stream)
    for _ in range(args.steps):
        for buf in car.flat:
            dist.all_reduce(buf)
    b1.record(stream)
    torch.cuda.synchronize()
    tb = torch.tensor([b0.elapsed_time(b1) / args.steps], device="cuda")
    dist.all_reduce(tb, op=dist.ReduceOp.MAX)
    base_ms = float(tb.item())

    # end to end with host buffers: pinned H2D of the gradient, reduce, D2H
    host_in = [torch.empty(b.numel(), dtype=torch.float32, pin_memory=True).normal_()
               for b in car.flat]
    host_out = [torch.empty(h.numel(), dtype=torch.float32, pin_memory=True) for h in host_in]
    torch.cuda.synchronize()
    dist.barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    for k in range(args.steps):
        for h, buf in zip(host_in, car.flat):
            buf.copy_(h, non_blocking=True)
        car.allreduce(10_000 + k)
        for h, buf in zip(host_out, car.flat):
            h.copy_(buf, non_blocking=True)
    x1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([x0.elapsed_time(x1) / args.steps], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())

    # the same step captured once as a CUDA graph (device-resident seeds, both
    # NCCL rounds inside the graph) and replayed.  Every rank must capture
    # successfully before any rank replays (a lone replay would wait on
    # peers that never join), so success is agreed over torch.distributed.
    graph_ms, graph_err = None, None
    if os.environ.get("GCX_BENCH_GRAPH", "1") != "0":
        gr = None
        torch.cuda.synchronize()  # no process-group work in flight during the capture
        dist.barrier()
        try:
            gr = car.capture(20_000)
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            graph_err = f"capture: {type(e).__name__}: {e}"[:300]
        ok = torch.tensor([1 if gr is not None else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 1:
            gr.replay()
            torch.cuda.synchronize()
            car.check_replay()
            dist.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(args.steps):
                gr.replay()
            g1.record(stream)
            torch.cuda.synchronize()
            car.check_replay()
            tg = torch.tensor([g0.elapsed_time(g1) / args.steps], device="cuda")
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
            graph_ms = float(tg.item())
        elif graph_err is None:
            graph_err = "another rank failed to capture"

    busbw = lambda ms_: (4 * n / (ms_ * 1e-3)) * 2 * (world - 1) / world / 1e9  # noqa: E731
    # the reference's CPU SRA on this host (rank 0 only, after the timed region)
    cb = None
    if rank == 0:
        s = cpu_sra_sample(world)
        cb = {k: s[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
    peak, peak_kind = measured_peaks()
    wire = car.wire_bytes_sent()
    dev_bytes = car.device_bytes_sent()
    if rank == 0:
        line = {
            "metric": metric, "value": busbw(ms), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 in, f64 codec math, u8 packed", "data": "synthetic (torch.randn * 1e-3)",
            "config": {"workload": "ResNet-50 per-layer gradient list (161 tensors, 25,557,032 "
                                   "floats), default filter, 4-bit/128, 64 MiB fused buffers, "
                                   "SRA average",
                       "parallelism": f"dp{world}", "buffers": len(car.buffers),
                       "convention": "busbw = (4n/t)*2(N-1)/N (nccl-tests)",
                       "aggregate_input_GBps": world * 4 * n / (ms * 1e-3) / 1e9,
                       "aggregate_note": "all ranks' gradient bytes reduced per second "
                                         "(N x 4n / t)",
                       "graph_ms_per_step": graph_ms,
                       "graph_busbw_GBps": busbw(graph_ms) if graph_ms else None,
                       "graph_note": "the step captured once as a CUDA graph "
                                     "(CompressedAllreduce.capture: device-resident seeds, "
                                     "NCCL rounds in the graph), K back-to-back replays "
                                     "on resident data" + (f"; {graph_err}" if graph_err else ""),
                       "nccl_fp32_allreduce_ms": base_ms,
                       "nccl_fp32_busbw_GBps": busbw(base_ms),
                       "speedup_vs_nccl_fp32": base_ms / ms,
                       "wire_bytes_sent_per_rank": wire, "device_bytes_sent_per_rank": dev_bytes,
                       "nvlink_GBps_on_compressed_bytes": dev_bytes / (ms * 1e-3) / 1e9,
                       "l2": "inputs refilled before every step (102 MB/rank, rotating RNG)"},
            "roofline": {"bound": "nvlink", "achieved": dev_bytes / (ms * 1e-3) / 1e9,
                         "peak": 770.0, "unit": "GB/s",
                         "frac": dev_bytes / (ms * 1e-3) / 1e9 / 770.0,
                         "traffic": dev_bytes,
                         "traffic_note": "bytes each rank sends per step over NVLink (both "
                                         "exchange rounds, from the piece tables); the kernels' "
                                         "DRAM traffic is in profiles/round2_launches_sra8_emul.csv",
                         "kernel": "whole SRA step (compressed bytes over NVLink)",
                         "peak_kind": "measured peer copy per direction (B200_PROFILING.md)"},
            "cpu_baseline": cb,
            "e2e": {"value": busbw(e2e_ms), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                    "d2h_bytes_per_step": 4 * n},
            "gpu_launches": car.launches_per_step() * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
