"""Per-rank compressed gradient allreduce for one process per GPU.

The production form of the reference engine's dense exchange
(/root/reference/proj/src/engine.cpp:147-238): per-layer codecs from the
filter rules and the compression plan, greedy 64 MiB fused buffers
(model.cpp:214-256), a per-buffer step seed H(H(step_seed, step), buffer),
and the SRA allreduce (average) of each buffer by a C++ DeviceReducer
(K1 -> all-to-all -> K2 -> all-gather -> K3) over a Transport:
``Communicator`` (NCCL over NVLink, one process per GPU) or
``LoopbackTransport`` (N ranks as threads of one process on one GPU — the
same reducer code, offsets and message matching, used to prove the per-rank
path bit-exact at N > 1 on a single B200).

Gradients live directly in the fused buffers (``views()`` hands out
per-layer views), so no gather/scatter copies are needed — the zero-copy
form of the reference's copy-in / copy-out (engine.cpp:210-217, :231-237).

Scheduling: every fused buffer has its own CUDA stream
and its own transport (``Transport.split()``: an independent NCCL
communicator), so buffer b+1's quantizer runs while buffer b's messages are
on the wire.  ``mark_ready(name)`` is the size trigger: a buffer is reduced
as soon as its last layer's gradient is ready, under the rest of the
backward pass.  (The reference's cycle-time cut, engine.hpp:31-34, never
fires: "a full step's submissions share one virtual instant, so only the
size cut ever triggers".)  torch is used only for device memory and streams.
"""
from __future__ import annotations

import json
import os

import torch

from . import _gcomm as G

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = {"weight": G.LayerKind.weight, "bias": G.LayerKind.bias, "norm": G.LayerKind.norm,
         "embedding": G.LayerKind.embedding, "other": G.LayerKind.other}


def load_layout(name: str):
    """Layer lists of the benchmark models (derived offline from torchvision /
    transformers parameter shapes; see layouts/*.json)."""
    with open(os.path.join(HERE, "layouts", f"{name}.json")) as f:
        d = json.load(f)
    return [(x["name"], int(x["elements"]), x["kind"]) for x in d["layers"]]


def resolve_codecs(layers, plan=None, filters=None):
    """engine.cpp:178-190 (static plan): filtered -> uncompressed, else plan."""
    if filters is None:
        filters = G.FilterRules()
    filters.compile()
    plan = plan or G.CompressionPlan()
    out = []
    for name, n, kind in layers:
        spec = G.LayerSpec(name, n, KINDS[kind])
        if filters.excluded(spec):
            out.append(G.LayerCodec(G.CodecMode.uncompressed, 4, 128, 0))
        else:
            out.append(plan.resolve(name))
    return out


def step_seed_of(base: int, step: int, buffer: int) -> int:
    """engine.cpp:208-209: H(H(cfg.step_seed, step), buffer_idx)."""
    return G.hash_combine(G.hash_combine(base, step), buffer)


class CompressedAllreduce:
    """Compressed SRA allreduce (average) of a model's gradients, per rank.

    ``comm``: this rank's Transport.  With ``pipeline`` (default) each fused
    buffer after the first gets ``comm.split()`` and its own stream; every
    rank must construct its CompressedAllreduce in the same order (the split
    is collective)."""

    def __init__(self, layers, comm, plan=None, filters=None, fuse_limit_bytes=64 << 20,
                 step_seed=1, device="cuda", pipeline=True):
        self.layers = layers
        self.comm = comm
        self.step_seed = step_seed
        self.codecs = resolve_codecs(layers, plan, filters)
        for c in self.codecs:
            if c.mode == G.CodecMode.topk:
                raise ValueError("the topk codec is not on the B200 path")
        sizes = [n for _, n, _ in layers]
        self.buffers = G.pack_fused_buffers(sizes, fuse_limit_bytes)
        self.pipeline = bool(pipeline) and len(self.buffers) > 1
        self.transports = [comm]
        for _ in self.buffers[1:]:
            self.transports.append(comm.split() if self.pipeline else comm)
        self.streams = ([torch.cuda.Stream(device=device) for _ in self.buffers]
                        if self.pipeline else None)
        self.flat = []
        self.reducers = []
        self._views = {}
        self._buffer_of = {}  # layer name -> buffers holding a piece of it
        for b, fb in enumerate(self.buffers):
            buf = torch.zeros(fb.total_elements, dtype=torch.float32, device=device)
            segs = []
            for s in fb.segments:
                c = self.codecs[s.tensor_index]
                segs.append(G.Segment(s.buffer_offset, s.length, c.mode, c.bits, c.bucket_size))
            self.flat.append(buf)
            self.reducers.append(G.DeviceReducer(self.transports[b], fb.total_elements, segs))
        for b, fb in enumerate(self.buffers):  # per-layer views (a split layer has several)
            for s in fb.segments:
                name = layers[s.tensor_index][0]
                self._views.setdefault(name, []).append(
                    (s.layer_offset, self.flat[b][s.buffer_offset:s.buffer_offset + s.length]))
                self._buffer_of.setdefault(name, []).append(b)
        self._pending = [len(fb.segments) for fb in self.buffers]
        self._launched = [False] * len(self.buffers)
        self._step = None
        self._origin = None
        self._dev_next = None  # device-resident seeds: the step the counters hold

    @property
    def elements(self) -> int:
        return sum(fb.total_elements for fb in self.buffers)

    def views(self):
        """name -> list of (layer_offset, view into the fused buffer)."""
        return self._views

    # -- whole-step form ------------------------------------------------------
    def allreduce(self, step: int, stream=None):
        """In-place average of every fused buffer across ranks, ordered after
        the work already on ``stream`` (default: the current stream), which
        waits for the result.  Raises the previous call's non-finite error
        (the reference's codec.cpp:43-45 message) before starting."""
        self.begin(step, stream)
        for b in range(len(self.buffers)):
            self._launch(b)
        self.end()

    # -- CUDA-graph form ---------------------------------------------------------
    def use_device_seeds(self, next_step: int):
        """Every reducer takes its step seed H(H(step_seed, step), buffer)
        (engine.cpp:208-209) from a device-resident counter starting at
        ``next_step`` and advanced on the device per call, so a captured step
        replays with fresh keys.  Steps must then run consecutively."""
        self.poll(wait=True)
        for b, r in enumerate(self.reducers):
            r.use_device_seeds(self.step_seed, b, next_step)
        self._dev_next = next_step

    def capture(self, next_step: int, stream=None):
        """Capture one whole step — every fused buffer's K1, exchange, owner
        step, exchange and K3 on its own stream — as a CUDA graph.  Each
        ``graph.replay()`` then averages the fused buffers in place for the
        next step (next_step, next_step + 1, ...) with no per-kernel host
        work; call ``check_replay()`` after a replay has completed to raise
        its non-finite / transport errors.  NCCL transport only (the
        loopback's rounds are host rendezvous)."""
        import torch
        self.use_device_seeds(next_step)
        graph = torch.cuda.CUDAGraph()
        # thread-local capture mode: other threads (NCCL's proxy, torch's
        # process-group watchdog) keep querying their events meanwhile
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
            origin = torch.cuda.current_stream()
            self._step, self._origin = next_step, origin
            self._pending = [len(fb.segments) for fb in self.buffers]
            self._launched = [False] * len(self.buffers)
            for b in range(len(self.buffers)):
                self._launch(b)
            if self.pipeline:
                for s in self.streams:
                    origin.wait_stream(s)
            self._step = None
        self._dev_next = None  # replays advance the counters on the device
        return graph

    def check_replay(self):
        for r in self.reducers:
            r.check_replay()

    def device_step(self) -> int:
        """The step the next call / replay reduces (device-resident seeds)."""
        return self.reducers[0].device_step()

    # -- readiness-driven form (size trigger) -----------------------------------
    def begin(self, step: int, stream=None):
        self.poll(wait=True)
        if self._dev_next is not None:
            if step != self._dev_next:
                raise ValueError(f"device-resident seeds hold step {self._dev_next}, "
                                 f"not {step}: steps must run consecutively")
            self._dev_next += 1
        self._step = step
        self._origin = stream or torch.cuda.current_stream()
        self._pending = [len(fb.segments) for fb in self.buffers]
        self._launched = [False] * len(self.buffers)

    def mark_ready(self, name: str):
        """The gradient of layer ``name`` is complete on the origin stream:
        a buffer whose last layer this is starts reducing right away."""
        for b in self._buffer_of[name]:
            self._pending[b] -= 1
            if self._pending[b] == 0 and not self._launched[b]:
                self._launch(b)

    def end(self):
        """Launch what is left and make the origin stream wait for all of it."""
        for b in range(len(self.buffers)):
            if not self._launched[b]:
                self._launch(b)
        if self.pipeline:
            for s in self.streams:
                self._origin.wait_stream(s)
        self._step = None

    def _launch(self, b: int):
        self._launched[b] = True
        buf, red = self.flat[b], self.reducers[b]
        seed = step_seed_of(self.step_seed, self._step, b)
        if self.pipeline:
            st = self.streams[b]
            st.wait_stream(self._origin)
        else:
            st = self._origin
        red.allreduce(buf.data_ptr(), buf.data_ptr(), buf.numel(), seed, G.ReduceOp.average,
                      st.cuda_stream)

    def poll(self, wait=True) -> bool:
        """Raise ValueError('non-finite gradient value at index i') if the last
        step saw a non-finite input, and transport errors.  -> all done."""
        return all([r.poll(wait) for r in self.reducers])

    def launches_per_step(self) -> int:
        return sum(r.launches_per_call() for r in self.reducers)

    def device_bytes_sent(self) -> int:
        return sum(r.device_bytes_sent() for r in self.reducers)

    def wire_bytes_sent(self) -> int:
        return sum(r.trace().bytes_sent[self.comm.rank()] if self.comm.size() > 1 else 0
                   for r in self.reducers)


def make_communicator(rank: int, world: int):
    """NCCL communicator for our kernels; the unique id travels over the
    already-initialised torch.distributed process group."""
    import torch.distributed as dist
    uid = [G.Communicator.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    return G.Communicator(rank, world, uid[0])


class CgxCommHook:
    """PyTorch DDP communication hook: each gradient bucket DDP hands over is
    averaged across ranks by the compressed SRA allreduce, in place.

    ``model.register_comm_hook(CgxCommHook(comm), cgx_comm_hook)``.  The bucket's
    flat buffer holds its parameters' gradients back to back; each parameter
    is a layer with the reference's filter rules and plan (engine.cpp:178-190):
    1-D parameters count as bias / norm and stay uncompressed by the default
    filter, as do layers under 4096 elements.

    DDP rebuilds its buckets once, after the first backward pass
    (``Reducer._rebuild_buckets``: the real gradient-ready order and a 1 MiB
    first bucket), so bucket k's parameters can change between steps.  A
    reducer is therefore keyed by the bucket's layout — (index, parameter
    sizes and kinds) — and every call checks dtype, contiguity, device and
    length against it.  Buckets are reduced on the current stream, in the
    order DDP hands them over; every bucket index has its own transport
    (``comm.split()``, in first-use order, which DDP makes identical on all
    ranks).  The per-bucket step seed follows engine.cpp:208-209 with the
    bucket index in place of the fused-buffer index.
    """

    def __init__(self, comm, plan=None, filters=None, step_seed=1):
        self.comm = comm
        self.plan = plan
        self.filters = filters
        self.step_seed = step_seed
        self.step = 0
        self.calls = 0
        self._reducers = {}
        self._transports = {}

    @staticmethod
    def _layout(bucket):
        return tuple((p.numel(), "weight" if p.dim() > 1 else "bias")
                     for p in bucket.parameters())

    def _reducer(self, bucket):
        idx = bucket.index()
        key = (idx, self._layout(bucket))
        red = self._reducers.get(key)
        if red is None:
            if idx not in self._transports:
                self._transports[idx] = self.comm if not self._transports else self.comm.split()
            layers = [(f"bucket{idx}.p{k}", n, kind) for k, (n, kind) in enumerate(key[1])]
            codecs = resolve_codecs(layers, self.plan, self.filters)
            segs, off = [], 0
            for (name, n, _), c in zip(layers, codecs):
                if c.mode == G.CodecMode.topk:
                    raise ValueError(f"{name}: the topk codec has no DDP bucket path")
                segs.append(G.Segment(off, n, c.mode, c.bits, c.bucket_size))
                off += n
            red = G.DeviceReducer(self._transports[idx], off, segs)
            self._reducers[key] = red
        return red

    def reduce(self, bucket):
        buf = bucket.buffer()
        if buf.dtype != torch.float32:
            raise ValueError(f"compressed allreduce needs float32 gradient buckets, got {buf.dtype}")
        if not buf.is_cuda or not buf.is_contiguous():
            raise ValueError("gradient bucket must be a contiguous CUDA tensor")
        red = self._reducer(bucket)
        red.poll(True)  # the previous call of this layout: raise its non-finite input
        seed = G.hash_combine(G.hash_combine(self.step_seed, self.step), bucket.index())
        red.allreduce(buf.data_ptr(), buf.data_ptr(), buf.numel(), seed, G.ReduceOp.average,
                      torch.cuda.current_stream().cuda_stream)
        self.calls += 1
        if bucket.is_last():
            self.step += 1
        fut = torch.futures.Future()
        fut.set_result(buf)
        return fut

    def poll(self, wait=True) -> bool:
        return all([r.poll(wait) for r in self._reducers.values()])


def cgx_comm_hook(state, bucket):
    """The function DDP calls per bucket (a named function, returning a
    torch.futures.Future[torch.Tensor]);
    ``state`` is the CgxCommHook holding the reducers."""
    return state.reduce(bucket)
