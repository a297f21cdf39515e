"""Per-rank compressed gradient allreduce for one process per GPU.

The production form of the reference engine's dense exchange
(/root/reference/proj/src/engine.cpp:147-238): per-layer codecs from the
filter rules and the compression plan, greedy 64 MiB fused buffers
(model.cpp:214-256), a per-buffer step seed H(H(step_seed, step), buffer),
and the SRA allreduce (average) of each buffer by a C++ DeviceReducer over
NCCL (K1 -> all-to-all -> K2 -> all-gather -> K3).

Gradients live directly in the fused buffers (``views()`` hands out
per-layer views), so no gather/scatter copies are needed — the zero-copy
form of the reference's copy-in / copy-out (engine.cpp:210-217, :231-237).
torch is used only for device memory and streams.
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


class CompressedAllreduce:
    def __init__(self, layers, comm, plan=None, filters=None, fuse_limit_bytes=64 << 20,
                 step_seed=1, device="cuda"):
        self.layers = layers
        self.comm = comm
        self.step_seed = step_seed
        self.codecs = resolve_codecs(layers, plan, filters)
        for c in self.codecs:
            if c.mode == G.CodecMode.topk:
                raise ValueError("the topk codec is not on the B200 path")
        sizes = [n for _, n, _ in layers]
        self.buffers = G.pack_fused_buffers(sizes, fuse_limit_bytes)
        self.flat = []
        self.reducers = []
        self._views = {}
        for fb in self.buffers:
            buf = torch.zeros(fb.total_elements, dtype=torch.float32, device=device)
            segs = []
            for s in fb.segments:
                c = self.codecs[s.tensor_index]
                segs.append(G.Segment(s.buffer_offset, s.length, c.mode, c.bits, c.bucket_size))
            self.flat.append(buf)
            self.reducers.append(G.DeviceReducer(comm, fb.total_elements, segs))
        # per-layer views (a split layer maps to several pieces)
        for b, fb in enumerate(self.buffers):
            for s in fb.segments:
                name = layers[s.tensor_index][0]
                self._views.setdefault(name, []).append(
                    (s.layer_offset, self.flat[b][s.buffer_offset:s.buffer_offset + s.length]))

    @property
    def elements(self) -> int:
        return sum(fb.total_elements for fb in self.buffers)

    def views(self):
        """name -> list of (layer_offset, view into the fused buffer)."""
        return self._views

    def allreduce(self, step: int, stream=None):
        """In-place average of every fused buffer across ranks."""
        st = (stream or torch.cuda.current_stream()).cuda_stream
        for b, (buf, red) in enumerate(zip(self.flat, self.reducers)):
            seed = G.hash_combine(G.hash_combine(self.step_seed, step), b)  # engine.cpp:208-209
            red.allreduce(buf.data_ptr(), buf.data_ptr(), seed, G.ReduceOp.average, st)

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
    filter, as do layers under 4096 elements.  One DeviceReducer per bucket
    index is built on first use (DDP keeps bucket layouts fixed after the
    first iteration); the per-bucket step seed follows engine.cpp:208-209
    with the bucket index in place of the fused-buffer index.
    """

    def __init__(self, comm, plan=None, filters=None, step_seed=1):
        self.comm = comm
        self.plan = plan
        self.filters = filters
        self.step_seed = step_seed
        self.step = 0
        self.calls = 0
        self._reducers = {}

    def _reducer(self, bucket):
        idx = bucket.index()
        red = self._reducers.get(idx)
        if red is None:
            layers = []
            for k, p in enumerate(bucket.parameters()):
                kind = "weight" if p.dim() > 1 else "bias"
                layers.append((f"bucket{idx}.p{k}", p.numel(), kind))
            codecs = resolve_codecs(layers, self.plan, self.filters)
            segs, off = [], 0
            for (name, n, _), c in zip(layers, codecs):
                if c.mode == G.CodecMode.topk:
                    raise ValueError(f"{name}: the topk codec has no DDP bucket path")
                segs.append(G.Segment(off, n, c.mode, c.bits, c.bucket_size))
                off += n
            red = G.DeviceReducer(self.comm, off, segs)
            self._reducers[idx] = red
        return red

    def reduce(self, bucket):
        buf = bucket.buffer()
        red = self._reducer(bucket)
        seed = G.hash_combine(G.hash_combine(self.step_seed, self.step), bucket.index())
        red.allreduce(buf.data_ptr(), buf.data_ptr(), seed, G.ReduceOp.average,
                      torch.cuda.current_stream().cuda_stream)
        self.calls += 1
        if bucket.is_last():
            self.step += 1
        fut = torch.futures.Future()
        fut.set_result(buf)
        return fut


def cgx_comm_hook(state, bucket):
    """The function DDP calls per bucket (a named function, returning a
    torch.futures.Future[torch.Tensor]);
    ``state`` is the CgxCommHook holding the reducers."""
    return state.reduce(bucket)
