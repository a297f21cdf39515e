"""CPU oracle for the compressed-allreduce hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It is the checker, never
the thing measured or shipped: ``paper_2111_08617_b200`` does not import it.

Two back ends, same signatures:

* ``Oracle()``     — ``liboracle.so`` built from ``cgx_oracle.c``, our plain-C
  restatement of ``/root/reference/proj/src/codec.cpp`` and
  ``src/collectives.cpp`` (citations inside the C file).
* ``RefOracle()``  — ``_ref/libgcomm_ref.so``, the reference sources compiled
  unmodified (``oracle/Makefile``), when present.

Parity pinning: the restatement is pinned by the Appendix-A known answers
(tests/test_oracle.py), by golden fixtures made with the compiled reference
(tests/golden/, oracle/make_golden.py) and, where ``_ref`` exists, by direct
comparison.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MODE_QUANTIZE, MODE_TOPK, MODE_UNCOMPRESSED = 0, 1, 2


class Segment(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("length", C.c_uint64), ("mode", C.c_int32),
                ("bits", C.c_int32), ("bucket", C.c_uint64)]


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _segs(segments):
    arr = (Segment * max(1, len(segments)))()
    for i, s in enumerate(segments):
        if isinstance(s, Segment):
            arr[i] = s
        else:
            off, ln, mode, bits, bucket = s
            arr[i] = Segment(off, ln, mode, bits, bucket)
    return arr


def _ptrs(arrs):
    return (C.POINTER(C.c_float) * len(arrs))(*[_f32p(a) for a in arrs])


def _threads():
    return max(1, min(32, len(os.sched_getaffinity(0))))


def bucket_count(n, bucket):
    return (n + bucket - 1) // bucket


def packed_size(n, bits):
    return (n * (bits + 1) + 7) // 8


class Oracle:
    """ctypes view of liboracle.so (the C restatement)."""

    LIB = os.path.join(HERE, "liboracle.so")

    def __init__(self, path: str | None = None):
        path = path or self.LIB
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        u64, i64, dbl, flt = C.c_uint64, C.c_int64, C.c_double, C.c_float
        L.oc_mix64.restype = u64
        L.oc_mix64.argtypes = [u64]
        L.oc_hash_combine.restype = u64
        L.oc_hash_combine.argtypes = [u64, u64]
        L.oc_uniform01.restype = dbl
        L.oc_uniform01.argtypes = [u64, u64, u64]
        L.oc_normal01.restype = flt
        L.oc_normal01.argtypes = [u64, u64]
        L.oc_fill_normal.argtypes = [C.POINTER(flt), u64, u64, flt]
        L.oc_fill_normal_range.argtypes = [C.POINTER(flt), u64, u64, u64, flt]
        L.oc_fnv1a64.restype = u64
        L.oc_fnv1a64.argtypes = [C.c_void_p, u64]
        L.oc_compressed_size.restype = u64
        L.oc_compressed_size.argtypes = [u64, C.c_int, u64]
        L.oc_serialized_size.restype = u64
        L.oc_serialized_size.argtypes = [u64, C.c_int, u64]
        L.oc_quantize.restype = i64
        L.oc_quantize.argtypes = [C.POINTER(flt), u64, C.c_int, u64, u64, C.POINTER(flt),
                                  C.POINTER(C.c_uint8)]
        L.oc_dequantize.argtypes = [C.POINTER(flt), C.POINTER(C.c_uint8), u64, C.c_int, u64,
                                    C.POINTER(flt)]
        L.oc_pack_levels.restype = C.c_int
        L.oc_pack_levels.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), u64, C.c_int,
                                     C.POINTER(C.c_uint8)]
        L.oc_unpack_levels.argtypes = [C.POINTER(C.c_uint8), u64, C.c_int,
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)]
        L.oc_serialize.argtypes = [u64, C.c_int, u64, u64, C.POINTER(flt), C.POINTER(C.c_uint8),
                                   C.POINTER(C.c_uint8)]
        L.oc_hop_seed.restype = u64
        L.oc_hop_seed.argtypes = [u64, u64, u64]
        L.oc_chunk_boundaries.argtypes = [u64, u64, C.POINTER(Segment), u64, C.POINTER(u64)]
        L.oc_sra_allreduce.restype = i64
        L.oc_sra_allreduce.argtypes = [C.POINTER(C.POINTER(flt)), u64, u64, C.POINTER(Segment),
                                       u64, u64, C.c_int, C.POINTER(flt)]
        L.oc_lossless_reference.argtypes = [C.POINTER(C.POINTER(flt)), u64, u64,
                                            C.POINTER(Segment), u64, C.c_int, C.POINTER(flt)]
        L.oc_sra_bytes_sent.restype = u64
        L.oc_sra_bytes_sent.argtypes = [u64, u64, u64, C.POINTER(Segment), u64]

    # util.hpp
    def mix64(self, z):
        return self.lib.oc_mix64(z)

    def hash_combine(self, a, b):
        return self.lib.oc_hash_combine(a, b)

    def uniform01(self, s, a, b):
        return self.lib.oc_uniform01(s, a, b)

    def normal01(self, s, i):
        return self.lib.oc_normal01(s, i)

    def normal_vector(self, n, seed, scale=1.0, out=None):
        if out is None:
            out = np.empty(n, np.float32)
        if n < (1 << 20):
            self.lib.oc_fill_normal(_f32p(out), n, seed, scale)
            return out
        # large vectors: ctypes releases the GIL, so threads fill slices
        from concurrent.futures import ThreadPoolExecutor
        step = 1 << 20
        base = out.ctypes.data
        fp = C.POINTER(C.c_float)

        def fill(lo):
            m = min(step, n - lo)
            self.lib.oc_fill_normal_range(C.cast(base + 4 * lo, fp), lo, m, seed, scale)

        with ThreadPoolExecutor(max_workers=_threads()) as ex:
            list(ex.map(fill, range(0, n, step)))
        return out

    def fnv1a64(self, arr):
        a = np.ascontiguousarray(arr)
        return self.lib.oc_fnv1a64(a.ctypes.data, a.nbytes)

    def hop_seed(self, s, hop, node):
        return self.lib.oc_hop_seed(s, hop, node)

    # codec.cpp
    def compressed_size(self, n, bits, bucket):
        return self.lib.oc_compressed_size(n, bits, bucket)

    def serialized_size(self, n, bits, bucket):
        return self.lib.oc_serialized_size(n, bits, bucket)

    def quantize(self, v, bits, bucket, seed):
        """-> (norms f32[nb], packed u8[P]); raises ValueError on non-finite input."""
        v = np.ascontiguousarray(v, np.float32)
        n = v.size
        norms = np.zeros(bucket_count(n, bucket), np.float32)
        packed = np.zeros(packed_size(n, bits), np.uint8)
        bad = self.lib.oc_quantize(_f32p(v), n, bits, bucket, seed, _f32p(norms), _u8p(packed))
        if bad >= 0:
            raise ValueError(f"non-finite gradient value at index {bad}")
        return norms, packed

    def dequantize(self, norms, packed, n, bits, bucket):
        out = np.empty(n, np.float32)
        norms = np.ascontiguousarray(norms, np.float32)
        packed = np.ascontiguousarray(packed, np.uint8)
        self.lib.oc_dequantize(_f32p(norms), _u8p(packed), n, bits, bucket, _f32p(out))
        return out

    def pack_levels(self, levels, signs, bits):
        levels = np.ascontiguousarray(levels, np.uint32)
        signs = np.ascontiguousarray(signs, np.uint8)
        out = np.zeros(packed_size(levels.size, bits), np.uint8)
        rc = self.lib.oc_pack_levels(levels.ctypes.data_as(C.POINTER(C.c_uint32)), _u8p(signs),
                                     levels.size, bits, _u8p(out))
        if rc:
            raise ValueError("level exceeds representable range")
        return out

    def unpack_levels(self, packed, n, bits):
        packed = np.ascontiguousarray(packed, np.uint8)
        levels = np.empty(n, np.uint32)
        signs = np.empty(n, np.uint8)
        self.lib.oc_unpack_levels(_u8p(packed), n, bits,
                                  levels.ctypes.data_as(C.POINTER(C.c_uint32)), _u8p(signs))
        return levels, signs

    def serialize(self, norms, packed, n, bits, bucket, seed):
        out = np.zeros(self.serialized_size(n, bits, bucket), np.uint8)
        self.lib.oc_serialize(n, bits, bucket, seed, _f32p(np.ascontiguousarray(norms)),
                              _u8p(np.ascontiguousarray(packed)), _u8p(out))
        return out

    # collectives.cpp
    def chunk_boundaries(self, d, nodes, segments):
        segs = _segs(segments)
        out = (C.c_uint64 * (nodes + 1))()
        self.lib.oc_chunk_boundaries(d, nodes, segs, len(segments), out)
        return list(out)

    def sra_allreduce(self, inputs, segments, step_seed, average=True):
        inputs = [np.ascontiguousarray(x, np.float32) for x in inputs]
        d = inputs[0].size
        out = np.empty(d, np.float32)
        bad = self.lib.oc_sra_allreduce(_ptrs(inputs), len(inputs), d, _segs(segments),
                                        len(segments), step_seed, 1 if average else 0,
                                        _f32p(out))
        if bad >= 0:
            raise ValueError(f"non-finite gradient value at index {bad}")
        return out

    def lossless_reference(self, inputs, segments, average=True):
        inputs = [np.ascontiguousarray(x, np.float32) for x in inputs]
        out = np.empty(inputs[0].size, np.float32)
        self.lib.oc_lossless_reference(_ptrs(inputs), len(inputs), inputs[0].size,
                                       _segs(segments), len(segments), 1 if average else 0,
                                       _f32p(out))
        return out

    def sra_bytes_sent(self, me, nodes, d, segments):
        return self.lib.oc_sra_bytes_sent(me, nodes, d, _segs(segments), len(segments))


class RefOracle:
    """The compiled, unmodified reference (oracle/_ref/libgcomm_ref.so)."""

    LIB = os.path.join(HERE, "_ref", "libgcomm_ref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.LIB)

    def __init__(self):
        L = self.lib = C.CDLL(self.LIB)
        u64, flt = C.c_uint64, C.c_float
        L.ref_last_error.restype = C.c_char_p
        L.ref_quantize.restype = C.c_int
        L.ref_quantize.argtypes = [C.POINTER(flt), u64, C.c_int, u64, u64, C.POINTER(flt),
                                   C.POINTER(C.c_uint8)]
        L.ref_dequantize.restype = C.c_int
        L.ref_dequantize.argtypes = [C.POINTER(flt), C.POINTER(C.c_uint8), u64, C.c_int, u64,
                                     C.POINTER(flt)]
        L.ref_serialize.restype = u64
        L.ref_serialize.argtypes = [C.POINTER(flt), u64, C.c_int, u64, u64, C.POINTER(C.c_uint8)]
        L.ref_allreduce_topo.restype = C.c_int
        L.ref_allreduce_topo.argtypes = [C.POINTER(C.POINTER(flt)), u64, u64, C.POINTER(Segment),
                                         u64, u64, C.c_int, C.c_int, C.POINTER(C.POINTER(flt)),
                                         C.POINTER(u64), C.POINTER(u64)]
        L.ref_allreduce.restype = C.c_int
        L.ref_allreduce.argtypes = [C.POINTER(C.POINTER(flt)), u64, u64, C.POINTER(Segment), u64,
                                    u64, C.c_int, C.POINTER(C.POINTER(flt)), C.POINTER(u64),
                                    C.POINTER(u64)]
        L.ref_topk_compress.restype = C.c_int
        L.ref_topk_compress.argtypes = [C.POINTER(flt), u64, u64, C.POINTER(flt), C.POINTER(u64),
                                        C.POINTER(flt)]
        L.ref_sparse_allreduce.restype = C.c_int
        L.ref_sparse_allreduce.argtypes = [u64, u64, C.POINTER(u64), C.POINTER(C.POINTER(u64)),
                                           C.POINTER(C.POINTER(flt)), C.c_int,
                                           C.POINTER(C.POINTER(flt)), C.POINTER(u64)]
        L.ref_hop_seed.restype = u64
        L.ref_hop_seed.argtypes = [u64, u64, u64]
        L.ref_engine_run.restype = C.c_int
        L.ref_engine_run.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_char_p), C.POINTER(u64),
                                     C.POINTER(C.c_int), C.POINTER(flt), C.c_int, u64,
                                     C.c_char_p, C.c_char_p, u64, u64, C.POINTER(u64),
                                     C.c_char_p, u64]

    def _check(self, rc):
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())

    def quantize(self, v, bits, bucket, seed):
        v = np.ascontiguousarray(v, np.float32)
        norms = np.zeros(bucket_count(v.size, bucket), np.float32)
        packed = np.zeros(packed_size(v.size, bits), np.uint8)
        self._check(self.lib.ref_quantize(_f32p(v), v.size, bits, bucket, seed, _f32p(norms),
                                          _u8p(packed)))
        return norms, packed

    def dequantize(self, norms, packed, n, bits, bucket):
        out = np.empty(n, np.float32)
        self._check(self.lib.ref_dequantize(_f32p(np.ascontiguousarray(norms, np.float32)),
                                            _u8p(np.ascontiguousarray(packed, np.uint8)), n,
                                            bits, bucket, _f32p(out)))
        return out

    def serialize(self, v, bits, bucket, seed):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(17 + packed_size(v.size, bits) + 4 * bucket_count(v.size, bucket) + 8,
                       np.uint8)
        n = self.lib.ref_serialize(_f32p(v), v.size, bits, bucket, seed, _u8p(out))
        return out[:n]

    def allreduce(self, inputs, segments, step_seed, average=True, topology="sra"):
        """-> (outputs per node, bytes_sent per node, counters dict)."""
        inputs = [np.ascontiguousarray(x, np.float32) for x in inputs]
        nodes, d = len(inputs), inputs[0].size
        outs = [np.empty(d, np.float32) for _ in range(nodes)]
        sent = (C.c_uint64 * nodes)()
        ctr = (C.c_uint64 * 5)()
        topo = {"sra": 0, "ring": 1, "tree": 2}[topology]
        self._check(self.lib.ref_allreduce_topo(_ptrs(inputs), nodes, d, _segs(segments),
                                                len(segments), step_seed, 1 if average else 0,
                                                topo, _ptrs(outs), sent, ctr))
        keys = ["compress_calls", "decompress_calls", "message_count", "rounds",
                "max_compress_depth"]
        return outs, list(sent), dict(zip(keys, list(ctr)))

    def topk_compress(self, v, k, residual):
        """-> (indices u64[k], values f32[k], new residual); codec.cpp:158-193."""
        v = np.ascontiguousarray(v, np.float32)
        r = np.array(residual, np.float32, copy=True)
        idx = np.zeros(max(k, 1), np.uint64)
        val = np.zeros(max(k, 1), np.float32)
        self._check(self.lib.ref_topk_compress(_f32p(v), v.size, k, _f32p(r),
                                               idx.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               _f32p(val)))
        return idx[:k], val[:k], r

    def sparse_allreduce(self, chunks, d, average=True):
        """chunks: [(indices, values)] per node -> (outputs, bytes_sent)."""
        nodes = len(chunks)
        ids = [np.ascontiguousarray(c[0], np.uint64) for c in chunks]
        vals = [np.ascontiguousarray(c[1], np.float32) for c in chunks]
        ks = (C.c_uint64 * nodes)(*[len(i) for i in ids])
        ip = (C.POINTER(C.c_uint64) * nodes)(*[i.ctypes.data_as(C.POINTER(C.c_uint64)) for i in ids])
        outs = [np.empty(d, np.float32) for _ in range(nodes)]
        sent = (C.c_uint64 * nodes)()
        self._check(self.lib.ref_sparse_allreduce(nodes, d, ks, ip, _ptrs(vals),
                                                  1 if average else 0, _ptrs(outs), sent))
        return outs, list(sent)

    def engine_run(self, nodes, layers, steps, tag, plan_json=None, adaptive_json=None,
                   step_seed=1, fuse_limit=0):
        """The reference Engine (src/engine.cpp) over SimNet.  layers: list of
        (name, elements, kind_int, scale).  -> (per-step digests of node 0's
        outputs, events JSONL)."""
        n = len(layers)
        names = (C.c_char_p * n)(*[x[0].encode() for x in layers])
        sizes = (C.c_uint64 * n)(*[x[1] for x in layers])
        kinds = (C.c_int * n)(*[x[2] for x in layers])
        scales = (C.c_float * n)(*[x[3] for x in layers])
        dig = (C.c_uint64 * steps)()
        ev = C.create_string_buffer(1 << 20)
        self._check(self.lib.ref_engine_run(nodes, n, names, sizes, kinds, scales, steps, tag,
                                            plan_json.encode() if plan_json else None,
                                            adaptive_json.encode() if adaptive_json else None,
                                            step_seed, fuse_limit, dig, ev, 1 << 20))
        return list(dig), ev.value.decode()


def engine_inputs(oracle, layers, nodes, step, tag):
    """The engine-parity input recipe shared with ref_engine_run: node r,
    layer t, step k -> scale_t * normal01(H(H(H(tag, k), r), t), i)."""
    out = []
    for r in range(nodes):
        row = []
        for t, (_, n, _, scale) in enumerate(layers):
            key = oracle.hash_combine(oracle.hash_combine(oracle.hash_combine(tag, step), r), t)
            row.append(oracle.normal_vector(n, key, scale))
        out.append(row)
    return out


def engine_inputs_flat(oracle, layers, step, tag, rank):
    """One rank's engine inputs (same recipe as engine_inputs), the layers
    concatenated into one float32 vector, filled by a thread pool (ctypes
    releases the GIL) so full-size models take seconds."""
    from concurrent.futures import ThreadPoolExecutor
    sizes = [x[1] for x in layers]
    total = int(sum(sizes))
    out = np.empty(total, np.float32)
    base = out.ctypes.data
    fp = C.POINTER(C.c_float)
    jobs, off = [], 0
    for t, (_, n, _, scale) in enumerate(layers):
        key = oracle.hash_combine(oracle.hash_combine(oracle.hash_combine(tag, step), rank), t)
        for lo in range(0, n, 1 << 20):
            jobs.append((off + lo, lo, min(1 << 20, n - lo), key, scale))
        off += n

    def fill(j):
        dst, lo, m, key, scale = j
        oracle.lib.oc_fill_normal_range(C.cast(base + 4 * dst, fp), lo, m, key, scale)

    with ThreadPoolExecutor(max_workers=_threads()) as ex:
        list(ex.map(fill, jobs))
    return out
