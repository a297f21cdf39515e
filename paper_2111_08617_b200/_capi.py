"""ctypes binding of the C-ABI in include/gcx.h (libgcx.so, sm_100a).

This is the reference-side FFI a Python caller would bind: plain pointers,
sizes and a stream handle.  There is no CPU fallback: importing this module
raises if libgcx.so is missing, and every call raises GcxError on a non-zero
status with the library's message.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgcx.so")

GCX_F_BIG_BUCKETS = 1
GCX_F_NEEDS_ZERO = 2
GCX_F_PIECE_SEEDS = 4
GCX_F_ODD_BUCKETS = 8
GCX_F_NORM_PASS = 16
GCX_F_LANE_GROUP = 32
GCX_F_KEY_PREFIX = 64
GCX_F_SPAN_ENC = 256
GCX_F_SEED_DEVICE = 1024
GCX_F_SPAN_DEC = 128
GCX_F_SPAN_DEC_WIDE = 512
GCX_TILE = 4096


class GcxError(RuntimeError):
    pass


NO_KEYS = 0xFFFFFFFFFFFFFFFF


class Piece(C.Structure):
    """gcx_piece (include/gcx.h)."""
    _fields_ = [("src", C.c_uint64), ("len", C.c_uint64), ("norms", C.c_uint64),
                ("packed", C.c_uint64), ("seed", C.c_uint64), ("bucket", C.c_uint32),
                ("bits", C.c_int32), ("keys", C.c_uint64)]

    def __init__(self, src=0, len=0, norms=0, packed=0, seed=0, bucket=0, bits=0,
                 keys=NO_KEYS):
        super().__init__(src, len, norms, packed, seed, bucket, bits, keys)


class KeyGroup(C.Structure):
    """gcx_keygroup (include/gcx.h)."""
    _fields_ = [("off", C.c_uint64), ("len", C.c_uint64), ("bucket", C.c_uint32),
                ("pad", C.c_uint32)]


assert C.sizeof(Piece) == 56 and C.sizeof(KeyGroup) == 24

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")

_lib = C.CDLL(LIB_PATH)
u64, i64, u32, i32, vp = C.c_uint64, C.c_int64, C.c_uint32, C.c_int, C.c_void_p


def _decl(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_decl("gcx_version", i32)
_decl("gcx_last_error", C.c_char_p)
_decl("gcx_compressed_size", u64, u64, i32, u64)
_decl("gcx_packed_bytes", u64, u64, i32)
_decl("gcx_packed_capacity", u64, u64, i32)
_decl("gcx_hop_seed", u64, u64, u64, u64)
_decl("gcx_uniform01", C.c_double, u64, u64, u64)
_decl("gcx_plan_tiles", i64, C.POINTER(Piece), u32, C.POINTER(u32), C.POINTER(u32))
_decl("gcx_quantize", i32, vp, u64, i32, u64, u64, vp, vp, vp, vp)
_decl("gcx_dequantize", i32, vp, vp, u64, i32, u64, vp, vp)
_decl("gcx_prefix_slots", u64, u64)
_decl("gcx_make_prefix", i32, u64, u64, vp, vp)
_decl("gcx_quantize_prefixed", i32, vp, u64, i32, u64, u64, vp, vp, vp, vp, vp)
_decl("gcx_encode_pieces", i32, vp, vp, u32, u32, u32, u64, vp, vp, vp, vp, vp)
_decl("gcx_decode_pieces", i32, vp, vp, u32, u32, u32, vp, vp, C.c_float, vp)
_decl("gcx_plan_keys", i64, C.POINTER(Piece), u32, C.POINTER(KeyGroup), u32, C.POINTER(u32))
_decl("gcx_make_keys", i32, vp, u32, u64, u64, vp, vp)
_decl("gcx_make_key_prefix", i32, vp, u32, u64, vp, vp)
_decl("gcx_make_keys_prefixed", i32, u64, u64, vp, vp, vp)
_decl("gcx_make_keys_prefixed_dev", i32, u64, vp, vp, vp, vp)
_decl("gcx_sra_step_seeds", i32, vp, vp)
_decl("gcx_fold_pieces", i32, vp, vp, u32, u32, u32, vp, u64, vp, u32, u32, vp, vp)
_decl("gcx_sra_fold_encode", i32, vp, vp, u32, u32, u32, vp, u64, vp, u32, u32, u64, vp, vp, vp,
      vp, vp)
_decl("gcx_sra_reduce", i32, vp, vp, u32, u32, u32, vp, u64, vp, u32, u32, u64, vp, vp,
      C.c_float, vp, vp, vp)
_decl("gcx_hash_bench", i32, u64, u64, u32, i32, vp, vp)
_decl("gcx_stats_accumulate", i32, vp, vp, u64, vp, vp)
_decl("gcx_add_f32", i32, vp, vp, u64, vp)
_decl("gcx_wire_layout", i64, C.POINTER(Piece), u32, C.POINTER(u64))
_decl("gcx_frame_pieces", i32, vp, vp, u32, vp, u64, u32, vp, vp)
_decl("gcx_unframe_pieces", i32, vp, vp, u32, vp, vp, vp, vp)
_decl("gcx_device_info", i32, i32, C.POINTER(i32), C.POINTER(i32))

EXPORTS = ["gcx_version", "gcx_last_error", "gcx_compressed_size", "gcx_packed_bytes",
           "gcx_packed_capacity", "gcx_hop_seed", "gcx_uniform01", "gcx_plan_tiles",
           "gcx_quantize", "gcx_dequantize", "gcx_encode_pieces", "gcx_decode_pieces",
           "gcx_sra_reduce", "gcx_sra_fold_encode", "gcx_hash_bench", "gcx_device_info", "gcx_plan_keys",
           "gcx_make_keys", "gcx_fold_pieces", "gcx_prefix_slots", "gcx_make_prefix",
           "gcx_quantize_prefixed", "gcx_make_key_prefix", "gcx_make_keys_prefixed",
           "gcx_make_keys_prefixed_dev", "gcx_sra_step_seeds",
           "gcx_stats_accumulate", "gcx_add_f32", "gcx_wire_layout", "gcx_frame_pieces",
           "gcx_unframe_pieces"]


def lib():
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise GcxError(f"gcx error {rc}: {_lib.gcx_last_error().decode()}")


def compressed_size(n: int, bits: int, bucket: int) -> int:
    return _lib.gcx_compressed_size(n, bits, bucket)


def packed_bytes(n: int, bits: int) -> int:
    return _lib.gcx_packed_bytes(n, bits)


def packed_capacity(n: int, bits: int) -> int:
    return _lib.gcx_packed_capacity(n, bits)


def hop_seed(step_seed: int, hop: int, node: int) -> int:
    return _lib.gcx_hop_seed(step_seed, hop, node)


def plan_tiles(pieces):
    """-> (ntiles, prefix list, flags)."""
    arr = (Piece * max(1, len(pieces)))(*pieces)
    prefix = (u32 * (len(pieces) + 1))()
    flags = u32(0)
    nt = _lib.gcx_plan_tiles(arr, len(pieces), prefix, C.byref(flags))
    if nt < 0:
        check(int(nt))
    return int(nt), list(prefix), int(flags.value)


def device_info(device: int = 0):
    sms, ctas = i32(0), i32(0)
    check(_lib.gcx_device_info(device, C.byref(sms), C.byref(ctas)))
    return sms.value, ctas.value
