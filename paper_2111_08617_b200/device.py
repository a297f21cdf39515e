"""Device-level (torch tensor) entry points over the C-ABI.

These are the zero-copy calls a PyTorch caller (bench, DDP-style hook) makes:
inputs and outputs stay in HBM, launches go on the current torch stream.
They mirror codec::quantize / codec::dequantize
(/root/reference/proj/src/codec.cpp:24-95) with caller-owned buffers.
"""
from __future__ import annotations

import torch

from . import _capi
from ._capi import check

_U64_MAX = 0xFFFFFFFFFFFFFFFF


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def bucket_count(n: int, bucket: int) -> int:
    return (n + bucket - 1) // bucket


def alloc_compressed(n: int, bits: int, bucket: int, device="cuda"):
    norms = torch.empty(bucket_count(n, bucket), dtype=torch.float32, device=device)
    packed = torch.empty(_capi.packed_capacity(n, bits), dtype=torch.uint8, device=device)
    return norms, packed


def quantize(x: torch.Tensor, bits: int, bucket: int, seed: int, norms=None, packed=None,
             bad=None, stream=None, reset_bad=True):
    """K1.  Returns (norms f32[nb], packed u8[capacity], bad u64[1]).

    ``bad`` holds UINT64_MAX unless a non-finite input was seen; then its low
    40 bits are the first bad index (call ``check_finite`` after syncing)."""
    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
    n = x.numel()
    if norms is None or packed is None:
        norms, packed = alloc_compressed(n, bits, bucket, x.device)
    if bad is None:
        bad = torch.full((1,), -1, dtype=torch.int64, device=x.device)
    elif not reset_bad:
        pass  # the caller preset it to UINT64_MAX
    elif stream is not None:
        with torch.cuda.stream(stream):
            bad.fill_(-1)
    else:
        bad.fill_(-1)
    check(_capi.lib().gcx_quantize(x.data_ptr(), n, bits, bucket, seed & _U64_MAX,
                                   norms.data_ptr(), packed.data_ptr(), bad.data_ptr(),
                                   _stream_ptr(stream)))
    return norms, packed, bad


def make_prefix(n: int, bucket: int, device="cuda", stream=None) -> torch.Tensor:
    """The seed-independent key prefixes T(i) of an n-element vector
    (gcx_make_prefix); build once per buffer shape, reuse every step."""
    table = torch.empty(_capi.lib().gcx_prefix_slots(n), dtype=torch.int64, device=device)
    check(_capi.lib().gcx_make_prefix(n, bucket, table.data_ptr(), _stream_ptr(stream)))
    return table


def quantize_prefixed(x: torch.Tensor, bits: int, bucket: int, seed: int, prefix: torch.Tensor,
                      norms=None, packed=None, bad=None, stream=None, reset_bad=True):
    """K1 with a prefix table: bit-identical to ``quantize``."""
    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
    n = x.numel()
    if norms is None or packed is None:
        norms, packed = alloc_compressed(n, bits, bucket, x.device)
    if bad is None:
        bad = torch.full((1,), -1, dtype=torch.int64, device=x.device)
    elif reset_bad:
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            bad.fill_(-1)
    check(_capi.lib().gcx_quantize_prefixed(x.data_ptr(), n, bits, bucket, seed & _U64_MAX,
                                            prefix.data_ptr(), norms.data_ptr(),
                                            packed.data_ptr(), bad.data_ptr(),
                                            _stream_ptr(stream)))
    return norms, packed, bad


def check_finite(bad: torch.Tensor) -> None:
    v = int(bad.item()) & _U64_MAX
    if v != _U64_MAX:
        raise ValueError(f"non-finite gradient value at index {v & ((1 << 40) - 1)}")


def dequantize(norms: torch.Tensor, packed: torch.Tensor, n: int, bits: int, bucket: int,
               out=None, stream=None) -> torch.Tensor:
    """K3 for one vector."""
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=packed.device)
    check(_capi.lib().gcx_dequantize(norms.data_ptr(), packed.data_ptr(), n, bits, bucket,
                                     out.data_ptr(), _stream_ptr(stream)))
    return out


def hash_bench(n: int, seed: int, bucket: int, sink: torch.Tensor, variant: int = 1,
               stream=None) -> None:
    check(_capi.lib().gcx_hash_bench(n, seed, bucket, variant, sink.data_ptr(),
                                     _stream_ptr(stream)))
