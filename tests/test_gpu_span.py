"""Span K1 (gcx_span.cu: warp tile of 4096, lane span of 128, TMA-staged rows,
bulk-stored packed words) against the oracle, bit for bit, on the edges the
kernel has: full tiles + ragged tail, n < one tile, exact multiples of a tile,
buckets 32/64/128/512, every width, inline keys and span-layout key prefixes,
zero / -0.0 / subnormal / non-finite inputs inside full tiles (the careful
bucket path), all-zero buckets, and input / output pointers that are only
4-byte aligned (no bulk copies).  Reference: codec.cpp:24-69."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import device
    return device


def _check(dev, oracle, v, bits, bucket, seed, prefixed, x_off=0, p_off=0):
    """Quantize v (placed x_off floats into a buffer, outputs p_off bytes into
    theirs) and compare with the oracle."""
    from paper_2111_08617_b200 import _capi
    n = v.size
    xb = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
    xb[x_off:x_off + n] = torch.from_numpy(v).cuda()
    x = xb[x_off:x_off + n]
    nb = (n + bucket - 1) // bucket
    norms = torch.full((nb,), -7.0, dtype=torch.float32, device="cuda")
    cap = _capi.packed_capacity(n, bits)
    pbuf = torch.full((cap + 32,), 0xAB, dtype=torch.uint8, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    if prefixed:
        table = dev.make_prefix(n, bucket)
        _capi.check(lib.gcx_quantize_prefixed(x.data_ptr(), n, bits, bucket, seed, table.data_ptr(),
                                              norms.data_ptr(), pbuf.data_ptr() + p_off,
                                              bad.data_ptr(), s))
    else:
        _capi.check(lib.gcx_quantize(x.data_ptr(), n, bits, bucket, seed, norms.data_ptr(),
                                     pbuf.data_ptr() + p_off, bad.data_ptr(), s))
    torch.cuda.synchronize()
    wn, wp = oracle.quantize(v, bits, bucket, seed)
    got_p = pbuf.cpu().numpy()[p_off:p_off + cap]
    assert (norms.cpu().numpy().view(np.uint32) == wn.view(np.uint32)).all()
    assert (got_p[: wp.size] == wp).all()
    assert (got_p[wp.size:] == 0).all()  # unused tail bits/bytes of the last word are zero
    return int(bad.item()) & 0xFFFFFFFFFFFFFFFF


@pytest.mark.parametrize("prefixed", [False, True])
@pytest.mark.parametrize("bucket", [32, 64, 128, 512])
@pytest.mark.parametrize("bits", range(1, 9))
def test_span_tiles_and_tail(dev, oracle, bits, bucket, prefixed):
    rng = np.random.default_rng(bits * 37 + bucket + prefixed)
    n = 3 * 4096 * 7 + int(rng.integers(1, 4096))  # full tiles over several warps + ragged tail
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6)).astype(np.float32)
    bad = _check(dev, oracle, v, bits, bucket, int(rng.integers(0, 2**63)), prefixed)
    assert bad == 0xFFFFFFFFFFFFFFFF


@pytest.mark.parametrize("n", [1, 31, 33, 127, 129, 4095, 4096, 4097, 8192, 4096 * 600])
@pytest.mark.parametrize("prefixed", [False, True])
def test_span_lengths(dev, oracle, n, prefixed):
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n).astype(np.float32)
    _check(dev, oracle, v, 4, 128, 42, prefixed)


@pytest.mark.parametrize("bucket", [32, 64, 128, 512])
@pytest.mark.parametrize("prefixed", [False, True])
def test_span_special_values_in_full_tiles(dev, oracle, bucket, prefixed):
    """Zeros, -0.0 and subnormals send their bucket down the careful path;
    all-zero buckets give all-zero fields (sign included, codec.cpp:50)."""
    rng = np.random.default_rng(bucket)
    n = 4096 * 40 + 77
    v = rng.standard_normal(n).astype(np.float32)
    v[rng.random(n) < 0.003] = 0.0
    v[rng.random(n) < 0.003] = np.float32(-0.0)
    sub = rng.random(n) < 0.001
    v[sub] = (rng.standard_normal(int(sub.sum())) * 1e-41).astype(np.float32)  # subnormals
    v[4096 * 3 + 128: 4096 * 3 + 256] = 0.0  # a whole zero bucket (and span)
    v[4096 * 5 + 256: 4096 * 5 + 384] = np.float32(-0.0)
    v[4096 * 9: 4096 * 9 + 128] = (rng.standard_normal(128) * 1e-40).astype(np.float32)
    _check(dev, oracle, v, 3, bucket, 1234567, prefixed)


def test_span_sparse_gradient(dev, oracle):
    """90 % zeros (an embedding-like gradient): every bucket is careful."""
    rng = np.random.default_rng(11)
    n = 4096 * 20 + 5
    v = rng.standard_normal(n).astype(np.float32)
    v[rng.random(n) < 0.9] = 0.0
    for prefixed in (False, True):
        _check(dev, oracle, v, 4, 128, 99, prefixed)


@pytest.mark.parametrize("prefixed", [False, True])
def test_span_non_finite_first_index(dev, oracle, prefixed):
    """The smallest non-finite index wins across tiles and warps (codec.cpp:43-45)."""
    n = 4096 * 50 + 100
    v = np.ones(n, np.float32)
    v[4096 * 37 + 5] = np.nan
    v[4096 * 12 + 1000] = np.inf
    v[4096 * 50 + 50] = -np.inf  # in the ragged tail
    from paper_2111_08617_b200 import _capi
    x = torch.from_numpy(v).cuda()
    table = dev.make_prefix(n, 128) if prefixed else None
    if prefixed:
        _, _, bad = dev.quantize_prefixed(x, 4, 128, 5, table)
    else:
        _, _, bad = dev.quantize(x, 4, 128, 5)
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match=f"index {4096 * 12 + 1000}"):
        dev.check_finite(bad)
    w = np.ones(4100, np.float32)
    w[4097] = np.nan  # only in the tail
    _, _, bad = dev.quantize(torch.from_numpy(w).cuda(), 4, 64, 5)
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="index 4097"):
        dev.check_finite(bad)
    assert _capi is not None


@pytest.mark.parametrize("x_off,p_off", [(1, 0), (0, 4), (3, 8), (2, 12)])
@pytest.mark.parametrize("prefixed", [False, True])
def test_span_unaligned_pointers(dev, oracle, x_off, p_off, prefixed):
    """Only 4-byte alignment is promised by the C-ABI: no bulk copies then."""
    rng = np.random.default_rng(x_off * 10 + p_off)
    n = 4096 * 9 + 1234
    v = rng.standard_normal(n).astype(np.float32)
    _check(dev, oracle, v, 5, 64, 77, prefixed, x_off=x_off, p_off=p_off)


def test_span_seeds_differ_only_in_keys(dev, oracle):
    """One prefix table serves every seed (the per-step use)."""
    rng = np.random.default_rng(3)
    n = 4096 * 13 + 999
    v = rng.standard_normal(n).astype(np.float32)
    table = dev.make_prefix(n, 128)
    x = torch.from_numpy(v).cuda()
    for seed in (0, 1, 2**63 + 5, 0xFFFFFFFFFFFFFFFF):
        norms, packed, bad = dev.quantize_prefixed(x, 4, 128, seed, table)
        torch.cuda.synchronize()
        wn, wp = oracle.quantize(v, 4, 128, seed)
        assert (packed.cpu().numpy()[: wp.size] == wp).all(), seed


@pytest.mark.parametrize("bits", range(1, 9))
@pytest.mark.parametrize("bucket", [128, 256, 512, 1024, 2048, 4096])
def test_span_decode_vs_oracle(dev, oracle, bits, bucket):
    """K3 span decode (one chunk of 128 per bucket slice; shuffle tables for
    widths 1-4, per-element values for 5-8): bit-exact dequantize
    (codec.cpp:71-95) over full tiles, a ragged tile and an output pointer
    that is only 4-byte aligned."""
    rng = np.random.default_rng(bits * 100 + bucket)
    for n in (4096 * 11 + int(rng.integers(1, 4096)), 100, 4096, 129):
        v = (rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20)).astype(np.float32)
        v[rng.random(n) < 0.01] = np.float32(-0.0)
        seed = int(rng.integers(0, 2**63))
        wn, wp = oracle.quantize(v, bits, bucket, seed)
        want = oracle.dequantize(wn, wp, n, bits, bucket)
        from paper_2111_08617_b200 import _capi
        cap = _capi.packed_capacity(n, bits)
        pk = np.zeros(cap, np.uint8)
        pk[: wp.size] = wp
        for off in (0, 1):
            obuf = torch.full((n + 4,), 7.0, dtype=torch.float32, device="cuda")
            out = obuf[off:off + n]
            dev.dequantize(torch.from_numpy(wn).cuda(), torch.from_numpy(pk).cuda(), n, bits, bucket,
                           out=out)
            torch.cuda.synchronize()
            got = obuf.cpu().numpy()
            assert (got[off:off + n].view(np.uint32) == want.view(np.uint32)).all(), (n, off)
            assert (got[off + n:] == 7.0).all() and (got[:off] == 7.0).all()


@pytest.mark.parametrize("bits", [5, 8])
def test_span_decode_tiny_norms(dev, oracle, bits):
    """Values whose dequantized magnitudes fall below the normal float range
    (the wide decode's exact correction + slow conversion path)."""
    rng = np.random.default_rng(bits)
    n = 4096 * 3 + 700
    v = (rng.standard_normal(n) * 1e-38).astype(np.float32)
    v[:2048] *= np.float32(1e-3)  # subnormal inputs
    wn, wp = oracle.quantize(v, bits, 512, 5)
    want = oracle.dequantize(wn, wp, n, bits, 512)
    from paper_2111_08617_b200 import _capi
    pk = np.zeros(_capi.packed_capacity(n, bits), np.uint8)
    pk[: wp.size] = wp
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    dev.dequantize(torch.from_numpy(wn).cuda(), torch.from_numpy(pk).cuda(), n, bits, 512, out=out)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all()
