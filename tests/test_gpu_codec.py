"""K1/K3 parity through the C-ABI on the GPU: bit-exact packed codes, norms
and dequantized values against the oracle."""
import json
import os

import numpy as np
import pytest

from tests.golden_inputs import make_input

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import device
    return device


def _gpu_codec(dev, v, bits, bucket, seed):
    x = torch.from_numpy(v).cuda()
    norms, packed, bad = dev.quantize(x, bits, bucket, seed)
    deq = dev.dequantize(norms, packed, v.size, bits, bucket)
    torch.cuda.synchronize()
    dev.check_finite(bad)
    nbytes = (v.size * (bits + 1) + 7) // 8
    return norms.cpu().numpy(), packed.cpu().numpy()[:nbytes], deq.cpu().numpy()


def test_golden_codec_cases_bit_exact(dev, oracle):
    with open(os.path.join(GOLD, "codec.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        v = make_input(c["n"], c["gen"])
        if c["n"] == 0:
            continue
        norms, packed, deq = _gpu_codec(dev, v, c["bits"], c["bucket"], c["seed"])
        assert oracle.fnv1a64(norms) == c["norms_fnv"], c
        assert oracle.fnv1a64(packed) == c["packed_fnv"], c
        assert oracle.fnv1a64(deq) == c["deq_fnv"], c


def test_c1_full_size_digests(dev, oracle):
    """C1 = 1e-3*normal01(0x5eed, i), n = 25,557,032, 4b/128, seed 42."""
    n = 25_557_032
    v = oracle.normal_vector(n, 0x5EED, 1e-3)
    norms, packed, deq = _gpu_codec(dev, v, 4, 128, 42)
    assert packed.size == 15_973_145 and norms.size == 199_665
    assert oracle.fnv1a64(packed) == 0x48061E58E8EFC214
    assert oracle.fnv1a64(norms) == 0xA0F211F9B3554F9A
    assert oracle.fnv1a64(deq) == 0x475F012FF75F72F5


@pytest.mark.parametrize("bits", range(1, 9))
@pytest.mark.parametrize("bucket", [1, 5, 64, 128, 512, 1024, 3000, 5000, 10000])
def test_random_matrix_vs_oracle(dev, oracle, bits, bucket):
    rng = np.random.default_rng(bits * 7919 + bucket)
    n = int(rng.integers(1, 60000))
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30)).astype(np.float32)
    v[rng.random(n) < 0.02] = np.float32(-0.0)
    v[rng.random(n) < 0.02] = 0.0
    seed = int(rng.integers(0, 2**63))
    norms, packed, deq = _gpu_codec(dev, v, bits, bucket, seed)
    wn, wp = oracle.quantize(v, bits, bucket, seed)
    assert (norms.view(np.uint32) == wn.view(np.uint32)).all()
    assert (packed == wp).all()
    wd = oracle.dequantize(wn, wp, n, bits, bucket)
    assert (deq.view(np.uint32) == wd.view(np.uint32)).all()


def test_error_bound_and_norm_bound(dev, oracle):
    """proj/tests/codec_test.cpp:78-96 on the GPU output."""
    n = 1_000_000
    v = oracle.normal_vector(n, 7)
    norms, packed, deq = _gpu_codec(dev, v, 3, 128, 99)
    bound = norms.astype(np.float64)[np.arange(n) // 128] / 7
    err = np.abs(deq.astype(np.float64) - v)
    assert (err <= bound * (1 + 1e-5)).all()
    assert (np.abs(deq) <= bound * 7 * (1 + 1e-5)).all()


def test_non_finite_reports_first_index(dev):
    v = np.ones(1000, np.float32)
    v[700] = np.inf
    v[901] = np.nan
    x = torch.from_numpy(v).cuda()
    _, _, bad = dev.quantize(x, 4, 128, 0)
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="index 700"):
        dev.check_finite(bad)


def test_dequant_exhaustive_levels(dev, oracle):
    """Every level of every width against random norms (A6 exactness)."""
    rng = np.random.default_rng(5)
    for bits in range(1, 9):
        s = (1 << bits) - 1
        nb = 4096
        norms = np.abs(rng.standard_normal(nb) * 10.0 ** rng.integers(-35, 35, nb)).astype(np.float32)
        bucket = s + 1
        n = nb * bucket
        levels = np.tile(np.arange(s + 1, dtype=np.uint32), nb)
        signs = (rng.random(n) < 0.5).astype(np.uint8)
        packed = oracle.pack_levels(levels, signs, bits)
        want = oracle.dequantize(norms, packed, n, bits, bucket)
        cap = np.zeros((packed.size + 3) // 4 * 4, np.uint8)
        cap[: packed.size] = packed
        got = dev.dequantize(torch.from_numpy(norms).cuda(), torch.from_numpy(cap).cuda(), n,
                             bits, bucket).cpu().numpy()
        assert (got.view(np.uint32) == want.view(np.uint32)).all(), bits


def test_key_table_encode_matches_inline(dev, oracle):
    """Pieces quantized under one seed share uniform01 keys per piece-local
    index and bucket size (codec.cpp:60; collectives.cpp:252-253 uses one seed
    per sender hop).  Encoding with a gcx_make_keys table must equal inline
    hashing byte for byte, and both the oracle per piece."""
    import ctypes as C
    from paper_2111_08617_b200 import _capi
    rng = np.random.default_rng(17)
    lens = [int(x) for x in rng.integers(1, 9000, 23)] + [8192, 8191, 1, 4096]
    pieces, off, src_off = [], 0, 0
    for k, n in enumerate(lens):
        bits = int(rng.integers(1, 9)) if k % 5 else 0
        bucket = int(rng.choice([7, 64, 128, 512, 2048, 5000])) if bits else 0
        nb = (n + bucket - 1) // bucket if bits else 0
        if bits:
            norms_off = off
            packed_off = (off + 4 * nb + 15) // 16 * 16
            off = (packed_off + _capi.packed_capacity(n, bits) + 15) // 16 * 16
        else:
            norms_off = packed_off = off
            off = (off + 4 * n + 15) // 16 * 16
        pieces.append(_capi.Piece(src_off, n, norms_off, packed_off, 0, bucket, bits))
        src_off += n
    x = (rng.standard_normal(src_off) * 10.0 ** rng.integers(-3, 3)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    seed = 0xABCDEF12345
    arr = (_capi.Piece * len(pieces))(*pieces)
    groups = (_capi.KeyGroup * len(pieces))()
    ng = C.c_uint32(0)
    total = _capi.lib().gcx_plan_keys(arr, len(pieces), groups, len(pieces), C.byref(ng))
    assert total > 0 and ng.value >= 5
    nt, prefix, flags = _capi.plan_tiles(list(arr))
    dev_pieces = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).cuda()
    dev_groups = torch.frombuffer(bytearray(bytes(groups)), dtype=torch.uint8).cuda()
    dev_prefix = torch.tensor(prefix, dtype=torch.int32).cuda()
    keys = torch.empty(total, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _capi.check(_capi.lib().gcx_make_keys(dev_groups.data_ptr(), ng.value, total, seed,
                                          keys.data_ptr(), st))
    # the two-step form an SRA reducer uses: stored prefixes, then one
    # finalizer per slot per step -> the same table word for word
    kpre = torch.empty(total, dtype=torch.int64, device="cuda")
    keys2 = torch.empty(total, dtype=torch.int64, device="cuda")
    _capi.check(_capi.lib().gcx_make_key_prefix(dev_groups.data_ptr(), ng.value, total,
                                                kpre.data_ptr(), st))
    _capi.check(_capi.lib().gcx_make_keys_prefixed(total, seed, kpre.data_ptr(), keys2.data_ptr(),
                                                   st))
    torch.cuda.synchronize()
    k1 = keys.cpu().numpy().view(np.uint32)
    k2 = keys2.cpu().numpy().view(np.uint32)
    for g in range(ng.value):  # every slot a piece can read (run padding is never read)
        t = groups[g].off + np.arange(groups[g].len, dtype=np.int64)
        pos = ((t >> 10) << 11) | (((t & 31) >> 2) << 7) | (((t >> 5) & 31) << 2) | (t & 3)
        assert (k1[pos] == k2[pos]).all() and (k1[pos + 1024] == k2[pos + 1024]).all()
    # spot-check table words against the reference RNG: slot s of run g holds
    # uniform01's key of piece-local index i = s - off (high word at key_pos)
    kw = keys.cpu().numpy().view(np.uint32)
    for g in range(ng.value):
        grp = groups[g]
        for i in (0, 1, 33, grp.len - 1):
            t = grp.off + i
            pos = ((t >> 10) << 11) | (((t & 31) >> 2) << 7) | (((t >> 5) & 31) << 2) | (t & 3)
            k53 = (int(kw[pos]) << 32 | int(kw[pos + 1024])) >> 11
            assert k53 * 2.0**-53 == _capi.lib().gcx_uniform01(seed, i // grp.bucket, i)
    outs = []
    for use_keys in (False, True):
        msg = torch.zeros(off + 64, dtype=torch.uint8, device="cuda")
        bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        _capi.check(_capi.lib().gcx_encode_pieces(
            dev_pieces.data_ptr(), dev_prefix.data_ptr(), len(pieces), nt, flags, seed,
            xd.data_ptr(), msg.data_ptr(), keys.data_ptr() if use_keys else None,
            bad.data_ptr(), st))
        torch.cuda.synchronize()
        assert int(bad.item()) == -1
        outs.append(msg.cpu().numpy())
    assert (outs[0] == outs[1]).all()
    for p in pieces:
        if p.bits == 0:
            assert (outs[1][p.norms:p.norms + 4 * p.len].view(np.float32) ==
                    x[p.src:p.src + p.len]).all()
            continue
        wn, wp = oracle.quantize(x[p.src:p.src + p.len], p.bits, p.bucket, seed)
        got_n = outs[1][p.norms:p.norms + 4 * wn.size].view(np.float32)
        assert (got_n.view(np.uint32) == wn.view(np.uint32)).all()
        assert (outs[1][p.packed:p.packed + wp.size] == wp).all()


@pytest.mark.parametrize("bits", [1, 2, 4, 5, 8])
@pytest.mark.parametrize("bucket", [32, 64, 96, 128, 256, 2048, 8192])
def test_dense_fast_paths_vs_oracle(dev, oracle, bits, bucket):
    """Zero-free inputs keep every group on K1b's 32-bit-compare fast path
    (bucket % 32 == 0: fused norms for 32/64/128, pre-pass otherwise) and K3's
    lane-per-chunk table path; ragged lengths end in a partial group."""
    rng = np.random.default_rng(bits * 131 + bucket)
    n = int(rng.integers(bucket, 70000)) | 1
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20)).astype(np.float32)
    v[v == 0] = np.float32(1e-3)
    seed = int(rng.integers(0, 2**63))
    norms, packed, deq = _gpu_codec(dev, v, bits, bucket, seed)
    wn, wp = oracle.quantize(v, bits, bucket, seed)
    assert (norms.view(np.uint32) == wn.view(np.uint32)).all()
    assert (packed == wp).all()
    wd = oracle.dequantize(wn, wp, n, bits, bucket)
    assert (deq.view(np.uint32) == wd.view(np.uint32)).all()


@pytest.mark.parametrize("bits", [2, 4, 7])
def test_ambiguous_key_compare_takes_exact_path(dev, oracle, bits):
    """K1b decides `uniform01 < p` on the key's top 32 bits and recomputes a
    group whose top word equals floor(frac(x) * 2^32).  Build such an element:
    bucket norm 1.0 (one dominant element), v0 tiny so x = v0 * s exactly, and
    v0 chosen so floor(x * 2^32) is the key's top word."""
    from paper_2111_08617_b200 import _capi
    v, hh, k53, seed = _ambiguous_vector(_capi.lib(), bits, 0x1234567 + bits)
    s = (1 << bits) - 1
    x = float(v[0]) * s
    assert int(np.floor(x * 2.0**32)) == hh  # the constructed tie on the top word
    norms, packed, deq = _gpu_codec(dev, v, bits, 128, seed)
    wn, wp = oracle.quantize(v, bits, 128, seed)
    assert wn[0] == np.float32(1.0)
    assert (packed == wp).all()
    # and the decision itself: level 0 rounds up iff k53 < x * 2^53
    up = k53 < x * 2.0**53
    assert (int(wp[0]) & s) == (1 if up else 0)


def _ambiguous_vector(lib, bits, seed, bucket=128):
    """-> (v, hh, k53, seed): element 0 of bucket 0 ties on the key's top word.
    The seed is advanced until the tie needs v0 < 2^-12, so the bucket norm
    stays exactly 1.0 and x = v0 * s is exact."""
    s = (1 << bits) - 1
    while True:
        k53 = int(lib.gcx_uniform01(seed, 0, 0) * 2.0**53)  # bucket 0, element 0
        hh = k53 >> 21
        if 0 < hh < min(s << 20, 1 << 22):  # float steps of v0 finer than the tie window
            break
        seed += 1
    v0 = np.float32((hh + 0.5) / s / 2.0**32)
    for _ in range(4096):  # walk to a float with floor(v0 * s * 2^32) == hh
        fl = int(np.floor(float(v0) * s * 2.0**32))
        if fl == hh:
            break
        v0 = np.nextafter(v0, np.float32(np.inf) if fl < hh else np.float32(0))
    v = np.full(bucket, np.float32(1e-12))
    v[0] = v0
    v[1] = np.float32(1.0)
    return v, hh, k53, seed


@pytest.mark.parametrize("bits,bucket,n,zeros", [
    (4, 128, 100_003, False), (4, 128, 65_537, True), (1, 32, 40_000, False),
    (8, 64, 33_333, True), (3, 512, 70_001, False), (5, 96, 50_000, True),
    (2, 1000, 30_000, False), (6, 8192, 50_000, False)])
def test_prefixed_quantize_matches_oracle(dev, oracle, bits, bucket, n, zeros):
    """gcx_quantize_prefixed (seed-independent key prefixes T(i) built once)
    is bit-identical to the reference codec for every kernel route: fused
    lane-per-bucket (32/64/128), pre-pass + lane-per-group (512, 8192),
    generic (96 is 32-aligned: lane-per-group; 1000: generic k_quant)."""
    rng = np.random.default_rng(bits * 1009 + bucket + n)
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8)).astype(np.float32)
    if zeros:
        v[rng.random(n) < 0.01] = 0.0
    x = torch.from_numpy(v).cuda()
    prefix = dev.make_prefix(n, bucket)
    for seed in (int(rng.integers(0, 2**63)), 7):
        norms, packed, bad = dev.quantize_prefixed(x, bits, bucket, seed, prefix)
        torch.cuda.synchronize()
        dev.check_finite(bad)
        wn, wp = oracle.quantize(v, bits, bucket, seed)
        assert (norms.cpu().numpy().view(np.uint32) == wn.view(np.uint32)).all()
        assert (packed.cpu().numpy()[: wp.size] == wp).all()


def test_wire_framing_is_the_reference_message(dev, oracle):
    """gcx_frame_pieces turns a device message into the reference's exact
    encode_pieces bytes (collectives.cpp:143-163: serialize() per quantized
    piece -- 17-byte header, norms, packed -- raw f32 otherwise), and
    gcx_unframe_pieces restores the device message; a header that disagrees
    with the layout is flagged."""
    import ctypes as C
    from paper_2111_08617_b200 import _capi
    rng = np.random.default_rng(31)
    lens = [int(x) for x in rng.integers(1, 7000, 17)] + [1, 4096, 4097]
    pieces, off, src_off = [], 0, 0
    for k, n in enumerate(lens):
        bits = int(rng.integers(1, 9)) if k % 4 else 0
        bucket = int(rng.choice([7, 64, 128, 1000])) if bits else 0
        if bits:
            nb = (n + bucket - 1) // bucket
            norms_off = off
            packed_off = (off + 4 * nb + 15) // 16 * 16
            off = (packed_off + _capi.packed_capacity(n, bits) + 15) // 16 * 16
        else:
            norms_off = packed_off = off
            off = (off + 4 * n + 15) // 16 * 16
        pieces.append(_capi.Piece(src_off, n, norms_off, packed_off, 0, bucket, bits))
        src_off += n
    x = (rng.standard_normal(src_off) * 0.1).astype(np.float32)
    seed = 0x5151_0001
    arr = (_capi.Piece * len(pieces))(*pieces)
    nt, prefix, flags = _capi.plan_tiles(list(arr))
    wire_off = (C.c_uint64 * len(pieces))()
    total = _capi.lib().gcx_wire_layout(arr, len(pieces), wire_off)
    dev_pieces = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).cuda()
    dev_prefix = torch.tensor(prefix, dtype=torch.int32).cuda()
    dev_woff = torch.tensor(list(wire_off), dtype=torch.int64).cuda()
    st = torch.cuda.current_stream().cuda_stream
    msg = torch.zeros(off + 64, dtype=torch.uint8, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    xd = torch.from_numpy(x).cuda()
    _capi.check(_capi.lib().gcx_encode_pieces(dev_pieces.data_ptr(), dev_prefix.data_ptr(),
                                              len(pieces), nt, flags, seed, xd.data_ptr(),
                                              msg.data_ptr(), None, bad.data_ptr(), st))
    wire = torch.zeros(total, dtype=torch.uint8, device="cuda")
    _capi.check(_capi.lib().gcx_frame_pieces(dev_pieces.data_ptr(), dev_woff.data_ptr(),
                                             len(pieces), msg.data_ptr(), seed, 0,
                                             wire.data_ptr(), st))
    torch.cuda.synchronize()
    want = []
    for p in pieces:
        part = x[p.src:p.src + p.len]
        if p.bits == 0:
            want.append(part.view(np.uint8))
        else:
            wn, wp = oracle.quantize(part, p.bits, p.bucket, seed)
            want.append(oracle.serialize(wn, wp, p.len, p.bits, p.bucket, seed))
    want = np.concatenate(want)
    assert want.size == total
    assert (wire.cpu().numpy() == want).all()
    # back to the device layout
    msg2 = torch.zeros_like(msg)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _capi.check(_capi.lib().gcx_unframe_pieces(dev_pieces.data_ptr(), dev_woff.data_ptr(),
                                               len(pieces), wire.data_ptr(), msg2.data_ptr(),
                                               err.data_ptr(), st))
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert torch.equal(msg, msg2)
    # a header whose element count disagrees with the layout is flagged
    k = next(i for i, p in enumerate(pieces) if p.bits)
    bad_wire = wire.clone()
    bad_wire[wire_off[k]] ^= 1
    _capi.check(_capi.lib().gcx_unframe_pieces(dev_pieces.data_ptr(), dev_woff.data_ptr(),
                                               len(pieces), bad_wire.data_ptr(), msg2.data_ptr(),
                                               err.data_ptr(), st))
    torch.cuda.synchronize()
    assert int(err.item()) == 1
