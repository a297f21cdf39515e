"""CPU-side tests of the host façade and the C-ABI boundary (no GPU needed).

Mirrors /root/reference/proj/tests/model_test.cpp and the format parts of
codec_test.cpp / collectives_test.cpp; checks that libgcx.so loads and
exports every symbol include/gcx.h declares.
"""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_2111_08617_b200 import _gcomm
    return _gcomm


def test_capi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "gcx.h")).read()
    declared = set(re.findall(r"\b(gcx_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 20
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2111_08617_b200", "libgcx.so"))
    for name in sorted(declared):
        assert hasattr(lib, name), name
    from paper_2111_08617_b200 import _capi
    assert set(_capi.EXPORTS) <= declared


def test_capi_host_helpers(oracle):
    from paper_2111_08617_b200 import _capi
    assert _capi.lib().gcx_version() == 2
    for n, bits, bucket in [(0, 4, 128), (128, 4, 128), (1 << 20, 4, 128), (100, 1, 64),
                            (25_557_032, 4, 128), (7, 8, 3)]:
        assert _capi.compressed_size(n, bits, bucket) == oracle.compressed_size(n, bits, bucket)
    assert _capi.hop_seed(7, 0, 0) == 0xD3855FAC7198D4DA
    assert _capi.hop_seed(7, 1, 3) == 0x095664549895F0FE
    assert _capi.lib().gcx_uniform01(42, 1, 130) == 0.26891814055097596
    # tile planning: one tile per 4096 elements for bucket 128; flags
    nt, prefix, flags = _capi.plan_tiles([_capi.Piece(0, 10000, 0, 0, 0, 128, 4)])
    assert nt == 3 and prefix == [0, 3]
    assert flags == 128 | 256 | (4 << 16) | (7 << 20)  # GCX_F_SPAN_DEC | GCX_F_SPAN_ENC, 4 bits, bucket 2^7
    nt, _, flags = _capi.plan_tiles([_capi.Piece(0, 10000, 0, 0, 0, 1000, 4)])
    # 4000-element tiles x 5 bits = 625 whole words: no zeroing; bucket 1000 takes
    # the generic K1b and the norm pre-pass
    assert flags == _capi.GCX_F_ODD_BUCKETS | _capi.GCX_F_NORM_PASS
    nt, _, flags = _capi.plan_tiles([_capi.Piece(0, 10000, 0, 0, 0, 999, 4)])
    assert flags & _capi.GCX_F_NEEDS_ZERO  # 3996-element tiles x 5 bits straddle words
    _, _, flags = _capi.plan_tiles([_capi.Piece(0, 10000, 0, 0, 0, 5000, 4)])
    assert flags & _capi.GCX_F_BIG_BUCKETS
    with pytest.raises(_capi.GcxError, match=r"bits must be in \[1, 8\]"):
        _capi.plan_tiles([_capi.Piece(0, 10, 0, 0, 0, 128, 9)])


def test_codec_formats(g, oracle):
    """codec_test.cpp:99-143 frozen bytes and sizes."""
    assert g.pack_levels(np.array([1, 0], np.uint32), np.array([0, 1], np.uint8), 1).tobytes() == b"\x09"
    p = g.QuantParams(4, 128, 0)
    assert g.compressed_size_bytes(128, p) == 84
    assert g.compressed_size_bytes(0, p) == 0
    assert g.compressed_size_bytes(1 << 20, p) == 688128
    assert g.compressed_size_bytes(100, g.QuantParams(1, 64, 0)) == (100 * 2 + 7) // 8 + 8
    rng = np.random.default_rng(1)
    for bits in range(1, 9):
        n = int(rng.integers(1, 400))
        lv = rng.integers(0, 1 << bits, n).astype(np.uint32)
        sg = rng.integers(0, 2, n).astype(np.uint8)
        packed = g.pack_levels(lv, sg, bits)
        assert (packed == oracle.pack_levels(lv, sg, bits)).all()
        lv2, sg2 = g.unpack_levels(packed, n, bits)
        assert (lv2 == lv).all() and (sg2 == sg).all()
    with pytest.raises(ValueError):
        g.QuantParams(0, 128, 0).validate()
    with pytest.raises(ValueError):
        g.QuantParams(9, 128, 0).validate()
    with pytest.raises(ValueError):
        g.QuantParams(4, 0, 0).validate()


def test_wire_roundtrip_and_truncation(g, oracle):
    """codec_test.cpp:190-214 on a chunk made by the oracle (no GPU)."""
    v = oracle.normal_vector(300, 8)
    norms, packed = oracle.quantize(v, 5, 64, 77)
    c = g.CompressedChunk()
    c.element_count = 300
    c.params = g.QuantParams(5, 64, 77)
    c.bucket_norms = norms
    c.packed_levels = packed
    wire = g.serialize(c)
    assert len(wire) == g.serialized_size_bytes(300, c.params)
    assert wire == oracle.serialize(norms, packed, 300, 5, 64, 77).tobytes()
    back = g.parse_chunk(wire)
    assert back.element_count == 300 and back.params.bits == 5 and back.params.seed == 77
    assert (back.bucket_norms == norms).all() and (back.packed_levels == packed).all()
    with pytest.raises(RuntimeError):
        g.parse_chunk(wire[:-1])
    with pytest.raises(RuntimeError):
        g.parse_chunk(wire[:10])


def test_filter_rules(g):
    """model_test.cpp: default filter excludes bias, norm and small layers."""
    L = g.LayerKind
    rules = g.FilterRules()
    rules.compile()
    layers = [g.LayerSpec("w", 8192, L.weight), g.LayerSpec("b", 8192, L.bias),
              g.LayerSpec("small_w", 1000, L.weight), g.LayerSpec("ln", 512, L.norm),
              g.LayerSpec("e", 4096, L.embedding)]
    assert [rules.excluded(x) for x in layers] == [False, True, True, True, False]
    r2 = g.FilterRules()
    r2.exclude_patterns = ["^decoder\\."]
    r2.compile()
    assert r2.excluded(g.LayerSpec("decoder.attn.w", 8192, L.weight))
    assert not r2.excluded(g.LayerSpec("encoder.attn.w", 8192, L.weight))
    bad = g.FilterRules()
    bad.exclude_patterns = ["([unterminated"]
    with pytest.raises(ValueError):
        bad.compile()
    r3 = g.FilterRules()
    r3.exclude_patterns = ["x"]
    with pytest.raises(RuntimeError):
        r3.excluded(layers[0])  # used before compile()


def test_plan_json(g):
    """model_test.cpp: plan json roundtrip, resolution, validation."""
    text = json.dumps({"defaults": {"bits": 4, "bucket": 128},
                       "layers": {"w1": {"bits": 2}, "w2": {"mode": "topk", "k": 64},
                                  "w3": {"mode": "uncompressed"}}})
    plan = g.CompressionPlan.from_json(text)
    assert plan.resolve("w1").bits == 2 and plan.resolve("w1").bucket_size == 128
    assert plan.resolve("w2").mode == g.CodecMode.topk and plan.resolve("w2").k == 64
    assert plan.resolve("w3").mode == g.CodecMode.uncompressed
    assert plan.resolve("other").bits == 4
    back = g.CompressionPlan.from_json(plan.to_json())
    assert back.resolve("w2").k == 64 and back.resolve("w1").bits == 2
    with pytest.raises(ValueError):
        g.CompressionPlan.from_json(json.dumps({"defaults": {"bits": 12}}))
    with pytest.raises(ValueError):
        g.CompressionPlan.from_json(json.dumps({"layers": {"x": {"mode": "topk"}}}))


def test_pack_fused_buffers(g):
    """model.cpp:214-256: greedy, oversized tensors split, split tail stays open."""
    MiB = 1 << 20
    el = lambda mib: mib * MiB // 4  # noqa: E731
    bufs = g.pack_fused_buffers([el(10), el(30), el(30), el(100), el(1)], 64 * MiB)
    got = [[(s.tensor_index, s.layer_offset, s.buffer_offset, s.length) for s in b.segments]
           for b in bufs]
    assert got == [
        [(0, 0, 0, el(10)), (1, 0, el(10), el(30))],
        [(2, 0, 0, el(30))],
        [(3, 0, 0, el(64))],
        [(3, el(64), 0, el(36)), (4, 0, el(36), el(1))],
    ]
    with pytest.raises(ValueError):
        g.pack_fused_buffers([0], 64 * MiB)
    with pytest.raises(ValueError):
        g.pack_fused_buffers([1], 3)


def test_chunk_boundaries_and_payloads(g, oracle):
    """collectives_test.cpp:214-232: cuts on the bucket grid; payloads
    101/185/185/254 bytes for d=1000, N=4, 4b/128."""
    segs = [g.Segment(0, 1000, g.CodecMode.quantize, 4, 128)]
    assert g.chunk_boundaries(1000, 4, segs) == [0, 128, 384, 640, 1000]
    sizes = [g.serialized_size_bytes(n, g.QuantParams(4, 128, 0)) for n in (128, 256, 256, 360)]
    assert sizes == [101, 185, 185, 254]
    # mixed layouts against the oracle's restatement
    rng = np.random.default_rng(2)
    for _ in range(50):
        d = int(rng.integers(50, 5000))
        cuts = sorted(set(int(x) for x in rng.integers(1, d, int(rng.integers(0, 6)))))
        edges = [0] + cuts + [d]
        segs, osegs = [], []
        for a, b in zip(edges[:-1], edges[1:]):
            if rng.random() < 0.3:
                segs.append(g.Segment(a, b - a, g.CodecMode.uncompressed, 4, 128))
                osegs.append((a, b - a, 2, 0, 0))
            else:
                bits, bucket = int(rng.integers(1, 9)), int(rng.choice([1, 7, 64, 128, 512]))
                segs.append(g.Segment(a, b - a, g.CodecMode.quantize, bits, bucket))
                osegs.append((a, b - a, 0, bits, bucket))
        for N in (2, 3, 5, 8):
            assert g.chunk_boundaries(d, N, segs) == oracle.chunk_boundaries(d, N, osegs)


def test_hop_seed_and_rounds(g):
    assert g.hop_seed(7, 0, 0) == 0xD3855FAC7198D4DA
    assert len({g.hop_seed(s, h, n) for s in range(3) for h in range(2) for n in range(4)}) == 24
    assert g.latency_rounds(g.Topology.sra, 8) == 2
    assert g.latency_rounds(g.Topology.sra, 1) == 0


def test_compute_entry_points_fail_loudly_without_gpu(g):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        g.quantize(np.ones(10, np.float32), g.QuantParams())


@pytest.mark.parametrize("nodes", [2, 3, 4, 5, 8])
def test_exchange_plans_pair_up_across_ranks(g, nodes):
    """sra_exchange_plan (what DeviceReducer hands its Transport) for every
    rank of a mixed layout: each round's sends and receives pair up one to
    one with equal sizes (NCCL grouped send/recv matching), the round-1
    message from r to owner c is r's copy of chunk c, round 2 carries the
    owner's aggregate, and receive slots never overlap."""
    rng = np.random.default_rng(nodes)
    segs, off = [], 0
    for _ in range(9):
        n = int(rng.integers(1, 40_000))
        if rng.random() < 0.3:
            segs.append(g.Segment(off, n, g.CodecMode.uncompressed, 0, 0))
        else:
            segs.append(g.Segment(off, n, g.CodecMode.quantize, int(rng.integers(1, 9)),
                                  int(rng.choice([32, 64, 128, 512, 100]))))
        off += n
    d = off
    plans = [g.sra_exchange_plan(d, nodes, me, segs) for me in range(nodes)]
    L = g.sra_layout(d, nodes, segs)
    msg = L["msg_bytes"]
    for rnd in range(2):
        sends = {(me, p): (reg, o, n) for me in range(nodes)
                 for p, reg, o, n in plans[me]["rounds"][rnd]["sends"]}
        recvs = {(src, me): (reg, o, n) for me in range(nodes)
                 for src, reg, o, n in plans[me]["rounds"][rnd]["recvs"]}
        assert set(sends) == set(recvs)
        for (a, b), (reg, o, n) in sends.items():
            assert recvs[(a, b)][2] == n
            owner = b if rnd == 0 else a
            assert n == msg[owner]
            assert reg == ("send" if rnd == 0 else "gather")
            assert o == plans[a]["gather_offset"][owner]
        for me in range(nodes):
            slots = sorted(o for _, reg, o, _ in plans[me]["rounds"][0]["recvs"])
            assert all(reg == "recv" for _, reg, _, _ in plans[me]["rounds"][0]["recvs"])
            stride = plans[me]["recv_stride"]
            assert slots == [k * stride for k in range(len(slots))]
            assert stride >= msg[me]
