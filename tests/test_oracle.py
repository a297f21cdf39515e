"""The oracle restatement pinned against the reference: SURVEY Appendix A
known answers, golden fixtures made by the compiled reference, and (when
oracle/_ref exists) the compiled reference directly."""
import json
import os

import numpy as np
import pytest

from tests.golden_inputs import make_input, mix64 as np_mix64

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_appendix_a_rng(oracle):
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert oracle.mix64(1) == 0x910A2DEC89025CC1
    assert oracle.hash_combine(1, 2) == 0xE06DD043328BD285
    assert oracle.uniform01(42, 0, 0) == 0.28203516835164866
    assert oracle.uniform01(42, 1, 130) == 0.26891814055097596
    assert oracle.hop_seed(7, 0, 0) == 0xD3855FAC7198D4DA
    assert oracle.hop_seed(7, 1, 3) == 0x095664549895F0FE
    assert np.float32(oracle.normal01(0x5EED, 0)) == np.float32(-0.2402201)
    assert np.float32(oracle.normal01(0x5EED, 1)) == np.float32(0.846494317)
    assert int(np_mix64(np.uint64(1))) == 0x910A2DEC89025CC1


def test_appendix_a_codec(oracle):
    v = np.array([oracle.normal01(123, i) for i in range(20)], np.float32)
    norms, packed = oracle.quantize(v, 4, 8, 1)
    assert packed.tobytes().hex() == "51ae007224719a33a71a26050d"
    assert [float(x).hex() for x in norms] == ["0x1.a092a20000000p+1", "0x1.2e8cb60000000p+1",
                                                "0x1.37b60a0000000p+0"]
    wire = oracle.serialize(norms, packed, 20, 4, 8, 1)
    assert wire.tobytes().hex() == ("1400000004080000000100000000000000514950405b46174005db9b"
                                    "3f51ae007224719a33a71a26050d")
    w = np.array([oracle.normal01(5, i) for i in range(300)], np.float32)
    want = {1: 0x443A645751F4B93F, 2: 0xFADD9C68827F7659, 3: 0xC0A49B30E95A0E29,
            5: 0x9CE860EF8C247B25, 8: 0x46D793339A9983B9}
    for bits, h in want.items():
        norms, packed = oracle.quantize(w, bits, 128, 99)
        assert oracle.fnv1a64(packed) == h
        assert float(norms[0]).hex() == "0x1.585a120000000p+3"


def test_frozen_pack_and_sizes(oracle):
    """proj/tests/codec_test.cpp:99-106, :130-143"""
    assert oracle.pack_levels([1, 0], [0, 1], 1).tobytes() == b"\x09"
    assert oracle.compressed_size(128, 4, 128) == 84
    assert oracle.compressed_size(0, 4, 128) == 0
    assert oracle.compressed_size(1 << 20, 4, 128) == 688128
    assert oracle.compressed_size(100, 1, 64) == (100 * 2 + 7) // 8 + 8


def _codec_cases():
    with open(os.path.join(GOLD, "codec.json")) as f:
        return json.load(f)["cases"]


def _sra_cases():
    with open(os.path.join(GOLD, "sra.json")) as f:
        return json.load(f)["cases"]


def test_golden_inputs_regenerate_bitwise(oracle):
    for c in _codec_cases():
        v = make_input(c["n"], c["gen"])
        assert oracle.fnv1a64(v) == c["input_fnv"], c


def test_oracle_matches_golden_codec(oracle):
    for c in _codec_cases():
        v = make_input(c["n"], c["gen"])
        norms, packed = oracle.quantize(v, c["bits"], c["bucket"], c["seed"])
        assert oracle.fnv1a64(norms) == c["norms_fnv"], c
        assert oracle.fnv1a64(packed) == c["packed_fnv"], c
        deq = oracle.dequantize(norms, packed, c["n"], c["bits"], c["bucket"])
        assert oracle.fnv1a64(deq) == c["deq_fnv"], c
        wire = oracle.serialize(norms, packed, c["n"], c["bits"], c["bucket"], c["seed"])
        assert oracle.fnv1a64(wire) == c["wire_fnv"], c


def test_oracle_matches_golden_sra(oracle):
    for c in _sra_cases():
        inputs = [make_input(c["d"], dict(c["gen"], seed=c["gen"]["seed"] + r))
                  for r in range(c["nodes"])]
        segs = [tuple(s) for s in c["segments"]]
        out = oracle.sra_allreduce(inputs, segs, c["step_seed"], c["average"])
        assert oracle.fnv1a64(out) == c["out_fnv"], c
        for me in range(c["nodes"]):
            assert oracle.sra_bytes_sent(me, c["nodes"], c["d"], segs) == c["bytes_sent"][me]


def test_sra_stage_counters_reference():
    """proj/tests/collectives_test.cpp:283-317 pins (N=8, d=2048): compress 64,
    decompress 120, messages 112, rounds 2; checked in the golden fixture of
    the compiled reference for the single-segment layouts."""
    for c in _sra_cases():
        if c["nodes"] == 8 and len(c["segments"]) == 1 and c["segments"][0][2] == 0:
            ctr = c["counters"]
            assert ctr["compress_calls"] == 8 * 7 + 8
            assert ctr["decompress_calls"] == 8 * 7 + 8 * 8
            assert ctr["message_count"] == 112 and ctr["rounds"] == 2


def test_oracle_rejects_non_finite(oracle):
    v = np.array([1.0, np.inf], np.float32)
    with pytest.raises(ValueError, match="index 1"):
        oracle.quantize(v, 4, 128, 0)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "oracle", "_ref", "libgcomm_ref.so")),
    reason="compiled reference not built")
def test_oracle_matches_compiled_reference(oracle):
    from oracle import RefOracle
    ref = RefOracle()
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(1, 5000))
        bits = int(rng.integers(1, 9))
        bucket = int(rng.choice([1, 3, 8, 64, 100, 128, 512, 1024, 4096]))
        v = (rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20)).astype(np.float32)
        v[rng.random(n) < 0.05] = 0.0
        seed = int(rng.integers(0, 2**63))
        a = oracle.quantize(v, bits, bucket, seed)
        b = ref.quantize(v, bits, bucket, seed)
        assert (a[0].view(np.uint32) == b[0].view(np.uint32)).all()
        assert (a[1] == b[1]).all()
