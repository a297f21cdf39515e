"""SRA allreduce parity on the GPU: the C++ façade's
collectives.allreduce (all nodes on one B200, K1 -> exchange -> K2 -> K3)
against the reference's run_sra, bit for bit, plus the reference's own
collectives_test.cpp properties."""
import json
import os

import numpy as np
import pytest

from tests.golden_inputs import make_input

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import _gcomm
    return _gcomm


MODES = {0: "quantize", 1: "topk", 2: "uncompressed"}


def _segments(g, segs):
    return [g.Segment(o, ln, getattr(g.CodecMode, MODES[m]), b or 4, bk or 128)
            for o, ln, m, b, bk in segs]


def _request(g, inputs, segs, step_seed, average):
    req = g.ReduceRequest()
    req.inputs = inputs
    req.segments = _segments(g, segs)
    req.op = g.ReduceOp.average if average else g.ReduceOp.sum
    req.step_seed = step_seed
    return req


def test_golden_sra_cases_bit_exact(g, oracle):
    with open(os.path.join(GOLD, "sra.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        inputs = [make_input(c["d"], dict(c["gen"], seed=c["gen"]["seed"] + r))
                  for r in range(c["nodes"])]
        res = g.allreduce(_request(g, inputs, c["segments"], c["step_seed"], c["average"]),
                          c["nodes"])
        outs = res.outputs
        assert len(outs) == c["nodes"]
        for o in outs:
            assert oracle.fnv1a64(o) == c["out_fnv"], c
        tr = res.trace
        assert list(tr.bytes_sent) == c["bytes_sent"], c
        ctr = c["counters"]
        assert tr.compress_calls == ctr["compress_calls"], c
        assert tr.decompress_calls == ctr["decompress_calls"], c
        assert tr.message_count == ctr["message_count"] and tr.rounds == ctr["rounds"]
        assert tr.max_compress_depth == ctr["max_compress_depth"], c


@pytest.mark.parametrize("nodes,want,sent", [(2, 0x948B0C51B738C804, 16_771_839),
                                             (4, 0xA4B0888C9775EAD6, 25_157_795),
                                             (8, 0x438C19827F791EE3, 29_350_875)])
def test_appendix_a_full_size_sra(g, oracle, nodes, want, sent):
    """single-segment 4b/128 SRA average of 25,557,032
    floats, step_seed 7, input[r] = 1e-3*normal01(hash_combine(0xa11, r), i)."""
    d = 25_557_032
    inputs = [oracle.normal_vector(d, oracle.hash_combine(0xA11, r), 1e-3) for r in range(nodes)]
    res = g.allreduce(_request(g, inputs, [(0, d, 0, 4, 128)], 7, True), nodes)
    for o in res.outputs:
        assert oracle.fnv1a64(o) == want
    assert res.trace.bytes_sent[0] == sent


def test_random_layouts_vs_oracle(g, oracle):
    rng = np.random.default_rng(11)
    for trial in range(25):
        nodes = int(rng.integers(2, 9))
        d = int(rng.integers(1, 30000))
        cuts = sorted(set(int(x) for x in rng.integers(1, max(2, d), int(rng.integers(0, 6)))))
        edges = [0] + [x for x in cuts if 0 < x < d] + [d]
        segs = []
        for a, b in zip(edges[:-1], edges[1:]):
            if rng.random() < 0.25:
                segs.append((a, b - a, 2, 0, 0))
            else:
                segs.append((a, b - a, 0, int(rng.integers(1, 9)),
                             int(rng.choice([1, 3, 32, 64, 100, 128, 512, 1024, 5000]))))
        inputs = [(rng.standard_normal(d) * 10.0 ** rng.integers(-3, 3)).astype(np.float32)
                  for _ in range(nodes)]
        step_seed = int(rng.integers(0, 2**63))
        average = bool(rng.random() < 0.7)
        want = oracle.sra_allreduce(inputs, segs, step_seed, average)
        res = g.allreduce(_request(g, inputs, segs, step_seed, average), nodes)
        for o in res.outputs:
            assert (o.view(np.uint32) == want.view(np.uint32)).all(), (trial, nodes, d, segs)


def test_lossless_matches_ordered_sum(g, oracle):
    """collectives_test.cpp:112-135 on integer-valued inputs (exact in any order)."""
    for nodes in (2, 4, 8):
        for d in (5, 64, 1000):
            inputs = [np.round(8.0 * oracle.normal_vector(d, 0x5EED + nodes * 131 + d + k))
                      .astype(np.float32) for k in range(nodes)]
            want = inputs[0].copy()
            for x in inputs[1:]:
                want += x
            res = g.allreduce(_request(g, inputs, [(0, d, 2, 0, 0)], 99, False), nodes)
            for o in res.outputs:
                assert (o == want).all()


def test_single_node_identity(g):
    """collectives_test.cpp:98-110: N=1 returns inputs untouched, no traffic."""
    x = np.array([1.5, -2.25, 0.0, 7.0], np.float32)
    res = g.allreduce(_request(g, [x], [(0, 4, 0, 4, 128)], 0, True), 1)
    assert (res.outputs[0] == x).all()
    assert res.trace.total_bytes_sent() == 0 and res.trace.rounds == 0


def test_mixed_segments_keep_plain_region_exact(g, oracle):
    """collectives_test.cpp:338-367: uncompressed segments equal the lossless fold."""
    nodes, d = 5, 6000
    inputs = [oracle.normal_vector(d, 300 + k) for k in range(nodes)]
    segs = [(0, 2000, 0, 3, 64), (2000, 1500, 2, 0, 0), (3500, 2500, 0, 6, 512)]
    res = g.allreduce(_request(g, inputs, segs, 5, True), nodes)
    exact = oracle.lossless_reference(inputs, segs, True)
    for o in res.outputs:
        assert (o[2000:3500] == exact[2000:3500]).all()
        assert not (o[:2000] == exact[:2000]).all()


def test_malformed_requests_rejected(g):
    """collectives_test.cpp:421-452: same exception types and messages."""
    x = [np.zeros(10, np.float32)] * 2
    with pytest.raises(ValueError, match="one input buffer per node"):
        g.allreduce(_request(g, x, [(0, 10, 2, 0, 0)], 0, False), 3)
    with pytest.raises(ValueError, match="contiguously"):
        g.allreduce(_request(g, x, [(1, 9, 2, 0, 0)], 0, False), 2)
    with pytest.raises(ValueError, match="cover 8 elements but buffers hold 10"):
        g.allreduce(_request(g, x, [(0, 8, 2, 0, 0)], 0, False), 2)
    with pytest.raises(ValueError, match="sparse path"):
        g.allreduce(_request(g, x, [(0, 10, 1, 4, 128)], 0, False), 2)
    with pytest.raises(ValueError, match="zero-length"):
        g.allreduce(_request(g, x, [(0, 0, 2, 0, 0), (0, 10, 2, 0, 0)], 0, False), 2)
    bad = [np.zeros(10, np.float32), np.zeros(10, np.float32)]
    bad[1][3] = np.nan
    with pytest.raises(ValueError, match="non-finite gradient value at index 3"):
        g.allreduce(_request(g, bad, [(0, 10, 0, 4, 128)], 0, False), 2)


def test_determinism_and_seed_sensitivity(g, oracle):
    """collectives_test.cpp:454-480."""
    nodes, d = 4, 4096
    inputs = [oracle.normal_vector(d, 40 + k) for k in range(nodes)]
    a = g.allreduce(_request(g, inputs, [(0, d, 0, 4, 128)], 11, True), nodes).outputs[0]
    b = g.allreduce(_request(g, inputs, [(0, d, 0, 4, 128)], 11, True), nodes).outputs[0]
    c = g.allreduce(_request(g, inputs, [(0, d, 0, 4, 128)], 12, True), nodes).outputs[0]
    assert (a == b).all() and not (a == c).all()


@pytest.mark.parametrize("topology", ["ring", "tree"])
def test_ring_and_tree_vs_compiled_reference(g, topology):
    """run_ring / run_tree (collectives.cpp:312-471) on the GPU — every hop's
    re-encode, the f32 folds in the reference's order, the owner/root's single
    broadcast encode — against the compiled reference, bit for bit, with the
    reference's byte, message, call, round and depth counters."""
    from oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    ref = RefOracle()
    rng = np.random.default_rng(23 if topology == "ring" else 29)
    for trial in range(14):
        nodes = [2, 3, 4, 5, 6, 7, 8][trial % 7]
        d = int(rng.integers(1, 20000))
        cuts = sorted(set(int(x) for x in rng.integers(1, max(2, d), int(rng.integers(0, 5)))))
        edges = [0] + [x for x in cuts if 0 < x < d] + [d]
        segs = []
        for a, b in zip(edges[:-1], edges[1:]):
            if rng.random() < 0.25:
                segs.append((a, b - a, 2, 0, 0))
            else:
                segs.append((a, b - a, 0, int(rng.integers(1, 9)),
                             int(rng.choice([1, 7, 32, 64, 128, 512, 1000]))))
        inputs = [(rng.standard_normal(d) * 10.0 ** rng.integers(-3, 3)).astype(np.float32)
                  for _ in range(nodes)]
        step_seed = int(rng.integers(0, 2**63))
        average = bool(rng.random() < 0.7)
        want, sent, ctr = ref.allreduce(inputs, segs, step_seed, average, topology)
        req = _request(g, inputs, segs, step_seed, average)
        req.topology = getattr(g.Topology, topology)
        res = g.allreduce(req, nodes)
        for k, o in enumerate(res.outputs):
            assert (o.view(np.uint32) == want[k].view(np.uint32)).all(), (trial, nodes, d, segs)
        tr = res.trace
        assert list(tr.bytes_sent) == sent, (trial, nodes, segs)
        assert tr.compress_calls == ctr["compress_calls"], (trial, ctr)
        assert tr.decompress_calls == ctr["decompress_calls"], (trial, ctr)
        assert tr.message_count == ctr["message_count"] and tr.rounds == ctr["rounds"], ctr
        assert tr.max_compress_depth == ctr["max_compress_depth"], (trial, ctr)


MIXED = [(2, 128, 70_000), (8, 128, 90_001), (3, 128, 66_000), (0, 0, 5_000), (4, 512, 80_000),
         (5, 128, 70_000), (4, 128, 100), (6, 64, 70_000), (1, 1024, 70_000), (4, 128, 75_000),
         (2, 128, 600_000)]


def mixed_segments(classes):
    segs, off = [], 0
    for bits, bucket, n in classes:
        segs.append((off, n, 2 if bits == 0 else 0, bits, bucket))
        off += n
    return segs, off


@pytest.mark.parametrize("nodes", [2, 3, 8])
def test_mixed_width_layout_vs_oracle(g, oracle, nodes):
    """A 1.3 M-element layout mixing (bits, bucket) classes the way the
    adaptive planner's per-layer widths do (plus raw and a 100-element
    piece): the oracle's SRA, bit for bit."""
    rng = np.random.default_rng(nodes)
    segs, d = mixed_segments(MIXED)
    inputs = [(rng.standard_normal(d) * 1e-3).astype(np.float32) for _ in range(nodes)]
    want = oracle.sra_allreduce(inputs, segs, 0xC4, True)
    res = g.allreduce(_request(g, inputs, segs, 0xC4, True), nodes)
    for o in res.outputs:
        assert (o.view(np.uint32) == want.view(np.uint32)).all()
