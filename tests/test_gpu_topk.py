"""TopK + error feedback, the reference's sparse codec (codec.cpp:158-214)
and sparse allreduce (collectives.cpp:533-603), on the GPU against the
compiled reference: indices, values, residuals and reduced outputs bit for
bit, including ties (lower index wins), signed zeros and multi-step feedback."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import _gcomm
    return _gcomm


@pytest.fixture(scope="module")
def ref():
    from oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return RefOracle()


def _vec(rng, n):
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3)).astype(np.float32)
    v[rng.random(n) < 0.1] = 0.0
    v[rng.random(n) < 0.05] = np.float32(-0.0)
    dup = rng.random(n) < 0.2  # ties in |acc|
    v[dup] = np.float32(0.5) * np.where(rng.random(dup.sum()) < 0.5, 1, -1)
    return v


def test_topk_compress_with_feedback_matches_reference(g, ref):
    rng = np.random.default_rng(41)
    for trial in range(12):
        n = int(rng.integers(1, 50000))
        k = int(rng.integers(1, n + 1))
        st = g.ErrorFeedbackState(n)
        want_r = np.zeros(n, np.float32)
        for step in range(3):  # residual carried across steps
            v = _vec(rng, n)
            c = g.topk_compress(v, k, st)
            wi, wv, want_r = ref.topk_compress(v, k, want_r)
            assert c.k == k and c.original_length == n
            assert (np.asarray(c.indices) == wi).all(), (trial, step)
            assert (np.asarray(c.values).view(np.uint32) == wv.view(np.uint32)).all()
            assert (np.asarray(st.residual).view(np.uint32) == want_r.view(np.uint32)).all()
            dense = g.topk_decompress(c)
            exp = np.zeros(n, np.float32)
            exp[wi.astype(np.int64)] = wv
            assert (dense.view(np.uint32) == exp.view(np.uint32)).all()


def test_sparse_allreduce_matches_reference(g, ref):
    rng = np.random.default_rng(43)
    for nodes in range(1, 9):
        d = int(rng.integers(1, 20000))
        chunks, pairs = [], []
        for r in range(nodes):
            k = int(rng.integers(1, d + 1))
            st = g.ErrorFeedbackState(d)
            c = g.topk_compress(_vec(rng, d), k, st)
            chunks.append(c)
            pairs.append((np.asarray(c.indices), np.asarray(c.values)))
        for average in (False, True):
            op = g.ReduceOp.average if average else g.ReduceOp.sum
            res = g.sparse_allreduce(chunks, op, nodes)
            want, sent = ref.sparse_allreduce(pairs, d, average)
            for k in range(nodes):
                assert (np.asarray(res.outputs[k]).view(np.uint32) ==
                        want[k].view(np.uint32)).all(), (nodes, average)
            if nodes > 1:
                assert list(res.trace.bytes_sent) == sent


def test_topk_errors_match_reference(g):
    v = np.ones(10, np.float32)
    with pytest.raises(ValueError, match=r"topk k must be in \[1, length\], got 0"):
        g.topk_compress(v, 0, g.ErrorFeedbackState(10))
    with pytest.raises(ValueError, match="got 11"):
        g.topk_compress(v, 11, g.ErrorFeedbackState(10))
    with pytest.raises(ValueError, match="error feedback state length"):
        g.topk_compress(v, 3, g.ErrorFeedbackState(9))
    v[6] = np.inf
    st = g.ErrorFeedbackState(10)
    with pytest.raises(ValueError, match="non-finite gradient value at index 6"):
        g.topk_compress(v, 3, st)
    assert (np.asarray(st.residual) == 0).all()  # state untouched
    c = g.SparseChunk()
    c.original_length, c.k = 5, 2
    c.indices = np.array([3, 1], np.uint64)
    c.values = np.array([1, 2], np.float32)
    with pytest.raises(RuntimeError, match="strictly increasing"):
        g.topk_decompress(c)
