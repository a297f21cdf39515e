"""Graph-replayable SRA steps: device-resident step seeds (GCX_F_SEED_DEVICE,
gcx_sra_step_seeds, DeviceReducer.use_device_seeds).

A step captured in a CUDA graph replays its kernels with the arguments of
the capture, so the per-step seeds (engine.cpp:208-209 step seed, hop seeds
collectives.cpp:252-253 / :283) must come from device memory: a one-thread
kernel derives them from a device-resident step counter and advances it.
These tests pin (1) that kernel against the host hash chain, (2) a captured
span-table K1 replayed three times against eager encodes with the host
seeds of consecutive steps, and (3) the production per-rank path in
device-seed mode against the compiled reference Engine's digests (the same
golden cases as tests/test_gpu_loopback.py).  Capturing a whole multi-rank
step needs the NCCL transport (the loopback's rounds are host rendezvous),
so on one GPU the exchange itself is not captured.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import _gcomm
    return _gcomm


def _host_hop_seed(oracle, base, step, buf, hop, node):
    s = oracle.hash_combine(oracle.hash_combine(base, step), buf)
    return oracle.hash_combine(s, oracle.hash_combine(hop, node))


def test_step_seeds_kernel_matches_host_chain(G, oracle):
    import torch

    from paper_2111_08617_b200 import _capi
    base, step, buf, me = 0x1234_5678_9ABC, 41, 3, 5
    state = torch.tensor([base, step, buf, me, 0, 0], dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for k in range(3):
        _capi.check(_capi.lib().gcx_sra_step_seeds(state.data_ptr(), st))
        h = [int(v) & (2**64 - 1) for v in state.cpu().tolist()]
        assert h[1] == step + k + 1
        for hop in (0, 1):
            want = _host_hop_seed(oracle, base, step + k, buf, hop, me)
            assert h[4 + hop] == want
            # the C-ABI's host hop seed agrees
            s = oracle.hash_combine(oracle.hash_combine(base, step + k), buf)
            assert _capi.lib().gcx_hop_seed(s, hop, me) == want


def _span_table(rng, lens, bits=4, bucket=128):
    from paper_2111_08617_b200 import _capi
    pieces, off, src = [], 0, 0
    for n in lens:
        nb = (n + bucket - 1) // bucket
        norms = off
        packed = (off + 4 * nb + 15) // 16 * 16
        off = (packed + _capi.packed_capacity(n, bits) + 15) // 16 * 16
        pieces.append(_capi.Piece(src, n, norms, packed, 0, bucket, bits))
        src += n
    return pieces, off, src


@pytest.mark.parametrize("lens", [[5000, 4096, 777, 12000],           # CTA-per-tile K1
                                  [400_000, 1_000_000, 3, 250_001]],  # k_span_pieces
                         ids=["short", "long"])
def test_graph_replay_span_encode_draws_fresh_seeds(G, oracle, lens):
    import torch

    from paper_2111_08617_b200 import _capi
    rng = np.random.default_rng(len(lens) + lens[0])
    pieces, msg_bytes, n = _span_table(rng, lens)
    nt, prefix, flags = _capi.plan_tiles(pieces)
    assert flags & _capi.GCX_F_SPAN_ENC
    arr = (_capi.Piece * len(pieces))(*pieces)
    dev_pieces = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).cuda()
    dev_prefix = torch.tensor(prefix, dtype=torch.int32).cuda()
    x = torch.from_numpy((rng.standard_normal(n) * 1e-3).astype(np.float32)).cuda()
    base, step0, buf, me = 77, 10, 1, 2
    state = torch.tensor([base, step0, buf, me, 0, 0], dtype=torch.int64, device="cuda")
    msg = torch.zeros(msg_bytes + 64, dtype=torch.uint8, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    lib = _capi.lib()

    def encode(st, seed, fl):
        _capi.check(lib.gcx_encode_pieces(dev_pieces.data_ptr(), dev_prefix.data_ptr(),
                                          len(pieces), nt, fl, seed, x.data_ptr(),
                                          msg.data_ptr(), None, bad.data_ptr(), st))

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up (kernel attributes) outside the capture
        encode(s.cuda_stream, 1, flags)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = torch.cuda.current_stream().cuda_stream
        _capi.check(lib.gcx_sra_step_seeds(state.data_ptr(), st))
        encode(st, state.data_ptr() + 4 * 8, flags | _capi.GCX_F_SEED_DEVICE)
    for k in range(3):
        msg.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = msg.cpu().numpy().copy()
        seed = _host_hop_seed(oracle, base, step0 + k, buf, 0, me)
        msg.zero_()
        encode(torch.cuda.current_stream().cuda_stream, seed, flags)
        torch.cuda.synchronize()
        want = msg.cpu().numpy()
        assert (got == want).all(), f"replay {k}"
        assert int(bad.item()) == -1
        if k == 0:  # and the oracle on the shortest piece
            p = min(pieces, key=lambda q: q.len)
            wn, wp = oracle.quantize(x.cpu().numpy()[p.src:p.src + p.len], p.bits, p.bucket,
                                     seed)
            assert (got[p.packed:p.packed + wp.size] == wp).all()
    assert int(state[1].item()) == step0 + 3


def test_device_seeds_reject_non_span_tables(G):
    import torch  # noqa: F401
    hub = G.LoopbackHub(2)
    # both chunks mix two widths: no table is a span table
    mixed = [G.Segment(k * 2048, 2048, G.CodecMode.quantize, 4 if k % 2 == 0 else 8, 128)
             for k in range(4)]
    red = G.DeviceReducer(hub.transport(0), 8192, mixed)
    with pytest.raises(ValueError, match="span tables"):
        red.use_device_seeds(1, 0, 0)


def test_device_seeds_per_rank_matches_reference_engine(G, oracle):
    """ResNet-50 (C2), N = 2 and 8, 3 steps: the per-rank path with every
    seed drawn on the device (what a replayed graph runs) gives the compiled
    reference Engine's digests, and the counters end at the next step."""
    import torch

    from oracle import engine_inputs_flat
    from paper_2111_08617_b200.ddp import CompressedAllreduce
    from tests.model_cases import cases, layers
    from tests.test_gpu_loopback import KIND_NAMES, flat_output, golden, run_ranks

    picked = [c for c in cases() if c["model"] == "resnet50" and c["nodes"] in (2, 8)]
    assert picked
    for case in picked:
        ml = layers(case["model"])
        spec = [(name, n, KIND_NAMES[k]) for name, n, k, _ in ml]
        N = case["nodes"]
        plan = G.CompressionPlan.from_json(case["plan"]) if case.get("plan") else None
        hub = G.LoopbackHub(N)

        def rank(r, stream):
            car = CompressedAllreduce(spec, hub.transport(r), plan=plan,
                                      step_seed=case.get("step_seed", 1))
            car.use_device_seeds(0)
            digests = []
            for k in range(case["steps"]):
                x = torch.from_numpy(engine_inputs_flat(oracle, ml, k, case["tag"], r))
                off = 0
                views = car.views()
                for name, n, _, _ in ml:
                    for lo, v in views[name]:
                        v.copy_(x[off + lo: off + lo + v.numel()], non_blocking=False)
                    off += n
                car.allreduce(k)
                car.poll(True)
                digests.append(oracle.fnv1a64(flat_output(car, ml).cpu().numpy()))
            with pytest.raises(ValueError, match="consecutively"):
                car.begin(case["steps"] + 5)
            return digests, car.device_step()

        res = run_ranks(N, rank)
        want = golden(case["name"])["digests"]
        for r, (dig, nxt) in enumerate(res):
            assert dig == want, (case["name"], r)
            assert nxt == case["steps"]
