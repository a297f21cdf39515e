"""The one-process-per-GPU path (NCCL communicator + DeviceReducer + the
per-rank fused-buffer engine in ddp.py) at world size 1 on the single GPU the
test tier has: it must build its NCCL communicator, piece tables and buffers
for the ResNet-50 layout and behave as the reference's N = 1 allreduce, the
identity (collectives.cpp:479-486).  The N > 1 per-rank path is proven
bit-exact by test_gpu_loopback.py (the same reducers over LoopbackTransport)."""
import pytest

pytestmark = pytest.mark.gpu


def test_world1_reducer_is_identity():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2111_08617_b200 import _gcomm as G
    from paper_2111_08617_b200.ddp import CompressedAllreduce, load_layout, make_communicator

    comm = make_communicator(0, 1)
    assert comm.rank() == 0 and comm.size() == 1
    layers = load_layout("resnet50")
    car = CompressedAllreduce(layers, comm)
    assert car.elements == 25_557_032 and len(car.buffers) == 2
    for b in car.flat:
        b.normal_()
    before = [b.clone() for b in car.flat]
    car.allreduce(step=0)
    torch.cuda.synchronize()
    for a, b in zip(before, car.flat):
        assert torch.equal(a, b)
    views = car.views()
    assert sum(v.numel() for parts in views.values() for _, v in parts) == car.elements
    assert car.launches_per_step() == 0  # N = 1: no kernels, no traffic
    red = G.DeviceReducer(comm, 1000, [G.Segment(0, 1000, G.CodecMode.quantize, 4, 128)])
    x = torch.randn(1000, device="cuda")
    y = torch.empty_like(x)
    red.allreduce(x.data_ptr(), y.data_ptr(), 1000, 7, G.ReduceOp.average,
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(x, y)


def test_ddp_comm_hook_world1():
    """CgxCommHook under torch DDP (NCCL process group of one rank): the hook
    runs on every bucket, builds its reducers from the buckets' parameters,
    and at N = 1 leaves the averaged gradients equal to plain autograd's."""
    import os

    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2111_08617_b200.ddp import CgxCommHook, cgx_comm_hook, make_communicator

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29633")
    own_pg = not dist.is_initialized()
    if own_pg:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        torch.manual_seed(0)
        net = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(),
                                  torch.nn.Linear(512, 64)).cuda()
        ref = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(),
                                  torch.nn.Linear(512, 64)).cuda()
        ref.load_state_dict(net.state_dict())
        model = DDP(net, device_ids=[0], bucket_cap_mb=1)
        hook = CgxCommHook(make_communicator(0, 1))
        model.register_comm_hook(hook, cgx_comm_hook)
        x = torch.randn(32, 256, device="cuda")
        for _ in range(2):
            model.zero_grad()
            ref.zero_grad()
            model(x).square().sum().backward()
            ref(x).square().sum().backward()
            torch.cuda.synchronize()
            for a, b in zip(model.module.parameters(), ref.parameters()):
                assert torch.equal(a.grad, b.grad)
        assert hook.calls >= 2 and hook.step == 2
    finally:
        if own_pg:
            dist.destroy_process_group()
