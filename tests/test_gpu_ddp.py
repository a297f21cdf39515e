"""The one-process-per-GPU path (NCCL communicator + DeviceReducer + the
per-rank fused-buffer engine in ddp.py) at world size 1 on the single GPU the
test tier has: it must build its NCCL communicator, piece tables and buffers
for the ResNet-50 layout and behave as the reference's N = 1 allreduce, the
identity (collectives.cpp:479-486).  The N > 1 exchange is proven bit-exact
by test_gpu_sra.py, which drives the same layout and kernels on one GPU."""
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
    red.allreduce(x.data_ptr(), y.data_ptr(), 7, G.ReduceOp.average,
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
