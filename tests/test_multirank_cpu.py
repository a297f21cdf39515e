"""N > 1 host logic on CPU with torch.distributed gloo, world_size 2 (the
driver's multi-process tier): every rank derives the same fused buffers,
codecs, SRA chunk layout and message sizes without talking to the others,
and the NCCL unique id travels over the process group the way
ddp.make_communicator sends it.  The device exchange itself needs GPUs
(tests/test_gpu_sra.py runs all ranks on one B200)."""
import os
import pickle

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_08617_b200 import _gcomm as G
        from paper_2111_08617_b200.ddp import load_layout, resolve_codecs

        layers = load_layout("resnet50")
        codecs = resolve_codecs(layers)
        bufs = G.pack_fused_buffers([n for _, n, _ in layers], 64 << 20)
        layouts = []
        for fb in bufs:
            segs = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                              codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
                    for s in fb.segments]
            L = G.sra_layout(fb.total_elements, world, segs)
            layouts.append((fb.total_elements, L["bounds"], L["msg_bytes"], L["wire_bytes"],
                            L["bytes_sent"], L["pieces"]))
        mine = pickle.dumps(layouts)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        same = all(x == gathered[0] for x in gathered)
        # unique id broadcast (bytes object over the group), as make_communicator does
        uid = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, uid[0])
        q.put((rank, same, len(set(ids)) == 1 and len(ids[0]) == 128, layouts[0][1], layouts[0][4],
               len(bufs)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_agree_on_layout_and_id():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, id_ok, bounds, sent, nbuf in res:
        assert same and id_ok
        assert nbuf == 2  # ResNet-50 -> 2 fused buffers
        assert bounds[0] == 0 and len(bounds) == world + 1
        assert len(sent) == world and all(b > 0 for b in sent)
