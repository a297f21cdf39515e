"""N > 1 host logic on CPU with torch.distributed gloo (the driver's
multi-process tier): every rank derives the same fused buffers, codecs, SRA
chunk layout and message sizes without talking to the others, the NCCL
unique id travels over the process group the way ddp.make_communicator sends
it, and the byte-level exchange plan every DeviceReducer hands its transport
(sra_exchange_plan: peers, regions, offsets, receive slots, sizes) is
executed over gloo point-to-point with real bytes: each rank's message for
owner c must land in owner c's receive slot for that sender (round 1) and
each owner's aggregate in every rank's gather region (round 2), exactly as
NCCL's grouped send/recv would place them.  The device kernels around the
exchange need a GPU (tests/test_gpu_loopback.py runs the ranks on one B200)."""
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
        plan_ok = _exchange_plan_over_gloo(G, bufs, codecs, rank, world)
        q.put((rank, same, len(set(ids)) == 1 and len(ids[0]) == 128, layouts[0][1], layouts[0][4],
               len(bufs), plan_ok))
    finally:
        dist.destroy_process_group()


def _pattern(sender, owner, rnd, n):
    """The bytes `sender` puts in its round-`rnd` message about chunk `owner`."""
    g = torch.Generator().manual_seed(1_000_003 * rnd + 1009 * sender + owner)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)


def _exchange_plan_over_gloo(G, bufs, codecs, rank, world):
    for fb in bufs:
        segs = [G.Segment(s.buffer_offset, s.length, codecs[s.tensor_index].mode,
                          codecs[s.tensor_index].bits, codecs[s.tensor_index].bucket_size)
                for s in fb.segments]
        P = G.sra_exchange_plan(fb.total_elements, world, rank, segs)
        goff = P["gather_offset"]
        stride = P["recv_stride"]
        regions = {"send": torch.zeros(P["gather_bytes"] + 16, dtype=torch.uint8),
                   "recv": torch.zeros(stride * (world - 1) + 16, dtype=torch.uint8),
                   "gather": torch.zeros(P["gather_bytes"] + 16, dtype=torch.uint8)}
        for rnd in range(2):
            R = P["rounds"][rnd]
            for peer, reg, off, n in R["sends"]:  # what K1 / the owner re-encode wrote
                owner = peer if rnd == 0 else rank
                regions[reg][off:off + n] = _pattern(rank, owner, rnd, n)
            reqs = []
            for peer, reg, off, n in R["sends"]:
                reqs.append(dist.isend(regions[reg][off:off + n].clone(), peer))
            bufs_in = []
            for peer, reg, off, n in R["recvs"]:
                t = torch.empty(n, dtype=torch.uint8)
                reqs.append(dist.irecv(t, peer))
                bufs_in.append((peer, reg, off, n, t))
            for r in reqs:
                r.wait()
            for peer, reg, off, n, t in bufs_in:
                regions[reg][off:off + n] = t
            for peer, reg, off, n, _ in bufs_in:
                if rnd == 0:  # sender `peer`'s share of my chunk, in its slot
                    slot = peer if peer < rank else peer - 1
                    if reg != "recv" or off != slot * stride:
                        return False
                    want = _pattern(peer, rank, 0, n)
                else:  # owner `peer`'s aggregate at its gather offset
                    if reg != "gather" or off != goff[peer]:
                        return False
                    want = _pattern(peer, peer, 1, n)
                if not torch.equal(regions[reg][off:off + n], want):
                    return False
            dist.barrier()
    return True


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_agree_on_layout_id_and_exchange_plan(world):
    port = 29500 + (os.getpid() % 1000) + 7 * world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, id_ok, bounds, sent, nbuf, plan_ok in res:
        assert same and id_ok and plan_ok
        assert nbuf == 2  # ResNet-50 -> 2 fused buffers
        assert bounds[0] == 0 and len(bounds) == world + 1
        assert len(sent) == world and all(b > 0 for b in sent)
