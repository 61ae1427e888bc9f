"""Cross-GPU KV migration over NCCL (two processes, one GPU each).  Skipped when fewer than 2
GPUs are visible (gpurun and the driver's round-end tests use one; an 8-GPU box runs it).

Both ranks send a node to each other in ONE halo_migrate_exchange call (the send-send pair that
deadlocks with ungrouped per-chunk ncclSend/ncclRecv), then a MOVE with the one-sided
halo_migrate_send / halo_migrate_recv.  Every received node must be bit-exact
(§3.3; north_star "migrated KV blocks must match bit-exactly").
"""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    try:
        import torch.distributed as dist

        import paper_2509_02121_b200 as halo
        from synth import make_config
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        obj = [halo.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        wls = [make_config("fanout", nreq=1, prefix=1000 + 1000 * r, layers=4, seed=50 + r)
               for r in range(world)]
        mine, peer = wls[rank], wls[1 - rank]
        pool = halo.Pool(4, 8, 32, 128, 4096, rank)
        k, v = mine.node_kv(0, f"cuda:{rank}")
        node = pool.register_prefix(-1, mine.nodes[0].ntok, k, v)
        pool.comm_init(obj[0], world, rank, chunk_bytes=4 << 20)
        (got,) = pool.migrate_exchange(sends=[(node, 1 - rank, 1)],
                                       recvs=[(1 - rank, -1, peer.nodes[0].ntok)])
        pk, pv = peer.node_kv(0, f"cuda:{rank}")
        ko, vo = torch.empty_like(pk), torch.empty_like(pv)
        pool.read_prefix(got, ko, vo)
        torch.cuda.synchronize()
        ok = torch.equal(ko.view(torch.int16), pk.view(torch.int16)) and \
            torch.equal(vo.view(torch.int16), pv.view(torch.int16))
        # rank 0 MOVEs its node to rank 1 (one-sided calls)
        if rank == 0:
            pool.migrate_send(node, 1, 0)
            torch.cuda.synchronize()
            try:
                pool.node_info(node)
                ok = False
            except halo.HaloError:
                pass
        else:
            got2 = pool.migrate_recv(0, -1, peer.nodes[0].ntok)
            pool.read_prefix(got2, ko, vo)
            torch.cuda.synchronize()
            ok = ok and torch.equal(ko.view(torch.int16), pk.view(torch.int16)) and \
                torch.equal(vo.view(torch.int16), pv.view(torch.int16))
        dist.barrier()
        pool.destroy()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:  # report to the parent instead of hanging it
        q.put((rank, False, repr(e)))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_rank_nccl_exchange_is_bit_exact():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, (rank, err)
