"""NEXT-1 execution across processes (CPU, gloo, world_size 3, 127.0.0.1): every rank runs
the same relocation planner call (halo_place_groups, Alg. 1) on the same inputs,
turns the move list into its own send / recv sequence (relocation.rank_actions) and executes
it with BLOCKING point-to-point transfers of each group's KV payload -- the host-side analogue
of halo_migrate_send / halo_migrate_recv over NCCL.  Checks: all ranks derive the same plan;
the transfers drain without deadlock even when moves form a cycle between ranks; afterwards
every rank holds exactly the groups the planner placed on it, bit-exact, and a MOVE source
has dropped its copy."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_02121_b200 import build as halo_build

WORLD = 3
# groups 0-2 live on rank 0, 3 on rank 1, 4-5 on rank 2; the e_v make the planner spread
# them, and the large kv_bytes on rank 2's groups keep those home (moves run both ways)
ITEMS = [{"exec_s": 9.0, "kv_bytes": 1e9, "home": 0}, {"exec_s": 8.0, "kv_bytes": 1e9, "home": 0},
         {"exec_s": 7.0, "kv_bytes": 1e9, "home": 0}, {"exec_s": 2.0, "kv_bytes": 1e9, "home": 1},
         {"exec_s": 6.0, "kv_bytes": 1e9, "home": 2}, {"exec_s": 1.0, "kv_bytes": 1e9, "home": 2},
         {"exec_s": 4.0, "kv_bytes": 2e9, "home": 1, "max_replicas": 3}]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def payload(item):
    """The group's 'KV': a deterministic int32 tensor (bit-exactness is checked)."""
    g = torch.Generator().manual_seed(1000 + item)
    return torch.randint(-2**31, 2**31 - 1, (4096 + 17 * item,), dtype=torch.int32, generator=g)


def _worker(rank, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import paper_2509_02121_b200 as halo
        from paper_2509_02121_b200.relocation import rank_actions
        halo.load_library()
        res = halo.place_groups(ITEMS, WORLD, beam_width=64, link_bytes_per_s=1e10)
        held = {i: payload(i) for i, it in enumerate(ITEMS) if it["home"] == rank}
        for kind, item, *rest in rank_actions(res["moves"], rank):
            if kind == "send":
                dst, mode = rest
                dist.send(held[item], dst=dst)
                if mode == 0:
                    del held[item]
            elif kind == "recv":
                buf = torch.empty_like(payload(item))
                dist.recv(buf, src=rest[0])
                held[item] = buf
        exact = all(torch.equal(v, payload(i)) for i, v in held.items())
        plans = [None] * WORLD
        dist.all_gather_object(plans, (res["masks"], res["moves"]))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, {"held": sorted(held), "exact": exact, "plans": plans, "masks": res["masks"],
                      "moves": res["moves"]}))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.fixture(scope="module")
def results():
    halo_build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    errs = {r: v for r, v in res.items() if isinstance(v, str)}
    assert not errs, errs
    return res


def test_every_rank_derives_the_same_plan(results):
    plans = results[0]["plans"]
    assert all(p == plans[0] for p in plans)
    assert len(results[0]["moves"]) > 0


def test_moves_execute_without_deadlock_and_land_bit_exact(results):
    masks = results[0]["masks"]
    for r in range(WORLD):
        want = sorted(i for i, m in enumerate(masks) if m >> r & 1)
        assert results[r]["held"] == want, (r, results[r]["held"], want)
        assert results[r]["exact"]


def test_moves_run_in_both_directions(results):
    moves = results[0]["moves"]
    pairs = {(m[1], m[2]) for m in moves if m[1] >= 0}
    # at least two distinct sources, so ranks both send and receive
    assert len({p[0] for p in pairs}) >= 2 or len({p[1] for p in pairs}) >= 2, pairs
