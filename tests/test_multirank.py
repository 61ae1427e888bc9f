"""N>1 host path on CPU: two ranks over gloo (world_size 2, 127.0.0.1).

Covers what bench.py and a multi-GPU deployment do on the host:
request-group placement (LPT over the K1/K2 roofline cost), kv-head ranges, planning each
rank's shard on a host-only pool (device=-1: the library's allocator/tree/planner, no
launches), and the max-over-ranks timing reduction.  The attention path itself has no
exchange step, so the per-rank plans must add up to the unsharded plan's work exactly.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_02121_b200 import sharding
from synth import make_config


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan_totals(wl):
    from paper_2509_02121_b200.loader import append_step, load
    ld = load(wl, device=-1)
    append_step(ld, wl, 0, device=-1)        # the decode step's token (append-then-attend)
    pl = ld.pool.plan(ld.req_ids)
    info = pl.info()
    k2_blocks = len(pl.export("req_blk"))   # paged blocks K2 streams (per kv head)
    pl.destroy()
    ld.pool.destroy()
    return [float(info["k1_flops"]), float(k2_blocks), float(info["k2_units"]),
            float(info["k1_tiles"]), float(info["nreq"])]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = {}
        # request-group sharding of C3 (64 templates over the ranks) and C2 (one tree)
        for name, kw in [("analytics", dict(templates=64, layers=1)), ("tree", dict(layers=1)),
                         ("ragged", {})]:
            wl = make_config(name, **kw)
            mine = sharding.rank_requests(wl, world, rank)
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            shard = sharding.subset_workload(wl, mine)
            tot = sharding.max_over_ranks([0.0], dist)  # exercised with a trivial value
            sums = _plan_totals(shard) if mine else [0.0] * 5
            import torch
            t = torch.tensor(sums, dtype=torch.float64)
            dist.all_reduce(t)
            out[name] = {"gathered": gathered, "sums": t.tolist(), "tot": tot}
        # kv-head sharding of C2 structure: plans on each head slice
        wl = make_config("tree", layers=1)
        hs = sharding.head_shard_workload(wl, world, rank)
        sums = _plan_totals(hs)
        import torch
        t = torch.tensor(sums, dtype=torch.float64)
        dist.all_reduce(t)
        out["heads"] = {"range": sharding.head_range(wl.hkv, world, rank), "sums": t.tolist()}
        out["max"] = sharding.max_over_ranks([float(rank), -float(rank), 3.0], dist)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception:  # surface the failure to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.fixture(scope="module")
def two_rank_results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    errs = {r: v for r, v in res.items() if isinstance(v, str)}
    assert not errs, errs
    return res


def test_request_groups_partition_the_batch(two_rank_results):
    for name, kw in [("analytics", dict(templates=64, layers=1)), ("tree", dict(layers=1)),
                     ("ragged", {})]:
        wl = make_config(name, **kw)
        g = two_rank_results[0][name]["gathered"]
        assert g == two_rank_results[1][name]["gathered"]
        allr = sorted(r for part in g for r in part)
        assert allr == list(range(wl.nreq)), name           # disjoint and complete
        # a prefix subtree never straddles ranks (its K1 tile needs all its requests)
        for nd in wl.nodes:
            users = {i for i, part in enumerate(g) for r in part if nd.ident in wl.path(r)}
            assert len(users) <= 1, (name, nd.ident, users)


def test_lpt_placement_is_balanced():
    wl = make_config("analytics", templates=64, layers=1)
    groups = sharding.subtree_groups(wl)
    for world in (2, 4, 8):
        where = sharding.place_groups([x.cost for x in groups], world)
        load = [sum(x.cost for x, w in zip(groups, where) if w == r) for r in range(world)]
        assert max(load) - min(load) <= max(x.cost for x in groups) + 1e-12
        assert len(set(where)) == world
    # unequal groups: the LPT bound holds
    costs = [7, 5, 4, 4, 3, 3, 2, 1]
    where = sharding.place_groups(costs, 3)
    load = [sum(c for c, w in zip(costs, where) if w == r) for r in range(3)]
    assert max(load) <= sum(costs) / 3 + max(costs)


def test_sharded_plans_add_up_to_the_unsharded_plan(two_rank_results):
    """No exchange on the attention path: every K1 FLOP, K2 byte and unit of the full batch
    is planned on exactly one rank (request groups) or one head slice (kv heads)."""
    for name, kw in [("analytics", dict(templates=64, layers=1)), ("tree", dict(layers=1)),
                     ("ragged", {})]:
        full = _plan_totals(make_config(name, **kw))
        sums = two_rank_results[0][name]["sums"]
        assert sums == two_rank_results[1][name]["sums"]
        assert sums[0] == pytest.approx(full[0], rel=1e-12)     # K1 FLOPs
        assert sums[2] == full[2] and sums[4] == full[4]        # K2 units, requests
        assert sums[1] == full[1]                                # K2 KV blocks
        # (K1 tile counts differ: each plan picks its own split-N to fill the SMs)
    full = _plan_totals(make_config("tree", layers=1))
    hs = two_rank_results[0]["heads"]["sums"]
    assert hs[0] == pytest.approx(full[0], rel=1e-12)
    assert hs[1] == 2 * full[1]           # every rank streams every block, for its heads
    assert hs[2] == full[2]
    assert two_rank_results[0]["heads"]["range"] == (0, 4)
    assert two_rank_results[1]["heads"]["range"] == (4, 8)


def test_max_over_ranks(two_rank_results):
    for r in (0, 1):
        assert two_rank_results[r]["max"] == [1.0, 0.0, 3.0]
    assert sharding.max_over_ranks([2.0, 1.0]) == [2.0, 1.0]   # single process: identity
    with pytest.raises(ValueError):
        sharding.head_range(8, 3, 0)
