"""Relocation planner: halo_place_groups runs PAPER.md Alg. 1 (beam
search with incremental cost, §3.2) with the §3.2 cost functions, and the
migration path executes its moves.

CPU pins of the planner (host logic, no device):
* with a beam wide enough to keep every partial assignment, Alg. 1 is exhaustive: its
  result equals the brute-force minimum of max_d C_a^d over all assignments (enumerated
  here from the cost definition, independently of the library's search);
* w = 1 is the greedy rule (each item in decreasing e_v to the worker that minimises the
  makespan, ties to the lower worker);
* limits: prohibitive relocation cost keeps every homed group home; replication happens
  under conditions (i)/(ii) only, and only when the k^beta speed-up beats the transfers;
* the move list realises the placement (MOVE/COPY), and the per-rank action lists pair up
  in order and cannot deadlock.
GPU: groups relocated between two pools by the planner's moves decode bit-identically to
the same groups on their home pool, and match the fp64 oracle."""
import itertools
import random

import numpy as np
import pytest
import torch

import oracle
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200 import build as halo_build
from paper_2509_02121_b200.relocation import execute_local, group_items, plan_relocation, rank_actions
from synth import make_config


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()


def prep(it, d, link):
    h = it.get("home", -1)
    if h == d:
        return 0.0
    return it.get("kv_bytes", 0.0) / link if h >= 0 else it.get("prep_s", 0.0)


def brute_force(items, D, link):
    """min over all single-worker assignments of max_d sum(e_v + p_v(d))."""
    best = None
    for assign in itertools.product(range(D), repeat=len(items)):
        load = [0.0] * D
        for it, d in zip(items, assign):
            load[d] += it["exec_s"] + prep(it, d, link)
        c = max(load)
        best = c if best is None else min(best, c)
    return best


def rand_items(rng, n, D, homes=True):
    return [{"exec_s": rng.choice([1.0, 2.0, 3.0, 5.0, 8.0]) * rng.uniform(0.5, 1.5),
             "kv_bytes": rng.uniform(0, 4e9), "prep_s": rng.uniform(0, 2.0),
             "home": rng.randrange(-1, D) if homes else -1} for _ in range(n)]


@pytest.mark.parametrize("seed", range(12))
def test_exhaustive_beam_equals_brute_force(seed):
    rng = random.Random(seed)
    D = rng.choice([2, 3])
    n = rng.choice([3, 4, 5, 6])
    link = rng.choice([1e9, 4e9, 1e10])
    items = rand_items(rng, n, D)
    res = halo.place_groups(items, D, beam_width=D ** n, link_bytes_per_s=link)
    bf = brute_force(items, D, link)
    assert res["cost"] == pytest.approx(bf, rel=1e-12)
    # the reported loads are those of the returned assignment
    load = [0.0] * D
    for it, ws in zip(items, res["workers"]):
        assert len(ws) == 1
        load[ws[0]] += it["exec_s"] + prep(it, ws[0], link)
    assert res["load"] == pytest.approx(load, rel=1e-12)
    assert res["cost"] == pytest.approx(max(load), rel=1e-12)
    # several items per iteration (|V_r| > 1) enumerate the same space
    res2 = halo.place_groups(items, D, beam_width=D ** n, ops_per_iter=2, link_bytes_per_s=link)
    assert res2["cost"] == pytest.approx(bf, rel=1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_width_one_is_greedy(seed):
    rng = random.Random(100 + seed)
    D, n, link = 4, 12, 2e9
    items = rand_items(rng, n, D)
    res = halo.place_groups(items, D, beam_width=1, link_bytes_per_s=link)
    order = sorted(range(n), key=lambda i: (-items[i]["exec_s"], i))
    load = [0.0] * D
    want = [None] * n
    for i in order:
        best = None
        for d in range(D):
            trial = list(load)
            trial[d] += items[i]["exec_s"] + prep(items[i], d, link)
            if best is None or max(trial) < best[0]:
                best = (max(trial), d, trial)
        want[i] = best[1]
        load = best[2]
    assert [w[0] for w in res["workers"]] == want
    # a wider beam never does worse than greedy
    wide = halo.place_groups(items, D, beam_width=64, link_bytes_per_s=link)
    assert wide["cost"] <= res["cost"] + 1e-12


def test_prohibitive_link_keeps_groups_home_and_free_link_balances():
    items = [{"exec_s": 4.0, "kv_bytes": 1e9, "home": 0} for _ in range(4)]
    stay = halo.place_groups(items, 2, beam_width=16, link_bytes_per_s=1.0)   # 1e9 s per move
    assert stay["workers"] == [[0]] * 4 and stay["moves"] == []
    assert stay["cost"] == pytest.approx(16.0)
    move = halo.place_groups(items, 2, beam_width=16, link_bytes_per_s=1e12)  # 1 ms per move
    assert sorted(len([w for w in move["workers"] if w == [d]]) for d in range(2)) == [2, 2]
    assert move["cost"] == pytest.approx(8.0 + 2e-3)
    assert all(m[3] == 0 and m[1] == 0 and m[2] == 1 for m in move["moves"])   # MOVE 0 -> 1
    assert len(move["moves"]) == 2


def test_replication_only_when_it_pays():
    big = [{"exec_s": 8.0, "kv_bytes": 1e9, "home": 0, "max_replicas": 4}]
    r = halo.place_groups(big, 4, beam_width=8, beta=1.0, link_bytes_per_s=1e11)
    assert r["workers"] == [[0, 1, 2, 3]]
    assert r["cost"] == pytest.approx(2.0 + 1e9 / 1e11)
    assert sorted(m[2] for m in r["moves"]) == [1, 2, 3] and all(m[3] == 1 for m in r["moves"])
    # beta = 0: replicas give no speed-up, so the transfers are pure loss
    r0 = halo.place_groups(big, 4, beam_width=8, beta=0.0, link_bytes_per_s=1e11)
    assert r0["workers"] == [[0]] and r0["moves"] == []
    # transfers dearer than the saving: 10 s per copy, 8/k + 10 > 8 for every k
    r1 = halo.place_groups(big, 4, beam_width=8, beta=1.0, link_bytes_per_s=1e8)
    assert r1["workers"] == [[0]]
    # condition (i): as many items as workers -> no replication even when it would pay
    four = [dict(big[0]) for _ in range(4)]
    r4 = halo.place_groups(four, 4, beam_width=64, beta=1.0, link_bytes_per_s=1e11)
    assert all(len(w) == 1 for w in r4["workers"])
    # condition (ii): a small item is never replicated
    mix = [dict(big[0]), {"exec_s": 0.5, "kv_bytes": 1e6, "home": 0, "max_replicas": 4}]
    rm = halo.place_groups(mix, 4, beam_width=64, beta=1.0, link_bytes_per_s=1e11)
    assert len(rm["workers"][1]) == 1


def test_moves_realise_the_placement():
    rng = random.Random(7)
    D = 4
    items = rand_items(rng, 10, D)
    for it in items:
        it["max_replicas"] = 3
    res = halo.place_groups(items[:3], D, beam_width=32, link_bytes_per_s=3e9)
    for i, it in enumerate(items[:3]):
        placed = set(res["workers"][i])
        mv = [m for m in res["moves"] if m[0] == i]
        h = it["home"]
        assert {m[2] for m in mv} == placed - {h}
        assert all(m[1] == h for m in mv)
        nmove = sum(m[3] == 0 for m in mv)
        assert nmove == (1 if (h >= 0 and h not in placed) else 0)
        for m in mv:
            assert m[4] == pytest.approx(prep(it, m[2], 3e9))


def test_errors():
    ok = [{"exec_s": 1.0}]
    with pytest.raises(halo.HaloError) as e:
        halo.place_groups(ok, 0)
    assert e.value.name == "HALO_EINVAL"
    for bad in ({"exec_s": -1.0}, {"exec_s": float("nan")}, {"exec_s": 1.0, "home": 5},
                {"exec_s": 1.0, "max_replicas": 0}):
        with pytest.raises(halo.HaloError) as e:
            halo.place_groups([bad], 2)
        assert e.value.name == "HALO_EINVAL"
    with pytest.raises(halo.HaloError) as e:
        halo.place_groups(ok * 3, 2, ops_per_iter=3)
    assert e.value.name == "HALO_EINVAL"
    with pytest.raises(halo.HaloError) as e:         # 2^20 candidate cap
        halo.place_groups(ok * 8, 8, beam_width=1 << 20, ops_per_iter=7)
    assert e.value.name == "HALO_EINVAL"


def _simulate(moves, world):
    """Step every rank through its action list; a transfer completes when both sides sit
    on it.  Returns True if all lists drain (no deadlock)."""
    acts = [rank_actions(moves, r) for r in range(world)]
    pos = [0] * world
    for _ in range(10 * len(moves) + 10):
        progressed = False
        for r in range(world):
            while pos[r] < len(acts[r]) and acts[r][pos[r]][0] == "prepare":
                pos[r] += 1
                progressed = True
            if pos[r] >= len(acts[r]):
                continue
            a = acts[r][pos[r]]
            peer = a[2]
            if pos[peer] < len(acts[peer]):
                b = acts[peer][pos[peer]]
                if a[0] == "send" and b[0] == "recv" and b[1] == a[1] and b[2] == r:
                    pos[r] += 1
                    pos[peer] += 1
                    progressed = True
        if all(pos[r] >= len(acts[r]) for r in range(world)):
            return True
        if not progressed:
            return False
    return False


@pytest.mark.parametrize("seed", range(6))
def test_rank_actions_pair_in_order_and_do_not_deadlock(seed):
    rng = random.Random(seed)
    world = 4
    items = rand_items(rng, 14, world)
    res = halo.place_groups(items, world, beam_width=8, link_bytes_per_s=2e10)
    for a in range(world):
        for b in range(world):
            sends = [x[1] for x in rank_actions(res["moves"], a) if x[0] == "send" and x[2] == b]
            recvs = [x[1] for x in rank_actions(res["moves"], b) if x[0] == "recv" and x[2] == a]
            assert sends == recvs
    assert _simulate(res["moves"], world)
    # an arbitrary interleaving of pairwise transfers in one global order is also safe
    moves = [(i, *rng.sample(range(world), 2), 1, 0.0) for i in range(40)]
    assert _simulate(moves, world)


def test_group_items_follow_the_workload():
    wl = make_config("tree", layers=4, root=512, roles=3, role_tok=128, per_role=20, suffix=31)
    groups, items = group_items(wl, [0], steps=10, fetch_bytes_per_s=5e10)
    assert len(groups) == 1 and len(items) == 1
    kv = (512 + 3 * 128) * wl.hkv * wl.d * 4 * wl.layers
    assert items[0]["kv_bytes"] == kv
    assert items[0]["prep_s"] == pytest.approx(kv / 5e10)
    assert items[0]["exec_s"] == pytest.approx(groups[0].cost * wl.layers * 10)
    wl2 = make_config("analytics", layers=2, templates=6, ctx=256, per_template=8, suffix=15)
    g2, it2 = group_items(wl2, [0] * 6)
    assert len(g2) == 6
    _, _, res = plan_relocation(wl2, [0] * 6, workers=3, link_bytes_per_s=1e12, beam_width=32,
                                steps=10000)   # a long decode horizon: moves are cheap
    assert sorted(len([w for w in res["workers"] if w == [d]]) for d in range(3)) == [2, 2, 2]


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_planner_moves_execute_and_decode_bit_identically():
    """Four templates live on pool 0 (worker 0).  The planner spreads them over two workers
    (pools 0 and 1 on this GPU, relocation = halo_prefix_clone); each group decodes
    bit-identically before and after the move, and matches the oracle."""
    torch.cuda.set_device(0)
    wl = make_config("analytics", layers=2, templates=4, ctx=300, per_template=40, suffix=20)
    from paper_2509_02121_b200.loader import blocks_needed, load
    ld = load(wl, 0)
    p0 = ld.pool
    p1 = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, blocks_needed(wl), 0)
    groups, items, res = plan_relocation(wl, [0] * 4, workers=2, link_bytes_per_s=1e12,
                                         beam_width=16, steps=10000)
    assert sorted(len(w) for w in res["workers"]) == [1, 1, 1, 1]
    assert sum(w == [1] for w in res["workers"]) == 2
    q = wl.q(0, "cuda")
    layer = 1

    def decode(pool, reqs, rows):
        pl = pool.plan(reqs)
        out = torch.empty((len(reqs), wl.hq, wl.d), device="cuda")
        pl.run(layer, q[layer][rows].contiguous(), out)
        torch.cuda.synchronize()
        pl.destroy()
        return out

    sk, sv = wl.suffix_kv("cuda")              # [L][sum S][Hkv][d]
    nk, nv = wl.new_kv(0, "cuda")              # [L][R][Hkv][d]
    off = wl.suffix_offsets

    def open_group(pool, nmap, rows):
        reqs = [pool.open_request(nmap[wl.requests[r].leaf]) for r in rows]
        tok = torch.tensor([t for r in rows for t in range(int(off[r]), int(off[r + 1]))], device="cuda")
        pool.append(reqs, [wl.requests[r].suffix for r in rows], sk.index_select(1, tok).contiguous(),
                    sv.index_select(1, tok).contiguous())
        idx = torch.tensor(rows, device="cuda")
        pool.append(reqs, [1] * len(rows), nk.index_select(1, idx).contiguous(),
                    nv.index_select(1, idx).contiguous())
        return reqs

    for rid in ld.req_ids:
        p0.close_request(rid)
    before = {}
    for gi, g in enumerate(groups):
        rows = list(g.requests)
        reqs = open_group(p0, ld.node_ids, rows)
        before[gi] = decode(p0, reqs, rows)
        for rid in reqs:
            p0.close_request(rid)
    maps = [dict(ld.node_ids), {}]
    execute_local([p0, p1], wl, groups, res["moves"], maps)
    pools = [p0, p1]
    for gi, g in enumerate(groups):
        w = res["workers"][gi][0]
        rows = list(g.requests)
        for n in g.nodes:
            assert n in maps[w] and (w == 0 or n not in maps[0])
        reqs = open_group(pools[w], maps[w], rows)
        after = decode(pools[w], reqs, rows)
        assert torch.equal(before[gi], after), gi
        ro, _ = oracle.decode_reference(wl, layer, steps=1, requests=rows)
        assert np.abs(after.cpu().numpy() - ro).max() <= 2e-3
        for rid in reqs:
            pools[w].close_request(rid)
    p1.destroy()
    p0.destroy()
