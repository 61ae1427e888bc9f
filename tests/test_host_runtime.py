"""CPU tests of the C-ABI library: symbol exports, and the host logic (block allocator,
prefix tree, requests, decode planner) on a host-only pool (device = -1: bookkeeping only,
no device memory and no kernels -- compute calls return HALO_EUNSUPPORTED)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2509_02121_b200 as halo
from paper_2509_02121_b200.abi import SIGNATURES, PlanOptions
from paper_2509_02121_b200 import build as halo_build
from synth import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "halo_attn.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(halo_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(halo.lib_path())
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(SIGNATURES), set(syms) ^ set(SIGNATURES)
    assert lib.halo_abi_version() == 1


def host_pool(layers=2, hkv=2, hq=8, d=128, cap=1000):
    return halo.Pool(layers, hkv, hq, d, cap, device=-1)


def test_pool_config_validation():
    for kw in [dict(hkv=3, hq=8), dict(d=96), dict(hkv=1, hq=16), dict(cap=0)]:
        with pytest.raises(halo.HaloError) as e:
            host_pool(**kw)
        assert e.value.name == "HALO_EINVAL"


def test_allocator_accounting_and_enomem_is_clean():
    p = host_pool(cap=10)
    assert p.stats() == (10, 0)
    a = p.register_prefix(-1, 33)  # 3 blocks
    assert p.stats() == (7, 3)
    r = p.open_request(a)
    p.append([r], [16 * 7])  # 7 blocks -> pool full
    assert p.stats() == (0, 10)
    with pytest.raises(halo.HaloError) as e:
        p.append([r], [1])
    assert e.value.name == "HALO_ENOMEM"
    assert p.request_info(r)["suffix_len"] == 112 and p.stats() == (0, 10)
    with pytest.raises(halo.HaloError):
        p.register_prefix(-1, 1)
    p.truncate([r], [17])
    assert p.request_info(r) == {"leaf": a, "suffix_len": 95, "nblocks": 6}
    assert p.stats() == (1, 9)
    p.close_request(r)
    assert p.stats() == (7, 3)
    p.release_prefix(a)
    assert p.stats() == (10, 0)
    p.destroy()


def test_tree_refcounts_and_errors():
    p = host_pool()
    root = p.register_prefix(-1, 40)
    child = p.register_prefix(root, 20)
    r = p.open_request(child)
    with pytest.raises(halo.HaloError) as e:
        p.release_prefix(root)
    assert e.value.name == "HALO_EBUSY"
    with pytest.raises(halo.HaloError) as e:
        p.release_prefix(child)
    assert e.value.name == "HALO_EBUSY"
    with pytest.raises(halo.HaloError) as e:
        p.open_request(12345)
    assert e.value.name == "HALO_ENOENT"
    with pytest.raises(halo.HaloError) as e:
        p.register_prefix(999, 5)
    assert e.value.name == "HALO_ENOENT"
    info = p.node_info(child)
    assert info["parent"] == root and info["ntok"] == 20 and len(info["blocks"]) == 2
    p.close_request(r)
    p.release_prefix(child)
    p.release_prefix(root)
    ids = {root, child, r}
    assert len(ids) == 3  # ids are unique across kinds
    p.destroy()


def test_append_handles_repeated_ids_and_fresh_suffix_blocks():
    p = host_pool()
    n = p.register_prefix(-1, 7)  # partial block: the suffix must start in a fresh block
    r = p.open_request(n)
    p.append([r, r, r], [5, 11, 1])
    inf = p.request_info(r)
    assert inf["suffix_len"] == 17 and inf["nblocks"] == 2
    assert p.stats()[1] == 3


def plan_of(wl, **opt):
    p = host_pool(wl.layers, wl.hkv, wl.hq, wl.d, cap=100000)
    from paper_2509_02121_b200.loader import load
    ld = load(wl, device=-1, pool=p)
    reqs = ld.req_ids
    # one decode step appends a token to each request
    p.append(reqs, [1] * len(reqs))
    o = PlanOptions(opt.get("min_rows", 0), opt.get("force_splits", 0), opt.get("max_splits", 0),
                    opt.get("chunk", 0))
    o.k2_whole_units = opt.get("whole_units", 0)
    return p, ld, p.plan(reqs, o)


def test_plan_dfs_ranges_are_contiguous_and_tiles_cover_every_row_token_once():
    wl = make_config("ragged")
    for min_rows, fs in [(1, 0), (1, 3), (64, 0), (16, 2)]:
        p, ld, pl = plan_of(wl, min_rows=min_rows, force_splits=fs)
        order = pl.export("req_order")
        assert sorted(order) == list(range(wl.nreq))
        # requests under any node are contiguous in DFS order
        pos = {int(r): i for i, r in enumerate(order)}
        for n in wl.nodes:
            under = [i for i in range(wl.nreq) if n.ident in wl.path(i)]
            if under:
                ps = sorted(pos[i] for i in under)
                assert ps == list(range(ps[0], ps[0] + len(ps)))
        tiles = pl.export("tiles")
        g = wl.g
        covered = {}
        for (req_off, nrows, head, t0, t1, blk_off, slot, node) in tiles:
            assert 0 < nrows <= 256 and t0 % 128 == 0 and t1 > t0
            for row in range(nrows):
                r = int(order[req_off + row // g])
                for t in sorted({int(t0), int(t1) - 1}):
                    key = (r, head * g + row % g, int(slot), t)
                    assert key not in covered
                    covered[key] = True
        nslots = pl.export("req_nslots")
        info = pl.info()
        assert info["max_slots"] == (max(nslots) if len(nslots) else 0)
        # K2 blocks per request = folded nodes' blocks + suffix blocks, counts add up
        off = pl.export("req_blk_off")
        blk = pl.export("req_blk")
        slot_tokens = {}
        for (req_off, nrows, head, t0, t1, blk_off, slot, node) in tiles:
            for row in range(nrows):
                r = int(order[req_off + row // g])
                slot_tokens[(r, int(slot))] = slot_tokens.get((r, int(slot)), 0) + 0
        for i in range(wl.nreq):
            cnt = sum(int((e >> 27) + 1) for e in blk[off[i]:off[i + 1]])
            k1_tok = 0
            for (req_off, nrows, head, t0, t1, blk_off, slot, node) in tiles:
                if head != 0:
                    continue
                rows_req = {int(order[req_off + row // g]) for row in range(nrows)}
                if i in rows_req:
                    k1_tok += t1 - t0
            assert cnt + k1_tok == wl.context_len(i, steps=1), (i, cnt, k1_tok)
            assert nslots[i] <= info["max_slots"]
        pl.destroy()
        p.destroy()


def test_plan_rejects_empty_context_and_unknown_ids():
    p = host_pool()
    r = p.open_request(-1)
    with pytest.raises(halo.HaloError) as e:
        p.plan([r])
    assert e.value.name == "HALO_EINVAL"
    with pytest.raises(halo.HaloError) as e:
        p.plan([777])
    assert e.value.name == "HALO_ENOENT"


def test_plan_split_choice_fills_the_sms():
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=15)
    p, ld, pl = plan_of(wl)
    info = pl.info()
    assert info["tensor_nodes"] == 1 and info["folded_nodes"] == 0
    assert 100 <= info["k1_tiles"] <= 296
    assert info["k1_flops"] == 4.0 * 256 * 4 * 2048 * 128 * 8
    # compute on a host-only pool is refused, not emulated
    with pytest.raises(halo.HaloError) as e:
        pl.run(0, 1, 1)
    assert e.value.name == "HALO_EUNSUPPORTED"
    with pytest.raises(halo.HaloError):
        p.destroy()  # plan still alive -> EBUSY
    pl.destroy()
    p.destroy()


def test_plan_rebuild_in_place():
    wl = make_config("ragged")
    p, ld, pl = plan_of(wl, min_rows=1)
    pl2 = p.plan(ld.req_ids[:5], reuse=pl)
    assert pl2 is pl and pl.info()["nreq"] == 5
    pl.destroy()


@pytest.mark.parametrize("cfg,kw,cb", [("ragged", {}, 0), ("ragged", {}, 3),
                                       ("ragged_suffix", {"layers": 1, "nreq": 40}, 0),
                                       ("fanout", {"layers": 1, "nreq": 256, "suffix": 255}, 0),
                                       ("toy", {}, 0), ("toy", {}, 16)])
def test_k2_chunk_schedule_covers_every_block_once(cfg, kw, cb):
    """K2's work queue: chunks of CB blocks tile [0, Btot); each unit is visited by exactly
    the chunks it intersects (its nseg pieces), zero-length units by exactly one chunk."""
    wl = make_config(cfg, **kw)
    p, ld, pl = plan_of(wl, min_rows=64, chunk=cb)
    boff = pl.export("unit_boff")
    u0, u1 = pl.export("chunk_u0"), pl.export("chunk_u1")
    nseg = pl.export("unit_nseg")
    clo = pl.export("chunk_lo")
    U, NC, Btot = len(boff) - 1, len(u0), int(boff[-1])
    assert len(clo) == NC + 1 and clo[0] == 0 and clo[-1] == Btot
    assert all(clo[i] < clo[i + 1] for i in range(NC)) or Btot == 0
    if cb:
        assert all(clo[i + 1] - clo[i] <= cb for i in range(NC))
    visits = [[] for _ in range(U)]
    covered = np.zeros(Btot, dtype=np.int32)
    for c in range(NC):
        lo, hi = clo[c], clo[c + 1]
        for u in range(u0[c], u1[c]):
            xs, xe = max(boff[u], lo), min(boff[u + 1], hi)
            if boff[u + 1] > boff[u]:
                assert xe > xs, (c, u)  # a chunk only lists units it intersects
            visits[u].append(c)
            covered[xs:xe] += 1
    assert np.all(covered == 1)
    for u in range(U):
        assert len(visits[u]) == nseg[u] >= 1, (u, visits[u], nseg[u])
        assert visits[u] == list(range(visits[u][0], visits[u][0] + nseg[u]))
    pl.destroy()
    p.destroy()


def test_prefill_plan_rows_are_causal_virtual_requests():
    """halo_prefill_plan (NEXT-4): one row per new prompt token; token t of request i sees
    the first len - ntok + t + 1 suffix tokens.  With few rows the causal part streams in K2
    (the row's block list grows with t); with enough rows (ntok x g >= min_rows) it becomes
    causal K1 tiles over the request's own blocks and K2 only merges."""
    p = host_pool(layers=1, hkv=2, hq=8, cap=400)
    a = p.register_prefix(-1, 100)
    r1, r2 = p.open_request(a), p.open_request(-1)
    p.append([r1, r2], [20, 40])
    # all in K2 (min_rows huge): the prefix is folded (+7 blocks on r1's rows)
    pl = p.prefill_plan([r1, r2], [20, 33], PlanOptions(100000, 0, 0, 0))
    info = pl.info()
    assert info["nreq"] == 53 and info["k1_tiles"] == 0
    nblk = np.diff(pl.export("req_blk_off"))
    want = [(n + 15) // 16 + 7 for n in range(1, 21)] + [(n + 15) // 16 for n in range(8, 41)]
    assert list(nblk) == want
    pl.destroy()
    # default: 20 x 4 = 80 and 33 x 4 = 132 rows >= 64 -> causal K1 tiles, nothing for K2
    pl = p.prefill_plan([r1, r2], [20, 33])
    info = pl.info()
    assert list(np.diff(pl.export("req_blk_off"))) == [0] * 53
    tiles = pl.export("tiles").reshape(-1, 8)
    causal = [t for t in tiles if t[7] == -1]
    assert len(causal) == 2 * 2                      # (r1, r2) x 2 kv heads, one m-tile each
    assert sorted(int(t[1]) for t in causal) == [80, 80, 132, 132]
    assert sorted(int(t[4]) for t in causal) == [20, 20, 40, 40]   # token range = visible max
    nsl = pl.export("req_nslots")
    assert list(nsl[:20]) == [2] * 20 and list(nsl[20:]) == [1] * 33   # prefix + causal slots
    # no K2 blocks: the merge runs as K3 alone, whose algorithmic bytes are the partial rows read
    # plus out / lse written (no q): sum_r slots_r * Hq * (d+1) * 4 + R * Hq * (d+1) * 4
    d, hq, R = 128, 8, 53
    assert info["k2_bytes"] == (int(nsl.sum()) + R) * hq * (d + 1) * 4
    pl.destroy()
    for bad in ([0, 1], [21, 1], [1, 41]):
        with pytest.raises(halo.HaloError) as e:
            p.prefill_plan([r1, r2], bad)
        assert e.value.name == "HALO_EINVAL"
    p.destroy()


def test_k2_schedule_spreads_blockless_units_over_warps():
    """Prefill rows whose causal part runs in K1 leave K2 with merge-only units: the item
    schedule (blocks + one merge item per unit) must still spread them over many chunks,
    each unit in exactly one chunk, chunk unit ranges tiling [0, U)."""
    p = host_pool(layers=1, hkv=2, hq=8, cap=4000)
    a = p.register_prefix(-1, 256)
    reqs = [p.open_request(a) for _ in range(64)]
    p.append(reqs, [40] * 64)
    pl = p.prefill_plan(reqs, [40] * 64)
    boff = pl.export("unit_boff")
    assert boff[-1] == 0                        # no blocks left for K2
    u0, u1, nseg, clo = pl.export("chunk_u0"), pl.export("chunk_u1"), pl.export("unit_nseg"), pl.export("chunk_lo")
    U = len(boff) - 1
    assert U == 64 * 40 * 2 and len(u0) >= 1000  # ~one merge per chunk at 148 x 12 warps
    assert all(n == 1 for n in nseg)
    cover = np.zeros(U, dtype=np.int32)
    for c in range(len(u0)):
        cover[u0[c]:u1[c]] += 1
    assert np.all(cover == 1) and np.all(clo == 0)
    pl.destroy()
    p.destroy()


def _k2_warp_blocks(pl, nwarps):
    """Blocks of K2 work per warp (warp w takes chunk w when chunks <= warps)."""
    clo = pl.export("chunk_lo")
    sizes = np.diff(clo)
    assert len(sizes) <= nwarps
    return sizes


def test_single_wave_k1_rule_lowers_splits_and_weights_early_k2_warps():
    """Planner section 7 (co-schedule model): a single-wave K1 beside a K2 that dominates the
    layer gets the split count of least modelled layer time (K1 on 40..75% of the SMs), and the
    K2 warps of the CTAs that start on the SMs K1 leaves idle (blockIdx < 148 - K1 CTAs) get the
    modelled weight w = (r_e T1 + r_pe T2) / (r_pl T2) times the blocks of the others (DESIGN.md,
    "K1/K2 co-schedule").  Shapes where K2 does not dominate keep the default split choice, and
    an explicit split cap disables the rule."""
    nsm, wide = 148, 12
    # C1: 256 requests x 2048-token prefix + 256-token suffixes -> 64 tiles (2 splits)
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=255)
    p, ld, pl = plan_of(wl)
    info = pl.info()
    assert info["k1_tiles"] == 64
    sizes = _k2_warp_blocks(pl, nsm * wide)
    early = (nsm - 64) * wide
    ratio = sizes[:early].mean() / sizes[early:].mean()
    # model: T1 = 3 + 2.75 * 8 = 25 us, E = 84 SMs, r_e = 44 GB/s per SM, B = 268 MB at 6.2 TB/s
    # -> T2 = (B - E r_e T1) / R = 28.3 us, w = (44 * 25 + 52 * 28.3) / (29 * 28.3) = 3.1
    assert 2.8 <= ratio <= 3.4, ratio
    assert sizes.sum() == 256 * 8 * 16  # every suffix block of every (request, kv head) once
    pl.destroy(); p.destroy()
    # small K2 (16-token suffixes): K1 keeps its default single wave of 128 tiles, equal shares
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=15)
    p, ld, pl = plan_of(wl)
    assert pl.info()["k1_tiles"] == 128
    pl.destroy(); p.destroy()
    # K1-bound fan-out (64 requests x 8192 tokens): K2 too small for the rule
    wl = make_config("fanout", layers=1, nreq=64, prefix=8192, suffix=255)
    p, ld, pl = plan_of(wl)
    assert pl.info()["k1_tiles"] == 128
    pl.destroy(); p.destroy()
    # explicit split cap: the rule is off
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=255)
    p, ld, pl = plan_of(wl, max_splits=4)
    assert pl.info()["k1_tiles"] == 128
    pl.destroy(); p.destroy()


def test_k2_launch_shape_whole_units_when_few_units_per_warp():
    """Planner 12b: with few (request, kv head) units per warp and no K1 beside K2 (here every
    prefix node folded into K2), whole units over the narrow shape (7 warps x 4 stages per SM)
    replace stream-K pieces -- C1 has 2048 units for 1776 wide warps, so nearly every unit
    would be cut in two (K2, "Unit ends"); k2_whole_units < 0 opts out.  Beside a
    co-scheduled K1 always wide."""
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=255)
    p, ld, pl = plan_of(wl)  # K1 tiles + co-schedule: wide
    info = pl.info()
    assert info["k1_tiles"] > 0 and info["k2_warps"] == 12
    pl.destroy(); p.destroy()
    p, ld, pl = plan_of(wl, min_rows=1 << 20)  # everything folded: K2 alone, whole units
    info = pl.info()
    assert info["k1_tiles"] == 0 and info["k2_warps"] == 7
    assert (pl.export("unit_nseg") == 1).all()  # whole units: no stream-K pieces
    pl.destroy(); p.destroy()
    p, ld, pl = plan_of(wl, min_rows=1 << 20, whole_units=-1)  # opted out: wide with pieces
    assert pl.info()["k2_warps"] == 12
    pl.destroy(); p.destroy()
    # many units per warp (C2: 8192 units): the wide shape
    wl = make_config("tree", layers=1)
    p, ld, pl = plan_of(wl, min_rows=1 << 20)
    assert pl.info()["k2_warps"] == 12
    pl.destroy(); p.destroy()
