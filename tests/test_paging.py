"""Host paging of prefix nodes (§3.3): offload /
fetch between the device pool and a pinned host arena, LRU eviction, and plan validity.

CPU tests run on host-only pools (bookkeeping: the same C++ code paths minus the copies);
the GPU tests check the copies bit-exactly and decode parity after a page-out / page-in."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200 import build as halo_build
from paper_2509_02121_b200.loader import append_step, load
from synth import make_config


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()


def err_name(fn, *a):
    with pytest.raises(halo.HaloError) as e:
        fn(*a)
    return e.value.name


# ------------------------------------------------------------------ CPU (host-only pools)

def test_offload_fetch_accounting_and_errors():
    p = halo.Pool(2, 2, 8, 128, 20, device=-1)
    a = p.register_prefix(-1, 40)          # 3 blocks
    r = p.open_request(a)
    p.append([r], [5])                     # 1 block
    assert p.stats() == (16, 4)
    assert err_name(p.offload_prefix, a) == "HALO_EUNSUPPORTED"   # no arena yet
    p.host_reserve(4)
    p.offload_prefix(a)
    assert p.residency(a)[0] is False
    assert p.stats() == (19, 1)
    assert p.node_info(a)["blocks"] == []
    assert err_name(p.offload_prefix, a) == "HALO_EINVAL"         # already offloaded
    assert err_name(p.plan, [r]) == "HALO_EBUSY"                 # plan reads an offloaded node
    b = p.register_prefix(-1, 33)          # 3 blocks: arena has 1 left
    assert err_name(p.offload_prefix, b) == "HALO_ENOMEM"
    assert p.residency(b)[0] is True and p.stats() == (16, 4)     # unchanged
    assert err_name(p.host_reserve, 8) == "HALO_EBUSY"            # nodes live in the arena
    p.fetch_prefix(a)
    assert p.residency(a)[0] is True and len(p.node_info(a)["blocks"]) == 3
    assert p.stats() == (13, 7)
    assert err_name(p.fetch_prefix, a) == "HALO_EINVAL"
    pl = p.plan([r])
    pl.destroy()
    p.offload_prefix(b)                    # arena space came back with the fetch
    p.close_request(r)
    p.release_prefix(a)
    p.release_prefix(b)                    # an offloaded node can be released
    assert p.stats() == (20, 0)
    p.host_reserve(2)                      # no offloaded nodes left: re-reserve allowed
    p.destroy()


def test_fetch_enomem_leaves_the_node_offloaded():
    p = halo.Pool(1, 1, 1, 64, 4, device=-1)
    p.host_reserve(8)
    a = p.register_prefix(-1, 48)          # 3 blocks
    p.offload_prefix(a)
    b = p.register_prefix(-1, 32)          # 2 blocks: 2 free device blocks remain
    assert err_name(p.fetch_prefix, a) == "HALO_ENOMEM"
    assert p.residency(a)[0] is False
    p.release_prefix(b)
    p.fetch_prefix(a)
    assert p.residency(a)[0] is True
    p.release_prefix(a)
    p.destroy()


def test_lru_evicts_least_recently_planned_first_and_spares_the_latest_plan():
    p = halo.Pool(1, 1, 4, 64, 64, device=-1)
    p.host_reserve(64)
    nodes = [p.register_prefix(-1, 16 * (i + 1)) for i in range(4)]   # 1..4 blocks
    reqs = [p.open_request(n) for n in nodes]
    p.append(reqs, [1] * 4)
    order = [2, 0, 3, 1]                   # plan use order: node 1 is the most recent
    for i in order:
        p.plan([reqs[i]]).destroy()
    ticks = [p.residency(n)[1] for n in nodes]
    assert [ticks[i] for i in order] == sorted(ticks)
    free0 = p.stats()[0]
    # ask for 3 more blocks: LRU is node 2 (3 blocks) -> exactly one eviction
    assert p.evict_lru(free0 + 3) == 1
    assert [p.residency(n)[0] for n in nodes] == [True, True, False, True]
    # ask for everything: nodes 0 and 3 go, node 1 (read by the latest plan) stays
    assert err_name(p.evict_lru, 10 ** 6) == "HALO_ENOMEM"
    assert [p.residency(n)[0] for n in nodes] == [False, True, False, False]
    for n in (0, 2, 3):
        p.fetch_prefix(nodes[n])
    p.destroy()


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_offload_fetch_round_trip_is_bit_exact_and_decodes_identically():
    torch.cuda.set_device(0)
    wl = make_config("tree", layers=3, root=500, roles=3, role_tok=130, per_role=30, suffix=20)
    ld = load(wl, 0)
    p = ld.pool
    p.host_reserve(64)
    append_step(ld, wl, 0, 0)
    q = wl.q(0, "cuda")
    plan = p.plan(ld.req_ids)
    o1 = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda")
    plan.run(2, q[2], o1)
    # page the root and one role out, make the pool reuse their blocks, page them back in
    root, role = ld.node_ids[0], ld.node_ids[2]
    p.offload_prefix(root)
    p.offload_prefix(role)
    with pytest.raises(halo.HaloError) as e:          # the plan predates the offload
        plan.run(2, q[2], o1)
    assert e.value.name == "HALO_EBUSY"
    junk = p.register_prefix(-1, 16 * 20, *[torch.full((wl.layers, 320, wl.hkv, wl.d), 7.0,
                                                        dtype=torch.bfloat16, device="cuda")] * 2)
    p.fetch_prefix(role)
    p.fetch_prefix(root)
    for n in wl.nodes:
        k, v = wl.node_kv(n.ident, "cuda")
        ko, vo = torch.empty_like(k), torch.empty_like(v)
        p.read_prefix(ld.node_ids[n.ident], ko, vo)
        torch.cuda.synchronize()
        assert torch.equal(ko.view(torch.int16), k.view(torch.int16)), n.ident
        assert torch.equal(vo.view(torch.int16), v.view(torch.int16)), n.ident
    plan = p.plan(ld.req_ids, reuse=plan)
    o2 = torch.empty_like(o1)
    plan.run(2, q[2], o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    ro, _ = oracle.decode_reference(wl, 2, steps=1)
    assert np.abs(o2.cpu().numpy() - ro).max() <= 2e-3
    plan.destroy()
    p.release_prefix(junk)
    p.destroy()


@pytest.mark.gpu
def test_lru_paging_under_memory_pressure_keeps_parity():
    """Two workflow templates share a pool too small for both: each step evicts the idle
    template (LRU) and prefetches the one the batch needs; outputs stay equal to the oracle."""
    torch.cuda.set_device(0)
    wl = make_config("analytics", layers=2, templates=2, ctx=1024, per_template=24, suffix=15)
    per_node = (1024 + 15) // 16
    cap = 2 * per_node + 2 * 24 * 2 + 8      # ~1.1 templates of prefix + all suffixes
    ld = load(wl, 0, capacity=2 * per_node + 2 * 24 * 3 + 16)
    p = ld.pool
    p.host_reserve(2 * per_node)
    append_step(ld, wl, 0, 0)
    groups = [[r for r in range(wl.nreq) if wl.requests[r].leaf == t] for t in range(2)]
    q = wl.q(0, "cuda")
    for it, t in enumerate([0, 1, 0, 1]):
        node = ld.node_ids[t]
        if not p.residency(node)[0]:
            free = p.stats()[0]
            if free < per_node:
                p.evict_lru(per_node)
            p.fetch_prefix(node)
        reqs = [ld.req_ids[r] for r in groups[t]]
        plan = p.plan(reqs)
        out = torch.empty((len(reqs), wl.hq, wl.d), device="cuda")
        plan.run(1, q[1][groups[t]].contiguous(), out)
        torch.cuda.synchronize()
        ro, _ = oracle.decode_reference(wl, 1, steps=1, requests=groups[t])
        assert np.abs(out.cpu().numpy() - ro).max() <= 2e-3, (it, t)
        plan.destroy()
        # the other template is now the LRU one: page it out to make room
        other = ld.node_ids[1 - t]
        if p.residency(other)[0]:
            p.offload_prefix(other)
    assert cap > 0
    p.destroy()


def test_prefetch_bookkeeping_on_host_only_pool():
    """halo_pool_prefetch fetches exactly the offloaded nodes on the requests' paths (parents
    first), nothing else; resident nodes and unknown requests behave as documented."""
    wl = make_config("tree", layers=2, root=64, roles=3, role_tok=32, per_role=4, suffix=5)
    ld = load(wl, device=-1)
    p = ld.pool
    p.host_reserve(64)
    root, r1, r2 = ld.node_ids[0], ld.node_ids[1], ld.node_ids[2]
    for n in (r2, r1, root):
        p.offload_prefix(n)
    reqs_r1 = [ld.req_ids[i] for i, r in enumerate(wl.requests) if r.leaf == 1]
    assert p.prefetch(reqs_r1) == 2          # root, then role 1
    assert p.residency(root)[0] and p.residency(r1)[0] and not p.residency(r2)[0]
    assert p.prefetch(reqs_r1) == 0
    assert err_name(p.prefetch, [123456]) == "HALO_ENOENT"
    p.destroy()


@pytest.mark.gpu
def test_background_prefetch_overlaps_decode_and_keeps_parity():
    """prefetch the next batch's offloaded template on a copy stream while the
    current batch decodes on the compute stream, then plan and run the next batch on the
    compute stream without a host synchronisation: the plan waits for the copies (node fetch
    events) and the outputs equal the pre-offload ones bit for bit (and the oracle)."""
    torch.cuda.set_device(0)
    wa = make_config("fanout", layers=4, nreq=128, prefix=2048, suffix=63, seed=11)
    wb = make_config("fanout", layers=4, nreq=128, prefix=1024, suffix=63, seed=12)
    from paper_2509_02121_b200.loader import blocks_needed
    la = load(wa, 0, capacity=blocks_needed(wa) + blocks_needed(wb))
    lb = load(wb, 0, pool=la.pool)
    p = la.pool
    p.host_reserve(2048 // 16 + 8)
    append_step(la, wa, 0, 0)
    append_step(lb, wb, 0, 0)
    qa, qb = wa.q(0, "cuda"), wb.q(0, "cuda")
    ref = torch.empty((wa.nreq, wa.hq, wa.d), device="cuda")
    pa = p.plan(la.req_ids)
    pa.run(3, qa[3], ref)
    pa.destroy()
    p.offload_prefix(la.node_ids[0])
    torch.cuda.synchronize()
    compute, copy = torch.cuda.Stream(), torch.cuda.Stream()
    ob = torch.empty((wb.nreq, wb.hq, wb.d), device="cuda")
    oa = torch.empty_like(ref)
    pb = p.plan(lb.req_ids, stream=compute)
    for rep in range(2):
        for l in range(4):
            pb.run(l, qb[l], ob, stream=compute)      # the current batch decodes ...
        if rep == 0:
            assert p.prefetch(la.req_ids, stream=copy) == 1   # ... while the next one's KV arrives
    pa = p.plan(la.req_ids, stream=compute)           # no host sync: the plan waits for the fetch
    pa.run(3, qa[3], oa, stream=compute)
    torch.cuda.synchronize()
    assert torch.equal(oa, ref)
    ro, _ = oracle.decode_reference(wa, 3, steps=1, requests=list(range(0, wa.nreq, 16)))
    assert np.abs(oa.cpu().numpy()[::16] - ro).max() <= 2e-3
    pa.destroy()
    pb.destroy()
    p.destroy()
