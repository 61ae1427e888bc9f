"""KV-block migration through NCCL (halo_migrate_exchange) on one B200: a 1-rank self-loop
communicator runs the exact migration pipeline -- K4 pack of the source blocks, ncclSend /
ncclRecv inside one ncclGroupStart/End per chunk round, K4 unpack into freshly allocated
blocks, registration of the received node -- with source and destination on the same GPU.

Paper: "cache snapshots can be migrated directly among GPUs via NVLink ... under scheduler
control" (PAPER.md:337 §3.3; :673 §4.5), overlapped with attention.
Bar (north_star): migrated KV blocks match bit-exactly; decoding against the migrated node
is bit-identical to decoding against the source and matches the fp64 oracle (2e-3 / 1e-3).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200 import build as halo_build
from paper_2509_02121_b200.loader import append_step, blocks_needed, load
from synth import make_config

pytestmark = pytest.mark.gpu

DEV = 0
OUT_TOL, LSE_TOL = 2e-3, 1e-3


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()
    torch.cuda.set_device(DEV)


def loopback(pool, **cfg):
    pool.comm_init(halo.comm_unique_id(), 1, 0, **cfg)


def assert_node_equals(pool, node, k, v):
    ko, vo = torch.empty_like(k), torch.empty_like(v)
    pool.read_prefix(node, ko, vo)
    torch.cuda.synchronize()
    assert torch.equal(ko.view(torch.int16), k.view(torch.int16)), "K not bit-exact"
    assert torch.equal(vo.view(torch.int16), v.view(torch.int16)), "V not bit-exact"


def torch_pool(wl, capacity):
    """A pool on torch-owned storage [layer][block][hkv*16*d] int16, so tests can compare raw
    slabs (halo_pool_config.k_storage / v_storage)."""
    shape = (wl.layers, capacity, wl.hkv * 16 * wl.d)
    ks = torch.zeros(shape, dtype=torch.int16, device="cuda")
    vs = torch.zeros(shape, dtype=torch.int16, device="cuda")
    return halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, capacity, DEV, k_storage=ks, v_storage=vs)


def slabs(pool, node):
    """Every (layer, block) slab of the node, K and V, raw (whole blocks, zero tail too)."""
    ks, vs = pool._keep
    blocks = torch.tensor(pool.node_info(node)["blocks"], dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    return ks[:, blocks].clone(), vs[:, blocks].clone()


def decode(pool, reqs, wl, layer):
    plan = pool.plan(reqs)
    q = wl.q(0, "cuda")
    out = torch.empty((len(reqs), wl.hq, wl.d), device="cuda")
    lse = torch.empty((len(reqs), wl.hq), device="cuda")
    plan.run(layer, q[layer], out, lse)
    torch.cuda.synchronize()
    plan.destroy()
    return out.cpu().numpy(), lse.cpu().numpy()


def open_like(pool, wl, leaf):
    """Open wl's requests under `leaf` with wl's initial suffixes + the step-0 token."""
    reqs = [pool.open_request(leaf) for _ in range(wl.nreq)]
    sk, sv = wl.suffix_kv("cuda")
    pool.append(reqs, [r.suffix for r in wl.requests], sk, sv)
    nk, nv = wl.new_kv(0, "cuda")
    pool.append(reqs, [1] * wl.nreq, nk, nv)
    return reqs


@pytest.mark.parametrize("mode", [1, 0])
def test_loopback_c1_template_bit_exact_and_decodes_identically(mode):
    """C1's 2048-token template (32 layers x 8 kv heads, 256 MiB of K+V) through NCCL."""
    wl = make_config("fanout", nreq=64)
    ld = load(wl, DEV, pool=torch_pool(wl, 2 * blocks_needed(wl, steps=2)))
    loopback(ld.pool)
    append_step(ld, wl, 0, DEV)
    layers = [0, 31]
    before = {l: decode(ld.pool, ld.req_ids, wl, l) for l in layers}
    src = ld.node_ids[0]
    src_slabs = slabs(ld.pool, src)
    if mode == 0:  # MOVE needs an unreferenced node: close the requests first
        for r in ld.req_ids:
            ld.pool.close_request(r)
    used0 = ld.pool.stats()[1]  # (blocks of closed requests may still be pending)
    (new,) = ld.pool.migrate_exchange(sends=[(src, 0, mode)], recvs=[(0, -1, 2048)])
    torch.cuda.synchronize()
    # every destination slab (all layers, K and V, whole blocks) equals its source slab
    dst_slabs = slabs(ld.pool, new)
    assert torch.equal(src_slabs[0], dst_slabs[0]) and torch.equal(src_slabs[1], dst_slabs[1])
    k, v = wl.node_kv(0, "cuda")
    assert_node_equals(ld.pool, new, k, v)
    info = ld.pool.node_info(new)
    assert info["ntok"] == 2048 and info["parent"] == -1 and len(info["blocks"]) == 128
    if mode == 0:
        with pytest.raises(halo.HaloError) as e:
            ld.pool.node_info(src)
        assert e.value.name == "HALO_ENOENT"
        assert ld.pool.stats()[1] == used0  # 128 blocks in, 128 blocks out
    else:
        assert ld.pool.stats()[1] == used0 + 128
    reqs2 = open_like(ld.pool, wl, new)
    for l in layers:
        o2, l2 = decode(ld.pool, reqs2, wl, l)
        assert np.array_equal(o2, before[l][0]) and np.array_equal(l2, before[l][1]), l
        ro, rl = oracle.decode_reference(wl, l, steps=1, requests=list(range(0, wl.nreq, 8)))
        assert np.abs(o2[::8] - ro).max() <= OUT_TOL
        assert np.abs(l2[::8] - rl).max() <= LSE_TOL
    ld.pool.destroy()


def test_loopback_move_of_a_32k_token_node():
    """The largest C4 node: 32768 tokens x 32 layers x 8 heads (4 GiB of K+V), MOVE."""
    wl = make_config("fanout", nreq=4, prefix=32768, suffix=15)
    ld = load(wl, DEV, capacity=2 * blocks_needed(wl, steps=2))
    loopback(ld.pool)
    append_step(ld, wl, 0, DEV)
    before = decode(ld.pool, ld.req_ids, wl, 5)
    for r in ld.req_ids:
        ld.pool.close_request(r)
    (new,) = ld.pool.migrate_exchange(sends=[(ld.node_ids[0], 0, 0)], recvs=[(0, -1, 32768)])
    k, v = wl.node_kv(0, "cuda")
    assert_node_equals(ld.pool, new, k, v)
    del k, v
    reqs2 = open_like(ld.pool, wl, new)
    o2, l2 = decode(ld.pool, reqs2, wl, 5)
    assert np.array_equal(o2, before[0]) and np.array_equal(l2, before[1])
    ro, rl = oracle.decode_reference(wl, 5, steps=1)
    assert np.abs(o2 - ro).max() <= OUT_TOL and np.abs(l2 - rl).max() <= LSE_TOL
    ld.pool.destroy()


@pytest.mark.parametrize("chunk_bytes", [64 << 10, 1 << 20, 0])
def test_exchange_many_nodes_ragged_chunks(chunk_bytes):
    """Several transfers of ragged sizes in ONE call (mixed MOVE / COPY, a child received under
    an existing parent), chunk sizes forcing 1 .. hundreds of rounds."""
    wl = make_config("ragged", layers=3)
    ld = load(wl, DEV, capacity=4 * blocks_needed(wl))
    loopback(ld.pool, chunk_bytes=chunk_bytes, copy_ctas=37)
    # leaves 4 (5 tokens, a root) and 5 (129 tokens, under 2) lose their requests -> MOVE
    ids = ld.node_ids
    for r, spec in zip(ld.req_ids, wl.requests):
        if spec.leaf in (4, 5):
            ld.pool.close_request(r)
    movable = [4, 5]
    sends, recvs, expect = [], [], []
    for n in sorted(ids):
        mode = 0 if n in movable else 1
        sends.append((ids[n], 0, mode))
        recvs.append((0, ids[0] if n != 0 else -1, wl.node(n).ntok))
        expect.append(n)
    new = ld.pool.migrate_exchange(sends=sends, recvs=recvs)
    assert len(new) == len(expect)
    for n, nid in zip(expect, new):
        k, v = wl.node_kv(n, "cuda")
        assert_node_equals(ld.pool, nid, k, v)
        info = ld.pool.node_info(nid)
        assert info["parent"] == (ids[0] if n != 0 else -1)
    for n in movable:
        with pytest.raises(halo.HaloError):
            ld.pool.node_info(ids[n])
    ld.pool.destroy()


def test_exchange_validation_leaves_the_pool_unchanged():
    wl = make_config("ragged", layers=2)
    ld = load(wl, DEV, capacity=blocks_needed(wl))
    p = ld.pool
    for r, spec in zip(ld.req_ids, wl.requests):
        if spec.leaf == 4:
            p.close_request(r)
    free = p.stats()[0]  # leave 10 free blocks: a 19-block receive must fail with ENOMEM
    z = torch.zeros((wl.layers, (free - 10) * 16, wl.hkv, wl.d), dtype=torch.bfloat16, device="cuda")
    p.register_prefix(-1, (free - 10) * 16, z, z)
    torch.cuda.synchronize()
    with pytest.raises(halo.HaloError) as e:   # no communicator yet
        p.migrate_exchange(sends=[(ld.node_ids[4], 0, 1)], recvs=[(0, -1, 5)])
    assert e.value.name == "HALO_ENCCL"
    loopback(p)
    before = p.stats()
    cases = [
        (dict(sends=[(ld.node_ids[4], 0, 1)]), "HALO_EINVAL"),                     # unmatched self send
        (dict(recvs=[(0, -1, 5)]), "HALO_EINVAL"),                                   # unmatched self recv
        (dict(sends=[(ld.node_ids[4], 0, 1)], recvs=[(0, -1, 6)]), "HALO_EINVAL"),   # ntok mismatch
        (dict(sends=[(123456, 0, 1)], recvs=[(0, -1, 5)]), "HALO_ENOENT"),
        (dict(sends=[(ld.node_ids[0], 0, 0)], recvs=[(0, -1, 301)]), "HALO_EBUSY"),  # MOVE of a parent
        (dict(sends=[(ld.node_ids[4], 0, 0), (ld.node_ids[4], 0, 0)],
              recvs=[(0, -1, 5), (0, -1, 5)]), "HALO_EINVAL"),                       # moved twice
        (dict(sends=[(ld.node_ids[4], 1, 1)], recvs=[(0, -1, 5)]), "HALO_EINVAL"),   # bad peer
        (dict(sends=[(ld.node_ids[4], 0, 0)], recvs=[(0, ld.node_ids[4], 5)]), "HALO_EINVAL"),
        (dict(sends=[(ld.node_ids[0], 0, 1)], recvs=[(0, 987654, 301)]), "HALO_ENOENT"),
        (dict(sends=[(ld.node_ids[0], 0, 1)], recvs=[(0, -1, 301)]), "HALO_ENOMEM"),  # 19 blocks > 10
    ]
    for kw, name in cases:
        with pytest.raises(halo.HaloError) as e:
            p.migrate_exchange(**kw)
        assert e.value.name == name, (kw, e.value)
        assert p.stats() == before
        for n in wl.nodes:
            p.node_info(ld.node_ids[n.ident])
    with pytest.raises(halo.HaloError) as e:  # one-sided helpers refuse self loops
        p.migrate_send(ld.node_ids[4], 0, 1)
    assert e.value.name == "HALO_EINVAL"
    p.destroy()


def test_migration_on_a_side_stream_beside_decode():
    """Decode on the compute stream while a 1k-token node migrates on a side stream (bounded
    NCCL and copy CTAs): decode outputs stay bit-identical, the migrated node bit-exact."""
    wl = make_config("fanout", nreq=64, layers=8)
    big = make_config("fanout", nreq=1, prefix=1024, layers=8, seed=77)
    cap = blocks_needed(wl, steps=2) + 4 * blocks_needed(big)
    ld = load(wl, DEV, capacity=cap)
    other = load(big, DEV, pool=ld.pool)
    p = ld.pool
    loopback(p, max_ctas=4, copy_ctas=64)
    append_step(ld, wl, 0, DEV)
    ref = [decode(p, ld.req_ids, wl, l) for l in range(wl.layers)]
    compute, side = torch.cuda.Stream(), torch.cuda.Stream()
    plan = p.plan(ld.req_ids, stream=compute)
    q = wl.q(0, "cuda")
    outs = torch.empty((wl.layers, wl.nreq, wl.hq, wl.d), device="cuda")
    lses = torch.empty((wl.layers, wl.nreq, wl.hq), device="cuda")
    torch.cuda.synchronize()
    news = []
    for rep in range(3):
        for l in range(wl.layers):
            plan.run(l, q[l], outs[l], lses[l], stream=compute)
        news += p.migrate_exchange(sends=[(other.node_ids[0], 0, 1)], recvs=[(0, -1, 1024)],
                                   stream=side)
    torch.cuda.synchronize()
    for l in range(wl.layers):
        assert np.array_equal(outs[l].cpu().numpy(), ref[l][0])
        assert np.array_equal(lses[l].cpu().numpy(), ref[l][1])
    k, v = big.node_kv(0, "cuda")
    for n in news:
        assert_node_equals(p, n, k, v)
    plan.destroy()
    p.destroy()
