"""Sharded execution checked against the fp64 oracle on one GPU.

The attention of one (request, q-head) row depends only on that row's keys,
so the multi-GPU partitionings have no exchange step.  Each GPU's share is emulated here by
its own pool on the same device, built exactly as a rank would build it:
  * kv-head sharding (C2): shard p holds kv heads [p H/P, (p+1) H/P) of every node and
    suffix block and serves their g H/P q-heads; the shards' outputs, concatenated along the
    head axis, must equal the unsharded oracle for every request (PAPER.md:236 replication
    with query partitioning is the request-axis analogue);
  * request-group sharding (C3, BASELINE configs[3]): sharding.rank_requests places whole
    template subtrees on 8 ranks by LPT (the paper's DP placement); every
    shard's requests are checked against the oracle of the shard's workload.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200 import build as halo_build
from paper_2509_02121_b200 import sharding
from paper_2509_02121_b200.loader import append_step, blocks_needed, load
from synth import make_config

pytestmark = pytest.mark.gpu

DEV = 0
OUT_TOL, LSE_TOL = 2e-3, 1e-3
_REF = {}


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()
    torch.cuda.set_device(DEV)


def head_shard_outputs(wl, P, layer):
    """Outputs of the P head shards of wl at `layer`, concatenated along the q-head axis."""
    outs, lses = [], []
    nodes_kv = {n.ident: wl.node_kv(n.ident, "cuda") for n in wl.nodes}
    sk, sv = wl.suffix_kv("cuda")
    nk, nv = wl.new_kv(0, "cuda")
    q = wl.q(0, "cuda")
    for p in range(P):
        lo, hi = sharding.head_range(wl.hkv, P, p)
        hkv, hq = hi - lo, wl.g * (hi - lo)
        pool = halo.Pool(wl.layers, hkv, hq, wl.d, blocks_needed(wl, steps=1), DEV)
        ids = {}
        depth = lambda n: 0 if wl.node(n).parent < 0 else 1 + depth(wl.node(n).parent)
        for n in sorted(wl.nodes, key=lambda x: (depth(x.ident), x.ident)):
            k, v = nodes_kv[n.ident]
            ids[n.ident] = pool.register_prefix(ids.get(n.parent, -1), n.ntok, k[:, :, lo:hi].contiguous(),
                                                v[:, :, lo:hi].contiguous())
        reqs = [pool.open_request(ids[r.leaf] if r.leaf >= 0 else -1) for r in wl.requests]
        pool.append(reqs, [r.suffix for r in wl.requests], sk[:, :, lo:hi].contiguous(), sv[:, :, lo:hi].contiguous())
        pool.append(reqs, [1] * wl.nreq, nk[:, :, lo:hi].contiguous(), nv[:, :, lo:hi].contiguous())
        plan = pool.plan(reqs)
        qs = q[layer][:, lo * wl.g:hi * wl.g].contiguous()
        out = torch.empty((wl.nreq, hq, wl.d), device="cuda")
        lse = torch.empty((wl.nreq, hq), device="cuda")
        plan.run(layer, qs, out, lse)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
        lses.append(lse.cpu().numpy())
        plan.destroy()
        pool.destroy()
    return np.concatenate(outs, axis=1), np.concatenate(lses, axis=1)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_head_sharded_c2_matches_the_unsharded_oracle(P):
    """C2's tree (4k root -> 16 roles x 1k -> 1024 requests, 256-token suffixes), its 8 kv heads
    split over P shards; all 1024 requests x 32 q-heads vs the oracle."""
    wl = make_config("tree", layers=2)
    layer = 1
    if "c2" not in _REF:
        _REF["c2"] = oracle.decode_reference(wl, layer, steps=1)
    ro, rl = _REF["c2"]
    o, l_ = head_shard_outputs(wl, P, layer)
    assert np.abs(o - ro).max() <= OUT_TOL
    assert np.abs(l_ - rl).max() <= LSE_TOL


@pytest.mark.parametrize("P", [2, 4])
def test_head_sharded_ragged_tree_matches_oracle(P):
    """A depth-3 ragged tree (partial blocks, prefix-less requests, empty initial suffixes),
    g = 4, its 4 kv heads over P shards, both layers, every request."""
    wl = make_config("ragged", layers=2, hq=16, hkv=4)
    for layer in range(2):
        ro, rl = oracle.decode_reference(wl, layer, steps=1)
        o, l_ = head_shard_outputs(wl, P, layer)
        assert np.abs(o - ro).max() <= OUT_TOL
        assert np.abs(l_ - rl).max() <= LSE_TOL


def test_group_sharded_c3_over_8_ranks_matches_oracle():
    """C3 (64 templates x 8k-token contexts, 256 requests each) placed on 8 ranks by
    sharding.rank_requests (LPT over the K1/K2 roofline cost); every rank's shard is loaded,
    planned and run like on its own GPU; 8 requests of every template are checked."""
    wl = make_config("analytics", templates=64, layers=1)
    seen = []
    for rank in range(8):
        mine = sharding.rank_requests(wl, 8, rank)
        assert len(mine) == 8 * 256          # 8 templates per rank
        seen += mine
        shard = sharding.subset_workload(wl, mine)
        ld = load(shard, DEV)
        append_step(ld, shard, 0, DEV)
        plan = ld.pool.plan(ld.req_ids)
        info = plan.info()
        assert info["tensor_nodes"] == 8
        q = shard.q(0, "cuda")
        out = torch.empty((shard.nreq, shard.hq, shard.d), device="cuda")
        lse = torch.empty((shard.nreq, shard.hq), device="cuda")
        plan.run(0, q[0], out, lse)
        torch.cuda.synchronize()
        sample = [i for i in range(shard.nreq) if i % 32 == rank % 32]
        ro, rl = oracle.decode_reference(shard, 0, steps=1, requests=sample)
        assert np.abs(out.cpu().numpy()[sample] - ro).max() <= OUT_TOL, rank
        assert np.abs(lse.cpu().numpy()[sample] - rl).max() <= LSE_TOL, rank
        plan.destroy()
        ld.pool.destroy()
    assert sorted(seen) == list(range(wl.nreq))
