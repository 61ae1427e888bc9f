"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by element.

Bar (north_star): max |out_gpu - o_oracle| <= 2e-3 on the fp32 output (bf16 KV inputs,
fp32 accumulation); max |lse_gpu - lse_oracle| <= 1e-3.  Migrated / cloned
blocks must be bit-exact; permutations and reruns bit-identical.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200 import build as halo_build
from paper_2509_02121_b200.abi import PlanOptions
from paper_2509_02121_b200.loader import append_step, load
from synth import make_config
from synth.gen import bf16_bits

pytestmark = pytest.mark.gpu

OUT_TOL = 2e-3
LSE_TOL = 1e-3
DEV = 0


@pytest.fixture(scope="module", autouse=True)
def built():
    halo_build.build()
    halo.load_library()
    torch.cuda.set_device(DEV)


def run_step(wl, opt=None, layers=None, reqs_perm=None):
    ld = load(wl, DEV)
    append_step(ld, wl, 0, DEV)
    order = list(range(wl.nreq)) if reqs_perm is None else list(reqs_perm)
    plan = ld.pool.plan([ld.req_ids[i] for i in order], opt)
    q = wl.q(0, f"cuda:{DEV}")[:, order].contiguous()
    L = wl.layers
    out = torch.full((L, len(order), wl.hq, wl.d), float("nan"), device=f"cuda:{DEV}")
    lse = torch.full((L, len(order), wl.hq), float("nan"), device=f"cuda:{DEV}")
    for l in (layers if layers is not None else range(L)):
        plan.run(l, q[l], out[l], lse[l])
    torch.cuda.synchronize()
    return ld, plan, out.cpu().numpy(), lse.cpu().numpy()


def cleanup(ld, plan):
    plan.destroy()
    ld.pool.destroy()


def check(wl, opt=None, layers=None, sample=None):
    layers = list(range(wl.layers)) if layers is None else layers
    ld, plan, out, lse = run_step(wl, opt, layers)
    info = plan.info()
    reqs = list(range(wl.nreq)) if sample is None else sample
    worst_o = worst_l = 0.0
    for l in layers:
        ro, rl = oracle.decode_reference(wl, l, steps=1, requests=reqs)
        eo = np.abs(out[l][reqs] - ro).max()
        el = np.abs(lse[l][reqs] - rl).max()
        worst_o, worst_l = max(worst_o, eo), max(worst_l, el)
    cleanup(ld, plan)
    assert np.isfinite(worst_o) and worst_o <= OUT_TOL, (worst_o, info)
    assert np.isfinite(worst_l) and worst_l <= LSE_TOL, (worst_l, info)
    return info, worst_o, worst_l


def opts(min_rows=0, splits=0, max_splits=0, chunk=0):
    return PlanOptions(min_rows, splits, max_splits, chunk)


def test_toy_c0_folded():
    info, *_ = check(make_config("toy"))
    assert info["tensor_nodes"] == 0 and info["folded_nodes"] == 1


def test_toy_c0_tensor_path_d64_g1():
    info, *_ = check(make_config("toy"), opts(min_rows=1))
    assert info["tensor_nodes"] == 1 and info["k1_tiles"] == 1


@pytest.mark.parametrize("min_rows,splits", [(1, 0), (1, 3), (16, 2), (0, 0), (100000, 0)])
def test_ragged_tree(min_rows, splits):
    """depth-3 tree, partial blocks, no-prefix requests, 0-token initial suffixes, g=4."""
    check(make_config("ragged"), opts(min_rows, splits))


@pytest.mark.parametrize("chunk", [1, 3, 16])
def test_k2_work_queue_chunking(chunk):
    """Units cut into many pieces by the K2 work queue merge back exactly (ragged suffixes,
    zero-length-suffix requests, folded nodes)."""
    check(make_config("ragged_suffix", layers=1, nreq=24, prefix=300, lo=1, hi=200),
          opts(chunk=chunk))
    check(make_config("ragged"), opts(min_rows=16, chunk=chunk))


def test_fanout_small_k1_multi_mtile():
    wl = make_config("fanout", layers=2, nreq=80, prefix=1000, suffix=40)
    info, *_ = check(wl)
    assert info["tensor_nodes"] == 1 and info["k1_tiles"] >= 24


def test_tree_two_levels():
    wl = make_config("tree", layers=2, root=700, roles=4, role_tok=300, per_role=40, suffix=20)
    info, *_ = check(wl)
    assert info["tensor_nodes"] == 5 and info["max_slots"] >= 2


def test_ragged_suffix_lengths():
    check(make_config("ragged_suffix", layers=1, nreq=40, prefix=512))


@pytest.mark.parametrize("alpha", [2.0, 4.0, 8.0])
def test_sharper_scores(alpha):
    """alpha = 2 and the stress alphas 4 / 8 (sharp, competing peaks; SURVEY.md §8(c) error
    budget): gated at the same 2e-3, since K1's P is fp16 (the budget's fp16-P column)."""
    check(make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, alpha_q=alpha))


@pytest.mark.parametrize("cfg,kw", [("fanout", dict(nreq=64, prefix=600, suffix=30)),
                                    ("tree", dict(root=300, roles=3, role_tok=130, per_role=30, suffix=20))])
def test_attention_sink(cfg, kw):
    """Attention-sink variant (+8 on token 0 of every root): most of the
    probability mass on one prefix token, in K1's first n-tile."""
    check(make_config(cfg, layers=1, sink=8.0, **kw))


def test_d64_g2():
    check(make_config("fanout", layers=1, nreq=70, prefix=333, suffix=17, hq=4, hkv=2, d=64))


def test_g8_and_g1():
    check(make_config("fanout", layers=1, nreq=40, prefix=260, suffix=9, hq=16, hkv=2))
    check(make_config("fanout", layers=1, nreq=130, prefix=260, suffix=9, hq=4, hkv=4),
          opts(min_rows=1))


def test_full_c1_at_bench_configuration():
    """C1 (BASELINE configs[1]) at full size: 256 requests, 2k prefix, 32 layers; every
    request at the first and last layer vs the oracle (the launch configuration bench.py
    times: default plan)."""
    wl = make_config("fanout")
    check(wl, layers=[0, 31])   # every request (C0-C2 all requests)


def test_request_permutation_and_rerun_are_bit_identical():
    wl = make_config("ragged")
    ld, plan, out, lse = run_step(wl, opts(min_rows=1, splits=2))
    # rerun the same plan
    q = wl.q(0, f"cuda:{DEV}")
    out2 = torch.empty((wl.nreq, wl.hq, wl.d), device=f"cuda:{DEV}")
    lse2 = torch.empty((wl.nreq, wl.hq), device=f"cuda:{DEV}")
    plan.run(1, q[1], out2, lse2)
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), out[1]) and np.array_equal(lse2.cpu().numpy(), lse[1])
    cleanup(ld, plan)
    perm = np.random.Generator(np.random.PCG64(5)).permutation(wl.nreq)
    ld, plan, outp, lsep = run_step(wl, opts(min_rows=1, splits=2), reqs_perm=perm)
    assert np.array_equal(outp, out[:, perm]) and np.array_equal(lsep, lse[:, perm])
    cleanup(ld, plan)


@pytest.mark.parametrize("hq,hkv,d,per", [(32, 8, 128, 70), (8, 8, 64, 150), (16, 2, 128, 37),
                                          (4, 2, 64, 70)])
def test_k1_q_by_tma_equals_manual_q_load(hq, hkv, d, per):
    """K1 loads a tile's Q rows by TMA when its requests are consecutive caller indices
    (box {64, g, 128/g}, rows request-major), else thread by thread.  Two templates: in
    template order every tile takes the TMA path (with a partial second sub-tile and, for
    the last template, rows past the last request, zero-filled out of bounds); with the two
    templates' requests interleaved no tile's requests are consecutive, so every tile loads
    Q thread by thread.  Both land the same bytes in shared memory: the rows are
    bit-identical, and match the oracle."""
    wl = make_config("analytics", layers=1, templates=2, ctx=300, per_template=per, suffix=9,
                     hq=hq, hkv=hkv, d=d)
    ld, plan, out, lse = run_step(wl, opts(min_rows=1))
    assert plan.info()["k1_tiles"] > 0
    cleanup(ld, plan)
    ro, rl = oracle.decode_reference(wl, 0, steps=1)
    assert np.abs(out[0] - ro).max() <= OUT_TOL and np.abs(lse[0] - rl).max() <= LSE_TOL
    inter = [i for pair in zip(range(per), range(per, 2 * per)) for i in pair]
    ld, plan, outp, lsep = run_step(wl, opts(min_rows=1), reqs_perm=inter)
    tiles = plan.export("tiles").reshape(-1, 8)
    order = plan.export("req_order")
    assert all(order[t[0] + 1] != order[t[0]] + 1 for t in tiles if t[1] > hq // hkv)  # manual path
    cleanup(ld, plan)
    assert np.array_equal(outp, out[:, inter]) and np.array_equal(lsep, lse[:, inter])


def test_physical_block_placement_is_bit_invisible():
    wl = make_config("tree", layers=1, root=300, roles=3, role_tok=100, per_role=30, suffix=40)
    ld, plan, out, lse = run_step(wl)
    cleanup(ld, plan)
    # same logical content, different physical blocks: fragment the pool first
    pool = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, 4000, DEV)
    junk = [pool.register_prefix(-1, 16 * (i % 3 + 1),
                                 *[torch.zeros(wl.layers, 16 * (i % 3 + 1), wl.hkv, wl.d,
                                               dtype=torch.bfloat16, device="cuda")] * 2)
            for i in range(40)]
    for j in junk[::2]:
        pool.release_prefix(j)
    torch.cuda.synchronize()
    ld2 = load(wl, DEV, pool=pool)
    append_step(ld2, wl, 0, DEV)
    plan2 = pool.plan(ld2.req_ids)
    q = wl.q(0, "cuda")
    out2 = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda")
    lse2 = torch.empty((wl.nreq, wl.hq), device="cuda")
    plan2.run(0, q[0], out2, lse2)
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), out[0]) and np.array_equal(lse2.cpu().numpy(), lse[0])
    plan2.destroy()
    pool.destroy()


def test_prefix_read_returns_registered_tensors():
    wl = make_config("ragged", layers=3)
    ld = load(wl, DEV)
    for n in wl.nodes:
        k, v = wl.node_kv(n.ident, "cuda")
        ko, vo = torch.empty_like(k), torch.empty_like(v)
        ld.pool.read_prefix(ld.node_ids[n.ident], ko, vo)
        torch.cuda.synchronize()
        assert torch.equal(ko.view(torch.int16), k.view(torch.int16))
        assert torch.equal(vo.view(torch.int16), v.view(torch.int16))
    ld.pool.destroy()


def test_clone_is_bit_exact_and_decodes_identically():
    """K4 pack/unpack relocation (the migration data path without NCCL)."""
    wl = make_config("fanout", layers=3, nreq=40, prefix=777, suffix=5)
    ld = load(wl, DEV)
    src = ld.node_ids[0]
    dst_pool = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, 1000, DEV)
    new = ld.pool.clone_prefix(src, dst_pool, -1)
    k, v = wl.node_kv(0, "cuda")
    ko, vo = torch.empty_like(k), torch.empty_like(v)
    dst_pool.read_prefix(new, ko, vo)
    torch.cuda.synchronize()
    assert torch.equal(ko.view(torch.int16), k.view(torch.int16))
    assert torch.equal(vo.view(torch.int16), v.view(torch.int16))
    # decode the same requests against the clone: bit-identical outputs
    append_step(ld, wl, 0, DEV)
    plan = ld.pool.plan(ld.req_ids)
    q = wl.q(0, "cuda")
    o1 = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda")
    plan.run(2, q[2], o1)
    reqs2 = [dst_pool.open_request(new) for _ in range(wl.nreq)]
    sk, sv = wl.suffix_kv("cuda")
    dst_pool.append(reqs2, [r.suffix for r in wl.requests], sk, sv)
    nk, nv = wl.new_kv(0, "cuda")
    dst_pool.append(reqs2, [1] * wl.nreq, nk, nv)
    plan2 = dst_pool.plan(reqs2)
    o2 = torch.empty_like(o1)
    plan2.run(2, q[2], o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    plan.destroy()
    plan2.destroy()
    dst_pool.destroy()
    ld.pool.destroy()


def test_decode_layers_with_host_buffers_matches_device_path():
    wl = make_config("fanout", layers=2, nreq=64, prefix=300, suffix=10)
    ld = load(wl, DEV)
    append_step(ld, wl, 0, DEV)
    plan = ld.pool.plan(ld.req_ids)
    q = wl.q(0, "cuda")
    od = torch.empty((2, wl.nreq, wl.hq, wl.d), device="cuda")
    ld_ = torch.empty((2, wl.nreq, wl.hq), device="cuda")
    plan.run_layers(2, q, od, ld_)
    qh = q.cpu().pin_memory()
    oh = torch.empty((2, wl.nreq, wl.hq, wl.d)).pin_memory()
    lh = torch.empty((2, wl.nreq, wl.hq)).pin_memory()
    plan.run_layers(2, qh, oh, lh)
    torch.cuda.synchronize()
    assert torch.equal(oh, od.cpu()) and torch.equal(lh, ld_.cpu())
    plan.destroy()
    ld.pool.destroy()


def test_truncate_then_append_is_a_stationary_step():
    """The bench keeps the batch stationary: roll back the decoded token, append again."""
    wl = make_config("fanout", layers=1, nreq=64, prefix=256, suffix=31)
    ld, plan, out, lse = run_step(wl)
    ld.pool.truncate(ld.req_ids, [1] * wl.nreq)
    append_step(ld, wl, 0, DEV)
    plan = ld.pool.plan(ld.req_ids, reuse=plan)
    q = wl.q(0, "cuda")
    o2 = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda")
    plan.run(0, q[0], o2)
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), out[0])
    cleanup(ld, plan)


def _decode_step_outputs(wl, host: bool):
    ld = load(wl, DEV)
    nk, nv = wl.new_kv(0, f"cuda:{DEV}")
    q = wl.q(0, f"cuda:{DEV}")
    L = wl.layers
    if host:
        nk, nv, q = nk.cpu().pin_memory(), nv.cpu().pin_memory(), q.cpu().pin_memory()
        out = torch.full((L, wl.nreq, wl.hq, wl.d), float("nan")).pin_memory()
        lse = torch.full((L, wl.nreq, wl.hq), float("nan")).pin_memory()
    else:
        out = torch.full((L, wl.nreq, wl.hq, wl.d), float("nan"), device=f"cuda:{DEV}")
        lse = torch.full((L, wl.nreq, wl.hq), float("nan"), device=f"cuda:{DEV}")
    plan = ld.pool.decode_step(ld.req_ids, nk, nv, q, out, lse)
    torch.cuda.synchronize()
    o, l_ = out.cpu().numpy(), lse.cpu().numpy()
    return ld, plan, o, l_


@pytest.mark.parametrize("host,layers", [(True, 3), (False, 3), (True, 9)])
def test_decode_step_pipelined_matches_oracle_and_run(host, layers):
    """halo_decode_step (append + plan + every layer; host copies in 4-layer H2D / 2-layer
    D2H chunks overlapped with the kernels -- 9 layers leave partial chunks in both
    directions) equals the oracle and is bit-identical to append + plan + halo_decode_run."""
    wl = make_config("ragged", layers=layers)
    ld, plan, o, l_ = _decode_step_outputs(wl, host)
    for layer in range(wl.layers):
        ro, rl = oracle.decode_reference(wl, layer, steps=1)
        assert np.abs(o[layer] - ro).max() <= OUT_TOL
        assert np.abs(l_[layer] - rl).max() <= LSE_TOL
    cleanup(ld, plan)
    ld2, plan2, o2, l2 = run_step(wl)
    assert np.array_equal(o, o2) and np.array_equal(l_, l2)
    cleanup(ld2, plan2)


def test_decode_step_reuses_its_plan_across_steps():
    wl = make_config("fanout", layers=2, nreq=48, prefix=200, suffix=14)
    ld = load(wl, DEV)
    L = wl.layers
    outs = []
    plan = None
    for step in range(3):
        nk, nv = wl.new_kv(step, "cuda")
        q = wl.q(step, "cuda")
        out = torch.empty((L, wl.nreq, wl.hq, wl.d), device="cuda")
        plan = ld.pool.decode_step(ld.req_ids, nk, nv, q, out, reuse=plan)
        outs.append(out)
    torch.cuda.synchronize()
    for layer in range(L):
        ro, _ = oracle.decode_reference(wl, layer, steps=3)
        assert np.abs(outs[2][layer].cpu().numpy() - ro).max() <= OUT_TOL
    cleanup(ld, plan)


def test_full_c2_tree_at_bench_configuration():
    """C2 (BASELINE configs[2]): 4k root -> 16 x 1k roles -> 1024 requests, two prefix levels
    merged with the suffix; the per-layer shapes bench.py's other_configs leg times."""
    wl = make_config("tree", layers=2)
    check(wl, layers=[1])       # all 1024 requests


def test_full_c3_analytics_sampled_at_bench_configuration():
    """C3 per GPU (BASELINE configs[3]): 8 templates x 8k-token contexts x 256 requests."""
    wl = make_config("analytics", layers=1)
    # a seeded sample of 512 requests covering every template of the GPU (64 per template)
    rng = np.random.Generator(np.random.PCG64(3))
    sample = sorted(int(t * 256 + r) for t in range(8) for r in rng.choice(256, 64, replace=False))
    check(wl, layers=[0], sample=sample)


def test_continuous_batching_requests_join_and_leave_between_steps():
    """Continuous batching ("continuous batching ...
    early stops and early joins"): requests under two templates join and finish between
    decode steps; every step is one halo_decode_step over the active set (plan rebuilt in
    place), and every active request's output equals the oracle over its own context:
    prefix path + initial suffix + the tokens of the steps it took part in."""
    wl = make_config("ragged_suffix", layers=2, nreq=48, prefix=300, lo=1, hi=90)
    # two templates: re-parent half of the requests onto a second root node
    from synth.workloads import NodeSpec, RequestSpec, Workload
    nodes = [NodeSpec(0, -1, 300), NodeSpec(1, -1, 170)]
    reqs = [RequestSpec(r.ident, r.ident % 2, r.suffix) for r in wl.requests]
    wl = Workload("churn", 2, 32, 8, 128, nodes, reqs, wl.seed)
    rng = np.random.Generator(np.random.PCG64(11))
    join = rng.integers(0, 4, wl.nreq)             # step at which request r joins
    leave = join + rng.integers(1, 5, wl.nreq)     # first step it no longer takes part in
    pool = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, 4000, DEV)
    node_ids = {}
    for n in wl.nodes:
        k, v = wl.node_kv(n.ident, "cuda")
        node_ids[n.ident] = pool.register_prefix(-1, n.ntok, k, v)
    rid, taken = {}, {r: [] for r in range(wl.nreq)}
    plan = None
    nsteps = int(leave.max())
    for step in range(nsteps):
        for r in range(wl.nreq):
            if leave[r] == step and r in rid:
                pool.close_request(rid.pop(r))
            if join[r] == step:
                rid[r] = pool.open_request(node_ids[wl.requests[r].leaf])
                if wl.requests[r].suffix:
                    kv = [wl.suffix_kv("cuda", layer=l, request=r) for l in range(wl.layers)]
                    k = torch.stack([x[0] for x in kv]).contiguous()
                    v = torch.stack([x[1] for x in kv]).contiguous()
                    pool.append([rid[r]], [wl.requests[r].suffix], k, v)
        active = sorted(rid)
        if not active:
            continue
        nk, nv = wl.new_kv(step, "cuda")
        q = wl.q(step, "cuda")
        idx = torch.tensor(active, device="cuda")
        out = torch.empty((wl.layers, len(active), wl.hq, wl.d), device="cuda")
        lse = torch.empty((wl.layers, len(active), wl.hq), device="cuda")
        plan = pool.decode_step([rid[r] for r in active], nk[:, idx].contiguous(), nv[:, idx].contiguous(),
                                q[:, idx].contiguous(), out, lse, reuse=plan)
        torch.cuda.synchronize()
        for r in active:
            taken[r].append(step)
        o, l_ = out.cpu().numpy(), lse.cpu().numpy()
        for layer in range(wl.layers):
            for i, r in enumerate(active):
                kb, vb = oracle.request_context(wl, r, layer, steps=0)
                for s in taken[r]:
                    k1, v1 = wl.new_kv(s, "cpu", layer, request=r)
                    kb = np.concatenate([kb, oracle._bits(k1)[None]])
                    vb = np.concatenate([vb, oracle._bits(v1)[None]])
                qb = oracle._bits(wl.q(step, "cpu", layer, request=r))
                ro, rl = oracle.attend(qb, kb, vb, 1.0 / np.sqrt(wl.d))
                assert np.abs(o[layer, i] - ro).max() <= OUT_TOL, (step, layer, r)
                assert np.abs(l_[layer, i] - rl).max() <= LSE_TOL, (step, layer, r)
    if plan is not None:
        plan.destroy()
    pool.destroy()


@pytest.mark.parametrize("min_rows,lo", [(0, 1), (1, 1), (100000, 1), (1, 16)])
def test_prefill_against_cached_prefixes_matches_oracle(min_rows, lo):
    """halo_prefill_plan (NEXT-4): a burst of prompt tokens per request attends causally to
    itself after the cached prefix path; every token row vs the oracle over its context.
    lo=16: every prompt's causal part runs as K1 tiles, so the plan has no K2 blocks and the
    merge runs as K3 alone (merge_only_kernel)."""
    wl = make_config("ragged", layers=2)
    ld = load(wl, DEV)
    rng = np.random.Generator(np.random.PCG64(3))
    sel = [i for i in range(wl.nreq) if i % 3 == 0]
    nnew = [int(x) for x in rng.integers(lo, 40, len(sel))]
    # the prompt tokens of request r are the decode-step tokens 0..n-1 of the workload
    nkv = [wl.new_kv(s, "cuda") for s in range(max(nnew))]      # [L][R][Hkv][d] per step
    qs = [wl.q(s, "cuda") for s in range(max(nnew))]
    ks, vs = [], []
    for r, n in zip(sel, nnew):
        ks.append(torch.stack([nkv[s][0][:, r] for s in range(n)], dim=1))
        vs.append(torch.stack([nkv[s][1][:, r] for s in range(n)], dim=1))
    ld.pool.append([ld.req_ids[r] for r in sel], nnew, torch.cat(ks, 1).contiguous(), torch.cat(vs, 1).contiguous())
    plan = ld.pool.prefill_plan([ld.req_ids[r] for r in sel], nnew, opts(min_rows=min_rows))
    if lo == 16 and wl.hq // wl.hkv >= 4:
        assert len(plan.export("req_blk")) == 0  # K3 alone
    rows = sum(nnew)
    qrows = torch.cat([torch.stack([qs[s][:, r] for s in range(n)], dim=1)
                       for r, n in zip(sel, nnew)], 1).contiguous()      # [L][rows][Hq][d]
    out = torch.empty((wl.layers, rows, wl.hq, wl.d), device="cuda")
    lse = torch.empty((wl.layers, rows, wl.hq), device="cuda")
    for layer in range(wl.layers):
        plan.run(layer, qrows[layer], out[layer], lse[layer])
    torch.cuda.synchronize()
    o, l_ = out.cpu().numpy(), lse.cpu().numpy()
    for layer in range(wl.layers):
        row = 0
        for r, n in zip(sel, nnew):
            kb, vb = oracle.request_context(wl, r, layer, steps=0)
            for t in range(n):
                k1, v1 = wl.new_kv(t, "cpu", layer, request=r)
                kb = np.concatenate([kb, oracle._bits(k1)[None]])
                vb = np.concatenate([vb, oracle._bits(v1)[None]])
                qb = oracle._bits(wl.q(t, "cpu", layer, request=r))
                ro, rl = oracle.attend(qb, kb, vb, 1.0 / np.sqrt(wl.d))
                assert np.abs(o[layer, row] - ro).max() <= OUT_TOL, (layer, r, t)
                assert np.abs(l_[layer, row] - rl).max() <= LSE_TOL, (layer, r, t)
                row += 1
    cleanup(ld, plan)


@pytest.mark.parametrize("shape", [1, 2])
def test_k2_forced_launch_shapes_on_every_head_layout(shape):
    """The planner picks K2's narrow shape (7 warps x 4 stages) only for C1-like batches;
    force each shape (halo_plan_options.k2_shape) on ragged trees, d=64/128 and g=1/2/4/8,
    stream-K pieces included."""
    def o(min_rows=0):
        return PlanOptions(min_rows, 0, 0, 0, shape)
    check(make_config("ragged"), o(min_rows=16))
    check(make_config("ragged_suffix", layers=1, nreq=40, prefix=300, lo=1, hi=300), o())
    check(make_config("fanout", layers=1, nreq=40, prefix=260, suffix=9, hq=16, hkv=2), o())
    check(make_config("fanout", layers=1, nreq=70, prefix=333, suffix=17, hq=4, hkv=2, d=64), o())
    check(make_config("fanout", layers=1, nreq=130, prefix=260, suffix=9, hq=4, hkv=4), o(min_rows=1))


def test_plan_options_sm_cap_and_k1_rule():
    """k2_sms caps K2's grid (a co-scheduled kernel keeps SMs), k1_sm_frac < 0 turns the
    single-wave K1 rule off, k2_early_weight set explicitly: all still match the oracle."""
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=63)
    check(wl, PlanOptions(0, 0, 0, 0, 0, 100, 0.0, 0.0))
    check(wl, PlanOptions(0, 0, 0, 0, 0, 0, -1.0, 0.0))
    check(wl, PlanOptions(0, 0, 0, 0, 0, 0, 0.0, 1.5))


def test_maximum_sizes_long_prefix_and_long_suffix():
    """Edge sizes: a 32k-token prefix node (the largest node of BASELINE configs[4]; split
    into many K1 tiles), a 16k-token private suffix (the longest context of PAPER.md:685,
    one K2 unit cut into many stream-K pieces), requests without a prefix, and a 1-token
    suffix; sampled rows vs the oracle."""
    from synth.workloads import NodeSpec, RequestSpec, Workload
    nodes = [NodeSpec(0, -1, 32768), NodeSpec(1, -1, 1000)]
    reqs = [RequestSpec(i, 0, 7) for i in range(70)] + [RequestSpec(70, 1, 16383),
                                                       RequestSpec(71, -1, 16383),
                                                       RequestSpec(72, -1, 0),
                                                       RequestSpec(73, 0, 0)]
    wl = Workload("maxsize", 1, 32, 8, 128, nodes, reqs, 9)
    check(wl, sample=[0, 33, 69, 70, 71, 72, 73])


def test_decode_run_is_cuda_graph_capturable():
    """halo_decode_run is documented graph-capturable: capture two layers (K1 + K2 with
    programmatic dependent launches) in a CUDA graph, replay, compare with eager runs."""
    wl = make_config("fanout", layers=2, nreq=64, prefix=600, suffix=30)
    ld = load(wl, DEV)
    append_step(ld, wl, 0, DEV)
    plan = ld.pool.plan(ld.req_ids)
    q = wl.q(0, "cuda")
    eager = torch.empty((2, wl.nreq, wl.hq, wl.d), device="cuda")
    for l in range(2):
        plan.run(l, q[l], eager[l])
    torch.cuda.synchronize()
    out = torch.zeros_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for l in range(2):
                plan.run(l, q[l], out[l], stream=s)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
    del g
    cleanup(ld, plan)


def test_plan_is_stale_after_blocks_are_given_back():
    """A plan records block ids: closing a request (or truncating, releasing, moving) makes
    plans built before it stale -- halo_decode_run returns EBUSY until it is re-planned."""
    wl = make_config("fanout", layers=1, nreq=8, prefix=100, suffix=20)
    ld = load(wl, DEV)
    append_step(ld, wl, 0, DEV)
    plan = ld.pool.plan(ld.req_ids[:4])
    q = wl.q(0, "cuda")[0][:4].contiguous()
    out = torch.empty((4, wl.hq, wl.d), device="cuda")
    plan.run(0, q, out)
    ld.pool.close_request(ld.req_ids[7])
    with pytest.raises(halo.HaloError) as e:
        plan.run(0, q, out)
    assert e.value.name == "HALO_EBUSY"
    ld.pool.plan(ld.req_ids[:4], reuse=plan)
    plan.run(0, q, out)
    torch.cuda.synchronize()
    cleanup(ld, plan)


@pytest.mark.parametrize("whole", [0, -1])
def test_k2_alone_uses_the_equal_share_schedule_and_matches_oracle(whole):
    """With the K1/K2 co-schedule on (C1 shape), K2 launched by itself after K1
    (halo_decode_run_stages K1 then K2) runs the plan's K2-alone schedule (C1: whole units over
    the narrow shape, no stream-K pieces; k2_whole_units = -1: wide, equal shares), K1+K2
    launched together the weighted wide one with pieces; both match the oracle."""
    wl = make_config("fanout", layers=1, nreq=256, prefix=2048, suffix=255)
    ld = load(wl, DEV)
    append_step(ld, wl, 0, DEV)
    po = PlanOptions(0, 0, 0, 0)
    po.k2_whole_units = whole
    plan = ld.pool.plan(ld.req_ids, po)
    assert plan.info()["k1_tiles"] == 64
    q = wl.q(0, "cuda")
    o1 = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda")
    o2 = torch.empty_like(o1)
    plan.run(0, q[0], o1)
    plan.run_stages(0, 1, q[0], o2)
    plan.run_stages(0, 2, q[0], o2)
    torch.cuda.synchronize()
    ro, _ = oracle.decode_reference(wl, 0, steps=1, requests=list(range(0, wl.nreq, 5)))
    for o in (o1, o2):
        assert np.abs(o.cpu().numpy()[::5] - ro).max() <= OUT_TOL
    cleanup(ld, plan)


def test_stream_k_pieces_beside_a_long_k1_park_and_merge():
    """Units cut into several stream-K pieces (64 requests x 8 kv heads = 512 units of 17
    blocks for ~1776 warps) while K1 runs long (an 8k-token prefix): the unit's first piece
    merges once the other pieces arrived, parking its state when K1 is still running (merged
    after griddepcontrol.wait); two layers, every request vs the oracle, and a rerun of the
    same plan is bit-identical."""
    wl = make_config("fanout", layers=2, nreq=64, prefix=8192, suffix=255)
    ld, plan, out, lse = run_step(wl)
    for l in range(2):
        ro, rl = oracle.decode_reference(wl, l, steps=1)
        assert np.abs(out[l] - ro).max() <= OUT_TOL and np.abs(lse[l] - rl).max() <= LSE_TOL
    q = wl.q(0, f"cuda:{DEV}")
    o2 = torch.empty((wl.nreq, wl.hq, wl.d), device=f"cuda:{DEV}")
    l2 = torch.empty((wl.nreq, wl.hq), device=f"cuda:{DEV}")
    plan.run(1, q[1], o2, l2)
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), out[1]) and np.array_equal(l2.cpu().numpy(), lse[1])
    cleanup(ld, plan)


def test_decode_step_host_buffers_back_to_back_steps_match_oracle():
    """halo_decode_step with pinned HOST inputs and outputs, four steps issued back to back
    with no synchronisation in between (the input staging is double-buffered: a step's uploads
    overlap the previous step's last layers and downloads); every step's output vs the oracle."""
    wl = make_config("fanout", layers=3, nreq=40, prefix=150, suffix=20)
    ld = load(wl, DEV)
    L = wl.layers
    steps = 4
    ins, outs = [], []
    for step in range(steps):
        nk, nv = wl.new_kv(step, "cpu")
        q = wl.q(step, "cpu")
        ins.append((nk.pin_memory(), nv.pin_memory(), q.pin_memory()))
        outs.append(torch.empty((L, wl.nreq, wl.hq, wl.d)).pin_memory())
    plan = None
    for step in range(steps):
        nk, nv, q = ins[step]
        plan = ld.pool.decode_step(ld.req_ids, nk, nv, q, outs[step], reuse=plan)
    torch.cuda.synchronize()
    for step in range(steps):
        for layer in range(L):
            ro, _ = oracle.decode_reference(wl, layer, steps=step + 1)
            assert np.abs(outs[step][layer].numpy() - ro).max() <= OUT_TOL, (step, layer)
    cleanup(ld, plan)


def test_decode_step_and_decode_layers_share_staging_without_races():
    """A plan used by halo_decode_step (double-buffered input staging) and halo_decode_layers
    (which stages host q in buffer 0) in alternation, every call with pinned host buffers and
    no synchronisation in between: each call's outputs equal the device-buffer reference."""
    wl = make_config("fanout", layers=2, nreq=32, prefix=120, suffix=12)
    ld = load(wl, DEV)
    L = wl.layers
    plan = None
    ins, outs = [], []
    for step in range(3):
        nk, nv = wl.new_kv(step, "cpu")
        q = wl.q(step, "cpu")
        ins.append((nk.pin_memory(), nv.pin_memory(), q.pin_memory()))
        outs.append((torch.empty((L, wl.nreq, wl.hq, wl.d)).pin_memory(),
                     torch.empty((L, wl.nreq, wl.hq, wl.d)).pin_memory()))
    for step in range(3):
        nk, nv, q = ins[step]
        plan = ld.pool.decode_step(ld.req_ids, nk, nv, q, outs[step][0], reuse=plan)
        plan.run_layers(L, q, outs[step][1])  # the same step's layers again through decode_layers
    torch.cuda.synchronize()
    for step in range(3):
        assert torch.equal(outs[step][0], outs[step][1]), step
        for layer in range(L):
            ro, _ = oracle.decode_reference(wl, layer, steps=step + 1)
            assert np.abs(outs[step][0][layer].numpy() - ro).max() <= OUT_TOL, (step, layer)
    cleanup(ld, plan)
