#!/usr/bin/env python
"""bench.py -- shared-prefix decode attention on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C1"): Llama-3-8B GQA (32 q / 8 kv heads, d=128, bf16
KV in 16-token paged blocks), 256 requests fanned out from one 2,048-token workflow-template
prefix, 256-token private suffixes, 32 layers, one B200 per rank.  Synthetic seeded data
(synth/), resident in HBM before the timed region.

A STEP is one decode step of the whole hot path over the batch:
  roll back last step's token (host bookkeeping) + append this step's token K/V for all 32
  layers (K5) + plan (host, uploaded) + for each of 32 layers: K1 (tcgen05 prefix
  attention over the shared node) and K2+K3 (paged suffix decode + LSE merge).
queries/s = requests x layers x steps / time  (1 query = one request's decode attention at
one layer over all its heads; SURVEY.md §8(c) reading 13).

N>1 (torchrun): weak scaling -- every rank runs its own independent C1 batch (request groups
partition across GPUs with no exchange on the attention path); time = max
over ranks.  KV migration (K4 pack + NCCL send/recv + K4 unpack) is measured in the same run
and reported under "migration" (N=1: same-GPU relocation through K4, no NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "shared-prefix decode attn queries/s; HBM GB/s & TC util vs peak; KV migrate GB/s"
UNIT = "queries/s"
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback
FALLBACK_BF16_TFLOPS = 1590.0
NVLINK_PEER_GBS = 770.0     # B200_PROFILING.md: measured peer copy per direction
TIMING_NOTE = ("CUDA events on the launching stream around every launch of the kernel, averaged "
               "over the K-step breakdown pass (same workload, right after the headline pass)")


def gate(torch, cycles=6_000_000):
    """Hold the stream for ~3 ms (a spin kernel) while the host enqueues a timed sequence, so no
    event interval holds host enqueue latency; a no-op where torch has no spin kernel."""
    if hasattr(torch.cuda, "_sleep"):
        torch.cuda._sleep(cycles)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", FALLBACK_HBM_GBS), d.get("bf16_tflops", FALLBACK_BF16_TFLOPS), \
            d.get("bf16_tflops_sustained"), "measured (MEASURED_PEAKS.json)"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in self.rows if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].startswith("Active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(self.rows[0][1]), "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((num(r[2]) or 0) for r in self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ oracle (CPU) legs
def oracle_sample(wl, budget_s: float, max_queries: int = 100000):
    """Time the fp64 oracle (as it stands) on a bounded sample of the same workload:
    (request, layer) queries in order, contexts gathered outside the timer, until
    `budget_s` seconds of oracle compute."""
    import numpy as np
    import oracle
    nthreads = host_cores()
    scale = 1.0 / np.sqrt(wl.d)
    t_total, done = 0.0, 0
    cache = {}
    for i in range(min(wl.nreq * wl.layers, max_queries)):
        layer, r = divmod(i, wl.nreq)
        k, v = oracle.request_context(wl, r, layer, steps=1, cache=cache)
        qb = oracle._bits(wl.q(0, "cpu", layer, request=r))
        t0 = time.perf_counter()
        oracle.attend(qb, k, v, scale, nthreads)
        t_total += time.perf_counter() - t0
        done += 1
        if t_total >= budget_s:
            break
    return done, t_total, nthreads


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle; the others exit 0 without work
    from synth import make_config
    wl = make_config(args.config)
    # each step = the oracle on a bounded sample (8 requests, layer 0)
    import numpy as np
    import oracle
    nthreads = host_cores()
    scale = 1.0 / np.sqrt(wl.d)
    ctx = []
    for r in range(8):
        k, v = oracle.request_context(wl, r, 0, steps=1)
        ctx.append((oracle._bits(wl.q(0, "cpu", 0, request=r)), k, v))

    def step():
        for qb, k, v in ctx:
            oracle.attend(qb, k, v, scale, nthreads)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = len(ctx) * args.steps / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator, synth/)",
        "config": {"workload": "C1 fanout: 256 req x 2048-token shared prefix + 256-token suffix, "
                               "Llama-3-8B GQA 32q/8kv d128, 32 layers",
                   "sample": "8 requests x layer 0 per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                         "sample": "8 requests of C1 at layer 0 per step (unshared fp64 attention)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ GPU leg
def setup_workload(halo, wl, dev, torch):
    """Load `wl` into a fresh pool (inputs resident in HBM), append this step's token, plan.
    Returns the loaded pool, the plan, its info and the step closure."""
    from paper_2509_02121_b200.loader import blocks_needed, load
    L, R, Hq, D = wl.layers, wl.nreq, wl.hq, wl.d
    ld = load(wl, dev, capacity=blocks_needed(wl, steps=2, slack=4096))
    pool, reqs = ld.pool, ld.req_ids
    nk, nv = wl.new_kv(0, f"cuda:{dev}")            # [L][R][Hkv][D] this step's token
    q = wl.q(0, f"cuda:{dev}")                      # [L][R][Hq][D]
    out = torch.empty((L, R, Hq, D), device=f"cuda:{dev}")
    lse = torch.empty((L, R, Hq), device=f"cuda:{dev}")
    ones = [1] * R
    pool.append(reqs, ones, nk, nv)
    # plan options (defaults; the env knobs are for A/B runs of bench.py only)
    popt = halo.PlanOptions(0, 0, int(os.environ.get("HALO_MAX_SPLITS", "0")), int(os.environ.get("HALO_K2_CHUNK", "0")))
    popt.k2_tail_pct = int(os.environ.get("HALO_K2_TAIL", "0"))
    plan = pool.plan(reqs, popt)
    info = plan.info()
    stream = torch.cuda.current_stream()

    def step(evs=None):
        pool.truncate(reqs, ones)                 # stationary batch: roll back, re-append
        pool.append(reqs, ones, nk, nv)
        pool.plan(reqs, popt, reuse=plan)
        if evs is not None:
            # breakdown pass: hold the stream (a ~3 ms spin kernel, outside every event pair)
            # while the host enqueues the step's 32 x (event, K1, event, K2, event), so no
            # interval between two events contains host enqueue latency
            if os.environ.get('HALO_BENCH_GATE', '1') == '1':
                gate(torch)
        for l in range(L):
            if evs is None:                       # headline pass: K1 -> K2 back to back (PDL)
                plan.run(l, q[l], out[l], lse[l])
                continue
            evs[l][0].record(stream)              # breakdown pass: an event around each kernel
            plan.run_stages(l, 1, q[l], out[l], lse[l])
            evs[l][1].record(stream)
            plan.run_stages(l, 2, q[l], out[l], lse[l])
            evs[l][2].record(stream)
    return ld, plan, info, step, (nk, nv, q, out, lse, ones, popt)


def time_steps(step, L, steps, warmup, world, dev, torch, dist, sample_clocks=False):
    """W untimed steps, then two timed passes of K steps, each between barriers + syncs with
    CUDA events on the launching stream, max over ranks:
      1. the headline pass: whole steps only (K1 and K2 of a layer back to back, so K2's
         programmatic dependent launch overlaps K1's tail);
      2. the breakdown pass: an event before K1, between K1 and K2 and after K2 of every
         layer (per-kernel launch durations for the rooflines; the events serialise the
         kernels, so this pass is a little slower than the first).  Each step's layers are
         enqueued behind a spin kernel, so no event interval holds host enqueue latency.
    Returns (pass-1 ms, pass-2 ms of the steps' layer spans, pass-2 K1 ms, pass-2 K2 ms,
    clock sampler)."""
    stream = torch.cuda.current_stream()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(L)]
           for _ in range(steps)]
    for w in range(warmup):
        # the last warm-up step runs the breakdown pass's launch sequence (K2 launched alone
        # uses the plan's K2-alone schedule, possibly another kernel instantiation): with lazy
        # module loading its first launch would otherwise load the kernel inside a timed
        # event interval (a 10-80 ms stall once per process)
        step(evs[0] if w == warmup - 1 else None)
    torch.cuda.synchronize()
    t = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    clk = ClockSampler(dev) if sample_clocks else None
    if clk:
        clk.__enter__()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]  # headline step edges
    for p in range(2):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t[2 * p].record(stream)
        for s in range(steps):
            if p == 0:
                marks[s].record(stream)
            step(evs[s] if p == 1 else None)
        if p == 0:
            marks[steps].record(stream)
        t[2 * p + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    if clk:
        clk.__exit__()
    ms = t[0].elapsed_time(t[1])
    ms_bd = sum(st[0][0].elapsed_time(st[L - 1][2]) for st in evs)  # first K1 .. last K2
    per_step = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(steps))
    time_steps.step_stats = {"median": per_step[len(per_step) // 2],
                             "p90": per_step[min(len(per_step) - 1, (9 * len(per_step)) // 10)],
                             "min": per_step[0], "max": per_step[-1], "rank": "this rank (rank 0)"}
    k1_ms = sum(e[0].elapsed_time(e[1]) for st in evs for e in st)
    k2_ms = sum(e[1].elapsed_time(e[2]) for st in evs for e in st)
    from paper_2509_02121_b200.sharding import max_over_ranks
    ms, ms_bd, k1_ms, k2_ms = max_over_ranks([ms, ms_bd, k1_ms, k2_ms], dist if world > 1 else None,
                                             f"cuda:{dev}")
    return ms, ms_bd, k1_ms, k2_ms, clk


def kernel_rooflines(info, k1_launch_ms, k2_launch_ms):
    hbm_peak, tc_peak, tc_sust, peak_src = peaks()
    k2_gbs = info["k2_bytes"] / (k2_launch_ms * 1e-3) / 1e9
    k1_tflops = info["k1_flops"] / (k1_launch_ms * 1e-3) / 1e12 if info["k1_flops"] else None
    return ({"bound": "hbm", "kernel": "suffix_decode_kernel (K2+K3)", "achieved": k2_gbs,
             "peak": hbm_peak, "unit": "GB/s", "frac": k2_gbs / hbm_peak,
             "algorithmic_bytes_per_launch": info["k2_bytes"], "avg_launch_ms": k2_launch_ms,
             "timing": TIMING_NOTE, "peak_source": peak_src},
            {"bound": "tensor", "kernel": "prefix_attn_kernel (K1)", "achieved": k1_tflops,
             "peak": tc_peak, "unit": "TFLOP/s", "frac": (k1_tflops / tc_peak) if k1_tflops else None,
             "algorithmic_flops_per_launch": info["k1_flops"], "avg_launch_ms": k1_launch_ms,
             "timing": TIMING_NOTE, "peak_source": peak_src,
             # K1 runs inside a long step at the chip's power cap: the sustained cuBLAS rate
             # (back to back for 4 s, MEASURED_PEAKS.json) is the like-for-like denominator
             "peak_sustained": tc_sust,
             "frac_sustained": (k1_tflops / tc_sust) if (k1_tflops and tc_sust) else None})


def measure_other_configs(halo, names, layers, steps, warmup, world, dev, torch, dist):
    """Per-launch K1/K2 rooflines on the other BASELINE configs (C2 tree, C3 analytics per
    GPU) with `layers` layers: same kernels and plan as C1; the per-layer work (and so the
    per-launch rooflines) is that of the full 32-layer config."""
    from synth import make_config
    res = {}
    for name in names:
        wl = make_config(name, layers=layers)
        ld, plan, info, step, bufs = setup_workload(halo, wl, dev, torch)
        ms, _, k1_ms, k2_ms, _ = time_steps(step, wl.layers, steps, warmup, world, dev, torch, dist)
        n = steps * wl.layers
        k2r, k1r = kernel_rooflines(info, k1_ms / n, k2_ms / n)
        layer_ms = (k1_ms + k2_ms) / n
        res[name] = {"requests": wl.nreq, "layers_run": wl.layers,
                     "prefix_nodes": len(wl.nodes), "k1_tiles": info["k1_tiles"],
                     "k2_units": info["k2_units"], "layer_ms": layer_ms,
                     "queries_per_s_kernels": wl.nreq / (layer_ms * 1e-3),
                     "roofline": k2r, "prefix_roofline": k1r,
                     "unshared_bytes_per_layer": info["unshared_bytes"]}
        plan.destroy()
        ld.pool.destroy()
        del bufs, step
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    return res


def measure_placed_c3(halo, layers, steps, warmup, world, rank, dev, torch, dist, link_gbs, nccl_ok):
    """BASELINE configs[3] (C3 batch analytics: 64 templates x 8k-token contexts, 256 requests
    each, over 8 GPUs "with cross-GPU prefix placement") at this N: 8 templates per GPU.  Each
    template's KV starts on GPU t % N (prefilled where it arrived); the relocation planner
    (halo_place_groups, Alg. 1 with the §3.2 costs) places the templates over the
    GPUs; the moves run through halo_migrate_exchange (NCCL) before the timed steps; then every
    GPU decodes the requests of the templates it holds (no exchange on the attention path).
    Aggregate queries/s = all requests x layers / max-over-ranks time."""
    from paper_2509_02121_b200.loader import blocks_needed
    from paper_2509_02121_b200.relocation import plan_relocation, rank_actions
    from synth import make_config
    T = 8 * world
    wl = make_config("analytics", templates=T, layers=layers)
    hbm, tc = peaks()[:2]
    homes = [0] * T
    groups, items, res = plan_relocation(wl, homes, workers=world, link_bytes_per_s=link_gbs * 1e9,
                                         beam_width=16, steps=256, tc_flops=tc * 1e12, hbm_bps=hbm * 1e9)
    held0 = [t for t in range(T) if homes[t] == rank]
    moves_ok = world == 1 or nccl_ok
    mine_after = [t for t in range(T) if res["masks"][t] >> rank & 1] if moves_ok else held0
    cap = sum((wl.nodes[t].ntok + 15) // 16 for t in set(held0) | set(mine_after))
    cap += sum((r.suffix + 2 + 15) // 16 for r in wl.requests if r.leaf in set(mine_after)) + 64
    pool = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, cap, dev)
    node = {}
    for t in held0:
        k, v = wl.node_kv(t, f"cuda:{dev}")
        node[t] = pool.register_prefix(-1, wl.nodes[t].ntok, k, v)
        del k, v
    torch.cuda.synchronize()
    moved_bytes, mig_ms = 0.0, 0.0
    acts = rank_actions(res["moves"], rank)
    if acts and world > 1:
        if moves_ok:
            uid = halo.comm_unique_id() if rank == 0 else b"\0" * 128
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            pool.comm_init(obj[0], world, rank)
            sends = [(node[it], dst, mode) for kind, it, *r in acts if kind == "send" for dst, mode in [r]]
            recv_items = [it for kind, it, *r in acts if kind == "recv"]
            recvs = [(r[0], -1, wl.nodes[it].ntok) for kind, it, *r in acts if kind == "recv"]
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            got = pool.migrate_exchange(sends=sends, recvs=recvs)
            e1.record()
            torch.cuda.synchronize()
            mig_ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{dev}")
            dist.all_reduce(mig_ms, op=dist.ReduceOp.MAX)
            mig_ms = mig_ms.item()
            for kind, it, *r in acts:
                if kind == "send" and r[1] == 0:
                    node.pop(it)
            for it, nid in zip(recv_items, got):
                node[it] = nid
            moved_bytes = sum(items[m[0]]["kv_bytes"] for m in res["moves"] if m[1] >= 0)
    reqs, idx = [], []
    for i, r in enumerate(wl.requests):
        if r.leaf in node and r.leaf in set(mine_after):
            reqs.append(pool.open_request(node[r.leaf]))
            idx.append(i)
    R = len(reqs)
    plan = None
    stream = torch.cuda.current_stream()
    if R:
        from synth.workloads import RequestSpec, Workload
        # this rank's requests (their initial suffixes and the step's token), resident in HBM
        sub = Workload("c3_shard", wl.layers, wl.hq, wl.hkv, wl.d, [], [RequestSpec(j, -1, wl.requests[i].suffix)
                       for j, i in enumerate(idx)], seed=wl.seed + 7)
        sk, sv = sub.suffix_kv(f"cuda:{dev}")
        pool.append(reqs, [wl.requests[i].suffix for i in idx], sk, sv)
        nk, nv = sub.new_kv(0, f"cuda:{dev}")
        pool.append(reqs, [1] * R, nk, nv)
        del sk, sv
        q = sub.q(0, f"cuda:{dev}")
        o = torch.empty((wl.layers, R, wl.hq, wl.d), device=f"cuda:{dev}")
        plan = pool.plan(reqs)

    def run_layers(evs=None):
        for l in range(wl.layers):
            if evs is not None:
                evs[l][0].record(stream)
            if plan is not None:
                plan.run_stages(l, 1, q[l], o[l]) if evs is not None else plan.run(l, q[l], o[l])
            if evs is not None:
                evs[l][1].record(stream)
                if plan is not None:
                    plan.run_stages(l, 2, q[l], o[l])
                evs[l][2].record(stream)
    ms, _, _, _, _ = time_steps(run_layers, wl.layers, steps, warmup, world, dev, torch, dist)
    if plan is not None:
        plan.destroy()
    from paper_2509_02121_b200.sharding import max_over_ranks
    step_ms = ms / steps  # (time_steps already reduced it over the ranks)
    out = {"workload": f"C3 batch analytics: {T} templates x 8192-token contexts x 256 requests, "
                       f"{layers} layers, relocation planner placement over {world} GPU(s)",
           "value": wl.nreq * wl.layers / (step_ms * 1e-3) if step_ms > 0 else None, "unit": "queries/s",
           "ms_per_step": step_ms, "templates_here": len(mine_after), "requests_here": R,
           "moves": len(res["moves"]), "bytes_moved": moved_bytes, "migration_ms": mig_ms,
           "migration_GB/s": moved_bytes / world / mig_ms / 1e6 if mig_ms > 0 else None,
           "planner_cost_s": res["cost"], "scaling": "weak",
           "placement": "relocation planner" if moves_ok else "home GPUs (gloo dry run: moves need NCCL)"}
    pool.destroy()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def measure_strong_scaling(halo, layers, steps, warmup, world, rank, dev, torch, dist):
    """C2 (consolidated agent-DAG tree: 4k root -> 16 roles x 1k -> 1024 requests) with the
    8 kv heads split 8/N per rank: every rank runs the same plan on its head slice (no
    exchange step), so the total work is fixed as N grows.  Headline-pass timing (K1 -> K2
    with PDL, the plan built once), max over ranks; queries/s = 1024 requests x layers /
    time of the layers."""
    from paper_2509_02121_b200.sharding import head_range, head_shard_workload
    from synth import make_config
    full = make_config("tree", layers=layers)
    wl = head_shard_workload(full, world, rank)
    ld, plan, info, step, bufs = setup_workload(halo, wl, dev, torch)
    q, out, lse = bufs[2], bufs[3], bufs[4]

    stream = torch.cuda.current_stream()

    def run_layers(evs=None):  # the layers only: with 4 layers the per-step host plan would dominate
        for l in range(wl.layers):
            if evs is None:
                plan.run(l, q[l], out[l], lse[l])
                continue
            evs[l][0].record(stream)
            plan.run_stages(l, 1, q[l], out[l], lse[l])
            evs[l][1].record(stream)
            plan.run_stages(l, 2, q[l], out[l], lse[l])
            evs[l][2].record(stream)
    ms, _, _, _, _ = time_steps(run_layers, wl.layers, steps, warmup, world, dev, torch, dist)
    ms /= steps
    lo, hi = head_range(full.hkv, world, rank)
    res = {"workload": f"C2 tree, 1024 requests, kv heads sharded {full.hkv // world} per GPU "
                       f"(total work fixed as N grows), {layers} layers",
           "value": full.nreq * wl.layers / (ms * 1e-3), "unit": "queries/s",
           "ms_per_step": ms, "n_gpus": world, "kv_heads_per_gpu": hi - lo,
           "scaling": "strong"}
    plan.destroy()
    ld.pool.destroy()
    del bufs, step
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="halo", choices=["halo", "reference"])
    ap.add_argument("--config", default="fanout")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-migration", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--other-configs", default="tree,tree_root,tree_roles,analytics",
                    help="BASELINE configs also measured per launch (C2 tree, C3 analytics); '' = none")
    ap.add_argument("--other-layers", type=int, default=4)
    ap.add_argument("--strong-layers", type=int, default=32, help="layers of the C2 strong-scaling leg")
    ap.add_argument("--layers", type=int, default=0, help="override the config's layer count (profiling)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: debug the N>1 path with several ranks on one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (rank 0 prints the line)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if int(os.environ.get("WORLD_SIZE", 1)) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', 1)}")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2509_02121_b200 as halo
    from paper_2509_02121_b200.loader import blocks_needed, load
    from synth import make_config

    rank, world, local = dist_env()
    # --dist-backend gloo (debug): exercise the multi-rank code path with several ranks on
    # one GPU (NCCL refuses two ranks per device); the NCCL migration leg is skipped then.
    dev = local % torch.cuda.device_count() if args.dist_backend == "gloo" else local
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
            args.no_migration = True
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    halo.load_library()

    wl = make_config(args.config, seed=1 + 1000 * rank, **({"layers": args.layers} if args.layers else {}))
    L, R, Hq, Hkv, D = wl.layers, wl.nreq, wl.hq, wl.hkv, wl.d
    ld, plan, info, step, (nk, nv, q, out, lse, ones, popt) = setup_workload(halo, wl, dev, torch)
    pool, reqs = ld.pool, ld.req_ids
    stream = torch.cuda.current_stream()
    ms, ms_bd, k1_ms, k2_ms, clk = time_steps(step, L, args.steps, args.warmup, world, dev, torch, dist,
                                       sample_clocks=True)
    step_stats = dict(time_steps.step_stats)  # the headline pass (later legs re-time)
    launches = args.steps * (3 + 2 * L)  # per step: slot upload + K5 append, plan upload, L x (K1, K2)
    ms_step = ms / args.steps
    value = R * L * world * args.steps / (ms / 1e3)

    k2_launch_ms = k2_ms / (args.steps * L)
    k1_launch_ms = k1_ms / (args.steps * L)
    k2_roof, k1_roof = kernel_rooflines(info, k1_launch_ms, k2_launch_ms)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    if k1_roof.get("frac") and 0 < info["k1_tiles"] < nsm:
        # C1's K1 is planned as one partial wave (the co-schedule leaves the other SMs to K2):
        # the rate per SM it occupies, for comparison with the multi-wave configs
        k1_roof["note"] = (f"single partial wave of {info['k1_tiles']} CTAs on {nsm} SMs by design "
                           f"(K2 streams on the rest); frac_per_occupied_sm = frac x {nsm}/{info['k1_tiles']}")
        k1_roof["frac_per_occupied_sm"] = k1_roof["frac"] * nsm / info["k1_tiles"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("suffix_decode_kernel", {}).get("dram_bytes_per_launch")

    extra = {}

    def guarded(key, fn):
        """The secondary legs must not cost the headline line: a failure is reported in place."""
        try:
            extra[key] = fn()
        except Exception as e:  # noqa: BLE001
            extra[key] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.synchronize()
    # ---- K2 alone with the wide stream-K schedule and equal per-warp shares (co-schedule
    # weights off, same K1 splits), for comparison: the breakdown pass above runs K2 alone
    # with the plan's K2-alone schedule (C1: whole units over the narrow shape) ----
    if not args.profile:
        def k2_equal():
            eopt = halo.PlanOptions(0, 0, int(os.environ.get("HALO_MAX_SPLITS", "0")), 0)
            eopt.k2_early_weight = 1.0
            ep = pool.plan(reqs, eopt)
            einfo = ep.info()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
            for rep in range(4):
                if rep == 3:
                    gate(torch)  # the timed layers enqueued behind a spin kernel
                for l in range(L):
                    ep.run_stages(l, 1, q[l], out[l], lse[l])
                    if rep == 3:
                        evs[l][0].record(stream)
                    ep.run_stages(l, 2, q[l], out[l], lse[l])
                    if rep == 3:
                        evs[l][1].record(stream)
            torch.cuda.synchronize()
            k2ms = sum(a.elapsed_time(b) for a, b in evs) / L
            ep.destroy()
            r = kernel_rooflines(einfo, k1_launch_ms, k2ms)[0]
            r["timing"] = ("CUDA events around each K2 launch (K1 before it, serialised), 32 layers; "
                           "wide shape, stream-K pieces, equal shares")
            return r
        guarded("roofline_k2_equal_shares", k2_equal)
        hbm_peak = peaks()[0]
        lay_bytes = info["k2_bytes"] + info["k1_bytes"]
        lay_ms = ms_step / L
        extra["layer_roofline"] = {"bound": "hbm", "what": "K1 + K2 algorithmic bytes per layer / headline "
                                   "time per layer (the kernels overlap under PDL)", "achieved": lay_bytes / lay_ms / 1e6,
                                   "peak": hbm_peak, "unit": "GB/s", "frac": lay_bytes / lay_ms / 1e6 / hbm_peak}
    # ---- e2e: the public API with HOST buffers (pinned), copies inside the timed region ----
    if not args.no_e2e and not args.profile:
        nk_h, nv_h = nk.cpu().pin_memory(), nv.cpu().pin_memory()
        q_h = q.cpu().pin_memory()
        out_h = torch.empty((L, R, Hq, D), pin_memory=True)
        e2e_steps = min(args.steps, 30)

        def e2e_step():
            pool.truncate(reqs, ones)             # stationary batch (host bookkeeping only)
            pool.decode_step(reqs, nk_h, nv_h, q_h, out_h, options=popt, reuse=plan)
        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        from paper_2509_02121_b200.sharding import max_over_ranks
        dt = max_over_ranks([dt], dist if world > 1 else None, f"cuda:{dev}")[0]
        h2d = nk_h.numel() * 2 * 2 + q_h.numel() * 2
        d2h = out_h.numel() * 4
        extra["e2e"] = {"value": R * L * world * e2e_steps / dt, "unit": UNIT,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "steps": e2e_steps, "how": "halo_decode_step (append one token per request + "
                        "plan + all layers; H2D in 4-layer and D2H in 2-layer chunks on library "
                        "copy streams, overlapped with the kernels) with pinned host buffers; "
                        "wall clock after sync"}
    if world > 1 and args.dist_backend == "gloo":
        extra["migration"] = {"skipped": "NCCL needs one GPU per rank (gloo dry run of the N>1 path)"}
        extra["paging"] = {"skipped": "gloo dry run"}
    # ---- migration (K4 + NCCL), measured in the same run ----
    if not args.no_migration and not args.profile:
        guarded("migration", lambda: measure_migration(halo, pool, ld, wl, world, rank, dev, torch, dist,
                                                       decode_step=step))
    # ---- host paging of the template node (NEXT-2) ----
    if not args.no_migration and not args.profile:
        guarded("paging", lambda: measure_paging(pool, ld, wl, torch, decode_step=step))
    # ---- cost-model relocation planner (NEXT-1), host-side ----
    if not args.profile:
        guarded("relocation", lambda: measure_relocation(halo, extra.get("migration", {})))
    # ---- continuous batching under churn (NEXT-3) ----
    if not args.no_e2e and not args.profile:
        guarded("continuous", lambda: measure_continuous(halo, wl, dev, torch, min(args.steps, 30)))
    # ---- shared-prefix prefill (NEXT-4) ----
    if not args.no_e2e and not args.profile:
        guarded("prefill", lambda: measure_prefill(halo, dev, torch, steps=min(args.steps, 10)))
    # ---- per-launch rooflines on the other configs (C2, C3) ----
    if args.other_configs and not args.profile:
        guarded("other_configs", lambda: measure_other_configs(
            halo, [x for x in args.other_configs.split(",") if x], args.other_layers,
            max(3, min(args.steps, 10)), 3, world, dev, torch, dist))
    # ---- strong scaling: C2 with its kv heads sharded over the ranks ----
    if args.other_configs and not args.profile:
        guarded("strong_scaling", lambda: measure_strong_scaling(
            halo, args.strong_layers, max(3, min(args.steps, 10)), 3, world, rank, dev, torch, dist))
    # ---- C3 with the relocation planner's placement (BASELINE configs[3]) ----
    if args.other_configs and not args.profile:
        link = NVLINK_PEER_GBS
        for e in extra.get("migration", {}).get("sweep", []) if isinstance(extra.get("migration"), dict) else []:
            if e.get("pairs_0_to_k"):
                link = e["pairs_0_to_k"][0]["GB/s"]
        guarded("c3_placed", lambda: measure_placed_c3(
            halo, args.other_layers, max(3, min(args.steps, 10)), 3, world, rank, dev, torch, dist, link,
            nccl_ok=world > 1 and args.dist_backend == "nccl"))
    # ---- CPU oracle baseline ----
    if rank == 0 and not args.no_cpu_baseline and not args.profile:
        n, t, cores = oracle_sample(wl, args.cpu_budget)
        extra["cpu_baseline"] = {"value": n / t, "unit": UNIT, "cores": cores, "kind": "oracle",
                                 "sample": f"first {n} (request, layer) queries of C1 (unshared "
                                           f"fp64 attention over 2304 tokens x 32 heads each), "
                                           f"{t:.1f} s of oracle time", "cpu_model": cpu_model()}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based generator, synth/); no weights needed",
            "config": {"workload": "C1 fanout: 256 req x 2048-token shared prefix + 256-token "
                                   "suffix, Llama-3-8B GQA 32q/8kv d128, 32 layers, 16-token blocks",
                       "requests_per_gpu": R, "layers": L, "prefix_tokens": wl.nodes[0].ntok,
                       "suffix_tokens": wl.requests[0].suffix + 1,
                       "parallelism": f"request-group sharding x{world} (no collective)",
                       "l2": "inputs exceed L2 (8.3 GiB KV touched per step vs 126 MB L2)",
                       "k1_tiles": info["k1_tiles"], "k2_units": info["k2_units"]},
            "roofline": dict(k2_roof, traffic=traffic),
            "prefix_roofline": k1_roof,
            "step_ms_distribution": step_stats,
            "step_breakdown_ms": {"pass": "breakdown pass (events around each kernel; K1 and K2 "
                                          "serialised; append + plan not included)",
                                  "layers": ms_bd / args.steps, "k1": k1_ms / args.steps,
                                  "k2": k2_ms / args.steps,
                                  "gaps": (ms_bd - k1_ms - k2_ms) / args.steps},
            "unshared_bytes_per_layer": info["unshared_bytes"],
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    plan.destroy()
    pool.destroy()
    if world > 1:
        dist.destroy_process_group()


def measure_prefill(halo, dev, torch, steps=10, prompt=64, layers=4):
    """Prefill of a `prompt`-token task prompt for each of the 256 C1 requests against the
    cached 2048-token template (halo_prefill_plan + halo_decode_run per layer): 16,384 query
    rows per kv head through K1 (tensor cores over the shared prefix) and the causal prompt
    part in K2.  Per-kernel CUDA events; `layers` layers (per-layer work of the full model)."""
    from paper_2509_02121_b200.loader import blocks_needed, load
    from synth import make_config
    wl = make_config("fanout", layers=layers, suffix=0)
    R, L = wl.nreq, wl.layers
    ld = load(wl, dev, capacity=blocks_needed(wl, steps=prompt + 2, slack=4096))
    pool = ld.pool
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(7)
    k = (torch.randn((L, R * prompt, wl.hkv, wl.d), device=f"cuda:{dev}", generator=g)).bfloat16()
    v = (torch.randn((L, R * prompt, wl.hkv, wl.d), device=f"cuda:{dev}", generator=g)).bfloat16()
    q = (torch.randn((L, R * prompt, wl.hq, wl.d), device=f"cuda:{dev}", generator=g)).bfloat16()
    out = torch.empty((L, R * prompt, wl.hq, wl.d), device=f"cuda:{dev}")
    pool.append(ld.req_ids, [prompt] * R, k, v)
    plan = pool.prefill_plan(ld.req_ids, [prompt] * R)
    info = plan.info()
    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps * L)]
    for _ in range(2):
        for l in range(L):
            plan.run(l, q[l], out[l])
    torch.cuda.synchronize()
    i = 0
    for _ in range(steps):
        for l in range(L):
            ev[i][0].record(stream)
            plan.run_stages(l, 1, q[l], out[l])
            ev[i][1].record(stream)
            plan.run_stages(l, 2, q[l], out[l])
            ev[i][2].record(stream)
            i += 1
    torch.cuda.synchronize()
    n = steps * L
    k1 = sum(e[0].elapsed_time(e[1]) for e in ev) / n
    k2 = sum(e[1].elapsed_time(e[2]) for e in ev) / n
    k2r, k1r = kernel_rooflines(info, k1, k2)
    if len(plan.export("req_blk")) == 0:  # every causal part in K1: the merge runs as K3 alone
        k2r["kernel"] = "merge_only_kernel (K3 alone: no suffix blocks in the plan)"
    plan.destroy()
    pool.destroy()
    return {"what": f"prefill of a {prompt}-token prompt for each of {R} requests against the cached "
                    f"{wl.nodes[0].ntok}-token template (rows = {R * prompt} tokens x {wl.hq} q-heads)",
            "layer_ms": k1 + k2, "tokens_per_s": R * prompt / ((k1 + k2) * 1e-3),
            "prefix_roofline": k1r, "suffix_roofline": k2r, "k1_tiles": info["k1_tiles"]}


def measure_continuous(halo, wl, dev, torch, steps, churn=0.125):
    """A serving loop on the C1 shape: each step `churn` of the 256 requests finish (closed)
    and as many new ones join under the template (opened + their 255-token prompt suffix
    appended), then one halo_decode_step over the batch (device-resident q / new K / V).
    Requests stay at most 1/churn steps, so suffix lengths spread over [255, 255 + 1/churn].
    Device time with CUDA events (host bookkeeping included in the stream gaps)."""
    from paper_2509_02121_b200.loader import blocks_needed, load
    L, R = wl.layers, wl.nreq
    ld = load(wl, dev, capacity=blocks_needed(wl, steps=int(1 / churn) + 4, slack=8192))
    pool = ld.pool
    tmpl = ld.node_ids[0]
    S = wl.requests[0].suffix
    sk, sv = wl.suffix_kv(f"cuda:{dev}")                  # [L][R*S][Hkv][d]
    sk = sk.view(L, R, S, wl.hkv, wl.d)[:, 0].contiguous()   # one prompt suffix, reused
    sv = sv.view(L, R, S, wl.hkv, wl.d)[:, 0].contiguous()
    nk, nv = wl.new_kv(0, f"cuda:{dev}")
    q = wl.q(0, f"cuda:{dev}")
    out = torch.empty((L, R, wl.hq, wl.d), device=f"cuda:{dev}")
    reqs = list(ld.req_ids)
    k_turn = max(1, int(R * churn))
    # the joiners' prompt K/V as a prefill would leave it (built once, outside the timing)
    skr, svr = sk.repeat(1, k_turn, 1, 1), sv.repeat(1, k_turn, 1, 1)
    plan = None
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(steps + 3):
        if it == 3:
            torch.cuda.synchronize()
            e0.record(stream)
        lo = (it * k_turn) % R
        for j in range(lo, lo + k_turn):                  # finish k requests, admit k new ones
            pool.close_request(reqs[j % R])
            reqs[j % R] = pool.open_request(tmpl)
        joined = [reqs[j % R] for j in range(lo, lo + k_turn)]
        pool.append(joined, [S] * k_turn, skr, svr)
        plan = pool.decode_step(reqs, nk, nv, q, out, reuse=plan)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    plan.destroy()
    pool.destroy()
    return {"what": f"C1 serving loop: {k_turn} of {R} requests finish and {k_turn} join per step "
                    f"(prompt suffix {S} tokens appended on join), then halo_decode_step",
            "steps": steps, "ms_per_step": ms, "value": R * L / (ms * 1e-3), "unit": UNIT}


def measure_paging(pool, ld, wl, torch, decode_step=None):
    """Offload (D2H) and fetch (H2D) of the C1 template node (256 MiB of K+V) through the
    library's pinned host arena (halo_prefix_offload / halo_prefix_fetch), CUDA events on the
    stream; the denominator is a plain pinned cudaMemcpy of the same bytes in this run.  The
    transfer-vs-recompute line is a derived estimate (prefill FLOPs of the 2048-token prefix
    through Llama-3-8B, 2 x 8.0e9 x tokens, at the measured bf16 peak), not a measurement."""
    node = ld.node_ids[0]
    ntok = wl.nodes[0].ntok
    nbytes = ntok * wl.layers * wl.hkv * wl.d * 2 * 2
    stream = torch.cuda.current_stream()
    pool.host_reserve((ntok + 15) // 16)

    def timed(fn, reps=3):
        best = None
        for i in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if i:
                best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
        return best
    t_off = t_fetch = None
    for _ in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        pool.offload_prefix(node, stream)
        e1.record(stream)
        pool.fetch_prefix(node, stream)
        e2.record(stream)
        torch.cuda.synchronize()
        a, b = e0.elapsed_time(e1), e1.elapsed_time(e2)
        t_off = a if t_off is None else min(t_off, a)
        t_fetch = b if t_fetch is None else min(t_fetch, b)
    h = torch.empty(nbytes // 4, pin_memory=True)
    d = torch.empty(nbytes // 4, device=stream.device)
    d2h = timed(lambda: h.copy_(d, non_blocking=True))
    h2d = timed(lambda: d.copy_(h, non_blocking=True))
    del h, d
    bg = None
    if decode_step is not None:
        bg = measure_background_prefetch(pool, wl, torch, decode_step, t_fetch)
    pool.host_reserve(0)
    _, tc_peak, _, _ = peaks()
    prefill_ms = 2 * 8.0e9 * ntok / (tc_peak * 1e12) * 1e3
    return {"what": "halo_prefix_offload / halo_prefix_fetch of the C1 template node (K+V, 32 layers)",
            "bytes": nbytes,
            "offload": {"ms": t_off, "GB/s": nbytes / t_off / 1e6,
                        "pcie_roofline": {"bound": "pcie", "achieved": nbytes / t_off / 1e6,
                                          "peak": nbytes / d2h / 1e6, "unit": "GB/s",
                                          "frac": d2h / t_off,
                                          "peak_source": "pinned cudaMemcpy D2H of the same bytes, this run"}},
            "fetch": {"ms": t_fetch, "GB/s": nbytes / t_fetch / 1e6,
                      "pcie_roofline": {"bound": "pcie", "achieved": nbytes / t_fetch / 1e6,
                                        "peak": nbytes / h2d / 1e6, "unit": "GB/s",
                                        "frac": h2d / t_fetch,
                                        "peak_source": "pinned cudaMemcpy H2D of the same bytes, this run"}},
            "recompute_estimate_ms": prefill_ms,
            "transfer_vs_recompute": prefill_ms / t_fetch,
            "background_prefetch": bg}


def measure_background_prefetch(pool, wl, torch, decode_step, t_fetch, steps=12):
    """PAPER.md:350 "prefetch upcoming caches ... just in time": a second 2048-token template
    (256 MiB of K+V) of the next batch sits in the host arena; halo_pool_prefetch brings it
    back on a copy stream while C1 decode steps run on the compute stream (no host sync; the
    next plan waits for the copy's event).  hidden = 1 - (decode slowdown) / (fetch time
    alone): 1.0 = the fetch cost the decode nothing."""
    import numpy as np
    ntok = wl.nodes[0].ntok
    dev = torch.cuda.current_device()
    k = torch.zeros((wl.layers, ntok, wl.hkv, wl.d), dtype=torch.bfloat16, device=f"cuda:{dev}")
    x = pool.register_prefix(-1, ntok, k, k)
    rq = pool.open_request(x)
    del k
    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=f"cuda:{dev}")

    def decode_window(with_fetch):
        pool.offload_prefix(x, compute)
        torch.cuda.synchronize()
        e0, e1, f1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(compute)
        if with_fetch:
            copy.wait_event(e0)
            pool.prefetch([rq], copy)
            f1.record(copy)
        for _ in range(steps):
            decode_step()
        e1.record(compute)
        torch.cuda.synchronize()
        dec = e0.elapsed_time(e1)
        fet = e0.elapsed_time(f1) if with_fetch else None
        if not with_fetch:
            pool.fetch_prefix(x, compute)
            torch.cuda.synchronize()
        return dec, fet
    for _ in range(2):
        decode_window(False)
        decode_window(True)
    alone = np.median([decode_window(False)[0] for _ in range(3)])
    both = [decode_window(True) for _ in range(3)]
    dec_b = float(np.median([b[0] for b in both]))
    fet_b = float(np.median([b[1] for b in both]))
    pool.close_request(rq)
    pool.release_prefix(x)
    torch.cuda.synchronize()
    slow = dec_b - alone
    return {"what": f"fetch of a 2048-token template (256 MiB) on a copy stream during {steps} C1 decode steps",
            "decode_ms_alone": float(alone), "decode_ms_with_prefetch": dec_b,
            "fetch_ms_alone": t_fetch, "fetch_done_ms_after_start": fet_b,
            "hidden_fraction": max(0.0, 1.0 - slow / t_fetch)}


def measure_relocation(halo, mig):
    """halo_place_groups (Alg. 1 + §3.2 costs) on the C3 batch: 64 templates x
    8192-token contexts (256 requests each, 32 layers) whose KV was all prefilled on worker
    0, placed over 8 workers for a 256-step decode horizon.  e_v from the K1/K2 rooflines at
    the measured peaks; p_v = template KV bytes / link rate (the NCCL GB/s measured above
    when N > 1, else the nominal per-direction NVLink rate).  Host time of the native
    planner, and the moves it emits (executed by halo_migrate_send/recv on a multi-GPU box)."""
    import time
    from paper_2509_02121_b200.relocation import plan_relocation
    from synth import make_config
    hbm, tc = peaks()[:2]
    link, link_src = NVLINK_PEER_GBS * 1e9, "measured NVLink peer copy per direction (B200_PROFILING.md)"
    for e in mig.get("sweep", []):  # N>1: this run's measured rank0 -> rank1 rate, largest node
        if e.get("pairs_0_to_k"):
            link, link_src = e["pairs_0_to_k"][0]["GB/s"] * 1e9, "this run: NCCL rank0 -> rank1"
    wl = make_config("analytics", templates=64)
    out = {}
    for w in (1, 8, 64):
        t0 = time.perf_counter()
        groups, items, res = plan_relocation(wl, [0] * 64, workers=8, link_bytes_per_s=link,
                                             beam_width=w, steps=256, tc_flops=tc * 1e12,
                                             hbm_bps=hbm * 1e9, max_replicas=8)
        dt = time.perf_counter() - t0
        moved = sum(items[m[0]]["kv_bytes"] for m in res["moves"])
        out[f"beam{w}"] = {"planner_ms": dt * 1e3, "makespan_s": res["cost"],
                           "moves": len(res["moves"]), "bytes_moved": moved,
                           "per_worker_groups": [sum(d in ws for ws in res["workers"]) for d in range(8)]}
    total = sum(it["exec_s"] for it in items)
    out.update({"what": "C3 batch (64 templates, all KV on worker 0) placed over 8 workers, "
                        "256 decode steps; planner = native beam search (host)",
                "link_GBps": link / 1e9, "link_source": link_src, "all_on_one_worker_s": total,
                "lower_bound_s": total / 8})
    return out


def _timed(fn, stream, torch, reps=3, warm=2):
    """Best of `reps` CUDA-event timings of fn() on `stream` after `warm` warm-up calls."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def _node_bytes(wl, ntok):
    return ntok * wl.layers * wl.hkv * wl.d * 2 * 2


def measure_migration(halo, pool, ld, wl, world, rank, dev, torch, dist, decode_step=None):
    """KV-block migration (PAPER.md:337 §3.3, :673 §4.5) of prefix nodes of 1k..32k tokens x
    32 layers x 8 kv heads (128 MiB..4 GiB of K+V: BASELINE configs[4], C4) through
    halo_migrate_exchange: K4 block pack -> ncclSend/ncclRecv (one group per 32-MiB chunk
    round) -> K4 unpack -> registration, timed with CUDA events on the migration stream.
    N=1: a 1-rank NCCL communicator (self send/recv): the whole pipeline on one GPU, NVLink
    not exercised; every byte moved costs 6 bytes of HBM traffic (pack r+w, NCCL r+w, unpack
    r+w), so it is reported against the HBM roofline, labelled "loopback".  N>1: rank 0 -> k
    pairs and the all-rank ring permutation, against the measured NVLink peer rate.  Both:
    the migration on a side stream concurrent with C1 decode steps on the compute stream
    (decode slowdown and migration GB/s under decode; PAPER.md:9, :59 overlap)."""
    hbm_peak = peaks()[0]
    stream = torch.cuda.current_stream()
    sizes = (1024, 2048, 4096, 8192, 16384, 32768)
    maxblk = (max(sizes) + 15) // 16
    mp = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, 2 * maxblk + 64, dev)
    uid = halo.comm_unique_id() if rank == 0 else b"\0" * 128
    if world > 1:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    mp.comm_init(uid, world, rank)
    res = {"chunk_bytes": 32 << 20}

    def make_node(ntok, seed):
        kx = torch.empty((wl.layers, ntok, wl.hkv, wl.d), dtype=torch.bfloat16, device=f"cuda:{dev}")
        g = torch.Generator(device=f"cuda:{dev}").manual_seed(seed)
        kx.normal_(generator=g)
        vx = torch.empty_like(kx).normal_(generator=g)
        n = mp.register_prefix(-1, ntok, kx, vx, stream)
        torch.cuda.synchronize()
        return n

    if world == 1:
        res["mode"] = ("loopback: 1-rank NCCL communicator on one GPU (self send/recv); pack -> NCCL "
                       "-> unpack -> register, the exact multi-GPU pipeline, NVLink not exercised")
        sweep = []
        for ntok in sizes:
            nd = make_node(ntok, ntok)
            nb = _node_bytes(wl, ntok)

            def loop():
                (n2,) = mp.migrate_exchange(sends=[(nd, 0, 1)], recvs=[(0, -1, ntok)], stream=stream)
                mp.release_prefix(n2)
            ms = _timed(loop, stream, torch)
            sweep.append({"tokens": ntok, "bytes": nb, "ms": ms, "loopback_GB/s": nb / ms / 1e6,
                          "hbm_roofline": {"bound": "hbm", "achieved": 6 * nb / ms / 1e6, "peak": hbm_peak,
                                           "unit": "GB/s", "frac": 6 * nb / ms / 1e6 / hbm_peak,
                                           "traffic_model": "6 bytes of HBM per byte moved"}})
            mp.release_prefix(nd)
        res["loopback_sweep"] = sweep
        # the K4 block pack alone (one chunk-free call: pool -> exchange layout of the C1 node)
        node, ntok = ld.node_ids[0], wl.nodes[0].ntok
        kx = torch.empty((wl.layers, ntok, wl.hkv, wl.d), dtype=torch.bfloat16, device=f"cuda:{dev}")
        vx = torch.empty_like(kx)
        nb = _node_bytes(wl, ntok)
        ms = _timed(lambda: pool.read_prefix(node, kx, vx, stream), stream, torch)
        res["pack_c1_template"] = {"what": "K4 gather of the C1 template (halo_prefix_read)", "bytes": nb,
                                   "ms": ms, "hbm_frac": 2 * nb / ms / 1e6 / hbm_peak}
        del kx, vx
    else:
        res["mode"] = f"NCCL over NVLink/NVSwitch, {world} ranks"
        pairs = []
        for ntok in (2048, 32768):
            nd = make_node(ntok, ntok + rank)
            nb = _node_bytes(wl, ntok)
            per_k = []
            for k in range(1, world):
                def pair():
                    if rank == 0:
                        mp.migrate_exchange(sends=[(nd, k, 1)], stream=stream)
                    elif rank == k:
                        (n2,) = mp.migrate_exchange(recvs=[(0, -1, ntok)], stream=stream)
                        mp.release_prefix(n2)
                ms = _ranked_timed(pair, stream, torch, dist, dev)
                per_k.append({"dst": k, "ms": ms, "GB/s": nb / ms / 1e6,
                              "nvlink_frac": nb / ms / 1e6 / NVLINK_PEER_GBS})
            pairs.append({"tokens": ntok, "bytes": nb, "pairs_0_to_k": per_k})

            def ring():
                (n2,) = mp.migrate_exchange(sends=[(nd, (rank + 1) % world, 1)],
                                            recvs=[((rank - 1) % world, -1, ntok)], stream=stream)
                mp.release_prefix(n2)
            ms = _ranked_timed(ring, stream, torch, dist, dev)
            pairs[-1]["ring_permutation"] = {"ms": ms, "per_gpu_send_GB/s": nb / ms / 1e6,
                                             "aggregate_GB/s": world * nb / ms / 1e6,
                                             "nvlink_frac": nb / ms / 1e6 / NVLINK_PEER_GBS}
            mp.release_prefix(nd)
        res["sweep"] = pairs
        res["nvlink_peak"] = {"GB/s": NVLINK_PEER_GBS, "source": "measured peer copy per direction "
                              "(B200_PROFILING.md; 900 nominal)"}
    if decode_step is not None:
        res["overlap"] = measure_overlap(mp, wl, world, rank, dev, torch, dist, decode_step)
    torch.cuda.synchronize()
    mp.destroy()
    if decode_step is not None:
        # the same with the migration's SM share bounded (NCCL maxCTAs, copy-kernel CTAs)
        cfg = {"max_ctas": 2, "copy_ctas": 2 * 148}
        mp = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, 2 * 512 + 64, dev)
        uid = halo.comm_unique_id() if rank == 0 else b"\0" * 128
        if world > 1:
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        mp.comm_init(uid, world, rank, **cfg)
        res["overlap_bounded"] = dict(measure_overlap(mp, wl, world, rank, dev, torch, dist, decode_step),
                                      comm_config=cfg)
        torch.cuda.synchronize()
        mp.destroy()
    return res


def _ranked_timed(fn, stream, torch, dist, dev, reps=3):
    """Best of `reps` (barrier; events around fn on `stream`; max over ranks)."""
    best = None
    for it in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{dev}")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if it > 0:  # the first call connects the peers
            best = ms.item() if best is None else min(best, ms.item())
    return best


def measure_overlap(mp, wl, world, rank, dev, torch, dist, decode_step, ntok=8192, dec_steps=20):
    """Migration on a side stream while C1 decode steps run on the compute stream (the
    deployment the paper describes: snapshots move under scheduler control while decode
    continues; compute-communication overlap, :9, :59).  Three passes: decode
    alone, migration alone, both (the migration loop sized to span the decode pass).  N=1:
    loopback (both ends on this GPU: the worst case for HBM contention); N>1: ring
    permutation.  NCCL CTAs / copy CTAs are the communicator's defaults."""
    compute = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=f"cuda:{dev}")
    kx = torch.empty((wl.layers, ntok, wl.hkv, wl.d), dtype=torch.bfloat16, device=f"cuda:{dev}")
    kx.normal_()
    nd = mp.register_prefix(-1, ntok, kx, kx, compute)
    del kx
    nb = _node_bytes(wl, ntok)
    dst, src = (rank + 1) % world, (rank - 1) % world

    def migrate():
        (n2,) = mp.migrate_exchange(sends=[(nd, dst, 1)], recvs=[(src, -1, ntok)], stream=side)
        mp.release_prefix(n2)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def span(events):
        return events[0].elapsed_time(events[1])

    for _ in range(3):
        decode_step()
        migrate()
    sync_all()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(compute)
    for _ in range(dec_steps):
        decode_step()
    ev[1].record(compute)
    sync_all()
    dec_alone = span(ev)
    ev[0].record(side)
    migrate()
    ev[1].record(side)
    sync_all()
    mig_one = span(ev)
    reps = max(1, int(round(dec_alone / mig_one)))
    evm = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(side)
    t0 = time.perf_counter()
    for _ in range(reps):
        migrate()
    host_ms = (time.perf_counter() - t0) * 1e3 / reps
    ev[1].record(side)
    sync_all()
    mig_alone = span(ev)
    # both: the host interleaves the enqueues (migrations spread evenly over the decode steps)
    # so the two streams really run side by side on the GPU
    evm[0].record(side)
    ev[0].record(compute)
    done = 0
    for i in range(dec_steps):
        decode_step()
        while done < reps * (i + 1) // dec_steps:
            migrate()
            done += 1
    ev[1].record(compute)
    evm[1].record(side)
    sync_all()
    dec_both, mig_both = span(ev), span(evm)
    vals = [dec_alone, dec_both, mig_alone, mig_both]
    if world > 1:
        from paper_2509_02121_b200.sharding import max_over_ranks
        vals = max_over_ranks(vals, dist, f"cuda:{dev}")
    dec_alone, dec_both, mig_alone, mig_both = vals
    mp.release_prefix(nd)
    return {"what": (f"{reps} x {ntok}-token node ({nb >> 20} MiB K+V) migrations on a side stream "
                     f"{'(loopback)' if world == 1 else '(ring permutation)'} concurrent with "
                     f"{dec_steps} C1 decode steps on the compute stream"),
            "decode_ms_per_step_alone": dec_alone / dec_steps,
            "decode_ms_per_step_with_migration": dec_both / dec_steps,
            "decode_slowdown_pct": 100.0 * (dec_both / dec_alone - 1.0),
            "migration_GB/s_alone": reps * nb / mig_alone / 1e6,
            "migration_GB/s_with_decode": reps * nb / mig_both / 1e6,
            "migration_ms_alone": mig_alone, "migration_ms_with_decode": mig_both,
            "host_enqueue_ms_per_migration": host_ms}


if __name__ == "__main__":
    main()
