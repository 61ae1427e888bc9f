"""Does K2-alone time at C1 depend on the pool's physical memory?  Loads the C1 workload into
several pools in one process (different physical pages) and times K2 launched alone after K1
(the bench's breakdown pass) on each.  Usage (GPU box): python tools/k2_layout_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    halo.load_library()
    wl = make_config("fanout", layers=int(os.environ.get("LAYERS", "8")))
    L = wl.layers
    q = wl.q(0, "cuda:0")
    out = torch.empty((L, wl.nreq, wl.hq, wl.d), device="cuda:0")
    s = torch.cuda.current_stream()
    keep = []
    for i in range(int(os.environ.get("POOLS", "4"))):
        ld = load(wl, 0, capacity=blocks_needed(wl, steps=2, slack=4096))
        nk, nv = wl.new_kv(0, "cuda:0")
        ld.pool.append(ld.req_ids, [1] * wl.nreq, nk, nv)
        popt = halo.PlanOptions(0, 0, 0, 0)
        popt.k2_whole_units = int(os.environ.get("WHOLE_UNITS", "1"))
        plan = ld.pool.plan(ld.req_ids, popt)
        ones = [1] * wl.nreq
        res = []
        for rep in range(int(os.environ.get("REPS", "3"))):
            if os.environ.get("HEADLINE"):  # the bench's headline pass first (K1 -> K2 under PDL)
                for _ in range(20):
                    for l in range(L):
                        plan.run(l, q[l], out[l])
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
            if os.environ.get("STEP"):  # the bench's step: roll back, re-append, re-plan
                ld.pool.truncate(ld.req_ids, ones)
                ld.pool.append(ld.req_ids, ones, nk, nv)
                ld.pool.plan(ld.req_ids, popt, reuse=plan)
            torch.cuda._sleep(4_000_000)
            for l in range(L):
                plan.run_stages(l, 1, q[l], out[l])
                evs[l][0].record(s)
                plan.run_stages(l, 2, q[l], out[l])
                evs[l][1].record(s)
            torch.cuda.synchronize()
            res.append(sum(a.elapsed_time(b) for a, b in evs) / L * 1e3)
        print(f"pool {i}: K2 alone " + " ".join(f"{x:.2f}" for x in res) + " us", flush=True)
        keep.append((ld, plan))


if __name__ == "__main__":
    main()
