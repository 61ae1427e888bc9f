"""Host time of the C1 step's library calls on a device pool (truncate, append, plan) next to
the same calls on a host-only pool (bookkeeping alone).  Usage: python tools/host_step_probe.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def run(device):
    wl = make_config("fanout")
    if device >= 0:
        ld = load(wl, device, capacity=blocks_needed(wl, steps=2, slack=4096))
        nk, nv = wl.new_kv(0, f"cuda:{device}")
    else:
        p = halo.Pool(wl.layers, wl.hkv, wl.hq, wl.d, blocks_needed(wl, steps=2, slack=4096), device=-1)
        ld = load(wl, device=-1, pool=p)
        nk = nv = None
    pool, reqs = ld.pool, ld.req_ids
    ones = [1] * len(reqs)
    pool.append(reqs, ones, nk, nv)
    popt = halo.PlanOptions(0, 0, 0, 0)
    plan = pool.plan(reqs, popt)
    t = {"truncate": 0.0, "append": 0.0, "plan": 0.0}
    N = 50
    for i in range(N + 5):
        a = time.perf_counter()
        pool.truncate(reqs, ones)
        b = time.perf_counter()
        pool.append(reqs, ones, nk, nv)
        c = time.perf_counter()
        pool.plan(reqs, popt, reuse=plan)
        d = time.perf_counter()
        if i >= 5:
            t["truncate"] += b - a
            t["append"] += c - b
            t["plan"] += d - c
    if device >= 0:
        torch.cuda.synchronize()
    print("device" if device >= 0 else "host-only", {k: round(v / N * 1e3, 3) for k, v in t.items()}, "ms",
          flush=True)


if __name__ == "__main__":
    run(0)
    run(-1)
