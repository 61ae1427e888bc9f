"""Where the C1 decode step's time goes beyond the 32 x (K1, K2) layers: CUDA events between
the step's phases (roll back + K5 append, plan + upload, layers) and host time per phase.
Usage (GPU box): python tools/step_probe.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    halo.load_library()
    wl = make_config("fanout")
    L, R = wl.layers, wl.nreq
    ld = load(wl, 0, capacity=blocks_needed(wl, steps=2, slack=4096))
    pool, reqs = ld.pool, ld.req_ids
    nk, nv = wl.new_kv(0, "cuda:0")
    q = wl.q(0, "cuda:0")
    out = torch.empty((L, R, wl.hq, wl.d), device="cuda:0")
    lse = torch.empty((L, R, wl.hq), device="cuda:0")
    ones = [1] * R
    pool.append(reqs, ones, nk, nv)
    popt = halo.PlanOptions(0, 0, 0, 0)
    plan = pool.plan(reqs, popt)
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    host = [0.0] * 4
    N = 40
    acc = [0.0] * 4
    for it in range(N + 5):
        t0 = time.perf_counter()
        ev[0].record(s)
        pool.truncate(reqs, ones)
        pool.append(reqs, ones, nk, nv)
        t1 = time.perf_counter()
        ev[1].record(s)
        pool.plan(reqs, popt, reuse=plan)
        t2 = time.perf_counter()
        ev[2].record(s)
        for l in range(L):
            plan.run(l, q[l], out[l], lse[l])
        t3 = time.perf_counter()
        ev[3].record(s)
        if it >= 5:
            host[0] += t1 - t0
            host[1] += t2 - t1
            host[2] += t3 - t2
    torch.cuda.synchronize()
    # device phases (last iteration only is recorded by the events; re-run a timed loop)
    for it in range(N):
        ev[0].record(s)
        pool.truncate(reqs, ones)
        pool.append(reqs, ones, nk, nv)
        ev[1].record(s)
        pool.plan(reqs, popt, reuse=plan)
        ev[2].record(s)
        for l in range(L):
            plan.run(l, q[l], out[l], lse[l])
        ev[3].record(s)
        torch.cuda.synchronize()
        acc[0] += ev[0].elapsed_time(ev[1])
        acc[1] += ev[1].elapsed_time(ev[2])
        acc[2] += ev[2].elapsed_time(ev[3])
    print(f"host ms/step: append {host[0] / N * 1e3:.3f}  plan {host[1] / N * 1e3:.3f}  "
          f"32 layer launches {host[2] / N * 1e3:.3f}")
    print(f"device ms/step (synchronised per step): append {acc[0] / N:.4f}  plan+upload {acc[1] / N:.4f}  "
          f"layers {acc[2] / N:.4f}")
    # pipelined steps: total per step
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for it in range(N):
        pool.truncate(reqs, ones)
        pool.append(reqs, ones, nk, nv)
        pool.plan(reqs, popt, reuse=plan)
        for l in range(L):
            plan.run(l, q[l], out[l], lse[l])
    e1.record(s)
    torch.cuda.synchronize()
    print(f"pipelined step {e0.elapsed_time(e1) / N:.4f} ms")
    e0.record(s)
    for it in range(N):
        for l in range(L):
            plan.run(l, q[l], out[l], lse[l])
    e1.record(s)
    torch.cuda.synchronize()
    print(f"layers only, pipelined {e0.elapsed_time(e1) / N:.4f} ms")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def layers_only(layers, frac):
    wl = make_config("fanout", layers=layers)
    ld = load(wl, 0, capacity=blocks_needed(wl, steps=2, slack=4096))
    pool, reqs = ld.pool, ld.req_ids
    nk, nv = wl.new_kv(0, "cuda:0")
    q = wl.q(0, "cuda:0")
    out = torch.empty((wl.layers, wl.nreq, wl.hq, wl.d), device="cuda:0")
    pool.append(reqs, [1] * wl.nreq, nk, nv)
    popt = halo.PlanOptions(0, 0, 0, 0)
    popt.k1_sm_frac = frac
    plan = pool.plan(reqs, popt)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        e0.record(s)
        for it in range(20):
            for l in range(wl.layers):
                plan.run(l, q[l], out[l])
        e1.record(s)
        torch.cuda.synchronize()
    info = plan.info()
    print(f"layers={layers} k1_sm_frac={frac}: k1_tiles={info['k1_tiles']} "
          f"{e0.elapsed_time(e1) / 20 / wl.layers * 1e3:.1f} us/layer")
    plan.destroy()
    pool.destroy()


if __name__ == "__main__" and len(sys.argv) > 1:
    for layers in (8, 32):
        for frac in (0.0, -1.0):
            layers_only(layers, frac)
