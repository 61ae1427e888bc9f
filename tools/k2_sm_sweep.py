"""K2 per-SM streaming cap and the K1/K2 co-schedule (round 2; tensor-core K2).

1. K2 alone on n SMs (halo_plan_options.k2_sms) for C1 and C3 (4 layers): GB/s of the
   algorithmic bytes; the slope at small n is the per-SM stream rate.
2. C1 headline-style layers (K1 then K2 under PDL) for K1-SM fractions x early weights.
Usage (GPU box): python tools/k2_sm_sweep.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.abi import PlanOptions  # noqa: E402
from paper_2509_02121_b200.loader import append_step, load  # noqa: E402
from synth import make_config  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    halo.load_library()
    for cfg in ("fanout", "analytics"):
        wl = make_config(cfg, layers=4)
        ld = load(wl, 0)
        append_step(ld, wl, 0, 0)
        q = wl.q(0, "cuda:0")
        out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
        for n in (148, 120, 96, 74, 64, 48, 32):
            opt = PlanOptions(0, 0, 0, 0)
            opt.k2_sms = n
            opt.k1_sm_frac = -1.0
            plan = ld.pool.plan(ld.req_ids, opt)
            info = plan.info()
            plan.run_stages(0, 1, q[0], out)
            ms = timed(lambda: [plan.run_stages(l, 2, q[l], out) for l in range(4)]) / 4
            print(f"{cfg} K2 alone on {n:3d} SMs: {ms * 1e3:7.1f} us  {info['k2_bytes'] / ms / 1e6:7.0f} GB/s  "
                  f"({info['k2_bytes'] / ms / 1e6 / n:5.1f} GB/s per SM)", flush=True)
            plan.destroy()
        if cfg == "fanout":
            for frac in (-1.0, 0.5, 0.65, 0.8):
                for w in (1.0, 1.2, 1.6, 2.0, 2.5, 3.0):
                    opt = PlanOptions(0, 0, 0, 0)
                    opt.k1_sm_frac = frac
                    opt.k2_early_weight = w
                    plan = ld.pool.plan(ld.req_ids, opt)
                    info = plan.info()
                    ms = timed(lambda: [plan.run(l, q[l], out) for l in range(4)]) / 4
                    print(f"fanout K1+K2 layer: k1_sm_frac={frac:5.2f} w={w:3.1f} k1_tiles={info['k1_tiles']:4d}: "
                          f"{ms * 1e3:6.1f} us/layer  {wl.nreq / ms * 1e3 / 1e6:6.3f} M q/s", flush=True)
                    plan.destroy()
        ld.pool.destroy()


if __name__ == "__main__":
    main()
