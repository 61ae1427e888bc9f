"""Default-plan decode throughput (K1 + K2 per layer under PDL, 8 layers) on fan-out shapes
around C1 -- the shapes round 1 tuned on (profiles/k2_shape_after_l2_r01.txt).
Usage (GPU box): python tools/fanout_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import append_step, load  # noqa: E402
from synth import make_config  # noqa: E402

SHAPES = [(256, 2048, 255), (256, 2048, 1023), (512, 2048, 255), (256, 1024, 255), (256, 4096, 255),
          (64, 8192, 255), (128, 2048, 255), (256, 2048, 15)]


def main():
    halo.load_library()
    L = 8
    for nreq, prefix, suffix in SHAPES:
        wl = make_config("fanout", layers=L, nreq=nreq, prefix=prefix, suffix=suffix)
        ld = load(wl, 0)
        append_step(ld, wl, 0, 0)
        plan = ld.pool.plan(ld.req_ids)
        info = plan.info()
        q = wl.q(0, "cuda:0")
        out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
        for _ in range(3):
            for l in range(L):
                plan.run(l, q[l], out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            for l in range(L):
                plan.run(l, q[l], out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * L)
        print(f"{nreq}x{prefix}+{suffix}: k1_tiles={info['k1_tiles']:4d} {us:7.1f} us/layer "
              f"{nreq / us:6.3f} M q/s", flush=True)
        plan.destroy()
        ld.pool.destroy()


if __name__ == "__main__":
    main()
