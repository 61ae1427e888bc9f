"""C1 K1+K2 layer time (PDL, as the headline runs) over K1 split counts (max_splits) and
K2 early weights (round 2 co-schedule study).  Usage (GPU box): python tools/k1k2_cosched_sweep.py"""
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
    L = int(os.environ.get("LAYERS", "8"))
    wl = make_config(os.environ.get("CFG", "fanout"), layers=L)
    ld = load(wl, 0)
    append_step(ld, wl, 0, 0)
    q = wl.q(0, "cuda:0")
    out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
    sl = [int(x) for x in os.environ.get("SPLITS", "1,2,3,4").split(",")]
    wl_ = [float(x) for x in os.environ.get("WEIGHTS", "1.0,1.5,2.0,2.7,3.5,5.0,8.0,12.0").split(",")]
    grid = [(s, w) for s in sl for w in wl_]
    for s, w in grid:
        opt = PlanOptions(0, 0, s, 0)
        opt.k1_sm_frac = -1.0
        opt.k2_early_weight = w
        opt.k2_shape = int(os.environ.get("K2_SHAPE", "0"))  # 0 planner, 1 wide, 2 narrow
        plan = ld.pool.plan(ld.req_ids, opt)
        info = plan.info()
        ms = timed(lambda: [plan.run(l, q[l], out) for l in range(L)]) / L
        print(f"{os.path.basename(halo.lib_path())} shape={info.get('k2_warps', '?')} splits={s} w={w:4.1f} k1_tiles={info['k1_tiles']:4d}: {ms * 1e3:6.1f} us/layer "
              f"{wl.nreq / ms * 1e3 / 1e6:6.3f} M q/s", flush=True)
        plan.destroy()
    ld.pool.destroy()


if __name__ == "__main__":
    main()
