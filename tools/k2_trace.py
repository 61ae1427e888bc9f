"""Per-warp timeline of K2 (debug build): start, first block arrived, end (us)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_02121_b200 import build as b  # noqa: E402

os.environ["HALO_LIB"] = b.build_trace()
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import append_step, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    wl = make_config(os.environ.get("CFG", "fanout"), layers=int(os.environ.get("LAYERS", "2")))
    ld = load(wl, 0)
    append_step(ld, wl, 0, 0)
    plan = ld.pool.plan(ld.req_ids)
    q = wl.q(0, "cuda:0")
    out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
    lib = halo.load_library()
    lib.halo_debug_k2_trace.argtypes = [ctypes.c_void_p]
    W = 148 * 12
    buf = torch.zeros(W * 4, dtype=torch.int64, device="cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    for it in range(4):
        plan.run_stages(1, 1, q[1], out)
        flush.zero_()
        buf.zero_()
        lib.halo_debug_k2_trace(ctypes.c_void_p(buf.data_ptr()))
        plan.run_stages(1, 2, q[1], out)
        lib.halo_debug_k2_trace(ctypes.c_void_p(0))
        torch.cuda.synchronize()
    t = buf.view(W, 4).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3
    print(f"warps={W} kernel span={t[:, 2].max():.2f} us")
    for name, col in [("start", 0), ("first data", 1), ("end", 2)]:
        v = t[:, col]
        print(f"{name:11s} min={v.min():7.2f} p10={np.percentile(v,10):7.2f} p50={np.median(v):7.2f} "
              f"p90={np.percentile(v,90):7.2f} max={v.max():7.2f}")
    ends = t[:, 2].reshape(-1, 12).max(axis=1)
    print("per-CTA end: min %.2f median %.2f max %.2f" % (ends.min(), np.median(ends), ends.max()))
    order = np.argsort(ends)
    print("slowest CTAs", order[-8:], ends[order[-8:]])
    print("fastest CTAs", order[:8], ends[order[:8]])


if __name__ == "__main__":
    main()
