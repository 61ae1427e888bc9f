"""Per-warp timeline of K2 (debug build with -DHALO_K2_TRACE): entry, first K/V stage
landed, K1 complete (griddepcontrol.wait returned), last K/V stage landed, start of the last
unit end (merge / finalize / publish), exit -- in us from the earliest entry.

Two runs on the chosen config (CFG=fanout|tree|analytics, LAYERS):
  alone : K2 by itself after an L2 flush (K1's partials already written)
  pdl   : K1 then K2 back to back (programmatic dependent launch), as the headline runs
Usage (GPU box): python tools/k2_trace.py
"""
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


def stats(name, v):
    v = v[np.isfinite(v)]
    if v.size == 0:
        return f"{name:12s} (none)"
    return (f"{name:12s} min={v.min():7.2f} p10={np.percentile(v, 10):7.2f} p50={np.median(v):7.2f} "
            f"p90={np.percentile(v, 90):7.2f} max={v.max():7.2f}")


def main():
    cfg = os.environ.get("CFG", "fanout")
    wl = make_config(cfg, layers=int(os.environ.get("LAYERS", "2")))
    ld = load(wl, 0)
    append_step(ld, wl, 0, 0)
    from paper_2509_02121_b200.abi import PlanOptions
    opt = PlanOptions(0, 0, int(os.environ.get("SPLITS", "0")), 0)
    opt.k2_early_weight = float(os.environ.get("EARLY_W", "0"))
    opt.k1_sm_frac = float(os.environ.get("K1_SM_FRAC", "0"))
    opt.k2_whole_units = int(os.environ.get("WHOLE_UNITS", "0"))
    plan = ld.pool.plan(ld.req_ids, opt)
    info = plan.info()
    q = wl.q(0, "cuda:0")
    out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
    lib = halo.load_library()
    lib.halo_debug_k2_trace.argtypes = [ctypes.c_void_p]
    W = 148 * 16
    buf = torch.zeros(W * 8, dtype=torch.int64, device="cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    print(f"{cfg}: k1_tiles={info['k1_tiles']} k2_units={info['k2_units']} k2_bytes={info['k2_bytes']:.3e}")
    for mode in ("alone", "pdl"):
        for it in range(4):
            if mode == "alone":
                plan.run_stages(1, 1, q[1], out)
            flush.zero_()
            buf.zero_()
            lib.halo_debug_k2_trace(ctypes.c_void_p(buf.data_ptr()))
            plan.run_stages(1, 2 if mode == "alone" else 3, q[1], out)
            lib.halo_debug_k2_trace(ctypes.c_void_p(0))
            torch.cuda.synchronize()
        t = buf.view(W, 8).cpu().numpy().astype(np.float64)
        used = t[:, 0] > 0
        t = t[used]
        t[t == 0] = np.nan
        t0 = np.nanmin(t[:, 0])
        t = (t - t0) / 1e3
        span = np.nanmax(t[:, 3])
        print(f"-- {mode}: warps={used.sum()} span={span:.2f} us  "
              f"(k2 bytes / span = {info['k2_bytes'] / span / 1e3:.0f} GB/s)")
        for name, col in [("entry", 0), ("first data", 1), ("k1 done", 2), ("last data", 4),
                          ("last unit end", 5), ("exit", 3)]:
            print(stats(name, t[:, col]))
        print(stats("end latency", t[:, 3] - t[:, 5]))
        print(stats("unit end", t[:, 6] - t[:, 5]))
        print(stats("final atomic", t[:, 3] - t[:, 6]))
        print(stats("tail after data", t[:, 3] - t[:, 4]))
        print(stats("busy", t[:, 3] - t[:, 0]))
        ncta_warps = int(os.environ.get("K2_WARPS", "0")) or None
        if ncta_warps:
            ends = t[:, 3][: (len(t) // ncta_warps) * ncta_warps].reshape(-1, ncta_warps).max(axis=1)
            starts = t[:, 0][: (len(t) // ncta_warps) * ncta_warps].reshape(-1, ncta_warps).min(axis=1)
            print("per-CTA exit: min %.2f median %.2f max %.2f" % (ends.min(), np.median(ends), ends.max()))
            early = starts < 2.0
            for name, sel in (("early CTAs", early), ("late CTAs", ~early)):
                if sel.any():
                    print(f"  {name:10s} n={sel.sum():3d} start p50 {np.median(starts[sel]):6.2f} "
                          f"exit min {ends[sel].min():6.2f} p50 {np.median(ends[sel]):6.2f} max {ends[sel].max():6.2f}")
    plan.destroy()
    ld.pool.destroy()


if __name__ == "__main__":
    main()
