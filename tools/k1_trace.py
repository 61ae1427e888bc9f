"""Timeline of one K1 CTA (debug build with -DHALO_K1_TRACE) on the C1 workload.

Usage (GPU box): python tools/k1_trace.py   -> prints per-tile event times (us from start).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_02121_b200 import build as b  # noqa: E402

os.environ["HALO_LIB"] = b.build_trace()
import ctypes  # noqa: E402

import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import append_step, load  # noqa: E402
from synth import make_config  # noqa: E402

EV = ["K issued", "V issued", "QK issue", "PV issue", "V full(conv)", "V conv done",
      "S full(smax)", "pass start", "P stored", None, "pass1 done", "exp done",
      "MMA Vconv ok", "B exp done", "B S full", "PV_B issue", "S loaded"]


def main():
    layers = int(os.environ.get("LAYERS", "1"))
    wl = make_config(os.environ.get("CFG", "fanout"), layers=layers)
    ld = load(wl, 0)
    append_step(ld, wl, 0, 0)
    plan = ld.pool.plan(ld.req_ids)
    q = wl.q(0, "cuda:0")
    out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
    buf = torch.zeros(24 * 64, dtype=torch.int64, device="cuda:0")
    lib = halo.load_library()
    lib.halo_debug_k1_trace.argtypes = [ctypes.c_void_p]
    for it in range(3):
        buf.zero_()
        lib.halo_debug_k1_trace(ctypes.c_void_p(buf.data_ptr()))
        plan.run_stages(0, 1, q[0], out)
        torch.cuda.synchronize()
    t = buf.view(24, 64).cpu()
    t0 = int(t[9, 0])
    print("tile0 info:", plan.export("tiles")[0].tolist())
    def at(e, n):
        return f"{(int(t[e, n]) - t0) / 1e3:.2f} us" if int(t[e, n]) else "- (TMA)"
    print(f"tmem+barriers {at(9, 3)}, producer past wait {at(9, 4)}, softmax past wait {at(9, 5)}, "
          f"q loaded by the softmax threads {at(9, 2)}, epilogue done {at(9, 1)}")
    nt = int((t[2] > 0).sum())
    evs = [e for e in range(len(EV)) if EV[e]]
    print("tile " + " ".join(f"{EV[e]:>12s}" for e in evs))
    for n in range(nt):
        print(f"{n:4d} " + " ".join(f"{(int(t[e, n]) - t0) / 1e3:12.2f}" if int(t[e, n]) else f"{'-':>12s}" for e in evs))


if __name__ == "__main__":
    main()
