"""Max |GPU - fp64 oracle| on the parity workloads of the error budget (GPU box; report)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_parity as T  # noqa: E402
from synth import make_config  # noqa: E402

T.halo_build.build()
T.halo.load_library()
import torch  # noqa: E402
torch.cuda.set_device(0)
cases = [("alpha1", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30)),
         ("alpha2", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, alpha_q=2.0)),
         ("alpha4", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, alpha_q=4.0)),
         ("alpha8", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, alpha_q=8.0)),
         ("sink", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, sink=8.0)),
         ("tree-sink", make_config("tree", layers=1, root=300, roles=3, role_tok=130, per_role=30,
                                   suffix=20, sink=8.0)),
         ("normal", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, dist="normal")),
         ("normal-a4", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, dist="normal", alpha_q=4.0)),
         ("outliers", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=30, dist="normal",
                                  k_outlier_dims=(3, 77))),
         ("C1-normal", make_config("fanout", layers=1, dist="normal")),
         ("suffix-only", make_config("fanout", layers=1, nreq=64, prefix=600, suffix=500, dist="normal"),
          T.opts(min_rows=100000))]
for case in cases:
    name, wl = case[0], case[1]
    info, eo, el = T.check(wl, case[2] if len(case) > 2 else None)
    print(f"{name:10s} max|out - oracle| = {eo:.2e}   max|lse - oracle| = {el:.2e}   "
          f"(k1_tiles {info['k1_tiles']}, k2_units {info['k2_units']})", flush=True)
raise SystemExit
for name, wl in cases:
    info, eo, el = T.check(wl)
    print(f"{name:10s} max|out - oracle| = {eo:.2e}   max|lse - oracle| = {el:.2e}   "
          f"(k1_tiles {info['k1_tiles']}, k2_units {info['k2_units']})", flush=True)
