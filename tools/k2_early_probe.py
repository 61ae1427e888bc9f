"""Single-wave K1 shapes (fan-out variants of C1, 32 layers) timed under the current env hooks
(HALO_MAX_SPLITS, HALO_K2_EARLY_W): one line per variant, q/s of the headline pass."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2509_02121_b200 as halo
from synth import make_config
import bench

halo.load_library()
tag = sys.argv[1]
res = {}
for (nreq, prefix, suffix) in [(256, 2048, 15), (256, 2048, 255), (256, 2048, 1023), (128, 2048, 255),
                               (512, 2048, 255), (256, 1024, 255), (256, 4096, 255), (64, 8192, 255)]:
    wl = make_config("fanout", layers=32, nreq=nreq, prefix=prefix, suffix=suffix)
    ld, plan, info, step, _ = bench.setup_workload(halo, wl, 0, torch)
    ms, *_ = bench.time_steps(step, wl.layers, 40, 5, 1, 0, torch, dist)
    qps = wl.nreq * wl.layers * 40 / (ms / 1e3)
    res[f"{nreq}x{prefix}+{suffix}"] = (round(qps / 1e6, 3), info["k1_tiles"] if isinstance(info, dict) else getattr(info, "k1_tiles", None))
    del ld, plan, step
    torch.cuda.empty_cache()
print(tag, json.dumps(res))
