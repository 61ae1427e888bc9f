# folded prefix nodes (shared by < 16 requests: n_req*g < 64 rows) streamed by K2 with the default
# L2 policy (HALO_K2_SHARED_NORMAL=1, default) vs evict_first like private suffix blocks (=0)
cat > /tmp/fold_probe.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
import paper_2509_02121_b200 as halo
from synth import make_config
import bench
halo.load_library()
res = {}
for name, kw in [("tree64x12", dict(layers=32, root=2048, roles=64, role_tok=1024, per_role=12, suffix=255)),
                 ("tree128x8", dict(layers=32, root=1024, roles=128, role_tok=512, per_role=8, suffix=127))]:
    wl = make_config("tree", **kw)
    ld, plan, info, step, _ = bench.setup_workload(halo, wl, 0, torch)
    ms, ms_bd, k1, k2, _ = bench.time_steps(step, wl.layers, 30, 5, 1, 0, torch, dist)
    res[name] = dict(qps=round(wl.nreq * wl.layers * 30 / (ms / 1e3) / 1e6, 3), k2_ms=round(k2 / 30 / wl.layers * 1e3, 2),
                     folded=info["folded_nodes"], k2_gb=round(info.get("k2_bytes", 0) / 1e9, 3))
    del ld, plan, step
    torch.cuda.empty_cache()
print(sys.argv[1], json.dumps(res))
PY
for rep in 1 2; do
  HALO_K2_SHARED_NORMAL=1 python /tmp/fold_probe.py normal 2>gpurun_out/fold_n.err
  HALO_K2_SHARED_NORMAL=0 python /tmp/fold_probe.py evict_first 2>gpurun_out/fold_e.err
done
