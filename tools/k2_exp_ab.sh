#!/bin/bash
# Where K2's time goes at C1 (timing-only builds, wrong outputs): exp1 = skip the per-block
# compute, exp2 = skip every unit end (merge / finalize / publish), exp3 = both; against the
# normal build (attn).  K2 launch time alone (breakdown pass) and the headline step.
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2509_02121_b200 import build as b
for v in (1, 2, 3):
    b.build(extra=[f"-DHALO_K2_EXP={v}"], lib=os.path.join(b.PKG, f"libhalo_exp{v}.so"))
PY
out=gpurun_out/k2exp.txt; : > $out
for pass in 1 2; do
for v in attn exp1 exp2 exp3; do
  HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 300 python bench.py --other-configs "" \
     --no-cpu-baseline --no-e2e --no-migration --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
e=d.get('roofline_k2_equal_shares',{})
print('$v', 'step %.4f ms' % d['ms_per_step'], 'k2 bd %.2f us' % (d['roofline']['avg_launch_ms']*1e3), 'k2 alone-eq %.2f us' % (e.get('avg_launch_ms',0)*1e3), 'k1 %.2f us' % (d['prefix_roofline']['avg_launch_ms']*1e3))" >> $out
done; done
cat $out
