#!/bin/bash
# A/B of K1 compile-time variants: builds libhalo_<name>.so for each "name=flags" in VARIANTS
# (e.g. VARIANTS="pp0=-DHALO_K1_PINGPONG=0 pp2=-DHALO_K1_PINGPONG=2") and compares their K1
# roofline fractions with the default build (attn) on C1 / C2 / C2 root / C2 roles / C3.
python - <<PY
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2509_02121_b200 import build as b
for kv in "$VARIANTS".split():
    name, flags = kv.split("=", 1)
    b.build(extra=flags.split(","), lib=os.path.join(b.PKG, f"libhalo_{name}.so"))
PY
out=gpurun_out/k1_variants_ab.txt; : > $out
names="attn $(for kv in $VARIANTS; do echo -n "${kv%%=*} "; done)"
for pass in 1 2; do
for v in $names; do
  HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 300 python bench.py --other-configs tree,tree_root,tree_roles,analytics \
     --no-cpu-baseline --no-e2e --no-migration --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$v', 'C1 %.3f' % d['prefix_roofline']['frac'], ' '.join('%s %.3f' % (k, v['prefix_roofline']['frac']) for k, v in d['other_configs'].items()), 'q/s %.3e' % d['value'])" >> $out
done; done
cat $out
