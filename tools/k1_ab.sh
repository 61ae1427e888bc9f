#!/bin/bash
# A/B of K1 variants: libhalo_k1old.so (previous K1) vs the current build; K1 roofline
# fractions on C1 / C2 / C2 root / C2 roles / C3 (bench other-configs), alternating passes.
out=gpurun_out/k1_ab.txt; : > $out
for pass in 1 2; do
for v in k1old attn; do
  HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 300 python bench.py --other-configs tree,tree_root,tree_roles,analytics \
     --no-cpu-baseline --no-e2e --no-migration --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$v', 'C1 %.3f' % d['prefix_roofline']['frac'], ' '.join('%s %.3f' % (k, v['prefix_roofline']['frac']) for k, v in d['other_configs'].items()), 'q/s %.3e' % d['value'])" >> $out
done; done
cat $out
