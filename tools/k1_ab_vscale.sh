#!/bin/bash
# A/B of K1 with the V-table scale (current) vs round-1 K1 (libhalo_ab_old.so, built from the
# previous revision): K1 roofline fractions of C1 / C2 / C3, three alternating passes.
out=gpurun_out/k1_ab_vscale.txt; : > $out
for pass in 1 2 3; do
for v in ab_old attn; do
  HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_${v}.so
  [ "$v" = attn ] && HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn.so
  HALO_LIB=$HALO_LIB timeout 300 python bench.py --other-configs tree,analytics --no-cpu-baseline --no-e2e --no-migration --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$v', 'C1 %.3f' % d['prefix_roofline']['frac'], ' '.join('%s %.3f' % (k, v['prefix_roofline']['frac']) for k, v in d['other_configs'].items()), 'q/s %.3e' % d['value'])" >> $out
done; done
cat $out
