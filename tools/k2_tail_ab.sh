#!/bin/bash
# A/B of K2's static-then-dynamic tail (halo_plan_options.k2_tail_pct via bench.py's
# HALO_K2_TAIL): C1 headline q/s and K2/K1 roofline fractions (breakdown pass), C2 and C3
# per-launch fractions; alternating passes.
out=gpurun_out/k2_tail_ab.txt; : > $out
for pass in 1 2; do
for t in -1 5 10 15 25; do
  HALO_K2_TAIL=$t timeout 300 python bench.py --other-configs tree,analytics --no-cpu-baseline --no-e2e --no-migration --steps 50 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('tail $t', 'q/s %.4e' % d['value'], 'K2 %.3f K1 %.3f' % (d['roofline']['frac'], d['prefix_roofline']['frac']), ' '.join('%s K2 %.3f' % (k, v['roofline']['frac']) for k, v in d['other_configs'].items()))" >> $out
done; done
cat $out
