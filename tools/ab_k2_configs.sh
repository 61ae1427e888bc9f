#!/bin/bash
# A/B (libhalo_prev.so vs current) of K2 across configs: C1 headline + K2-alone roofline, C2
# tree and C3 analytics K2 rooflines (bench other-configs, 4 layers).
for pass in 1 2; do for v in prev attn; do
HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 400 python bench.py --other-configs tree,analytics --no-cpu-baseline --no-e2e --no-migration --steps 50 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); o=d['other_configs']
print('$v', 'C1 %.4e K2 %.3f layer %.3f' % (d['value'], d['roofline']['frac'], d['layer_roofline']['frac']), 'C2 K2 %.3f' % o['tree']['roofline']['frac'], 'C3 K2 %.3f' % o['analytics']['roofline']['frac'])"
done; done
