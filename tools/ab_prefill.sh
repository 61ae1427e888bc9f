#!/bin/bash
# A/B (previous build vs current) of the legs a K3-merge change moves: prefill (merge-only
# K2 units: prompt rows), C2 tree (two partial slots per request) -- K2 roofline fractions.
for pass in 1 2; do for v in prev attn; do
HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 400 python bench.py --other-configs tree --no-cpu-baseline --no-migration --steps 30 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; t=d['other_configs']['tree']
print('$v', 'C1 %.3e' % d['value'], 'prefill layer_ms %.3f K2 %.3f K1 %.3f' % (p['layer_ms'], p['suffix_roofline']['frac'], p['prefix_roofline']['frac']), 'tree K2 %.3f layer_ms %.4f' % (t['roofline']['frac'], t['layer_ms']))"
done; done
