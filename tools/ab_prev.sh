#!/bin/bash
# A/B of the previous build (libhalo_prev.so) against the current one on the default C1 bench
# line (no extras), alternating passes: value, ms/step, K2 roofline (alone), layer roofline, W.
PASSES=${PASSES:-2}
for pass in $(seq $PASSES); do for v in prev attn; do
HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 300 python bench.py --other-configs "" --no-cpu-baseline --no-e2e --no-migration --steps ${STEPS:-100} 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['layer_roofline']['frac'], d['clocks']['power_w_max'])"
done; done
