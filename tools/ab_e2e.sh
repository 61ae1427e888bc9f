#!/bin/bash
# A/B (libhalo_prev.so vs current) of the end-to-end leg (halo_decode_step with pinned host
# buffers, C1) and the continuous-batching leg.
for pass in 1 2 3; do for v in prev attn; do
HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_$v.so timeout 400 python bench.py --other-configs "" --no-cpu-baseline --no-migration --steps 30 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'C1 %.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], 'continuous %.4e' % d['continuous']['value'])"
done; done
