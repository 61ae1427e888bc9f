#!/bin/bash
# Run-to-run spread of the default C1 bench line (headline, K2-alone roofline, equal-share
# K2, K1, breakdown gaps); GATE=0/1 toggles the breakdown pass's spin-kernel gate.
for i in 1 2 3 4; do for gate in ${GATES:-1}; do
HALO_BENCH_GATE=$gate timeout 300 python bench.py --other-configs "" --no-cpu-baseline --no-e2e --no-migration --steps 100 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('gate=$gate', 'q/s %.4e' % d['value'], 'K2 alone %.2f us roofline %.3f' % (d['roofline']['avg_launch_ms'] * 1e3, d['roofline']['frac']), 'eq %.3f' % d['roofline_k2_equal_shares']['frac'], 'K1 %.3f' % d['prefix_roofline']['frac'], 'layers %.3f gaps %.3f' % (b['layers'], b['gaps']), 'MHz %s W %.0f' % (d['clocks']['sm_mhz'], d['clocks']['power_w_max']))"
done; done
