# narrow K2 shape only for short units (< 8 blocks): fan-out probe, C1 headline
python tools/k2_early_probe.py short_narrow 2>/dev/null
python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', round(d['value']/1e6,3), 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3))"
