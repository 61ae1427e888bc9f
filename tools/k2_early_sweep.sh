# C1 headline vs K2 early-CTA weight (HALO_K2_EARLY_W) x K1 split cap (HALO_MAX_SPLITS) x K2 shape
set -x
run() {  # name, env...
  name=$1; shift
  env "$@" python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/early_$name.json 2> gpurun_out/early_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/early_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'), d['step_breakdown_ms'])"
}
run base X=0
for s in 4 3 2; do
  for w in 1.5 2 3 4; do
    run s${s}_w${w} HALO_MAX_SPLITS=$s HALO_K2_EARLY_W=$w
  done
done
for s in 4 2; do
  for w in 1 2 3; do
    run wide_s${s}_w${w} HALO_K2_FORCE_WIDE=1 HALO_MAX_SPLITS=$s HALO_K2_EARLY_W=$w
  done
done
