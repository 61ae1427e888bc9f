# K2 launch shape under the single-wave K1 rule (C1): default (weighted cuts -> wide + pieces) vs forced narrow
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/shape_$name.json 2> gpurun_out/shape_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/shape_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/shape_$name.err
}
run default X=0
run rule_off HALO_K1_SM_FRAC=0
for w in 1.0 1.1 1.2 1.3; do run narrow_w$w HALO_K2_FORCE_NARROW=1 HALO_K2_EARLY_W=$w; done
run default2 X=0
