# K2 register parking (HALO_K2_PARK) A/B on C1, with split caps / early weights around the default rule
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/park_$name.json 2> gpurun_out/park_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/park_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/park_$name.err
}
run park1_default X=0
run park0_default HALO_K2_PARK=0
run park1_rule_off HALO_K1_SM_FRAC=0
run park0_rule_off HALO_K2_PARK=0 HALO_K1_SM_FRAC=0
for w in 1.35 1.5 1.7; do run park1_s3_w$w HALO_MAX_SPLITS=3 HALO_K2_EARLY_W=$w; done
for w in 1.2 1.5 1.8 2.2; do run park1_s2_w$w HALO_MAX_SPLITS=2 HALO_K2_EARLY_W=$w; done
run park1_s4_w1.3 HALO_MAX_SPLITS=4 HALO_K2_EARLY_W=1.3
