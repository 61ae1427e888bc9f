# finer sweep around HALO_MAX_SPLITS=2, HALO_K2_EARLY_W=1.5 (tools/k2_early_sweep.sh); base repeated for noise
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/early2_$name.json 2> gpurun_out/early2_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/early2_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))"
}
run base1 X=0
for w in 1.2 1.35 1.5 1.7; do run s2_w$w HALO_MAX_SPLITS=2 HALO_K2_EARLY_W=$w; done
for w in 1.2 1.35; do run s3_w$w HALO_MAX_SPLITS=3 HALO_K2_EARLY_W=$w; done
for w in 1.15 1.3; do run s4_w$w HALO_MAX_SPLITS=4 HALO_K2_EARLY_W=$w; done
for w in 1.2 1.5; do run wide_s2_w$w HALO_K2_FORCE_WIDE=1 HALO_MAX_SPLITS=2 HALO_K2_EARLY_W=$w; done
run base2 X=0
