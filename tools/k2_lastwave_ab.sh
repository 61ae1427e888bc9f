# C2 (tree, 384 K1 tiles = 2.6 waves): weight the K2 CTAs that start beside K1's partial last wave
run() {
  name=$1; shift
  env "$@" python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --config tree --other-configs "" > gpurun_out/lw_$name.json 2> gpurun_out/lw_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/lw_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/lw_$name.err
}
for rep in 1 2; do
run base$rep X=0
for w in 1.1 1.2 1.35; do run w${w}_$rep HALO_K2_EARLY_LASTWAVE=1 HALO_K2_EARLY_W=$w; done
done
