# C1 early-weight check around the default (1.2) with the L2 policy
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/wf_$name.json 2> gpurun_out/wf_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/wf_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/wf_$name.err
}
[ -n "$1" ] || for rep in 1 2; do
run w1.2_$rep X=0
run w1.1_$rep HALO_K2_EARLY_W=1.1
run w1.0_$rep HALO_K2_EARLY_W=1.0
done
# (second pass) the wide shape without weights at 96 K1 CTAs: is it the shape or the weights?
if [ "$1" = wide ]; then
for rep in 1 2; do
run wide_w1.0_$rep HALO_K2_FORCE_WIDE=1 HALO_K2_EARLY_W=1.0
run wide_w1.2_$rep HALO_K2_FORCE_WIDE=1
done
fi
# (third pass) rule off (128 K1 CTAs): narrow (planner's choice) vs forced wide, with the L2 policy
if [ "$1" = norule ]; then
for rep in 1 2; do
run norule_narrow_$rep HALO_K1_SM_FRAC=0
run norule_wide_$rep HALO_K1_SM_FRAC=0 HALO_K2_FORCE_WIDE=1
done
fi
