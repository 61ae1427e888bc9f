# wide K2 shape by default (narrow only with HALO_K2_AUTO_NARROW=1): rule on/off, old behaviour
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/wd_$name.json 2> gpurun_out/wd_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/wd_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/wd_$name.err
}
for rep in 1 2; do
run rule_$rep X=0
run norule_$rep HALO_K1_SM_FRAC=0
run old_norule_$rep HALO_K1_SM_FRAC=0 HALO_K2_AUTO_NARROW=1
done
python tools/k2_early_probe.py wide_rule 2>/dev/null
HALO_K1_SM_FRAC=0 python tools/k2_early_probe.py wide_norule 2>/dev/null
