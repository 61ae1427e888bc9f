# C1 early-weight check around the default (1.2) with the L2 policy
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/wf_$name.json 2> gpurun_out/wf_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/wf_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/wf_$name.err
}
for rep in 1 2; do
run w1.2_$rep X=0
run w1.1_$rep HALO_K2_EARLY_W=1.1
run w1.0_$rep HALO_K2_EARLY_W=1.0
done
