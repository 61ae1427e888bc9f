# end-of-session: GPU tests, rule on/off with the L2 hint, the default bench line, ncu refresh
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/fin_$name.json 2> gpurun_out/fin_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/fin_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/fin_$name.err
}
run rule X=0
run norule HALO_K1_SM_FRAC=0
run rule_w1.35 HALO_K2_EARLY_W=1.35
run s2_w1.2 HALO_MAX_SPLITS=2 HALO_K2_EARLY_W=1.2
run rule2 X=0
run norule2 HALO_K1_SM_FRAC=0
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; head -c 300 gpurun_out/bench_full.json; echo
bash tools/round_ncu.sh > gpurun_out/round_ncu.log 2>&1
ls gpurun_out/*.ncu-rep
