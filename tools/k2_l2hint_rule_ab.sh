# with the K2 L2 evict_first hint (default): single-wave K1 rule on/off, and the no-hint build
run() {
  name=$1; shift
  env "$@" python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/l2r_$name.json 2> gpurun_out/l2r_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/l2r_$name.json')); print('$name', round(d['value']/1e6,3), 'Mq/s', 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3), 'tiles', d['config'].get('k1_tiles'))" || tail -3 gpurun_out/l2r_$name.err
}
run hint_rule X=0
run hint_norule HALO_K1_SM_FRAC=0
run nohint_rule HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_nohint.so
run nohint_norule HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_nohint.so HALO_K1_SM_FRAC=0
run hint_rule_w1.35 HALO_K2_EARLY_W=1.35
run hint_s2_w1.2 HALO_MAX_SPLITS=2 HALO_K2_EARLY_W=1.2
run hint_rule2 X=0
run hint_norule2 HALO_K1_SM_FRAC=0
