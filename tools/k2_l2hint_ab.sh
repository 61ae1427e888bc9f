# A/B: K2 suffix K/V bulk copies with an L2 evict_first policy (libhalo_attn_ef.so, -DHALO_K2_L2_EVICT_FIRST)
for rep in 1 2; do
for v in base ef; do
  if [ $v = ef ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_ef.so; else unset HALO_LIB; fi
  python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/l2h_${v}_$rep.json 2> gpurun_out/l2h_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/l2h_${v}_$rep.json')); o=d.get('other_configs',{})
print('$v$rep', round(d['value']/1e6,3), 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3),
      'C2', round(o['tree']['queries_per_s_kernels']/1e6,3), round(o['tree']['roofline']['frac'],3),
      'C3', round(o['analytics']['queries_per_s_kernels']/1e6,3), round(o['analytics']['roofline']['frac'],3))" || tail -3 gpurun_out/l2h_${v}_$rep.err
done
done
export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_ef.so
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/l2h_parity.log 2>&1; tail -1 gpurun_out/l2h_parity.log
