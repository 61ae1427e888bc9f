# A/B repeat: default lib (K2 L2 evict_first hint) vs libhalo_attn_nohint.so, alternating, with C2/C3
for rep in 1 2; do
for v in hint nohint; do
  if [ $v = nohint ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_nohint.so; else unset HALO_LIB; fi
  python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/l2b_${v}_$rep.json 2> gpurun_out/l2b_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/l2b_${v}_$rep.json')); o=d.get('other_configs',{})
print('$v$rep', round(d['value']/1e6,3), 'k2', round(d['roofline']['frac'],3), 'k1', round(d['prefix_roofline']['frac'],3),
      'C2', round(o['tree']['queries_per_s_kernels']/1e6,3), round(o['tree']['roofline']['frac'],3),
      'C3', round(o['analytics']['queries_per_s_kernels']/1e6,3), round(o['analytics']['roofline']['frac'],3))" || tail -3 gpurun_out/l2b_${v}_$rep.err
done
done
nvidia-smi --query-gpu=name,serial,clocks.max.sm,clocks.max.mem --format=csv
