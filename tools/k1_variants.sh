for v in "" nopp; do
  if [ -n "$v" ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_$v.so; else unset HALO_LIB; fi
  python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/bench_k1_$v.json 2> gpurun_out/bench_k1_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_k1_$v.json'));print('$v', round(d['value']), 'k1', round(d['prefix_roofline']['frac'],3), [ (k, round(v['prefix_roofline']['frac'],3)) for k,v in d['other_configs'].items()])"
done
