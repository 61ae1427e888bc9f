python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in "" w12s2bf w8s3 w8s2 w8s3bf; do
  if [ -n "$v" ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_$v.so; else unset HALO_LIB; fi
  python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python -c "
import json,sys;d=json.load(open('gpurun_out/bench_$v.json'));print('$v', round(d['value']), d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['step_breakdown_ms'])" 
done
