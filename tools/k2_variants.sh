for v in "" w7s4 w8s3; do
  if [ -n "$v" ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_$v.so; else unset HALO_LIB; fi
  python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/bench_k2_$v.json 2> gpurun_out/bench_k2_$v.err
done
