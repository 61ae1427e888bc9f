#!/bin/bash
# A/B of K1 build variants: default lib vs libhalo_attn_<v>.so (HALO_LIB), bench K1 fractions + parity.
for v in "" "$@"; do
  if [ -n "$v" ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_$v.so; else unset HALO_LIB; fi
  python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/k1ab_$v.json 2> gpurun_out/k1ab_$v.err
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/k1ab_parity_$v.log 2>&1
done
