#!/bin/bash
# K1 A/B: split P.V (default lib) vs no split (libhalo_attn_nosplit.so), and the K1 tile order.
run() {  # name, env...
  local name=$1; shift
  env "$@" python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/k1ab2_$name.json 2> gpurun_out/k1ab2_$name.err
}
run split
run nosplit HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_nosplit.so
run split_mouter HALO_K1_TILE_ORDER=mouter
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/k1ab2_parity.log 2>&1; tail -1 gpurun_out/k1ab2_parity.log
CFG=fanout python tools/k1_trace.py > gpurun_out/k1trace_fanout.log 2>&1
CFG=analytics python tools/k1_trace.py > gpurun_out/k1trace_analytics.log 2>&1
