#!/bin/bash
# A/B of K2 schedules on the GPU box: static vs dynamic (narrow / wide launch shape).
# Writes gpurun_out/ab_<variant>.json (bench line) and k2 traces per variant.
for v in static dyn dynwide; do
  case $v in
    static) export HALO_K2_SCHED=static; unset HALO_K2_SHAPE;;
    dyn) export HALO_K2_SCHED=dyn; unset HALO_K2_SHAPE;;
    dynwide) export HALO_K2_SCHED=dyn; export HALO_K2_SHAPE=wide;;
  esac
  python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-migration > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  for c in fanout analytics; do CFG=$c LAYERS=2 python tools/k2_trace.py > gpurun_out/k2trace_${c}_$v.log 2>&1; done
done
