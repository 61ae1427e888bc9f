#!/bin/bash
# K2 alone on a restricted number of SMs (HALO_K2_SMS): its per-SM streaming capability.
for n in 148 128 112 96 84 72 64; do
  for c in fanout analytics; do
    HALO_K2_SMS=$n CFG=$c LAYERS=2 python tools/k2_trace.py > gpurun_out/k2sms_${c}_$n.log 2>&1
  done
done
grep -H "alone" gpurun_out/k2sms_*.log
