#!/bin/bash
# C1 headline vs K1 split cap (HALO_MAX_SPLITS: fewer, longer K1 tiles -> fewer partial slots)
for s in 0 1 2 3; do
  HALO_MAX_SPLITS=$s python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/splits_$s.json 2> gpurun_out/splits_$s.err
done
