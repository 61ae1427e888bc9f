# ncu evidence for one round (one GPU): the launch list of a short bench run, and one
# `ncu --set full` capture each of K2 (C1 and C3) and K1 (C1 and C3) at the bench configuration.
# `bench.py --profile --steps 2 --warmup 3` launches 5 x 32 headline K2s (K1 -> K2 under PDL,
# the co-scheduled schedule) and then 2 x 32 breakdown K2s (K2 launched alone after K1: the
# schedule the bench's `roofline` times) -- `-s 170` picks a breakdown launch, `-s 40` a
# headline one.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefix_attn|suffix_decode|kv_" --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 3 --warmup 3 --other-configs "" > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_decode -s 170 -c 1 -o gpurun_out/k2full -f \
    python bench.py --profile --steps 2 --warmup 3 --other-configs "" > gpurun_out/k2full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_decode -s 40 -c 1 -o gpurun_out/k2full_pdl -f \
    python bench.py --profile --steps 2 --warmup 3 --other-configs "" > gpurun_out/k2full_pdl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_decode -s 8 -c 1 -o gpurun_out/k2full_c3 -f \
    python bench.py --profile --config analytics --layers 2 --steps 1 --warmup 3 --other-configs "" > gpurun_out/k2full_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefix_attn -s 40 -c 1 -o gpurun_out/k1full -f \
    python bench.py --profile --steps 2 --warmup 3 --other-configs "" > gpurun_out/k1full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefix_attn -s 4 -c 1 -o gpurun_out/k1full_c3 -f \
    python bench.py --profile --config analytics --layers 2 --steps 1 --warmup 3 --other-configs "" > gpurun_out/k1full_c3.log 2>&1
ls -la gpurun_out
