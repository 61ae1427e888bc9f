# one GPU: ncu --set full capture of K1 on C3 (analytics, 2 layers)
ncu --set full --clock-control none --import-source on -k regex:prefix_attn -s 4 -c 1 -o gpurun_out/k1prof -f python bench.py --profile --config analytics --layers 2 --steps 1 --warmup 3 --other-configs "" > gpurun_out/k1prof.log 2>&1; tail -2 gpurun_out/k1prof.log
