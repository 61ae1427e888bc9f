# one GPU: parity tests, then an ncu --set full capture of K2 (3 launches after warm-up)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
ncu --set full --clock-control none --import-source on -k regex:suffix_decode -s 40 -c 2 -o gpurun_out/k2prof -f python bench.py --profile --steps 2 --warmup 3 > gpurun_out/k2prof.log 2>&1; tail -2 gpurun_out/k2prof.log
