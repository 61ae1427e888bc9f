# One GPU, end of a measurement cycle: GPU tests, the default bench line, then the ncu
# captures of tools/round_ncu.sh (launch list + `--set full` of K1 and K2 at C1 and C3).
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
bash tools/round_ncu.sh
