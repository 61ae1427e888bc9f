#!/bin/bash
# compute-sanitizer over a subset of the GPU parity tests (small configs): memcheck (out-of-
# bounds / misaligned accesses, leaks of device allocations are not checked: torch caches),
# racecheck (shared-memory hazards) and synccheck (barrier misuse).  Logs to gpurun_out/.
T="tests/test_gpu_parity.py::test_toy_c0_folded tests/test_gpu_parity.py::test_toy_c0_tensor_path_d64_g1 tests/test_gpu_parity.py::test_d64_g2 tests/test_gpu_parity.py::test_g8_and_g1 tests/test_gpu_parity.py::test_tree_two_levels tests/test_gpu_parity.py::test_ragged_suffix_lengths tests/test_gpu_parity.py::test_prefix_read_returns_registered_tensors"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $T -m gpu -x -q -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3 >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
