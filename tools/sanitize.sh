#!/bin/bash
# compute-sanitizer (memcheck: out-of-bounds / misaligned accesses; racecheck: shared-memory
# hazards; synccheck: barrier misuse) over GPU tests that cover every kernel and path:
# small trees (K1 d=64/128, g=1..8, K2 folded), C1-size batches (256 requests x 2k prefix,
# default plan, SM cap, K1 rule off), K2 stream-K with 1-block chunks, K2 launched alone (the
# whole-unit narrow schedule at C1), prefill (causal K1),
# V beyond fp16 range (scaled converters), host paging (fetch + V-table recompute), and
# NCCL loopback migration (pack / unpack).  Logs in gpurun_out/sanitize_*.log.
P=tests/test_gpu_parity.py
T="$P::test_toy_c0_folded $P::test_toy_c0_tensor_path_d64_g1 $P::test_d64_g2 $P::test_g8_and_g1
$P::test_tree_two_levels $P::test_ragged_suffix_lengths $P::test_prefix_read_returns_registered_tensors
$P::test_plan_options_sm_cap_and_k1_rule $P::test_k2_work_queue_chunking[1]
$P::test_k2_alone_uses_the_equal_share_schedule_and_matches_oracle
$P::test_prefill_against_cached_prefixes_matches_oracle[1]
tests/test_gpu_inputs.py::test_v_beyond_fp16_range_huge_tiny_and_growing[1-3]
tests/test_paging.py::test_offload_fetch_round_trip_is_bit_exact_and_decodes_identically
tests/test_migration.py::test_exchange_many_nodes_ragged_chunks[1048576]"
: > gpurun_out/sanitize_summary.txt
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $T -m gpu -x -q -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3 >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
