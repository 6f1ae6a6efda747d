# compute-sanitizer over small cases of every kernel family (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_engine_parity.py::test_trajectory_parity_graph_replay tests/test_engine_parity.py::test_variants_are_result_neutral tests/test_markov.py::test_markov_steps_bit_exact tests/test_distributed.py::test_virtual_ranks_match_single_engine tests/test_graphgen.py::test_device_generator_matches_host_rows tests/test_graphgen.py::test_ba_device_structure tests/test_graphgen.py::test_er_device_structure_and_law tests/test_analysis.py::test_device_records_match_reference tests/test_analysis.py::test_device_fidelity_matches_reference tests/test_analysis.py::test_device_column_quantiles_match_numpy"
for TOOL in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $TOOL --error-exitcode 99 --print-limit 20 python -m pytest $T -q -x -m gpu -p no:cacheprovider > gpurun_out/sanitize_$TOOL.log 2>&1; echo "$TOOL rc=$?"
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$TOOL.log | tail -3
done
