# compute-sanitizer over small cases of every kernel family (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_engine_parity.py::test_trajectory_parity_graph_replay tests/test_engine_parity.py::test_variants_are_result_neutral tests/test_markov.py::test_markov_steps_bit_exact tests/test_distributed.py::test_virtual_ranks_match_single_engine tests/test_graphgen.py::test_device_generator_matches_host_rows tests/test_graphgen.py::test_ba_device_structure tests/test_graphgen.py::test_er_device_structure_and_law tests/test_analysis.py::test_device_records_match_reference tests/test_analysis.py::test_device_fidelity_matches_reference tests/test_analysis.py::test_device_column_quantiles_match_numpy"
# round 2: the f32 fold with the mask and the one-launch edge-merge (hub pre-pass with release/acquire tags),
# lockstep ensembles and batched seed selection, the bulk exchange (mailbox staging / apply), IPC transport
T="$T tests/test_engine_parity.py::test_gather_forms_bit_exact tests/test_ensemble.py::test_lockstep_equals_stream_runner tests/test_ensemble.py::test_batched_init_equals_per_trial_init tests/test_distributed.py::test_edge_balanced_virtual_ranks_match_single_engine"
T=${TESTS:-$T}
for TOOL in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $TOOL --error-exitcode 99 --print-limit 20 python -m pytest $T -q -x -m gpu -p no:cacheprovider > gpurun_out/sanitize_$TOOL.log 2>&1; echo "$TOOL rc=$?"
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$TOOL.log | tail -3
done
