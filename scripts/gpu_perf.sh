# perf iteration: quick parity + bench + launch list + one full ncu capture of the step kernel
set -x
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider --deselect tests/test_full_size.py > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-steps 3 ${BENCH_ARGS} > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-e2e --cpu-steps 1 ${BENCH_ARGS} > /dev/null 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 6 -c 1 -o gpurun_out/prof_$TAG -f python bench.py --steps 10 --warmup 3 --no-e2e --cpu-steps 1 ${BENCH_ARGS} > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
