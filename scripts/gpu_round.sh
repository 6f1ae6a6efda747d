# full round evidence: smoke, gpu tests, bench (json), launch list, one ncu --set full capture of the step kernel
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-e2e --cpu-steps 1 ${BENCH_ARGS} > /dev/null 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 6 -c 1 -o gpurun_out/prof_$TAG -f python bench.py --steps 10 --warmup 3 --no-e2e --cpu-steps 1 ${BENCH_ARGS} > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
