# quick round-start check: smoke, gpu tests, bench lines for the named workloads
mkdir -p gpurun_out
TAG=${TAG:-q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
for W in ${WORKLOADS:-c2}; do
  timeout 900 python bench.py --workload $W ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "bench $W rc=$?"
  cat gpurun_out/bench_${TAG}_$W.json
done
