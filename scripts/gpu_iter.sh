# quick iteration: selected gpu tests + benches of the given workloads
set -x
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 900 python -m pytest ${TESTS:-tests} -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_$TAG.log
for W in ${WORKLOADS:-c2}; do
  timeout 900 python bench.py --workload $W ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "bench $W rc=$?"
  cat gpurun_out/bench_${TAG}_$W.json; tail -3 gpurun_out/bench_${TAG}_$W.err
done
