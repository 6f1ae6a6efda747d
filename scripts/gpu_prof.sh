# one ncu --set full capture of the step kernel per workload
mkdir -p gpurun_out
TAG=${TAG:-prof}
for W in ${WORKLOADS:-c2}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_step -s ${SKIP:-6} -c 1 -o gpurun_out/prof_${TAG}_$W -f \
    python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --cpu-steps 0 ${BENCH_ARGS} > gpurun_out/ncu_${TAG}_$W.log 2>&1; echo "ncu $W rc=$?"
  tail -2 gpurun_out/ncu_${TAG}_$W.log
done
