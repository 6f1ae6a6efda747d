# end-of-iteration evidence: full gpu tests, smoke, bench lines for every workload,
# reference arm, launch list and ncu captures of the headline kernel
set -x
mkdir -p gpurun_out
TAG=${TAG:-fin}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo "bench c2 rc=$?"
for W in ${WORKLOADS:-c3 c4 c5 c1}; do
  timeout 900 python bench.py --workload $W --cpu-steps 10 > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "bench $W rc=$?"
done
timeout 900 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_${TAG}_ref_c2.json 2> gpurun_out/bench_${TAG}_ref_c2.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_${TAG}_c2.csv python bench.py --steps 20 --warmup 3 --no-e2e --cpu-steps 0 > /dev/null 2>&1; echo "list rc=$?"
WORKLOADS="${PROF:-c2}" TAG=$TAG bash scripts/gpu_prof.sh
