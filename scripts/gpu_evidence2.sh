# round-2 evidence: library sha, bench lines per workload, one ncu --set full
# capture of the dominant kernel per workload, launch list of the headline
mkdir -p gpurun_out
TAG=${TAG:-ev}
sha256sum paper_2604_22092_b200/libflashspread_b200.so | cut -c1-16 > gpurun_out/lib_sha16_$TAG.txt
for W in ${WORKLOADS:-c2}; do
  timeout 900 python bench.py --workload $W ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "bench $W rc=$?"
done
for W in ${PROF:-}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_step}" -s ${SKIP:-6} -c 1 -o gpurun_out/prof_${TAG}_$W -f \
    python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --cpu-steps 0 > gpurun_out/ncu_${TAG}_$W.log 2>&1; echo "ncu $W rc=$?"
done
if [ -n "$LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_${TAG}_$LAUNCHES.csv python bench.py --workload $LAUNCHES --steps 20 --warmup 3 --no-e2e --cpu-steps 0 > /dev/null 2>&1; echo "list rc=$?"
fi
