# one ncu --set full capture of kernel regex $K in `bench.py --workload $W` (after $SKIP matching launches),
# digested on the box (summary + hot source lines); the report is kept only if KEEP is set
mkdir -p gpurun_out
TAG=${TAG:-one}
R=gpurun_out/prof_${TAG}_$W
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${K:-k_step} -s ${SKIP:-5} -c 1 -o $R -f \
  python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --cpu-steps 0 ${BENCH_ARGS} > gpurun_out/ncu_${TAG}_$W.log 2>&1; echo "ncu $W rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > gpurun_out/${TAG}_${W}_ncu_summary.txt 2>&1
python scripts/ncu_hot.py $R.ncu-rep 40 > gpurun_out/${TAG}_${W}_ncu_hot.txt 2>&1
[ -z "$KEEP" ] && rm -f $R.ncu-rep
head -40 gpurun_out/${TAG}_${W}_ncu_summary.txt
