# round-2 evidence, all from one build (lib sha recorded): smoke, gpu tests,
# bench lines for every workload (with CPU baselines), the reference arm, the
# launch list of the headline command, and one `ncu --set full` capture of the
# dominant kernel per workload, digested on the box (summary + hot source lines
# + ncu_summary.json); the reports themselves stay on the box
mkdir -p gpurun_out
TAG=${TAG:-r2ev}
sha256sum paper_2604_22092_b200/libflashspread_b200.so | cut -c1-16 > gpurun_out/lib_sha16_$TAG.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
  tail -2 gpurun_out/pytest_gpu_$TAG.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo "bench c2 rc=$?"
  for W in ${WORKLOADS:-c3 c4 c5 c2s c3f c3c ens m2 c1}; do
    timeout 900 python bench.py --workload $W --cpu-steps ${CPU_STEPS:-10} > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "bench $W rc=$?"
  done
  timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_ref_c2.json 2> gpurun_out/bench_${TAG}_ref_c2.err; echo "ref rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_${TAG}_c2.csv python bench.py --steps 20 --warmup 3 --no-e2e --cpu-steps 0 > /dev/null 2>&1; echo "list rc=$?"
  # the C4 step kernel over the bench window (its per-launch times grow with the epidemic)
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_step_incr$" --csv --log-file gpurun_out/launches_${TAG}_c4.csv python bench.py --workload c4 --steps 50 --warmup 3 --no-e2e --cpu-steps 0 > /dev/null 2>&1; echo "list c4 rc=$?"
  timeout 900 python bench.py --partitioned --workload c5 --steps 50 --warmup 3 --cpu-steps 0 > gpurun_out/bench_${TAG}_c5_partitioned_world1.json 2> gpurun_out/bench_${TAG}_c5p.err; echo "c5 partitioned rc=$?"
fi
for W in ${PROF:-c2 c3 c4 c5 c2s c3f c3c ens}; do
  case $W in c2s|c3f|c3c) K="^k_step$";; ens) K="^k_step_incr_persist$";; *) K="^k_step_incr$";; esac
  R=gpurun_out/prof_${TAG}_$W
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-6} -c 1 -o $R -f \
    python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --cpu-steps 0 > gpurun_out/ncu_${TAG}_$W.log 2>&1; echo "ncu $W rc=$?"
  python scripts/ncu_hot.py $R.ncu-rep 40 > gpurun_out/${TAG}_${W}_ncu_hot.txt 2>&1
done
OUT=gpurun_out python scripts/ncu_to_summary.py $TAG ${PROF:-c2 c3 c4 c5 c2s c3f c3c ens}
rm -f gpurun_out/prof_${TAG}_*.ncu-rep
du -sh gpurun_out
