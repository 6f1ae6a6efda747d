# A/B of the in-tree library against ab_libs/$BASE (FS_LIB_PATH) on one box:
# optional parity subset, then bench value / warm / per-window e2e for $WORKLOADS, interleaved
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "$PYTEST_K" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
fi
for rep in 1 2; do
for W in ${WORKLOADS:-c2 c3 c4}; do
  for V in new base; do
    if [ $V = base ]; then export FS_LIB_PATH=$PWD/ab_libs/${BASE:-base.so}; else unset FS_LIB_PATH; fi
    timeout 600 python bench.py --workload $W --cpu-steps 0 ${BENCH_ARGS:---no-e2e} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d.get(\"e2e\") or {}; print(\"$W $V\", round(d[\"value\"],2), round(d[\"ms_per_step\"]*1e3,2), round(d[\"value_l2_warm\"][\"value\"],2), e.get(\"value\") and round(e[\"value\"],2))"
  done
done
done
unset FS_LIB_PATH
if [ -n "$E2E" ]; then for V in new base; do
  if [ $V = base ]; then export FS_LIB_PATH=$PWD/ab_libs/${BASE:-base.so}; else unset FS_LIB_PATH; fi
  echo "e2e windows $V"; python scripts/e2e_batches.py 2>&1 | tail -2
done; unset FS_LIB_PATH; fi
