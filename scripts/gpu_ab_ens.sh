# A/B of the ensemble workload: in-tree library (1024 / 512-thread member CTAs) against ab_libs/base.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ensemble.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_ab_ens.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ab_ens.log
for rep in 1 2; do
  for V in new new512 base; do
    unset FS_LIB_PATH FS_PERSIST_BLOCK
    [ $V = base ] && export FS_LIB_PATH=$PWD/ab_libs/base.so
    [ $V = new512 ] && export FS_PERSIST_BLOCK=512
    timeout 600 python bench.py --workload ens --cpu-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ens $V', round(d['value'],3), [round(w*1e3,2) for w in d['engine']['wall_s']])"
  done
done
unset FS_LIB_PATH FS_PERSIST_BLOCK
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:persist --csv python scripts/prof_ens.py 2>/dev/null | grep -c persist
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:persist -c 3 --csv python scripts/prof_ens.py 2>/dev/null | grep persist | tail -3 | cut -c1-300
