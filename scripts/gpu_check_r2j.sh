# full GPU suite + smoke + ensemble phases + short bench lines on the in-tree build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_r2j.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r2j.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2j.log 2>&1; echo "smoke rc=$?"
unset FS_PERSIST_BLOCK; python scripts/ens_phases.py 2>&1 | tail -3
for W in ens c2 c3; do
  timeout 600 python bench.py --workload $W --cpu-steps 0 2>/dev/null > gpurun_out/bench_r2j_$W.json
  python -c "import json; d=json.loads(open('gpurun_out/bench_r2j_$W.json').read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('$W', round(d['value'],3), e.get('value') and round(e['value'],2))"
done
