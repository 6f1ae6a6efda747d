# f32 mask prefilter: parity suite, then c2s with and without the prefilter
mkdir -p gpurun_out
TAG=${TAG:-f32m}
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_$TAG.log
for W in c2s c3f; do
timeout 600 python bench.py --workload $W --cpu-steps 0 --no-e2e > gpurun_out/bench_${TAG}_$W.json 2> gpurun_out/bench_${TAG}_$W.err; echo "$W rc=$?"
FS_NO_F32_MASK=1 timeout 600 python bench.py --workload $W --cpu-steps 0 --no-e2e > gpurun_out/bench_${TAG}_${W}_nomask.json 2> gpurun_out/bench_${TAG}_${W}_nomask.err; echo "$W nomask rc=$?"
done
FS_MERGE_FUSED=1 timeout 600 python bench.py --workload c3f --cpu-steps 0 --no-e2e > gpurun_out/bench_${TAG}_c3f_fused.json 2> gpurun_out/bench_${TAG}_c3f_fused.err; echo "c3f fused rc=$?"
for f in gpurun_out/bench_${TAG}_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],2), round(d['ms_per_step']*1e3,1), (d.get('value_l2_warm') or {}).get('value'))"; done
