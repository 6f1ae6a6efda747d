# A/B: workloads with and without an env toggle (quick, no e2e/cpu)
mkdir -p gpurun_out
TAG=${TAG:-ab}
for W in ${WORKLOADS:-c4}; do
  for V in "" "$TOGGLE"; do
    env $V timeout 900 python bench.py --workload $W --steps ${STEPS:-100} --no-e2e --cpu-steps 0 > gpurun_out/ab_${TAG}_${W}_${V:-base}.json 2> gpurun_out/ab_${TAG}_${W}_${V:-base}.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${TAG}_${W}_${V:-base}.json')); print('$W', '${V:-base}', round(d['value'],3), 'G-NUPS', round(d['ms_per_step'],4), 'ms', 'warm', round(d['value_l2_warm']['value'],3))" || tail -3 gpurun_out/ab_${TAG}_${W}_${V:-base}.err
  done
done
