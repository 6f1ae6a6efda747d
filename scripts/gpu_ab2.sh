# A/B/C/... of env variants on one box: VARIANTS="A=1 B=2|C=3" (| separates variants, "" = base)
mkdir -p gpurun_out
TAG=${TAG:-ab2}
IFS='|' read -ra VS <<< "base|${VARIANTS}"
for R in 1 2; do
for W in ${WORKLOADS:-c2}; do
  for V in "${VS[@]}"; do
    E=""; [ "$V" != "base" ] && E="$V"
    env $E timeout 900 python bench.py --workload $W --steps ${STEPS:-200} ${E2E:---no-e2e} --cpu-steps 0 > gpurun_out/ab2.json 2> gpurun_out/ab2.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab2.json')); e=d.get('e2e') or {}; print('rep $R', '$W', '$V', round(d['value'],2), 'G-NUPS', round(d['ms_per_step']*1e3,2), 'us', 'warm', round(d['value_l2_warm']['value'],2), 'e2e', round(e.get('value',0),2), round(e.get('wall_s',0),3))" || tail -3 gpurun_out/ab2.err
  done
done
done
