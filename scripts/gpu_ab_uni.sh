# same-box A/B of the uniform-S-age kernel (FS_NO_UNI=1 switches it off)
mkdir -p gpurun_out
TAG=${TAG:-ab}
for W in ${WORKLOADS:-c2 c4}; do
  for V in off on; do
    if [ $V = off ]; then export FS_NO_UNI=1; else unset FS_NO_UNI; fi
    timeout 900 python bench.py --workload $W --cpu-steps 0 ${BENCH_ARGS} > gpurun_out/ab_${TAG}_${W}_$V.json 2> gpurun_out/ab_${TAG}_${W}_$V.err; echo "bench $W $V rc=$?"
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${TAG}_${W}_$V.json')); print('$W $V', round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us warm', round(d['value_l2_warm']['value'],2), 'e2e', d['e2e'] and round(d['e2e']['value'],2), d['e2e'] and d['e2e'].get('final_R'))" 2>&1 | tail -1
  done
done
unset FS_NO_UNI
