# sweep the streaming kernel's CTA size / slot count (quick bench, no e2e)
mkdir -p gpurun_out
for B in 512 768; do for S in 2 3 4; do
  FS_TMA_BLOCK=$B FS_TMA_SLOTS=$S timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-steps 1 > gpurun_out/sw_${B}_${S}.json 2>gpurun_out/sw_${B}_${S}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sw_${B}_${S}.json')); print('block $B slots $S', round(d['value'],2), 'warm', round(d['value_l2_warm']['value'],2), round(d['value_l2_warm']['ms_per_step']*1e3,1),'us')" || tail -3 gpurun_out/sw_${B}_${S}.err
done; done
