# round evidence for the headline kernel: launch list (serialised, cold) of the
# timed bench command, and one ncu --set full capture per workload
mkdir -p gpurun_out
TAG=${TAG:-ev}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_${TAG}_c2.csv python bench.py --steps 20 --warmup 3 --no-e2e --cpu-steps 0 > /dev/null 2>&1; echo "list rc=$?"
WORKLOADS="${WORKLOADS:-c2 c4 c5}" TAG=$TAG bash scripts/gpu_prof.sh
