set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-steps 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --cpu-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_full_size.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/pytest_gpu.log
