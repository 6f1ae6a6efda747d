# lockstep ensembles: tests, the ens bench, and a C2 regression check
mkdir -p gpurun_out
TAG=${TAG:-ens}
timeout 900 python -m pytest tests/test_ensemble.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --workload ens --cpu-steps 0 > gpurun_out/bench_${TAG}_ens.json 2> gpurun_out/bench_${TAG}_ens.err; echo "ens rc=$?"
tail -3 gpurun_out/bench_${TAG}_ens.err
timeout 600 python bench.py --cpu-steps 0 --no-e2e > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo "c2 rc=$?"
