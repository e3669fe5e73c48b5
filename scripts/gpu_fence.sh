cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./scripts/cd_bench > gpurun_out/cd_bench.log 2>&1; echo "rc=$?" >> gpurun_out/cd_bench.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rf -k "not cfg5_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in cfg2 cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
echo done
