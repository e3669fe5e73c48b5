cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./scripts/cd_bench > gpurun_out/cd_bench.log 2>&1; echo "rc=$?" >> gpurun_out/cd_bench.log
if [ "$1" = "test" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
echo done
