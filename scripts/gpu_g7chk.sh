cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rf -k "not full_size and not cfg5_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --config logit --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_logit.log 2>&1
echo done
