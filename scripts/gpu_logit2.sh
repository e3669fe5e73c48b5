cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_logistic.py -q -x --timeout 600 -rf > gpurun_out/pytest_logit.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_logit.log
timeout 900 python bench.py --config logit --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_logit.log 2>&1
echo done
