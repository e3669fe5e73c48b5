cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_outofcore.py -q --timeout 600 -rf > gpurun_out/pytest_ooc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ooc.log
timeout 900 python bench.py --config cfg3 --resident host --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_host.log 2>&1
timeout 900 python bench.py --config cfg4 --resident host --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_host.log 2>&1
echo done
