cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_outofcore.py tests/test_gpu_sharded.py -q --timeout 600 -rf > gpurun_out/pytest_ooc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ooc.log
echo done
