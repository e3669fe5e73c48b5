cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -rf -k concurrent > gpurun_out/pytest_conc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_conc.log
echo done
