cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_logistic.py -q -x -k single_cta --timeout 600 -rf > gpurun_out/pytest_single.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_single.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_batch_mma -s 20 -c 1 -o gpurun_out/prof_bmma2 python scripts/cv_small.py 200000 > gpurun_out/ncu_bmma.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_bmma.log
echo done
