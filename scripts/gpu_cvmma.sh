cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -rf -k "cv" > gpurun_out/pytest_cv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cv.log
BL_CV_MMA=0 timeout 600 python scripts/cv_small.py 200000 > gpurun_out/cv_fma.log 2>&1
BL_CV_MMA=1 timeout 600 python scripts/cv_small.py 200000 > gpurun_out/cv_mma.log 2>&1
echo done
