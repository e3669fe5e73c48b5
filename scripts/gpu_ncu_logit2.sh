cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_logistic.py -q -x --timeout 600 -rf > gpurun_out/pytest_logit.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_logit.log
timeout 600 ncu --kernel-name-base demangled -k regex:k_cd_logit_gram -s 150 -c 1 --set full --import-source on -o gpurun_out/prof_logit_gram python scripts/logit_small.py > gpurun_out/ncu_logit.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_logit.log
echo done
