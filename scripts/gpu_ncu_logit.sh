cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/logit_small.py > gpurun_out/logit_small.log 2>&1
timeout 600 ncu --kernel-name-base demangled -k regex:k_cd_logit -s 60 -c 1 --set full --import-source on -o gpurun_out/prof_logit python scripts/logit_small.py > gpurun_out/ncu_logit.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_logit.log
echo done
