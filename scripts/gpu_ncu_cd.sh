cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --target-processes all --kernel-name-base demangled -k regex:gram7 -s 6 -c 1 --set full --import-source on -o gpurun_out/prof_cd_cfg2 ./scripts/cd_bench > gpurun_out/ncu_cd.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_cd.log
echo done
