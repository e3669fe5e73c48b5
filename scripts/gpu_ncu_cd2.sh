cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cd_gram7 -s 150 -c 1 -o gpurun_out/prof_cd_cfg2_s4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cd.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_cd.log
echo done
