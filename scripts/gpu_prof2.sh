cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_fp -s 2 -c 1 -o gpurun_out/prof_scan_cfg2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_i8 -s 2 -c 1 -o gpurun_out/prof_scan_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_fp -s 2 -c 1 -o gpurun_out/prof_scan_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cd_gram7 -s 100 -c 1 -o gpurun_out/prof_cd_cfg2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cd.log 2>&1
echo done
