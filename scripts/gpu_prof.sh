cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg4.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_fp -s 40 -c 2 -o gpurun_out/prof_scan_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
