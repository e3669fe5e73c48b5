cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg5.log
echo done
