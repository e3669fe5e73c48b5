cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in cfg2 cfg3 cfg4 cfg1; do
  for cd in auto residual; do
    timeout 600 python bench.py --config $cfg --cd $cd --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/perf_${cfg}_${cd}.log 2>&1; echo "rc=$?" >> gpurun_out/perf_${cfg}_${cd}.log
  done
done
echo done
