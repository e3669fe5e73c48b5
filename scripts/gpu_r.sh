cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 4 8 16; do
  BL_CD_CLUSTER=$r timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_r$r.log 2>&1
done
echo done
