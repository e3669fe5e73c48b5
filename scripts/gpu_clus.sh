cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for R in 8 16; do for c in cfg2 cfg3; do BL_CD_CLUSTER=$R timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_${c}_R$R.log 2>&1; done; done
echo done
