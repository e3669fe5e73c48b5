cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in 4; do for c in cfg2 cfg3 cfg4; do BL_SCAN_C=$C timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_${c}_C$C.log 2>&1; done; done
echo done
