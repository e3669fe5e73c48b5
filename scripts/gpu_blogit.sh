cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config logit --steps 3 --warmup 3 --ref-seconds 8 > gpurun_out/bench_logit.log 2>&1
echo done
