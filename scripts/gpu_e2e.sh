cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e.log 2>&1
echo done
