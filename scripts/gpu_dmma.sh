cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/dmma_peak > gpurun_out/dmma_peak.log 2>&1
./scripts/fp64_peak >> gpurun_out/dmma_peak.log 2>&1
echo done
