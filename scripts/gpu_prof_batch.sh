cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/cv_small.py 200000 > gpurun_out/cv_small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_batch -s 20 -c 1 -o gpurun_out/prof_batch python scripts/cv_small.py 200000 > gpurun_out/ncu_batch.log 2>&1
echo done
