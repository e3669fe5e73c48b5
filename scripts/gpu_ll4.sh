cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ll4.log 2>&1
echo done
