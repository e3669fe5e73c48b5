python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4_pytest.log
bash scripts/bench_all.sh s4
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 4000 --csv --log-file gpurun_out/s4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4_ncu_launch.log 2>&1; echo "ncu rc=$?"
