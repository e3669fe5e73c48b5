cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size" --timeout 1400 -rf > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
for c in cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log; done
echo done
