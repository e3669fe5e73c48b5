cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -rf -k "cv or cfg5 or path_parity or sharded" > gpurun_out/pytest_cv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cv.log
timeout 900 python scripts/cfg5_single.py > gpurun_out/cfg5_single.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
echo done
