#!/usr/bin/env bash
# The GPU checks of a development round, run on a B200 box through gpurun:
#   gpurun --timeout 3000 -- 'bash scripts/gpu.sh [tests|slow|bench|ncu|sanitize|all]'
# Outputs land in gpurun_out/ (scratch; summaries worth keeping are copied to profiles/).
set -u
mode=${1:-all}
mkdir -p gpurun_out
if [[ $mode == tests || $mode == all ]]; then
  python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "tests rc=$?"
fi
if [[ $mode == slow || $mode == all ]]; then
  python -m pytest tests -m "gpu and slow" -x -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_slow.log 2>&1
  echo "slow rc=$?"
fi
if [[ $mode == bench || $mode == all ]]; then
  for cfg in cfg3 cfg2 cfg4; do
    python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
    echo "bench $cfg rc=$?"
  done
fi
if [[ $mode == ncu ]]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
fi
