#!/usr/bin/env bash
# Bench lines of every BASELINE config (and the NEXT rows) for DESIGN's tables:
#   gpurun --timeout 3000 -- 'bash scripts/bench_all.sh r02'
tag=${1:-r02}
mkdir -p gpurun_out
for spec in "cfg3" "cfg2" "cfg4" "logit" "cfg1"; do
  python bench.py --config $spec --steps 5 --warmup 3 > gpurun_out/${tag}_bench_$spec.json 2> gpurun_out/${tag}_bench_$spec.err
  echo "$spec rc=$?"
done
python bench.py --config cfg3 --resident host --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg3_host.json 2> gpurun_out/${tag}_bench_cfg3_host.err
echo "cfg3 host rc=$?"
python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg5.json 2> gpurun_out/${tag}_bench_cfg5.err
echo "cfg5 rc=$?"
