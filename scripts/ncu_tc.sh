#!/usr/bin/env bash
# ncu capture of the tcgen05 batched scan in the stand-alone checker (gpurun; output in gpurun_out/)
tag=${1:-tc}
./scripts/tc_check.bin 10000 200000 11 2 > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scan_batch_tc -s 1 -c 1 -o gpurun_out/${tag}_prof \
    ./scripts/tc_check.bin 10000 200000 11 2 > gpurun_out/${tag}_ncu.log 2>&1
echo rc=$?
