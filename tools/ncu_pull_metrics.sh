#!/bin/bash
# ncu LSU metrics of the pull SpMV (warm cache) -> gpurun_out/prof_$1
export SSO_STORAGE=3
python tools/ncu_target.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:spmv_pull -s 20 -c 1 \
    -o gpurun_out/prof_$1 python tools/ncu_target.py > gpurun_out/ncu_$1.log 2>&1; echo rc=$?
