#!/bin/bash
# Round evidence on one B200: GPU tests, bench (+ reference arm), ncu launch list and a
# full ncu capture of the CG kernels.  Outputs under gpurun_out/.
set -u
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"
python bench.py --steps 1 --warmup 0 --no-cpu --no-alt > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-alt > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_target.py > gpurun_out/plain_target.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spmv_pull|cg_update|cg_pupdate|quad_assemble|quad_grad" -s 6 -c 8 \
    -o gpurun_out/prof_round python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
