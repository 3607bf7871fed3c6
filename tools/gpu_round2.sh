#!/bin/bash
# Round-2 evidence on one B200 (outputs under gpurun_out/r2/).
set -u
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/smi.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dfma_peak.cu -o /tmp/dfma && /tmp/dfma > $O/fp64_peak.json
timeout 900 python -m pytest tests -m gpu -q -s -rf > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_c3b.json 2> $O/bench_c3b.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --workload C1 --steps 1000 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 rc=$?"
timeout 300 python bench.py --workload C2 --steps 300 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu --virtual-parts 8 > $O/bench_c4_vp8.json 2> $O/bench_c4_vp8.err; echo "c4 vp8 rc=$?"
timeout 300 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_target.py > $O/san_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 300 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_target.py > $O/san_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 300 compute-sanitizer --tool synccheck python tools/sanitize_target.py > $O/san_synccheck.log 2>&1; echo "synccheck rc=$?"
timeout 300 compute-sanitizer --tool initcheck python tools/sanitize_target.py > $O/san_initcheck.log 2>&1; echo "initcheck rc=$?"
python bench.py --steps 1 --warmup 0 --no-cpu --no-alt > $O/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-alt > $O/ncu_launch.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_target.py > $O/plain_target.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv_pull|cg_update_fused|quad_assemble|quad_grad" -s 6 -c 6 \
    -o $O/prof_round2 python tools/ncu_target.py > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
