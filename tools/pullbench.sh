#!/bin/bash
# quick storage comparison on C3b (development helper)
python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric or pull" > gpurun_out/t_pull.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_pull.log
for v in "$@"; do
  SSO_PULL_VARIANT=$v python bench.py --steps 3 --warmup 3 --no-cpu --storage 3 > gpurun_out/bench_st3v$v.log 2>&1
  echo "variant $v: $(tail -1 gpurun_out/bench_st3v$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"]["cg_iters"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"])')"
done
