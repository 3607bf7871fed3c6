#!/bin/bash
# C5 designs/s (bench.py, no CPU leg): prints the value only
python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu --no-alt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'])"
