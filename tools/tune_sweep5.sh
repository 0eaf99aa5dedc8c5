#!/bin/bash
run() { echo -n "$* : "; env "$@" python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-precond-bench 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'], 4))"; }
run NG_TUNE_X=0
run NG_TUNE_SIDE_PRIORITY=0
run CUDA_DEVICE_MAX_CONNECTIONS=16
run NG_TUNE_TC_STAGES=3
run NG_TUNE_X=0
