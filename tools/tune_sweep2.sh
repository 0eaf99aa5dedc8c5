#!/bin/bash
# One-at-a-time sweep of the GEMM tile knobs on the config-3 bench (frames/s, ms/step).
run() { echo -n "$* : "; env "$@" python bench.py --steps 150 --no-cpu-baseline --no-e2e --no-precond-bench 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'], 4))"; }
run NG_TUNE_X=0
run NG_TUNE_UPD_BN=128
run NG_TUNE_UPD_BN=32
run NG_TUNE_APPLY_BN=64
run NG_TUNE_BWD_BN=128
run NG_TUNE_BWD_SPLITS=3
run NG_TUNE_BWD_SPLITS=4
run NG_TUNE_FWD_BN=64
run NG_TUNE_X=0
