#!/bin/bash
run() { echo -n "$* : "; env "$@" python bench.py --steps 200 --no-cpu-baseline --no-e2e --no-precond-bench 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'], 4))"; }
for rep in 1 2; do
run NG_TUNE_X=0
run NG_TUNE_FWD_PNORM_BN=160
done
