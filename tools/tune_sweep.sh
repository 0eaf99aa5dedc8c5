#!/bin/bash
# Sweep the GEMM tuning knobs on the plain (non-refresh) step and the full step.
# Usage (on a GPU box): bash tools/tune_sweep.sh > gpurun_out/sweep.txt
cd "$(dirname "$0")/.."
run() {
  local tag="$1"; shift
  local plain full
  plain=$(env "$@" python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-precond-bench \
          --update-period 100000 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')
  full=$(env "$@" python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-precond-bench \
          2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')
  echo "$tag plain_ms=$plain full_ms=$full"
}
if [ $# -gt 0 ]; then
  for v in "$@"; do run "$v" $v; done
  exit 0
fi
run default X=1
run fwd64 NG_TUNE_FWD_BN=64
run upd128 NG_TUNE_UPD_BN=128
run upd32 NG_TUNE_UPD_BN=32
run apply64 NG_TUNE_APPLY_BN=64
run stages3 NG_TUNE_TC_STAGES=3
run stages6 NG_TUNE_TC_STAGES=6
run bwdsp3 NG_TUNE_BWD_SPLITS=3
run bwd128 NG_TUNE_BWD_BN=128
