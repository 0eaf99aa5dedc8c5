#!/bin/bash
# Round-end measurement pass on one B200 (run from the repo root under gpurun), outputs in
# gpurun_out/final/:
#   bash tools/final_profile.sh bench   bench lines for every workload / mode, timelines, the
#                                       ncu launch list of bench.py
#   bash tools/final_profile.sh ncu     ncu --set full of ~4 steady-state steps; the report
#                                       stays in /tmp (hundreds of MB), its raw page is exported
O=gpurun_out/final
mkdir -p $O
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.out 2> $O/$name.err; echo "$name rc=$?"; tail -1 $O/$name.out > $O/$name.json; }
if [ "$1" = bench ]; then
  run bench python bench.py
  run bench_config5 python bench.py --workload config5
  run bench_fp32 python bench.py --precision fp32
  run bench_simple python bench.py --precond simple
  run bench_none python bench.py --precond none
  run bench_reference python bench.py --impl reference
  timeout 300 python tools/refresh_timeline.py 60 > $O/refresh_timeline.txt 2>&1
  timeout 300 python tools/step_timeline.py 40 > $O/step_timeline.txt 2>&1
  timeout 300 python tools/eig_bench.py > $O/eig_bench.txt 2>&1
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 24 --warmup 10 > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
fi
if [ "$1" = ncu ]; then
  timeout 2000 ncu --set full --clock-control none --launch-skip 1600 --launch-count 180 -o /tmp/full \
    python bench.py --steps 24 --warmup 10 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
  ncu -i /tmp/full.ncu-rep --page raw --csv > $O/full_raw.csv 2> $O/full_raw.err; echo "export rc=$?"
  rm -f /tmp/full.ncu-rep
fi
ls -la $O
du -sh gpurun_out
