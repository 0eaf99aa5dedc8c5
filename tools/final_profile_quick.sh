#!/bin/bash
# Round-end re-measurement of the final code (subset of final_profile.sh bench): the default
# bench line, config 5, the FP32-grade mode, timelines and the ncu launch list, in
# gpurun_out/final2/.
O=gpurun_out/final2
mkdir -p $O
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.out 2> $O/$name.err; echo "$name rc=$?"; tail -1 $O/$name.out > $O/$name.json; }
run bench python bench.py
run bench_config5 python bench.py --workload config5
run bench_fp32 python bench.py --precision fp32
timeout 300 python tools/refresh_timeline.py 60 > $O/refresh_timeline.txt 2>&1
timeout 300 python tools/step_timeline.py 40 > $O/step_timeline.txt 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 24 --warmup 10 > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
ls -la $O
