mkdir -p gpurun_out/n1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc_gemm|pnorm_back|softmax|renorm|seg_reduce|finalize" --launch-skip 600 --launch-count 24 -o /tmp/p1 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-precond-bench > gpurun_out/n1/ncu.log 2>&1; echo ncu rc=$?
ncu -i /tmp/p1.ncu-rep --page raw --csv > gpurun_out/n1/raw.csv 2>gpurun_out/n1/raw.err
ncu -i /tmp/p1.ncu-rep --page details --csv > gpurun_out/n1/details.csv 2>>gpurun_out/n1/raw.err
cp /tmp/p1.ncu-rep gpurun_out/n1/ 2>/dev/null
ls -la gpurun_out/n1
