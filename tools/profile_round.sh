set -x
mkdir -p gpurun_out/r15
timeout 600 python bench.py > gpurun_out/r15/bench.log 2> gpurun_out/r15/bench.err; echo bench $?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r15/launches.csv python bench.py > gpurun_out/r15/bench_under_ncu.log 2>&1; echo launches $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 3 -c 1 -o gpurun_out/r15/merge python bench.py --steps 1 --warmup 3 --pairs 32 --no-cpu-baseline --no-c5 --no-c3 --e2e-steps 1 > gpurun_out/r15/ncu_merge.log 2>&1; echo merge $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_scan -s 3 -c 1 -o gpurun_out/r15/tc_scan python bench.py --steps 1 --warmup 3 --pairs 32 --no-cpu-baseline --no-c5 --no-c3 --e2e-steps 1 > gpurun_out/r15/ncu_tc.log 2>&1; echo tc $?
ls -la gpurun_out/r15
