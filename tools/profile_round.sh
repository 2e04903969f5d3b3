# Round-2 evidence (run under gpurun from the repo root): GPU tests of the
# tensor route, the default bench line, the ncu launch list of the same
# command, and one `ncu --set full` capture per kernel class summarised by
# tools/ncu_summary.py.  Outputs land in gpurun_out/r2p/.
set -x
O=gpurun_out/${PROF_OUT:-r2p}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_route.py tests/test_gpu_exact.py tests/test_gpu_c5.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; rc=$?; echo tests $rc; tail -1 $O/tests.log
[ $rc -eq 0 ] || exit 1
timeout 600 python bench.py > $O/bench.log 2> $O/bench.err; echo bench $?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py > $O/bench_under_ncu.log 2>&1; echo launches $?
SMALL="python bench.py --steps 1 --warmup 3 --pairs 32 --no-cpu-baseline --no-c5 --no-c3 --no-other-backends --e2e-steps 1 --parity-pairs 0"
for k in ${PROF_KERNELS:-tc_scan merge_kernel gather_kernel pack_kernel harvest_kernel rescan_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/$k $SMALL > $O/ncu_$k.log 2>&1; echo $k $?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flashmatch4 -s 30 -c 1 -o $O/flashmatch4 python tools/fm_time.py > $O/ncu_fm.log 2>&1; echo fm $?
ls -la $O
