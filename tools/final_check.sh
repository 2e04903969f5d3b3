mkdir -p gpurun_out/fin
# synccheck cannot run kernels inside a conditional (WHILE) graph body: it
# reports barrier errors and kills even a trivially correct kernel there
# (tools/ubench_cond_sync.cu; memcheck and plain runs are clean), and
# racecheck crashes the host process at the loop graph's first launch, so
# both check the same kernels with the loop graph off; memcheck runs with it on
for t in memcheck racecheck synccheck; do
  g=1; [ $t != memcheck ] && g=0
  FNL_LOOP_GRAPH=$g timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/fin/sanitize_$t.log 2>&1; echo $t $?; tail -1 gpurun_out/fin/sanitize_$t.log
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fin/gpu_tests.log 2>&1; echo tests $?; tail -1 gpurun_out/fin/gpu_tests.log
timeout 600 python bench.py > gpurun_out/fin/bench.log 2> gpurun_out/fin/bench.err; echo bench $?
