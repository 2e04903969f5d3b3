# A/B of an env knob on one box: GPU tests of the tensor route under the build
# default, then the C2 bench step (no CPU baseline / C3 / C5) for each value,
# interleaved twice.  usage: bash tools/ab_env.sh VAR val1 val2 [tests...]
VAR=$1; A=$2; B=$3; shift 3
mkdir -p gpurun_out/ab
if [ $# -gt 0 ]; then
  timeout 900 python -m pytest "$@" -x -q -p no:cacheprovider > gpurun_out/ab/tests.log 2>&1; echo tests $?; tail -1 gpurun_out/ab/tests.log
fi
for v in $A $B $A $B; do
  env $VAR=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c5 --no-c3 --no-other-backends --e2e-steps 1 > gpurun_out/ab/bench_$v.log 2> gpurun_out/ab/bench_$v.err
  python - "$VAR" "$v" <<'PY'
import json,sys
try:
    d=json.loads(open(f"gpurun_out/ab/bench_{sys.argv[2]}.log").read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e); sys.exit(0)
kb=d["config"]["kernel_breakdown_rank0"]
print(sys.argv[1], sys.argv[2], "pairs/s", round(d["value"]), "ms", round(d["ms_per_step"],3), "score", kb["score"]["ms"], "pack", kb["pack"]["ms"], kb["pack"].get("hbm_gbs"), "merge", kb["merge"]["ms"], "frac", round(d["roofline"]["frac"],3), "clk", d["clocks"]["sm_mhz"])
PY
done
