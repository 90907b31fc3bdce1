# A/B of environment-variable variants of the single-GPU bench on one box.
# usage: bash tools/ab_env.sh VAR v1 v2 ...   (two interleaved repetitions; AB_ARGS: extra bench flags)
var=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env "$var=$v" python bench.py --steps ${AB_STEPS:-30} --warmup 5 --no-cpu-baseline --no-c2 ${AB_ARGS:-} 2>/dev/null |
      AB_TAG="$var=$v" python -c '
import json, os, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
s = d["stage_ms"]
print(os.environ["AB_TAG"], round(d["ms_per_step"], 3), "wgrad", s.get("wgrad1"), s.get("wgrad2"), "fwd", s.get("gemm1_fwd"), s.get("gemm2_fwd"), "dgrad", s.get("dgrad2"), s.get("dgrad1"), "clk", d["clocks"]["sm_mhz"])'
  done
done
