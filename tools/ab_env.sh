# A/B of environment-variable variants of the single-GPU bench on one box.
# usage: bash tools/ab_env.sh VAR v1 v2 ...   (two interleaved repetitions)
var=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env "$var=$v" python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null |
      AB_TAG="$var=$v" python -c '
import json, os, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(os.environ["AB_TAG"], round(d["ms_per_step"], 4), d["stage_ms"], d["clocks"]["sm_mhz"])'
  done
done
