# A/B of libraries (TED_LIB) on the C2 single-GPU workload, gate stages only
for rep in 1 2; do
  for v in "$@"; do
    TED_LIB=$v python bench.py --workload c2 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null |
      AB_TAG="$v" python -c '
import json, os, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); s = d["stage_ms"]
print(os.environ["AB_TAG"], round(d["ms_per_step"], 4), {k: s[k] for k in ("gate", "gate_dw", "gate_dx", "colsum", "combine_fwd", "combine_bwd", "route_dispatch")})'
  done
done
