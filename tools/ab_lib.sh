# Same-box A/B of library builds on the single-GPU C3 bench.
# usage: bash tools/ab_lib.sh lib1.so lib2.so ...   ("default" = the in-tree build)
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset TED_LIB; else export TED_LIB=$lib; fi
    python bench.py --steps ${AB_STEPS:-30} --warmup 5 --no-cpu-baseline --no-c2 ${AB_ARGS:-} 2>/dev/null |
      AB_TAG="$lib" python -c '
import json, os, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
s = d["stage_ms"]
print(os.environ["AB_TAG"], round(d["ms_per_step"], 3), "wgrad1", s.get("wgrad1"), "wgrad2", s.get("wgrad2"),
      "frac", round(d["roofline"]["frac"], 3), "clk", d["clocks"]["sm_mhz"])'
  done
done
unset TED_LIB
