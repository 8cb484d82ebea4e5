#!/bin/bash
# A/B of environment toggles on the C5 batch bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ' =' '__')
  env $cfg timeout 600 python bench.py --workload batch --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/abb_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
n=sys.argv[1]
l=[x for x in open(f"gpurun_out/abb_{n}.log") if x.startswith("{")]
if not l: print(n, "FAILED", open(f"gpurun_out/abb_{n}.log").read()[-800:]); sys.exit()
d=json.loads(l[-1])
print(n, "value %.1f" % d["value"], "ms %.1f" % d["ms_per_step"], "agg_frac %.3f" % d["roofline"]["frac"], "solves/step", d["roofline"]["solves_per_step"])
PY
done
