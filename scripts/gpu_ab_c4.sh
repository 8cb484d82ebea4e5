#!/bin/bash
# A/B of environment toggles on the C4 bench line (no CPU baseline).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ' =' '__')
  env $cfg timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/abc4_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
n=sys.argv[1]
l=[x for x in open(f"gpurun_out/abc4_{n}.log") if x.startswith("{")]
if not l: print(n, "FAILED", open(f"gpurun_out/abc4_{n}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); c=d["config"]
print(n, "value %.3f" % d["value"], "ms %.1f" % d["ms_per_step"], "adj_it", c["mean_adjoint_iterations"], "e2e %.3f" % d["e2e"]["value"], "fwd_ms %.1f bwd_ms %.1f" % (c.get("forward_ms", 0), c.get("backward_ms", 0)))
PY
done
