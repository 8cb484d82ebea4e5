#!/bin/bash
# A/B of environment toggles on the C3 bench line (no CPU baseline).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ' =' '__')
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
n=sys.argv[1]
l=[x for x in open(f"gpurun_out/ab_{n}.log") if x.startswith("{")]
if not l: print(n, "FAILED", open(f"gpurun_out/ab_{n}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); c=d["config"]
print(n, "value %.2f" % d["value"], "ms %.3f" % d["ms_per_step"], "solve_us %.1f" % (1e3*d["roofline"]["ms_per_launch"]), "frac %.3f" % d["roofline"]["frac"], "adj_it", c["mean_adjoint_iterations"], "e2e %.2f" % d["e2e"]["value"], "launches", d["gpu_launches"], "fwd_ms %.3f bwd_ms %.3f" % (c.get("forward_ms", 0), c.get("backward_ms", 0)))
PY
done
