#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_aa_solve -s 80 -c 2 -o gpurun_out/aasolve_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_aasolve.log 2>&1
ls -la gpurun_out | head
