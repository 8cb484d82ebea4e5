#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + one full capture of the solve.
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rowdot\|k_zreduce\|k_coltile\|k_xreduce -s 60 -c 4 -o gpurun_out/solve_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_local\|k_bapply -s 10 -c 2 -o gpurun_out/local_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_local.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_aa_solve\|k_gather_perm\|k_aa_dots -s 60 -c 3 -o gpurun_out/small_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1
ls -la gpurun_out
