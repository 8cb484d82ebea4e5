#!/bin/bash
# Round-2 closing measurement session, third pass (after the static-layout prefetches in the z folds
# and the 32-block per-sample CG kernels):
# GPU tests + smoke, bench lines (C3 with the CPU baseline, reference arm, C4,
# C5 lockstep), refactorization phases, launch lists of the C3 and C5 steps,
# full captures of the C3 backbone kernels and of k_local at C3 and C5 sizes,
# compute-sanitizer memcheck over the round-2 paths.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
HETERODYN_REFACTOR_TRACE=1 timeout 600 python scripts/time_refactor.py > gpurun_out/refactor.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_batch.py 64 1 2 > gpurun_out/ncu_launch_c5.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowdot|k_zreduce|k_coltile|k_cpcg_apply|k_bapply|k_dpcg_rz|k_dpcg_p|k_pcg_xr|k_local" -s 300 -c 10 -o gpurun_out/r02f_backbone python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_backbone.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_local|k_inverse_values" -c 2 -o gpurun_out/r02f_local_c5 python scripts/prof_batch.py 64 1 1 > gpurun_out/ncu_local_c5.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
ls -la gpurun_out
