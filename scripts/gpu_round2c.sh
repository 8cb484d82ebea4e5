#!/bin/bash
# Round-2 final measurement session (after block CG for the contact columns and
# the recycled-subspace deflation of the backbone CG): bench lines (C3 with the
# CPU baseline, reference arm, C4, C5 lockstep), launch lists of the C3 and C4
# steps, full captures of the C3 backbone iteration's kernels and of the C4
# block-CG iteration, compute-sanitizer over the new kernels.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowdot|k_zreduce|k_coltile|k_cpcg_apply|k_bapply|k_dpcg_rz|k_dpcg_p|k_pcg_xr" -s 300 -c 8 -o gpurun_out/r02c_backbone python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_backbone.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowdot_mma|k_coltile_mma|k_bcg|k_bapply_cols|k_cpcg_apply" -s 400 -c 8 -o gpurun_out/r02c_c4_block python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --launch-timeout 0 python scripts/sanitize_round2.py > gpurun_out/sanitizer_memcheck.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --launch-timeout 0 python scripts/sanitize_round2.py > gpurun_out/sanitizer_racecheck.txt 2>&1
ls -la gpurun_out
