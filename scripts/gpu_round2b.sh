#!/bin/bash
# Round-2 measurement session: full GPU tests, smoke, bench lines (C3 + CPU
# baseline, reference arm, C4, C5 lockstep), ncu launch list of the C3 step,
# full captures of the C3 backbone / local kernels, the C5 lockstep solve and
# the device refactorization fronts.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload batch --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowdot|k_zreduce|k_coltile|k_bb_dots|k_bb_mix|k_bapply|k_gather_sorted" -s 200 -c 7 -o gpurun_out/r02_backbone python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_backbone.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_local|k_differential|k_energy" -s 3 -c 3 -o gpurun_out/r02_local python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_local.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none -k regex:"k_rowdot|k_coltile|k_seg_bb|k_bapply|k_local" -s 40 -c 6 -o gpurun_out/r02_c5 python scripts/prof_batch.py 64 1 1 > gpurun_out/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_mf_level|k_inverse" -s 60 -c 4 -o gpurun_out/r02_refactor python scripts/time_refactor.py > gpurun_out/ncu_refactor.log 2>&1
ls -la gpurun_out
