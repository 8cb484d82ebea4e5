#!/bin/bash
# Round-2 measurements: FP64 peak, bench lines (C3, C4, C5), contact-kernel captures.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
./scripts/micro/dfma_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload batch --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ncp|k_setup|k_corrected" -s 60 -c 3 -o gpurun_out/c4_ncp python scripts/time_contact_steps.py C4 9 > gpurun_out/ncu_ncp.log 2>&1
ls -la gpurun_out
