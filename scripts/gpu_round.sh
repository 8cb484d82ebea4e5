#!/bin/bash
# One GPU session: parity tests, smoke, bench lines (C3, reference, C4, C5),
# ncu launch list + full captures, in-graph timeline and phase times.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --workload batch --steps 2 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/bench_c5.log
timeout 300 python scripts/prof_trace.py C3 > gpurun_out/trace_c3.txt 2>&1
HETERODYN_PHASES=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/phases.txt 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowdot|k_zreduce|k_coltile|k_bb_dots|k_bb_mix|k_bapply|k_gather_pp" -s 200 -c 7 -o gpurun_out/backbone_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_local|k_differential|k_energy" -s 3 -c 3 -o gpurun_out/local_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_local.log 2>&1
HETERODYN_NO_COND_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:c2<\(int\)4" -s 4 -c 2 -o gpurun_out/c4_columns python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out
