#!/bin/bash
# Quick GPU check: parity tests, smoke, bench line (BENCH_ARGS), optional extra command (EXTRA).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "${BENCH_ARGS}" ]; then timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; fi
if [ -n "${EXTRA}" ]; then bash -c "${EXTRA}" > gpurun_out/extra.log 2>&1; echo "extra rc=$?" >> gpurun_out/extra.log; fi
tail -n 5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -n 2 gpurun_out/bench.log 2>/dev/null | cut -c1-600
