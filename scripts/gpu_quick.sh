#!/usr/bin/env bash
# Quick GPU round-trip (run under gpurun): GPU tests with durations, smoke,
# the default bench line and a C4 single-pair timing.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=40 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
VEQ_PROF=1 timeout 600 python scripts/dbg_c4.py 4096 128 1 > gpurun_out/c4.log 2>&1
tail -45 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; head -c 700 gpurun_out/bench.json; echo; tail -3 gpurun_out/bench.err; tail -4 gpurun_out/c4.log
