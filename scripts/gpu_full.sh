#!/usr/bin/env bash
# Full GPU round-trip (run under gpurun): every GPU test, smoke, the default
# bench line (C3) and the C5 line with its reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1200 python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload c5 --impl reference > gpurun_out/bench_c5_ref.json 2> gpurun_out/bench_c5_ref.err
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for f in bench_c3 bench_c5 bench_c5_ref; do head -c 400 gpurun_out/$f.json; echo; tail -2 gpurun_out/$f.err; done
