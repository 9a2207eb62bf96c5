mkdir -p gpurun_out
VEQ_STEP_PROF=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sp.json 2> gpurun_out/bench_sp.err
grep "^\[step\]" gpurun_out/bench_sp.err | tail -4
