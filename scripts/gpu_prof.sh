mkdir -p gpurun_out
VEQ_PROF=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
grep "veq prof" gpurun_out/bench_prof.err | tail -6
