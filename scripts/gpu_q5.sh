mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;l=json.load(open('gpurun_out/bench.json'));print(round(l['value']), round(l['ms_per_step'],1), {k:round(v,1) for k,v in l['phases_ms'].items()}, round(l['e2e']['value']))" || tail -3 gpurun_out/bench.err
VEQ_PROF=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
grep "veq prof\] items" gpurun_out/bench_prof.err | tail -1 | cut -c1-400
timeout 600 python scripts/dbg_c4.py 4096 128 1 > gpurun_out/c4.log 2>&1; tail -2 gpurun_out/c4.log
