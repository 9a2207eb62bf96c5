mkdir -p gpurun_out
VEQ_PROF=1 VEQ_STEP_PROF=1 timeout 600 python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c2sp.json 2> gpurun_out/c2sp.err
grep "^\[step\]\|veq load" gpurun_out/c2sp.err | tail -6
python -c "
import json;l=json.load(open('gpurun_out/c2sp.json'));print(round(l['value']), round(l['ms_per_step'],1), {k:round(v,2) for k,v in l['phases_ms'].items()})"
