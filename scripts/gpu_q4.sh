mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;l=json.load(open('gpurun_out/bench.json'));print(round(l['value']), round(l['ms_per_step'],1), {k:round(v,1) for k,v in l['phases_ms'].items()}, round(l['e2e']['value']))" || tail -3 gpurun_out/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_warp -s 2 -c 1 -f -o gpurun_out/prof_c3_eval python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_eval.log 2>&1
tail -2 gpurun_out/ncu_eval.log
