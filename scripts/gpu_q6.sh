mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for W in c2 c3; do
timeout 900 python bench.py --workload $W --no-cpu-baseline > gpurun_out/b_$W.json 2> gpurun_out/b_$W.err
python -c "
import json;l=json.load(open('gpurun_out/b_$W.json'));print('$W', round(l['value']), round(l['ms_per_step'],1), round(l['e2e']['value']))" || tail -3 gpurun_out/b_$W.err
done
