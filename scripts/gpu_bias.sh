mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for b in 0 64 256 1024; do
VEQ_LATE_BIAS=$b timeout 900 python bench.py --steps 16 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json;l=json.load(open('gpurun_out/b.json'));print('bias $b', round(l['value']), round(l['ms_per_step'],1), round(l['phases_ms']['eval'],1))" || tail -3 gpurun_out/b.err
done
timeout 900 python scripts/dbg_c4.py 4096 128 1 > gpurun_out/c4.log 2>&1; tail -2 gpurun_out/c4.log
