mkdir -p gpurun_out
for c in 4 8 16; do
  timeout 900 python bench.py --ctas $c --steps $((64 / c)) --no-cpu-baseline > gpurun_out/ctas_$c.json 2> gpurun_out/ctas_$c.err
  python -c "
import json;l=json.load(open('gpurun_out/ctas_$c.json'));print($c, round(l['value']), round(l['ms_per_step'],1), {k:round(v,1) for k,v in l['phases_ms'].items()}, round(l['e2e']['value']))" || tail -3 gpurun_out/ctas_$c.err
done
