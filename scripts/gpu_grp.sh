mkdir -p gpurun_out
for cfg in "1 0" "2 0" "2 1024" "2 4096" "2 16384"; do
  set -- $cfg
  VEQ_EVAL_GROUPS=$1 VEQ_GROUP_DELAY=$2 timeout 900 python bench.py --steps 16 --no-cpu-baseline > gpurun_out/grp.json 2> gpurun_out/grp.err
  python -c "
import json;l=json.load(open('gpurun_out/grp.json'));print('$1 $2', round(l['value']), round(l['ms_per_step'],1), round(l['phases_ms']['eval'],1))" || tail -3 gpurun_out/grp.err
done
