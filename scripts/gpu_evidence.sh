#!/usr/bin/env bash
# One GPU round-trip of bench evidence for a workload (run under gpurun):
# bench line (with cpu_baseline), the reference arm, the ncu launch list of
# one timed step and one ncu --set full capture per listed kernel.
# Usage: bash scripts/gpu_evidence.sh c3 "k_eval_warp k_exec_warp"
W=${1:-c3}
KS=${2:-k_eval_warp}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1200 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
timeout 900 python bench.py --workload $W --impl reference > gpurun_out/bench_${W}_ref.json 2> gpurun_out/bench_${W}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_bench_$W.log 2>&1
for K in $KS; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-1} -c 1 -f -o gpurun_out/prof_${W}_$K \
    python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_${W}_$K.log 2>&1
done
head -c 400 gpurun_out/bench_$W.json; echo; head -c 300 gpurun_out/bench_${W}_ref.json; tail -2 gpurun_out/bench_$W.err
