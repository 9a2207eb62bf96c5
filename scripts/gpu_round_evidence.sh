#!/usr/bin/env bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, smoke, and for
# C3 (default), C5, C4 and C2: the bench line with cpu_baseline, the reference
# arm, the ncu launch list of one step and an ncu --set full capture of the
# dominant kernel(s).
mkdir -p gpurun_out/ev
O=gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for W in c3 c5 c4 c2; do
  timeout 1500 python bench.py --workload $W > $O/bench_$W.json 2> $O/bench_$W.err
  timeout 1200 python bench.py --workload $W --impl reference > $O/bench_${W}_ref.json 2> $O/bench_${W}_ref.err
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$W.csv \
    python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_bench_$W.log 2>&1
done
# full captures: eval (pass 1 of the timed step: launch index 2) and the warp executor
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_warp -s 2 -c 1 -f -o $O/prof_c3_eval \
  python bench.py --workload c3 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full_c3_eval.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_exec_warp -s 1 -c 1 -f -o $O/prof_c3_exec \
  python bench.py --workload c3 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full_c3_exec.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_eval_warp -s 2 -c 1 -f -o $O/prof_c5_eval \
  python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full_c5_eval.log 2>&1
timeout 1800 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats \
  --section WarpStateStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:k_eval_warp -c 2 -f -o $O/prof_c4_eval \
  python scripts/dbg_c4.py 4096 128 1 > $O/ncu_c4_eval.log 2>&1
# keep what travels back under 64 MiB: raw counters of every capture as CSV,
# one full report (C3 eval) for source-level reading
for R in prof_c3_eval prof_c3_exec prof_c5_eval prof_c4_eval; do
  [ -f $O/$R.ncu-rep ] && ncu -i $O/$R.ncu-rep --page raw --csv > $O/$R.raw.csv 2>/dev/null
done
rm -f $O/prof_c3_exec.ncu-rep $O/prof_c5_eval.ncu-rep $O/prof_c4_eval.ncu-rep
du -sh $O
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log
for W in c3 c5 c4 c2; do head -c 250 $O/bench_$W.json; echo; head -c 200 $O/bench_${W}_ref.json; echo; done
