mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_exec_warp -s 1 -c 1 -f -o gpurun_out/prof_exec \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_exec.log 2>&1
ncu -i gpurun_out/prof_exec.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/exec_src.csv 2>/dev/null
rm -f gpurun_out/prof_exec.ncu-rep
gzip -f gpurun_out/exec_src.csv; ls -la gpurun_out/exec_src.csv.gz
