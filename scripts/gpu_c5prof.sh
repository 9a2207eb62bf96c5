mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_c5_variants.py tests/test_gpu_pipeline.py tests/test_integration.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_c5.log 2>&1
VEQ_PROF=1 VEQ_STEP_PROF=1 timeout 1500 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5p.json 2> gpurun_out/bench_c5p.err
tail -3 gpurun_out/pytest_c5.log; grep -v "^\[veq prof\]" gpurun_out/bench_c5p.err | tail -14; head -c 300 gpurun_out/bench_c5p.json
