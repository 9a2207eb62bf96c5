mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_c5_variants.py tests/test_gpu_pipeline.py -q -m gpu -x --durations=8 > gpurun_out/pytest_c5.log 2>&1
timeout 1500 python bench.py --workload c5 --steps 2 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -14 gpurun_out/pytest_c5.log; head -c 1500 gpurun_out/bench_c5.json; echo; tail -5 gpurun_out/bench_c5.err
