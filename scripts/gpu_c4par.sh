mkdir -p gpurun_out
timeout 900 python scripts/dbg_c4.py 4096 128 1 > gpurun_out/c4.log 2>&1; tail -2 gpurun_out/c4.log
timeout 900 python scripts/dbg_c4.py 4096 128 4 > gpurun_out/c4b.log 2>&1; tail -2 gpurun_out/c4b.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
