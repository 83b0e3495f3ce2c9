timeout 900 python -m pytest tests/test_fast_mode.py -q > gpurun_out/r2c_fast.log 2>&1
tail -40 gpurun_out/r2c_fast.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2c_gpu_all.log 2>&1; tail -15 gpurun_out/r2c_gpu_all.log
