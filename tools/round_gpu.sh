python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 1000 python bench.py > gpurun_out/head5.json 2> gpurun_out/head5.err
bash tools/prof_r1d.sh
