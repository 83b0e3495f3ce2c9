python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2a_c2.json 2> gpurun_out/r2a_c2.err
tail -3 gpurun_out/r2a_pytest_gpu.log; tail -1 gpurun_out/r2a_smoke.log; cat gpurun_out/r2a_c2.json | head -c 600
