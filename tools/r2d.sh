timeout 600 python -m pytest tests/test_lattice.py tests/test_phrases.py -x -q > gpurun_out/r2d_lat.log 2>&1; tail -15 gpurun_out/r2d_lat.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or c5" --durations=5 > gpurun_out/r2d_c3c5.log 2>&1; tail -15 gpurun_out/r2d_c3c5.log
timeout 600 python bench.py --search fast --streams 0 --no-cpu > gpurun_out/r2d_c2_fast.json 2> gpurun_out/r2d_c2_fast.err
python -c "import json; d=json.load(open('gpurun_out/r2d_c2_fast.json')); print(d['value'], json.dumps(d['lattice']))" || tail -5 gpurun_out/r2d_c2_fast.err
