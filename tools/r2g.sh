timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2g.log 2>&1; tail -3 gpurun_out/r2g.log
timeout 900 python bench.py --lattice 0 --no-cpu > gpurun_out/r2g_c2.json 2> gpurun_out/r2g_c2.err; python -c "import json; d=json.load(open('gpurun_out/r2g_c2.json')); print(d['value'], json.dumps(d['streaming']['gpu']))" || tail -3 gpurun_out/r2g_c2.err
