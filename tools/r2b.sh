# fast-mode bring-up: fast tests, full gpu suite, C2 bench in both modes (no side legs)
timeout 900 python -m pytest tests/test_fast_mode.py -x -q > gpurun_out/r2b_fast.log 2>&1
tail -30 gpurun_out/r2b_fast.log
timeout 600 python bench.py --search fast --streams 0 --lattice 0 > gpurun_out/r2b_c2_fast.json 2> gpurun_out/r2b_c2_fast.err
timeout 600 python bench.py --search exact --streams 0 --lattice 0 --no-cpu > gpurun_out/r2b_c2_exact.json 2> gpurun_out/r2b_c2_exact.err
python - <<'PY'
import json
for m in ("fast","exact"):
    try:
        d=json.load(open(f"gpurun_out/r2b_c2_{m}.json"))
        print(m, d["value"], d["e2e"]["value"], d.get("parity"), json.dumps(d["stage_profile"])[:600])
    except Exception as e: print(m, "ERR", e, open(f"gpurun_out/r2b_c2_{m}.err").read()[-2000:])
PY
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gpu_all.log 2>&1; tail -5 gpurun_out/r2b_gpu_all.log
