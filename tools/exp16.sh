for f in "-DCTW_LOAD_DIV=8" "-DCTW_LOAD_DIV=2" ""; do
  CTW_NVCC_FLAGS="$f" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
  timeout 300 python bench.py --batch 512 --no-cpu --streams 0 --lattice 0 --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],1), round(d['value']), d['workload_stats']['max_slots'])"
done
