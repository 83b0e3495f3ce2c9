# C4 streaming p50/p99 with and without the per-step CUDA graph (two runs each)
for mode in graph plain graph plain; do
  if [ $mode = plain ]; then export CTW_NO_GRAPH=1; else unset CTW_NO_GRAPH; fi
  python bench.py --steps 1 --warmup 3 --no-cpu --lattice 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['streaming']['gpu']; print('$mode', round(g['p50_total_ms'],3), round(g['p99_total_ms'],3), g['breakdown_s']['advance_s'], g['breakdown_s'].get('step_graphs'))"
done
