for f in "-DCTW_MINB=3" "-DCTW_MINB=4" "-DCTW_MINB=1"; do
  CTW_NVCC_FLAGS="$f" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
  for c in 4 8; do
  CTW_CLUSTER=$c timeout 300 python bench.py --batch 512 --no-cpu --streams 0 --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['stage_profile']; print('$f', 'C', $c, round(d['ms_per_step'],1), p['cycles_per_lane_frame'], round(d['value']), {k:p[k] for k in ['emit','eps','beam_count','select','records','reset']})"
  done
done
