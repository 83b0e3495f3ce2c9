# cluster-port correctness + speed sweep
set -x
python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
for c in 8 1; do
  CTW_CLUSTER=$c timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
done
for c in 8 4 2 1; do
  for n in 37 512; do
    CTW_CLUSTER=$c timeout 300 python bench.py --batch $n --no-cpu --streams 0 --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['stage_profile']; print('C', $c, 'N', $n, round(d['ms_per_step'],1), p['cycles_per_lane_frame'], round(d['value']), {k:p[k] for k in ['emit','eps','beam_count','select','records','reset']}, d.get('parity'))"
  done
done
