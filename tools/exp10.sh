python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
for t in 1 2; do
timeout 300 python bench.py --batch 512 --no-cpu --streams 0 --lattice 0 --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['stage_profile']; print(round(d['ms_per_step'],1), round(d['value']), {k:p[k] for k in ['emit','eps','records']}, p['cycles_per_lane_frame'])"
done
