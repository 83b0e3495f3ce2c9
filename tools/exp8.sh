python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
for t in 1 2; do timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed|Error" | head -5; done
python tools/dbg_golden.py c1_utt0 30 | tail -1
CTW_CLUSTER=1 timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed" | head -3
for c in 8 4; do
  CTW_CLUSTER=$c timeout 300 python bench.py --batch 512 --no-cpu --streams 0 --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['stage_profile']; print('C', $c, round(d['ms_per_step'],1), p['cycles_per_lane_frame'], round(d['value']), {k:p[k] for k in ['emit','eps','beam_count','select','records','reset']})"
done
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; cat gpurun_out/bench_full.json; tail -2 gpurun_out/bench_full.err
