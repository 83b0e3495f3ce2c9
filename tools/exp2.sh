for bs in 1024 256; do
  CTW_NVCC_FLAGS="-DCTW_BS=$bs" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
  for n in 18 37; do
    timeout 300 python bench.py --batch $n --no-cpu --streams 0 --steps 1 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['stage_profile']; print($bs, $n, round(d['ms_per_step'],1), p['cycles_per_lane_frame'], {k:p[k] for k in ['emit','eps','beam_count','select','records','reset']})"
  done
done > gpurun_out/exp2.txt 2>&1
cat gpurun_out/exp2.txt
