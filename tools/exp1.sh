for bs in 512 1024; do
  CTW_NVCC_FLAGS="-DCTW_BS=$bs" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
  for n in 148 512; do
    timeout 300 python bench.py --batch $n --no-cpu --streams 0 --steps 2 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($bs, $n, d['ms_per_step'], d['stage_profile']['cycles_per_lane_frame'], d['value'], d['stage_profile'])"
  done
done > gpurun_out/exp1.txt 2>&1
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/exp1.txt
cat gpurun_out/exp1.txt
