# full ncu capture of one steady-state 512-lane x 80-frame k_decode_chunk launch
python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 4 -c 1 \
  -o gpurun_out/r1_full python bench.py --batch 512 --frames 80 --steps 1 --warmup 4 --no-cpu --streams 0 > gpurun_out/r1_full.log 2>&1
tail -n 2 gpurun_out/r1_full.log
