# Round-1 evidence for profiles/: (1) launch list + DRAM bytes of the bench command,
# (2) full ncu capture of one 512-lane x 80-frame k_decode_chunk launch.
python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --csv --log-file gpurun_out/r1_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --streams 0 > gpurun_out/r1_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 2 -c 1 \
  -o gpurun_out/r1_full python bench.py --batch 512 --frames 80 --steps 1 --warmup 3 --no-cpu --streams 0 > gpurun_out/r1_full.log 2>&1
tail -2 gpurun_out/r1_launches.log gpurun_out/r1_full.log
