# Round-1 evidence on the round-final kernel: launch list + DRAM bytes of the bench command, and
# one full capture of a steady-state 512-lane x 80-frame launch.
python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --csv --log-file gpurun_out/r1f_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --streams 0 --lattice 0 > gpurun_out/r1f_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 4 -c 1 \
  -o gpurun_out/r1f_full python bench.py --batch 512 --frames 80 --steps 1 --warmup 4 --no-cpu --streams 0 --lattice 0 > gpurun_out/r1f_full.log 2>&1
tail -n 1 gpurun_out/r1f_launches.log gpurun_out/r1f_full.log
