# ncu evidence for one kernel variant: launch list of the bench command (per-launch
# time + DRAM bytes) and one --set full capture of a steady-state 512-lane x 80-frame
# launch.   usage: bash tools/prof.sh TAG [fast|exact]
TAG=${1:?tag}; SEARCH=${2:-fast}
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --search $SEARCH --steps 1 --warmup 3 --no-cpu --streams 0 --lattice 0 > gpurun_out/${TAG}_launches.log 2>&1
# (the first decode call also runs a few small grow re-runs: skip past them
# into the steady warm-up launches)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 6 -c 1 \
  -o gpurun_out/${TAG}_full python bench.py --search $SEARCH --batch 512 --frames 80 --steps 1 --warmup 8 --no-cpu \
  --streams 0 --lattice 0 > gpurun_out/${TAG}_full.log 2>&1
tail -n 2 gpurun_out/${TAG}_launches.log gpurun_out/${TAG}_full.log
ls -la gpurun_out/${TAG}_*
