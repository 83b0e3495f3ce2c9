# ncu full capture of the lattice kernel on 64 C2 utterances (fast decode)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 0 -c 1 \
  -o gpurun_out/${1:-prof_lat} python bench.py --batch 64 --lattice 64 --no-cpu --streams 0 --steps 1 --warmup 3 > gpurun_out/${1:-prof_lat}.log 2>&1
tail -n 2 gpurun_out/${1:-prof_lat}.log
