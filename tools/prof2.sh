# ncu full capture of the cluster frame kernel: 512 lanes x 40 frames
python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
CTW_CLUSTER=${C:-4} timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 2 -c 1 \
  -o gpurun_out/prof_${TAG:-c4} python bench.py --batch ${NB:-512} --frames ${NF:-40} --steps 1 --warmup 3 --no-cpu --streams 0 > gpurun_out/prof_${TAG:-c4}.log 2>&1
tail -2 gpurun_out/prof_${TAG:-c4}.log
