# ncu full capture of k_decode_chunk: 1024-thread variant, 148 lanes x 30 frames
CTW_NVCC_FLAGS="${CTW_NVCC_FLAGS:--DCTW_BS=1024}" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 2 -c 1 \
  -o gpurun_out/prof_${TAG:-bs1024} python bench.py --batch ${NB:-148} --frames ${NF:-30} --steps 1 --warmup 3 --no-cpu --streams 0 > gpurun_out/prof_${TAG:-bs1024}.log 2>&1
tail -3 gpurun_out/prof_${TAG:-bs1024}.log
