# ncu full capture of one steady streaming step's frame kernel (6 lanes x 12
# frames, the wide 16 x 1024-thread shape) from tools/stream_timeline.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 25 -c 1 \
  -o gpurun_out/${1:-prof_stream} python tools/stream_timeline.py 6 10 > gpurun_out/${1:-prof_stream}.log 2>&1
tail -n 2 gpurun_out/${1:-prof_stream}.log
