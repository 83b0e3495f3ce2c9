# DRAM bytes of k_decode_chunk for library variants (ncu, 512 x 80 launch, 2nd launch)
for lib in "$@"; do
  CTW_B200_LIB=$(realpath $lib) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_decode_chunk -s 2 -c 2 --csv python tools/ab.py --child $lib --batch 512 --frames 80 --steps 1 --warmup 2 --search fast 2>/dev/null | grep -E "dram__bytes|lts__t_sector_hit|gpu__time" | awk -F'","' -v L=$(basename $lib) '{print L, $(NF-2), $(NF-1), $NF}'
done
