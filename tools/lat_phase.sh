# lattice stage phase times (CTW_LAT_TIMING) on 64 C2 utterances, optionally
# for several CTW_LAT_RANKS values: bash tools/lat_phase.sh [ranks ...]
if [ $# -eq 0 ]; then set -- auto; fi
for r in "$@"; do
  if [ "$r" = auto ]; then unset CTW_LAT_RANKS; else export CTW_LAT_RANKS=$r; fi
  echo "== ranks $r"
  CTW_LAT_TIMING=1 python tools/lat_timing2.py 64 2>&1 | grep -v "^ " | grep "kernel\|n=64" | tail -3
done
