# Lattice-leg A/B of library variants: tools/ab_lat.sh lib1.so lib2.so ...
for lib in "$@"; do
  CTW_B200_LIB=$(realpath $lib) python bench.py --steps 1 --warmup 3 --no-cpu --streams 0 --lattice 512 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); l=d['lattice']; print('$lib', round(d['value']), round(l['lattice_stage_s'],3), round(l['decode_lattice_s'],3), l['best_equals_decode'], l['nbest1_equals_best'], round(l['nbest10_host_s'],3), round(l['nbest10_pool_s'],3), l['nbest_pool_identical'])"
done
