for f in "" "-DLAT_BS=1024" "-DLAT_BS=256"; do
  CTW_NVCC_FLAGS="$f" python -m paper_2311_04996_b200.build -f >/dev/null 2>&1
  timeout 300 python bench.py --batch 64 --lattice 64 --no-cpu --streams 0 --steps 1 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); l=d['lattice']; print('$f', round(l['lattice_stage_s'],3), round(l['rtfx_decode_plus_lattice']), l['arcs_per_frame_mean'])"
done
