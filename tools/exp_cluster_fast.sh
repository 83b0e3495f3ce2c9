# fast mode: ranks per lane sweep (CTW_CLUSTER) on C2
for R in 8 4 2 16; do
  CTW_CLUSTER=$R timeout 600 python bench.py --search fast --streams 0 --lattice 0 --no-cpu > gpurun_out/expc_$R.json 2> gpurun_out/expc_$R.err
  python -c "import json,sys; d=json.load(open('gpurun_out/expc_$R.json')); print('R=$R', round(d['value']), d['stage_profile']['cycles_per_lane_frame'], d['stage_profile']['eps_passes_per_frame'])" || tail -3 gpurun_out/expc_$R.err
done
