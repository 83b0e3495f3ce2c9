set -x
for cl in 8 16; do
CTW_CLUSTER=$cl timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --streams 0 --lattice 0 2>gpurun_out/exp_$cl.err | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print($cl, d['value'], d['workload_stats'], d['stage_profile']['cycles_per_lane_frame'])"
done
