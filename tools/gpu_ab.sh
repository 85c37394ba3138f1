#!/bin/bash
# A/B of an environment toggle on the bench (same box, alternating runs)
# Usage (under gpurun): bash tools/gpu_ab.sh TAG "ENV=0" "ENV=1" [reps]
TAG=$1; A=$2; B=$3; REPS=${4:-2}
mkdir -p gpurun_out
for r in $(seq $REPS); do
  for cfg in "$A" "$B"; do
    env $cfg timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_ab.json 2> gpurun_out/${TAG}_ab.err
    python -c "import json;d=json.load(open('gpurun_out/${TAG}_ab.json'));print('$cfg', 'value %.1f ms %.4f e2e %.1f conv %.3f elt_ms %.3f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['all_convs_frac'], d['roofline']['elementwise']['ms_per_step']))" 2>&1 | tail -1
  done
done
