#!/bin/bash
# A/B of two builds of librn.so (ab/base.so vs ab/new.so) on the bench, alternating, same box.
# Usage (under gpurun): bash tools/gpu_ab_so.sh TAG [reps]
TAG=$1; REPS=${2:-2}
mkdir -p gpurun_out
for r in $(seq $REPS); do
  for v in base new; do
    cp ab/$v.so paper_2104_05035_b200/librn.so
    timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_ab.json 2> gpurun_out/${TAG}_ab.err
    python -c "import json;d=json.load(open('gpurun_out/${TAG}_ab.json'));print('$v', 'value %.1f ms %.4f e2e %.1f elt_ms %.3f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['elementwise']['ms_per_step']))" 2>&1 | tail -1
  done
done
cp ab/new.so paper_2104_05035_b200/librn.so
