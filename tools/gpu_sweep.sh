#!/bin/bash
# context measurements beside the headline bench line: batch and depth sweep (device-timed, 1 GPU)
TAG=${1:-sw}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "18 8" "18 16" "18 32" "34 8" "34 32"; do
  set -- $cfg
  timeout 600 python bench.py --depth $1 --batch $2 --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${TAG}_r$1_b$2.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_r$1_b$2.json'));print('r$1 b$2', round(d['value'],1), 'samples/s', round(d['ms_per_step'],3), 'ms/step', 'e2e', round(d['e2e']['value'],1), 'pair-frac', round(d['roofline']['frac'],3), 'all-conv-frac', round(d['roofline']['all_convs']['frac'],3))"
done
