#!/bin/bash
# A/B of env switches on the default bench: bash tools/ab_env.sh "ENV1=a ENV2=b" "ENV1=c" ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu-baseline --f32-steps 0 --steps 30 > /tmp/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/ab.json'));e=d['roofline']['elementwise']['by_family'];print('[$cfg]',round(d['value'],1),round(d['ms_per_step'],4),'bn_apply',round(e['bn_apply']['ms_per_step'],3),'bn_bwd',round(e['bn_bwd_apply']['ms_per_step'],3))"
done
done
