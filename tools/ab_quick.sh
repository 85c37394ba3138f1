#!/bin/bash
# quick GPU check of a change: op-level parity + 3 default bench runs (value, ms/step)
python -m pytest tests/test_gpu_ops.py tests/test_gpu_units.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
 python bench.py --no-cpu-baseline --f32-steps 0 --steps 30 > /tmp/ab.json 2>/dev/null
 python -c "import json;d=json.load(open('/tmp/ab.json'));print(round(d['value'],1),round(d['ms_per_step'],4))"
done
