#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list, ncu --set full of the top conv kernels.
# Usage (under gpurun): bash tools/gpu_round.sh [tag] [what...]   what ∈ tests smoke bench launches full
set -x
TAG=${1:-r1}; shift
WHAT=${@:-tests smoke bench launches full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for w in $WHAT; do case $w in
tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" ;;
bench) timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json ;;
launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 2 > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?";
  python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1 ;;
full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel|wgrad_tc_kernel" -s 60 -c 4 -o gpurun_out/${TAG}_full python tools/profile_step.py 2 > gpurun_out/${TAG}_full.log 2>&1; echo "full rc=$?" ;;
esac; done
