#!/bin/bash
# ncu --set full captures of selected kernels of the r18 step (demangled-name regexes)
# Usage: bash tools/gpu_ncu.sh TAG "regex1" skip1 "regex2" skip2 ...
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
i=0
while [ $# -ge 2 ]; do
  re=$1; sk=$2; shift 2
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s $sk -c 1 \
    -o gpurun_out/${TAG}_k$i python tools/profile_step.py 2 > gpurun_out/${TAG}_k$i.log 2>&1
  echo "k$i $re rc=$?"; i=$((i+1))
done
