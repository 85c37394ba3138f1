#!/bin/bash
# Round-end evidence: bench JSON, CUPTI per-kernel table, ncu launch list of one
# step, ncu --set full of the dominant kernels.  Usage: bash tools/gpu_profiles.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
RN_PDL=0 KPROF_NOSIDE=1 KPROF_NOGRAPH=1 timeout 300 python tools/kprof.py 5 8 gpurun_out/${TAG}_kprof.txt > /dev/null 2>&1  # PDL off: CUPTI durations would include the griddepcontrol.wait of early-launched kernels
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python tools/profile_step.py 2 > gpurun_out/${TAG}_launches.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1
for spec in "conv_pair_kernel:2" "wgrad_tc_kernel<\(int\)64, \(int\)3:2" "conv_tc_kernel<\(int\)128, \(int\)6:6" "bn_apply_part_k:2"; do
  re=${spec%:*}; sk=${spec##*:}; nm=$(echo "$re" | tr -dc 'a-z_')
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s $sk -c 1 \
    -o gpurun_out/${TAG}_full_${nm} python tools/profile_step.py 2 > gpurun_out/${TAG}_full_${nm}.log 2>&1
done
cat gpurun_out/${TAG}_bench.json
