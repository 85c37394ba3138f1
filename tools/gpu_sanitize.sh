#!/bin/bash
# compute-sanitizer over the tcgen05/TMA conv kernels and one tiny bf16 step (summaries -> gpurun_out/)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_convs.py > gpurun_out/san_${tool}_convs.txt 2>&1
  echo "convs $tool rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_${tool}_convs.txt)"
done
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_tiny.py 18 64 24 28 24 2 1 bf16 1 > gpurun_out/san_${tool}_step.txt 2>&1
  echo "r18 bf16 step $tool rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_${tool}_step.txt)"
done
