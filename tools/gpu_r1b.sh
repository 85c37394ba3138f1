set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2104_05035_b200/csrc mma_rate.cu -o mma_rate -lcuda && ./mma_rate > ../../gpurun_out/r1b_mma_rate.txt 2>&1; cd ../..
python tools/bench_conv.py > gpurun_out/r1b_bench_conv.txt 2>&1
for k in conv_halo_kernel "conv_tc_kernel<64" "conv_tc_kernel<128" "wgrad_tc_kernel<64" "wgrad_tc_kernel<128" sgd_repack_all_k stem_wgrad_k wg_reduce_add bn_finalize_k; do
  n=$(echo $k | tr -dc 'a-z0-9_')
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -o gpurun_out/r1b_$n python tools/profile_step.py 2 > gpurun_out/r1b_$n.log 2>&1
done
