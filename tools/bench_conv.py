"""Micro-benchmark of every r18 convolution class through rn_op_conv3d (batch 8,
full 91x109x91 sizes): CUDA-event time per launch and TFLOP/s.
Usage: python tools/bench_conv.py [ops=0,1,2] [impl=0]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.net import conv_out  # noqa: E402  (shape arithmetic only)
from paper_2104_05035_b200 import rn  # noqa: E402

CONVS = [("s1_k3", 23, 28, 23, 64, 64, 3, 1, 1), ("s2_k3_s2", 23, 28, 23, 64, 128, 3, 2, 1),
         ("s2_proj", 23, 28, 23, 64, 128, 1, 2, 0), ("s2_k3", 12, 14, 12, 128, 128, 3, 1, 1),
         ("s3_k3_s2", 12, 14, 12, 128, 256, 3, 2, 1), ("s3_k3", 6, 7, 6, 256, 256, 3, 1, 1),
         ("s4_k3_s2", 6, 7, 6, 256, 512, 3, 2, 1), ("s4_k3", 3, 4, 3, 512, 512, 3, 1, 1),
         ("att1_mask_k3", 12, 14, 12, 64, 64, 3, 1, 1), ("att1_mconv", 23, 28, 23, 64, 64, 1, 1, 0)]
ops = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2").split(",")]
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
only = sys.argv[3].split(",") if len(sys.argv) > 3 else None
N = 8
for name, Di, Hi, Wi, Ci, Co, k, s, p in CONVS:
    if only and name not in only:
        continue
    Do, Ho, Wo = (conv_out(v, k, s, p) for v in (Di, Hi, Wi))
    geom = [N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p]
    x = torch.randn(N, Di, Hi, Wi, Ci, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, k ** 3, Ci, device="cuda") * 0.05).to(torch.bfloat16)
    dy = torch.randn(N, Do, Ho, Wo, Co, device="cuda").to(torch.bfloat16)
    y = torch.empty(N, Do, Ho, Wo, Co, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty_like(x)
    dw = torch.empty(Co, k ** 3, Ci, device="cuda")
    flops = 2.0 * N * Do * Ho * Wo * Co * Ci * k ** 3
    out = []
    for op in ops:
        a, b, o = [(x, w, y), (dy, w, dx), (x, dy, dw)][op]
        for _ in range(3):
            rn.op_conv3d(rn.RN_BF16, op, geom, a, b, o, impl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        R = 10
        for _ in range(R):
            rn.op_conv3d(rn.RN_BF16, op, geom, a, b, o, impl)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / R
        out.append(f"{['fprop', 'dgrad', 'wgrad'][op]} {us:7.1f} us {flops / us / 1e6:6.0f} TF/s")
    print(f"{name:14s} {flops / 1e9:6.1f} GF  " + "  ".join(out))
