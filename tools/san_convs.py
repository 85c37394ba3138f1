"""Small conv launches through rn_op_conv3d for compute-sanitizer (racecheck /
synccheck / memcheck) on the hand-written tcgen05 / TMA / mbarrier pipelines:
CTA-pair (impl 4), haloed (3), generic implicit GEMM (2: stride 1 and stride 2,
64/128 channels, split-K), tensor-core wgrad.  Usage: python tools/san_convs.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_05035_b200 import rn  # noqa: E402

torch.manual_seed(0)
dev = torch.device("cuda", 0)


def run(op, N, Di, Hi, Wi, Ci, Co, k, s, p, impl):
    Do, Ho, Wo = ((v + 2 * p - k) // s + 1 for v in (Di, Hi, Wi))
    geom = [N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p]
    w = torch.randn(Co, k * k * k, Ci, device=dev).to(torch.bfloat16)
    if op == 0:
        a = torch.randn(N, Di, Hi, Wi, Ci, device=dev).to(torch.bfloat16)
        out = torch.empty(N, Do, Ho, Wo, Co, device=dev, dtype=torch.bfloat16)
        rn.op_conv3d(rn.RN_BF16, 0, geom, a, w, out, impl)
    elif op == 1:
        a = torch.randn(N, Do, Ho, Wo, Co, device=dev).to(torch.bfloat16)
        out = torch.empty(N, Di, Hi, Wi, Ci, device=dev, dtype=torch.bfloat16)
        rn.op_conv3d(rn.RN_BF16, 1, geom, a, w, out, impl)
    else:
        a = torch.randn(N, Di, Hi, Wi, Ci, device=dev).to(torch.bfloat16)
        dy = torch.randn(N, Do, Ho, Wo, Co, device=dev).to(torch.bfloat16)
        out = torch.empty(Co, k * k * k, Ci, device=dev, dtype=torch.float32)
        rn.op_conv3d(rn.RN_BF16, 2, geom, a, dy, out, impl)
    torch.cuda.synchronize()
    print(f"op {op} impl {impl} geom {geom}: ok", flush=True)


run(0, 1, 4, 16, 16, 64, 64, 3, 1, 1, 4)     # CTA pair fprop
run(1, 1, 4, 16, 16, 64, 64, 3, 1, 1, 4)     # CTA pair dgrad
run(0, 1, 4, 16, 16, 64, 64, 3, 1, 1, 3)     # haloed
run(0, 1, 6, 7, 6, 128, 128, 3, 1, 1, 2)     # generic, split-K
run(1, 1, 12, 14, 12, 64, 128, 3, 2, 1, 2)   # stride-2 dgrad (parity classes)
run(0, 1, 12, 14, 12, 64, 128, 3, 2, 1, 2)   # stride-2 fprop
run(2, 1, 6, 8, 8, 64, 64, 3, 1, 1, 0)       # tensor-core wgrad
