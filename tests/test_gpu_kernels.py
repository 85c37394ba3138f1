"""Kernel-level parity through the C ABI (rn_op_conv3d): every convolution
class of the r18 step at the full 91x109x91 sizes (batch 2), tcgen05 and SIMT,
against the oracle's float64 convolution on the same bf16-valued inputs.
Tolerance: fp32 accumulation + one bf16 rounding of the output ->
per-tensor relative L2 error <= 4e-3 AND element-wise |err| <= 2^-7 |ref| +
2^-9 max|ref| (bf16 outputs; fp32 weight gradients: 1e-4 rel-L2 and 1e-3 |ref|
+ 1e-5 max|ref|).  impl 5 runs the persistent kernel
on CTA pairs (cta_group::2) for every launch it takes, split-K included; impl 6
the streaming mma.sync kernel of the 64 -> 64 1x1x1 convs (k_conv1x1.cu)."""
import numpy as np
import pytest
import torch

from oracle import net as O
from paper_2104_05035_b200 import rn

pytestmark = pytest.mark.gpu

# (name, Di,Hi,Wi, Ci, Co, k, s, p) — the r18 conv classes (reading X2-X5)
CONVS = [
    ("s1_k3", 23, 28, 23, 64, 64, 3, 1, 1),
    ("s2_k3_s2", 23, 28, 23, 64, 128, 3, 2, 1),
    ("s2_proj", 23, 28, 23, 64, 128, 1, 2, 0),
    ("s2_k3", 12, 14, 12, 128, 128, 3, 1, 1),
    ("s3_k3_s2", 12, 14, 12, 128, 256, 3, 2, 1),
    ("s3_k3", 6, 7, 6, 256, 256, 3, 1, 1),
    ("s4_k3_s2", 6, 7, 6, 256, 512, 3, 2, 1),
    ("s4_k3", 3, 4, 3, 512, 512, 3, 1, 1),
    ("att1_mask_k3", 12, 14, 12, 64, 64, 3, 1, 1),
    ("att1_mconv", 23, 28, 23, 64, 64, 1, 1, 0),
]


def bf16_vals(shape, rng, scale=1.0):
    t = torch.from_numpy((rng.standard_normal(shape) * scale).astype(np.float32)).to(torch.bfloat16)
    return t


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def elem_ok(a, b, r=2.0 ** -7, t=2.0 ** -9):
    """Element-wise: |a - b| <= r |b| + t max|b| at every element (bf16 outputs: one
    rounding is <= 2^-9 |b|; fp32 accumulation adds far less) -- a single wrong voxel
    row or channel fails it, which the norm-wise check would not see."""
    err = np.abs(a - b)
    bound = r * np.abs(b) + t * np.abs(b).max()
    return bool((err <= bound).all()), float((err / bound).max())


@pytest.mark.parametrize("impl", [6, 5, 4, 3, 2, 1])
@pytest.mark.parametrize("cv", CONVS, ids=[c[0] for c in CONVS])
def test_conv_fprop_dgrad(cv, impl):
    name, Di, Hi, Wi, Ci, Co, k, s, p = cv
    if impl in (3, 4) and not (Ci == 64 and Co == 64 and k == 3 and s == 1):
        pytest.skip("haloed / CTA-pair kernels: 64->64 stride-1 3x3x3 only")
    if impl == 6 and not (Ci == 64 and Co == 64 and k == 1 and s == 1):
        pytest.skip("streaming 1x1x1 kernel: 64->64 stride-1 1x1x1 only")
    N = 2
    Do, Ho, Wo = (O.conv_out(v, k, s, p) for v in (Di, Hi, Wi))
    rng = np.random.default_rng(0)
    x = bf16_vals((N, Di, Hi, Wi, Ci), rng)
    w = bf16_vals((Co, k * k * k, Ci), rng, scale=(2.0 / (Co * k ** 3)) ** 0.5)
    dy = bf16_vals((N, Do, Ho, Wo, Co), rng)
    geom = [N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p]
    y = torch.empty((N, Do, Ho, Wo, Co), dtype=torch.bfloat16, device="cuda")
    dx = torch.empty((N, Di, Hi, Wi, Ci), dtype=torch.bfloat16, device="cuda")
    xd, wd, dyd = x.cuda(), w.cuda(), dy.cuda()
    rn.op_conv3d(rn.RN_BF16, 0, geom, xd, wd, y, impl)
    rn.op_conv3d(rn.RN_BF16, 1, geom, dyd, wd, dx, impl)
    torch.cuda.synchronize()
    # oracle on the same bf16 values, float64
    wc = w.float().numpy().astype(np.float64).reshape(Co, k, k, k, Ci).transpose(0, 4, 1, 2, 3)
    xn = x.float().numpy().astype(np.float64)
    dyn = dy.float().numpy().astype(np.float64)
    y_ref = O.conv3d(xn, wc, s, p)
    dx_ref, _ = O.conv3d_backward(xn, wc, dyn, s, p)
    yg, dxg = y.float().cpu().numpy(), dx.float().cpu().numpy()
    assert rel(yg, y_ref) < 4e-3
    assert rel(dxg, dx_ref) < 4e-3
    assert elem_ok(yg, y_ref)[0], elem_ok(yg, y_ref)
    assert elem_ok(dxg, dx_ref)[0], elem_ok(dxg, dx_ref)


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("cv", CONVS, ids=[c[0] for c in CONVS])
def test_conv_wgrad(cv, impl):
    name, Di, Hi, Wi, Ci, Co, k, s, p = cv
    N = 2
    Do, Ho, Wo = (O.conv_out(v, k, s, p) for v in (Di, Hi, Wi))
    rng = np.random.default_rng(1)
    x = bf16_vals((N, Di, Hi, Wi, Ci), rng)
    dy = bf16_vals((N, Do, Ho, Wo, Co), rng)
    geom = [N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p]
    dw = torch.empty((Co, k ** 3, Ci), dtype=torch.float32, device="cuda")
    rn.op_conv3d(rn.RN_BF16, 2, geom, x.cuda(), dy.cuda(), dw, impl)
    torch.cuda.synchronize()
    xn = x.float().numpy().astype(np.float64)
    dyn = dy.float().numpy().astype(np.float64)
    _, dw_ref = O.conv3d_backward(xn, np.zeros((Co, Ci, k, k, k)), dyn, s, p, need_dx=False)
    got = dw.cpu().numpy().reshape(Co, k, k, k, Ci).transpose(0, 4, 1, 2, 3)
    assert rel(got, dw_ref) < 1e-4
    assert elem_ok(got, dw_ref, 1e-3, 1e-5)[0], elem_ok(got, dw_ref, 1e-3, 1e-5)


@pytest.mark.parametrize("cv", CONVS, ids=[c[0] for c in CONVS])
def test_conv_bench_batch(cv):
    """The launch configuration bench.py times: batch 8 (BASELINE configs[1]) and
    the plan's own dispatch (impl 0: CTA pair for 64->64 stride 1, tcgen05 with its
    batch-8 tiling / ring depth / split-K / parity classes otherwise) for fprop,
    dgrad and wgrad, against the float64 oracle on the same bf16 values."""
    name, Di, Hi, Wi, Ci, Co, k, s, p = cv
    N = 8
    Do, Ho, Wo = (O.conv_out(v, k, s, p) for v in (Di, Hi, Wi))
    rng = np.random.default_rng(2)
    x = bf16_vals((N, Di, Hi, Wi, Ci), rng)
    w = bf16_vals((Co, k * k * k, Ci), rng, scale=(2.0 / (Co * k ** 3)) ** 0.5)
    dy = bf16_vals((N, Do, Ho, Wo, Co), rng)
    geom = [N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p]
    y = torch.empty((N, Do, Ho, Wo, Co), dtype=torch.bfloat16, device="cuda")
    dx = torch.empty((N, Di, Hi, Wi, Ci), dtype=torch.bfloat16, device="cuda")
    dw = torch.empty((Co, k ** 3, Ci), dtype=torch.float32, device="cuda")
    xd, wd, dyd = x.cuda(), w.cuda(), dy.cuda()
    rn.op_conv3d(rn.RN_BF16, 0, geom, xd, wd, y, 0)
    rn.op_conv3d(rn.RN_BF16, 1, geom, dyd, wd, dx, 0)
    rn.op_conv3d(rn.RN_BF16, 2, geom, xd, dyd, dw, 0)
    torch.cuda.synchronize()
    wc = w.float().numpy().astype(np.float64).reshape(Co, k, k, k, Ci).transpose(0, 4, 1, 2, 3)
    xn = x.float().numpy().astype(np.float64)
    dyn = dy.float().numpy().astype(np.float64)
    y_ref = O.conv3d(xn, wc, s, p)
    dx_ref, dw_ref = O.conv3d_backward(xn, wc, dyn, s, p)
    yg, dxg = y.float().cpu().numpy(), dx.float().cpu().numpy()
    assert rel(yg, y_ref) < 4e-3
    assert rel(dxg, dx_ref) < 4e-3
    assert elem_ok(yg, y_ref)[0], elem_ok(yg, y_ref)
    assert elem_ok(dxg, dx_ref)[0], elem_ok(dxg, dx_ref)
    got = dw.cpu().numpy().reshape(Co, k, k, k, Ci).transpose(0, 4, 1, 2, 3)
    assert rel(got, dw_ref) < 1e-4
    assert elem_ok(got, dw_ref, 1e-3, 1e-5)[0], elem_ok(got, dw_ref, 1e-3, 1e-5)
