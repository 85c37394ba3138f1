"""Pins for the oracle's primitive ops (CPU only).  Each test checks the oracle
against something other than itself: brute-force loops, closed forms,
invariants, adjoint identities, or PyTorch CPU float64 (independent library)."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import net as O

rng = np.random.default_rng(123)


def brute_conv(x, w, s, p):
    """7-nested-loop direct convolution (definition)."""
    N, D, H, W, Ci = x.shape
    Co, _, k, _, _ = w.shape
    Do, Ho, Wo = ((v + 2 * p - k) // s + 1 for v in (D, H, W))
    y = np.zeros((N, Do, Ho, Wo, Co))
    for n in range(N):
        for od in range(Do):
            for oh in range(Ho):
                for ow in range(Wo):
                    for co in range(Co):
                        acc = 0.0
                        for kd in range(k):
                            for kh in range(k):
                                for kw in range(k):
                                    i, j, l = od * s + kd - p, oh * s + kh - p, ow * s + kw - p
                                    if 0 <= i < D and 0 <= j < H and 0 <= l < W:
                                        for ci in range(Ci):
                                            acc += x[n, i, j, l, ci] * w[co, ci, kd, kh, kw]
                        y[n, od, oh, ow, co] = acc
    return y


@pytest.mark.parametrize("s,k,p", [(1, 3, 1), (2, 3, 1), (2, 1, 0), (1, 1, 0)])
def test_conv_bruteforce(s, k, p):
    x = rng.standard_normal((2, 5, 4, 6, 2))
    w = rng.standard_normal((3, 2, k, k, k))
    np.testing.assert_allclose(O.conv3d(x, w, s, p), brute_conv(x, w, s, p), rtol=1e-12, atol=1e-12)


def test_conv_special_cases():
    x = rng.standard_normal((2, 4, 5, 3, 3))
    w1 = rng.standard_normal((4, 3, 1, 1, 1))
    np.testing.assert_allclose(O.conv3d(x, w1, 1, 0), x @ w1[:, :, 0, 0, 0].T, rtol=1e-13)
    delta = np.zeros((3, 3, 3, 3, 3))
    for c in range(3):
        delta[c, c, 1, 1, 1] = 1.0
    np.testing.assert_array_equal(O.conv3d(x, delta, 1, 1), x)


@pytest.mark.parametrize("s,k,p", [(1, 3, 1), (2, 3, 1), (2, 1, 0)])
def test_conv_vs_torch_and_adjoint(s, k, p):
    x = rng.standard_normal((2, 7, 6, 5, 3))
    w = rng.standard_normal((4, 3, k, k, k))
    y = O.conv3d(x, w, s, p)
    yt = F.conv3d(torch.from_numpy(x).permute(0, 4, 1, 2, 3), torch.from_numpy(w), stride=s, padding=p)
    np.testing.assert_allclose(y, yt.permute(0, 2, 3, 4, 1).numpy(), rtol=1e-12, atol=1e-12)
    dy = rng.standard_normal(y.shape)
    dx, dw = O.conv3d_backward(x, w, dy, s, p)
    lhs = np.sum(y * dy)
    assert abs(lhs - np.sum(x * dx)) < 1e-10 * max(1, abs(lhs))      # <conv(x),dy> = <x, dgrad(dy)>
    assert abs(lhs - np.sum(w * dw)) < 1e-10 * max(1, abs(lhs))      # <conv(x),dy> = <w, wgrad(x,dy)>


def test_bn_closed_forms():
    x = 3.0 + 2.0 * rng.standard_normal((3, 4, 5, 2, 4))
    g = rng.standard_normal(4)
    b = rng.standard_normal(4)
    y, c = O.bn_forward(x, g, b)
    var = x.var(axis=(0, 1, 2, 3))
    np.testing.assert_allclose(y.mean(axis=(0, 1, 2, 3)), b, atol=1e-12)
    np.testing.assert_allclose(y.var(axis=(0, 1, 2, 3)), g * g * var / (var + O.BN_EPS), rtol=1e-10)
    dy = rng.standard_normal(x.shape)
    dx, dg, db = O.bn_backward(dy, c, g)
    np.testing.assert_allclose(dx.sum(axis=(0, 1, 2, 3)), 0, atol=1e-10)
    # sum dx*xhat = gamma*invstd*(eps/(var+eps))*sum dy*xhat (zero up to the eps term)
    sdx = (dy * c["xhat"]).sum(axis=(0, 1, 2, 3))
    np.testing.assert_allclose((dx * c["xhat"]).sum(axis=(0, 1, 2, 3)),
                               g * c["invstd"] * O.BN_EPS / (var + O.BN_EPS) * sdx, rtol=1e-6, atol=1e-12)
    # library routine: torch batch_norm autograd
    xt = torch.from_numpy(x).permute(0, 4, 1, 2, 3).requires_grad_()
    gt = torch.from_numpy(g).requires_grad_()
    bt = torch.from_numpy(b).requires_grad_()
    rm, rv = torch.zeros(4, dtype=torch.float64), torch.ones(4, dtype=torch.float64)
    yt = F.batch_norm(xt, rm, rv, gt, bt, training=True, momentum=0.1, eps=1e-5)
    np.testing.assert_allclose(yt.permute(0, 2, 3, 4, 1).detach().numpy(), y, rtol=1e-12, atol=1e-12)
    yt.backward(torch.from_numpy(dy).permute(0, 4, 1, 2, 3))
    np.testing.assert_allclose(xt.grad.permute(0, 2, 3, 4, 1).numpy(), dx, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(gt.grad.numpy(), dg, rtol=1e-10)
    np.testing.assert_allclose(bt.grad.numpy(), db, rtol=1e-10)
    np.testing.assert_allclose(rv.numpy(), 0.9 + 0.1 * c["var_unbiased"], rtol=1e-12)
    np.testing.assert_allclose(rm.numpy(), 0.1 * c["mu"], rtol=1e-12)


def brute_maxpool(x):
    N, D, H, W, C = x.shape
    Do, Ho, Wo = ((v - 1) // 2 + 1 for v in (D, H, W))
    y = np.zeros((N, Do, Ho, Wo, C))
    am = np.zeros((N, Do, Ho, Wo, C), dtype=int)
    for n in range(N):
        for od in range(Do):
            for oh in range(Ho):
                for ow in range(Wo):
                    for c in range(C):
                        best, bi = -np.inf, -1
                        for t in range(27):
                            kd, kh, kw = t // 9, (t // 3) % 3, t % 3
                            i, j, l = 2 * od + kd - 1, 2 * oh + kh - 1, 2 * ow + kw - 1
                            if 0 <= i < D and 0 <= j < H and 0 <= l < W and x[n, i, j, l, c] > best:
                                best, bi = x[n, i, j, l, c], t
                        y[n, od, oh, ow, c], am[n, od, oh, ow, c] = best, bi
    return y, am


def test_maxpool_bruteforce_and_torch():
    x = rng.standard_normal((2, 5, 6, 7, 3))
    x[0, 1, 1, 1, 0] = x[0, 1, 1, 2, 0]          # a tie inside one window
    y, am = O.maxpool3(x)
    yb, ab = brute_maxpool(x)
    np.testing.assert_array_equal(y, yb)
    np.testing.assert_array_equal(am, ab)
    dy = rng.standard_normal(y.shape)
    dx = O.maxpool3_backward(dy, am, x.shape)
    xt = torch.from_numpy(x).permute(0, 4, 1, 2, 3).requires_grad_()
    yt = F.max_pool3d(xt, 3, 2, 1)
    yt.backward(torch.from_numpy(dy).permute(0, 4, 1, 2, 3))
    np.testing.assert_allclose(xt.grad.permute(0, 2, 3, 4, 1).numpy(), dx, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("din,dout", [((12, 14, 12), (23, 28, 23)), ((3, 4, 3), (6, 7, 6)), ((8, 8, 8), (16, 16, 16))])
def test_trilinear_vs_torch_adjoint_constant(din, dout):
    x = rng.standard_normal((2,) + din + (3,))
    y = O.upsample_trilinear(x, dout)
    yt = F.interpolate(torch.from_numpy(x).permute(0, 4, 1, 2, 3), size=dout, mode="trilinear", align_corners=False)
    np.testing.assert_allclose(y, yt.permute(0, 2, 3, 4, 1).numpy(), rtol=1e-12, atol=1e-13)
    dy = rng.standard_normal(y.shape)
    dx = O.upsample_trilinear_backward(dy, din)
    assert abs(np.sum(y * dy) - np.sum(x * dx)) < 1e-10
    c = np.full((1,) + din + (1,), 2.5)
    np.testing.assert_allclose(O.upsample_trilinear(c, dout), 2.5, rtol=1e-14)


def test_attention_and_ce_special_cases():
    assert O.sigmoid(np.array(0.0)) == 0.5        # m = 0 -> out = 1.5 T
    z = np.zeros((3, 2))
    loss, dz = O.softmax_ce(z, np.array([0, 1, 1]))
    assert abs(loss - math.log(2.0)) < 1e-15
    assert abs(loss - 0.6931471805599453) < 1e-15
    np.testing.assert_allclose(dz.sum(axis=1), 0, atol=1e-16)
    np.testing.assert_allclose(dz, np.array([[-0.5, 0.5], [0.5, -0.5], [0.5, -0.5]]) / 3)


def test_gradcam_last_pins():
    """Grad-CAM at the last conv layer: (a) the gradient it uses
    matches central finite differences of the class score y_c = FC(GAP(A))_c;
    (b) a constant activation gives a constant map ReLU(sum_k alpha_k a_k);
    (c) a negative evidence map is zeroed (ReLU)."""
    rng = np.random.default_rng(3)
    N, d, h, w, C = 2, 3, 4, 3, 5
    A = rng.standard_normal((N, d, h, w, C))
    W = rng.standard_normal((2, C))
    V = d * h * w

    def score(Ax, c):  # y_c for one sample
        return float(Ax.reshape(-1, C).mean(axis=0) @ W[c])
    eps = 1e-6
    for c in (0, 1):
        k, vox = 2, (1, 2, 0)
        Ap, Am = A[0].copy(), A[0].copy()
        Ap[vox + (k,)] += eps
        Am[vox + (k,)] -= eps
        fd = (score(Ap, c) - score(Am, c)) / (2 * eps)
        assert abs(fd - W[c, k] / V) < 1e-8
    const = np.ones((1, d, h, w, C)) * 0.7
    m = O.gradcam_last(const, W, 1, (7, 9, 5))
    ref = max(0.0, float(0.7 * W[1].sum() / V))
    np.testing.assert_allclose(m, ref, rtol=1e-12, atol=1e-15)
    neg = -np.abs(np.ones((1, d, h, w, C)))
    Wp = np.abs(W)
    assert np.all(O.gradcam_last(neg, Wp, 0, (5, 5, 5)) == 0.0)
