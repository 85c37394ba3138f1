"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
cpu_baseline / --impl reference).  The product path (paper_2104_05035_b200/) never
imports this package and this package never imports the product.

Plain, slow, float64 NumPy implementation of ONE synchronous training step of
3D-ResAttNet (forward, backward, SGD) as the paper describes it:

* network (§4.3.1; concrete readings X1-X11 in DESIGN.md):
  stem Conv block (3x3x3 conv + BN + ReLU [+ maxpool]), residual network layers
  (two Conv blocks + skip), residual self-attention modules
  out = (1 + sigmoid(mask)) * trunk, global-average-pool + FC + cross-entropy
  (P:486).
* gradient flow between partitions / layers by the chain rule.
* data-parallel objective and gradient (Eqs. 9-11): the global
  gradient is (1/m) sum over replicas of each replica's mean gradient; with
  micro-batching (reading X18) each replica's gradient is the mean over its
  micro-batches.  BN statistics are per replica / micro-batch (reading X9).
* SGD update w <- w - gamma * g (plain SGD, reading X14).

Layout: activations are float64 arrays [N, D, H, W, C] (channels last).  The
convolution is written as the sum over the k^3 kernel offsets of a shifted
slice times the W_k channel matrix (one library matmul per offset) — no
blocking or fusion beyond that.

Parity status: pinned in tests/test_oracle_net.py against brute-force 7-loop
convolution, adjoint identities, closed forms (BN, CE, attention), PyTorch CPU
float64 autograd (an independent library routine) and central finite
differences.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BN_EPS = 1e-5          # reading X8 (PyTorch BatchNorm3d default, P:351 PyTorch 1.2)
BN_MOMENTUM = 0.1      # reading X8
N_CLASSES = 2          # binary tasks


# ----------------------------------------------------------------------------
# Network description (readings X2-X6)
# ----------------------------------------------------------------------------

def conv_out(n: int, k: int, s: int, p: int) -> int:
    return (n + 2 * p - k) // s + 1


@dataclass
class Unit:
    kind: str                  # 'stem' | 'block' | 'att' | 'head'
    cin: int
    cout: int
    stride: int
    in_dims: tuple
    out_dims: tuple
    extra: dict = field(default_factory=dict)


def arch(depth: int):
    """depth 0 = tiny (BASELINE configs[0]), 18, 34 (Table 2, reading X3)."""
    if depth == 0:
        return dict(stem_stride=1, stem_pool=False, blocks=[1], att_after=[0])
    if depth == 18:
        return dict(stem_stride=2, stem_pool=True, blocks=[2, 2, 2, 2], att_after=[0, 1, 2])
    if depth == 34:
        return dict(stem_stride=2, stem_pool=True, blocks=[3, 4, 6, 3], att_after=[0, 1, 2])
    raise ValueError(depth)


def build_units(depth: int, base_width: int, in_dims) -> list:
    a = arch(depth)
    units = []
    d = tuple(in_dims)
    s = a["stem_stride"]
    d1 = tuple(conv_out(v, 3, s, 1) for v in d)
    d2 = tuple(conv_out(v, 3, 2, 1) for v in d1) if a["stem_pool"] else d1
    units.append(Unit("stem", 1, base_width, s, d, d2, dict(conv_dims=d1, pool=a["stem_pool"])))
    c = base_width
    d = d2
    for si, nb in enumerate(a["blocks"]):
        width = base_width * (2 ** si)
        for bi in range(nb):
            stride = 2 if (si > 0 and bi == 0) else 1
            do = tuple(conv_out(v, 3, stride, 1) for v in d)
            units.append(Unit("block", c, width, stride, d, do))
            c, d = width, do
        if si in a["att_after"]:
            dm = tuple(conv_out(v, 3, 2, 1) for v in d)
            units.append(Unit("att", c, c, 1, d, d, dict(mask_dims=dm)))
    units.append(Unit("head", c, N_CLASSES, 1, d, (1, 1, 1)))
    return units


def block_param_shapes(prefix, cin, cout, stride):
    t = [(prefix + ".conv1", (cout, cin, 3, 3, 3), "conv"),
         (prefix + ".bn1.gamma", (cout,), "bn_gamma"), (prefix + ".bn1.beta", (cout,), "bn_beta"),
         (prefix + ".conv2", (cout, cout, 3, 3, 3), "conv"),
         (prefix + ".bn2.gamma", (cout,), "bn_gamma"), (prefix + ".bn2.beta", (cout,), "bn_beta")]
    if stride != 1 or cin != cout:
        t += [(prefix + ".proj", (cout, cin, 1, 1, 1), "conv"),
              (prefix + ".projbn.gamma", (cout,), "bn_gamma"), (prefix + ".projbn.beta", (cout,), "bn_beta")]
    return t


def param_tensors(units) -> list:
    """Canonical parameter order: list of (name, shape, kind)."""
    out = []
    for ui, u in enumerate(units):
        p = f"u{ui}"
        if u.kind == "stem":
            out += [(p + ".conv", (u.cout, 1, 3, 3, 3), "conv"),
                    (p + ".bn.gamma", (u.cout,), "bn_gamma"), (p + ".bn.beta", (u.cout,), "bn_beta")]
        elif u.kind == "block":
            out += block_param_shapes(p, u.cin, u.cout, u.stride)
        elif u.kind == "att":
            c = u.cout
            out += block_param_shapes(p + ".trunk", c, c, 1)
            out += block_param_shapes(p + ".mask", c, c, 1)
            out += [(p + ".mconv1", (c, c, 1, 1, 1), "conv"),
                    (p + ".mbn.gamma", (c,), "bn_gamma"), (p + ".mbn.beta", (c,), "bn_beta"),
                    (p + ".mconv2", (c, c, 1, 1, 1), "conv"),
                    (p + ".mconv2.bias", (c,), "bias")]
        elif u.kind == "head":
            out += [(p + ".fc.weight", (N_CLASSES, u.cin), "fc_w"), (p + ".fc.bias", (N_CLASSES,), "bias")]
    return out


def bn_layers(units) -> list:
    """Names of BN layers in canonical order (running statistics state)."""
    return [n[: -len(".gamma")] for n, s, k in param_tensors(units) if k == "bn_gamma"]


# ----------------------------------------------------------------------------
# Primitive ops, forward and backward (chain rule)
# ----------------------------------------------------------------------------

def conv3d(x, w, stride, pad):
    """x [N,D,H,W,Ci], w [Co,Ci,k,k,k] -> [N,Do,Ho,Wo,Co];
    y[n,o,co] = sum_{kd,kh,kw,ci} x[n, s*o + k - p, ci] * w[co,ci,k] (zero padding)."""
    N, D, H, W, Ci = x.shape
    Co, _, k, _, _ = w.shape
    Do, Ho, Wo = (conv_out(v, k, stride, pad) for v in (D, H, W))
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (pad, pad), (0, 0)))
    y = np.zeros((N, Do, Ho, Wo, Co))
    s = stride
    for kd in range(k):
        for kh in range(k):
            for kw in range(k):
                sl = xp[:, kd:kd + s * (Do - 1) + 1:s, kh:kh + s * (Ho - 1) + 1:s, kw:kw + s * (Wo - 1) + 1:s, :]
                y += (sl.reshape(-1, Ci) @ w[:, :, kd, kh, kw].T).reshape(N, Do, Ho, Wo, Co)
    return y


def conv3d_backward(x, w, dy, stride, pad, need_dx=True):
    """Returns (dx, dw) for y = conv3d(x, w)."""
    N, D, H, W, Ci = x.shape
    Co, _, k, _, _ = w.shape
    _, Do, Ho, Wo, _ = dy.shape
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (pad, pad), (0, 0)))
    dxp = np.zeros_like(xp) if need_dx else None
    dw = np.zeros_like(w)
    s = stride
    dy2 = dy.reshape(-1, Co)
    for kd in range(k):
        for kh in range(k):
            for kw in range(k):
                idx = (slice(None), slice(kd, kd + s * (Do - 1) + 1, s), slice(kh, kh + s * (Ho - 1) + 1, s),
                       slice(kw, kw + s * (Wo - 1) + 1, s), slice(None))
                sl = xp[idx]
                dw[:, :, kd, kh, kw] = dy2.T @ sl.reshape(-1, Ci)
                if need_dx:
                    dxp[idx] += (dy2 @ w[:, :, kd, kh, kw]).reshape(N, Do, Ho, Wo, Ci)
    dx = dxp[:, pad:pad + D, pad:pad + H, pad:pad + W, :] if need_dx else None
    return dx, dw


def bn_forward(x, gamma, beta):
    """Train-mode batch norm over (N,D,H,W) per channel (reading X8)."""
    axes = (0, 1, 2, 3)
    mu = x.mean(axis=axes)
    var = ((x - mu) ** 2).mean(axis=axes)            # biased, used to normalise
    invstd = 1.0 / np.sqrt(var + BN_EPS)
    xhat = (x - mu) * invstd
    y = gamma * xhat + beta
    cnt = x.size // x.shape[-1]
    var_unbiased = var * cnt / (cnt - 1) if cnt > 1 else var
    return y, dict(xhat=xhat, invstd=invstd, mu=mu, var_unbiased=var_unbiased)


def bn_backward(dy, cache, gamma):
    axes = (0, 1, 2, 3)
    xhat, invstd = cache["xhat"], cache["invstd"]
    dgamma = (dy * xhat).sum(axis=axes)
    dbeta = dy.sum(axis=axes)
    mdy = dy.mean(axis=axes)
    mdyx = (dy * xhat).mean(axis=axes)
    dx = gamma * invstd * (dy - mdy - xhat * mdyx)
    return dx, dgamma, dbeta


def bn_backward_coefs(dy, cache, gamma, h=None):
    """bn_backward's dx written as A*dy + B*h + Cc per channel (h = the BN input:
    x-hat = (h - mu) * invstd), with dgamma / dbeta:
    dx = gamma*invstd*(dy - mean(dy) - xhat*mean(dy*xhat)) = A dy + B h + Cc.
    h (optional): the values x-hat is formed from (default: the forward's x-hat)."""
    axes = (0, 1, 2, 3)
    xhat, invstd, mu = cache["xhat"], cache["invstd"], cache["mu"]
    if h is not None:
        xhat = (h - mu) * invstd
    dgamma = (dy * xhat).sum(axis=axes)
    dbeta = dy.sum(axis=axes)
    mdy = dy.mean(axis=axes)
    mdyx = (dy * xhat).mean(axis=axes)
    A = gamma * invstd
    B = -A * invstd * mdyx
    Cc = -A * mdy + A * invstd * mu * mdyx
    return A, B, Cc, dgamma, dbeta


# stem widths whose pooled bf16 backward runs at the pooled resolution (reading X23c)
STEM_POOLED_BWD_WIDTHS = (8, 16, 32, 64)


def relu(x):
    return np.maximum(x, 0.0)


def maxpool3(x):
    """MaxPool3d(k=3, s=2, p=1) with -inf padding; returns (y, argmax) where argmax
    is the window offset 0..26 ((kd*3+kh)*3+kw) of the FIRST maximum (reading X10)."""
    N, D, H, W, C = x.shape
    Do, Ho, Wo = (conv_out(v, 3, 2, 1) for v in (D, H, W))
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (1, 1), (0, 0)), constant_values=-np.inf)
    y = np.full((N, Do, Ho, Wo, C), -np.inf)
    am = np.zeros((N, Do, Ho, Wo, C), dtype=np.int64)
    for kd in range(3):
        for kh in range(3):
            for kw in range(3):
                sl = xp[:, kd:kd + 2 * (Do - 1) + 1:2, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2, :]
                better = sl > y                      # strict: first maximum wins
                y = np.where(better, sl, y)
                am = np.where(better, (kd * 3 + kh) * 3 + kw, am)
    return y, am


def maxpool3_backward(dy, am, in_shape):
    N, D, H, W, C = in_shape
    _, Do, Ho, Wo, _ = dy.shape
    dxp = np.zeros((N, D + 2, H + 2, W + 2, C))
    for kd in range(3):
        for kh in range(3):
            for kw in range(3):
                sel = (am == (kd * 3 + kh) * 3 + kw)
                idx = (slice(None), slice(kd, kd + 2 * (Do - 1) + 1, 2), slice(kh, kh + 2 * (Ho - 1) + 1, 2),
                       slice(kw, kw + 2 * (Wo - 1) + 1, 2), slice(None))
                dxp[idx] += np.where(sel, dy, 0.0)
    return dxp[:, 1:D + 1, 1:H + 1, 1:W + 1, :]


def linear_interp_matrix(n_in: int, n_out: int) -> np.ndarray:
    """1-D linear interpolation matrix, align_corners=False, output size given
    (reading X11): src = max((o + 1/2) * n_in/n_out - 1/2, 0), i0 = floor(src),
    i1 = min(i0 + 1, n_in - 1), lambda = src - i0."""
    M = np.zeros((n_out, n_in))
    scale = n_in / n_out
    for o in range(n_out):
        src = max((o + 0.5) * scale - 0.5, 0.0)
        i0 = int(math.floor(src))
        i0 = min(i0, n_in - 1)
        i1 = min(i0 + 1, n_in - 1)
        lam = src - i0
        M[o, i0] += 1.0 - lam
        M[o, i1] += lam
    return M


def upsample_trilinear(x, out_dims):
    """Separable trilinear interpolation = the product of three 1-D linear maps."""
    Md = linear_interp_matrix(x.shape[1], out_dims[0])
    Mh = linear_interp_matrix(x.shape[2], out_dims[1])
    Mw = linear_interp_matrix(x.shape[3], out_dims[2])
    return np.einsum("ad,bh,cw,ndhwk->nabck", Md, Mh, Mw, x, optimize=True)


def upsample_trilinear_backward(dy, in_dims):
    Md = linear_interp_matrix(in_dims[0], dy.shape[1])
    Mh = linear_interp_matrix(in_dims[1], dy.shape[2])
    Mw = linear_interp_matrix(in_dims[2], dy.shape[3])
    return np.einsum("ad,bh,cw,nabck->ndhwk", Md, Mh, Mw, dy, optimize=True)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


# ----------------------------------------------------------------------------
# Units: forward with cache, backward
# ----------------------------------------------------------------------------

class Params:
    """Name -> float64 array view over the canonical list."""

    def __init__(self, tensors, arrays):
        self.names = [t[0] for t in tensors]
        self.d = {n: np.asarray(a, dtype=np.float64) for n, a in zip(self.names, arrays)}

    def __getitem__(self, k):
        return self.d[k]


class BNState:
    """Running statistics (reading X8): r <- (1-momentum) r + momentum * stat,
    unbiased variance for the running variance."""

    def __init__(self, names, channels):
        self.mean = {n: np.zeros(c) for n, c in zip(names, channels)}
        self.var = {n: np.ones(c) for n, c in zip(names, channels)}

    def update(self, name, cache):
        self.mean[name] = (1 - BN_MOMENTUM) * self.mean[name] + BN_MOMENTUM * cache["mu"]
        self.var[name] = (1 - BN_MOMENTUM) * self.var[name] + BN_MOMENTUM * cache["var_unbiased"]


# Storage rounding (reading X23 (ii)): with Net(..., store="bf16")
# every value the RN_BF16 GPU path STORES in bf16 (conv outputs, BN-apply
# outputs, pooled / upsampled / attention tensors, every activation gradient,
# conv weight copies) is rounded to bf16 (round-to-nearest-even of the fp32
# value) at that point; the arithmetic stays float64.  store="f64" (default)
# makes Q and QW the identity, i.e. the plain definition.
def _bf16_round(a):
    f = np.asarray(a, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def _identity(a):
    return a


Q = _identity     # rounding of stored activations / gradients
QW = _identity    # rounding of the conv weights the kernels read


def block_forward(P, pre, x, stride, bns):
    c = {}
    c["x"] = x
    h1 = Q(conv3d(x, QW(P[pre + ".conv1"]), stride, 1))
    y1, c["bn1"] = bn_forward(h1, P[pre + ".bn1.gamma"], P[pre + ".bn1.beta"])
    a1 = Q(relu(y1))
    c["a1"] = a1
    h2 = Q(conv3d(a1, QW(P[pre + ".conv2"]), 1, 1))
    y2, c["bn2"] = bn_forward(h2, P[pre + ".bn2.gamma"], P[pre + ".bn2.beta"])
    if (pre + ".proj") in P.d:
        hp = Q(conv3d(x, QW(P[pre + ".proj"]), stride, 0))
        skip, c["bnp"] = bn_forward(hp, P[pre + ".projbn.gamma"], P[pre + ".projbn.beta"])
        c["proj"] = True
    else:
        skip = x
        c["proj"] = False
    z = y2 + skip
    out = Q(relu(z))
    c["out"] = out
    for k, n in (("bn1", ".bn1"), ("bn2", ".bn2"), ("bnp", ".projbn")):
        if k in c:
            bns.append((pre + n, c[k]))
    return out, c


def block_backward(P, pre, dout, c, stride, G, dx_acc=None):
    """dx_acc: gradient already accumulated into the input (attention: the mask
    branch); the result is dx_acc + this block's input gradient."""
    dz = dout * (c["out"] > 0)
    dh2, G[pre + ".bn2.gamma"], G[pre + ".bn2.beta"] = bn_backward(dz, c["bn2"], P[pre + ".bn2.gamma"])
    dh2 = Q(dh2)
    da1, G[pre + ".conv2"] = conv3d_backward(c["a1"], QW(P[pre + ".conv2"]), dh2, 1, 1)
    da1 = Q(da1)
    dy1 = da1 * (c["a1"] > 0)
    dh1, G[pre + ".bn1.gamma"], G[pre + ".bn1.beta"] = bn_backward(dy1, c["bn1"], P[pre + ".bn1.gamma"])
    dh1 = Q(dh1)
    dx, G[pre + ".conv1"] = conv3d_backward(c["x"], QW(P[pre + ".conv1"]), dh1, stride, 1)
    acc = 0.0 if dx_acc is None else dx_acc
    if c["proj"]:
        dhp, G[pre + ".projbn.gamma"], G[pre + ".projbn.beta"] = bn_backward(dz, c["bnp"], P[pre + ".projbn.gamma"])
        dhp = Q(dhp)
        dxp, G[pre + ".proj"] = conv3d_backward(c["x"], QW(P[pre + ".proj"]), dhp, stride, 0)
        dx = Q(Q(acc + dx) + dxp)
    else:
        dx = Q(acc + dx + dz)
    return dx


def unit_forward(P, ui, u, x, bns):
    pre = f"u{ui}"
    c = {}
    if u.kind == "stem":
        c["x"] = x
        c["h_raw"] = conv3d(x, P[pre + ".conv"], u.stride, 1)  # stem reads fp32 master weights
        h = Q(c["h_raw"])
        y, c["bn"] = bn_forward(h, P[pre + ".bn.gamma"], P[pre + ".bn.beta"])
        bns.append((pre + ".bn", c["bn"]))
        a = relu(y)
        c["a"] = a
        if u.extra["pool"]:
            out, c["am"] = maxpool3(a)
            out = Q(out)
        else:
            out = Q(a)
            c["a"] = out
        return out, c
    if u.kind == "block":
        return block_forward(P, pre, x, u.stride, bns)
    if u.kind == "att":
        T, c["trunk"] = block_forward(P, pre + ".trunk", x, 1, bns)
        u0, c["am"] = maxpool3(x)
        c["x_shape"] = x.shape
        um, c["mask"] = block_forward(P, pre + ".mask", u0, 1, bns)
        c["um_dims"] = um.shape[1:4]
        up = Q(upsample_trilinear(um, T.shape[1:4]))
        c["up"] = up
        h = Q(conv3d(up, QW(P[pre + ".mconv1"]), 1, 0))
        y, c["mbn"] = bn_forward(h, P[pre + ".mbn.gamma"], P[pre + ".mbn.beta"])
        bns.append((pre + ".mbn", c["mbn"]))
        r = Q(relu(y))
        c["r"] = r
        m = Q(conv3d(r, QW(P[pre + ".mconv2"]), 1, 0) + P[pre + ".mconv2.bias"])
        sg = sigmoid(m)
        c["sg"], c["T"] = sg, T
        return Q((1.0 + sg) * T), c
    if u.kind == "head":
        c["x_shape"] = x.shape
        g = x.mean(axis=(1, 2, 3))                     # GAP
        c["g"] = g
        z = g @ P[pre + ".fc.weight"].T + P[pre + ".fc.bias"]
        return z, c
    raise ValueError(u.kind)


def unit_backward(P, ui, u, dout, c, G):
    pre = f"u{ui}"
    if u.kind == "stem":
        if u.extra["pool"] and (Q is _identity or u.cout in STEM_POOLED_BWD_WIDTHS):
            # reading X23c: the pooled stem's backward neither reads the stored h nor
            # stores anything at the conv resolution — the pool adjoint da and dh are
            # not rounded, and the backward takes the conv's unrounded output h_raw
            # (x-hat of the BN sums and the h-term of dh; mu / invstd stay those of the
            # forward).  With store="f64" this IS bn_backward.
            da = maxpool3_backward(dout, c["am"], c["a"].shape)
            dy = da * (c["a"] > 0)
            A, B, Cc, G[pre + ".bn.gamma"], G[pre + ".bn.beta"] = bn_backward_coefs(
                dy, c["bn"], P[pre + ".bn.gamma"], h=c["h_raw"])
            dh = A * dy + B * c["h_raw"] + Cc
        else:
            da = Q(maxpool3_backward(dout, c["am"], c["a"].shape)) if u.extra["pool"] else dout
            dy = da * (c["a"] > 0)
            dh, G[pre + ".bn.gamma"], G[pre + ".bn.beta"] = bn_backward(dy, c["bn"], P[pre + ".bn.gamma"])
            dh = Q(dh)
        _, G[pre + ".conv"] = conv3d_backward(c["x"], P[pre + ".conv"], dh, u.stride, 1, need_dx=False)
        return None
    if u.kind == "block":
        return block_backward(P, pre, dout, c, u.stride, G)
    if u.kind == "att":
        sg, T = c["sg"], c["T"]
        dT = Q(dout * (1.0 + sg))
        dm = dout * T * sg * (1.0 - sg)
        G[pre + ".mconv2.bias"] = dm.sum(axis=(0, 1, 2, 3))
        dm = Q(dm)
        dr, G[pre + ".mconv2"] = conv3d_backward(c["r"], QW(P[pre + ".mconv2"]), dm, 1, 0)
        dr = Q(dr)
        dy = dr * (c["r"] > 0)
        dh, G[pre + ".mbn.gamma"], G[pre + ".mbn.beta"] = bn_backward(dy, c["mbn"], P[pre + ".mbn.gamma"])
        dh = Q(dh)
        dup, G[pre + ".mconv1"] = conv3d_backward(c["up"], QW(P[pre + ".mconv1"]), dh, 1, 0)
        dup = Q(dup)
        dum = Q(upsample_trilinear_backward(dup, c["um_dims"]))
        du0 = block_backward(P, pre + ".mask", dum, c["mask"], 1, G)
        dx_mask = Q(maxpool3_backward(du0, c["am"], c["x_shape"]))
        return block_backward(P, pre + ".trunk", dT, c["trunk"], 1, G, dx_acc=dx_mask)
    if u.kind == "head":
        dz = dout
        G[pre + ".fc.weight"] = dz.T @ c["g"]
        G[pre + ".fc.bias"] = dz.sum(axis=0)
        dg = dz @ P[pre + ".fc.weight"]
        N, D, H, W, C = c["x_shape"]
        return Q(np.broadcast_to(dg[:, None, None, None, :] / (D * H * W), c["x_shape"]).copy())
    raise ValueError(u.kind)


def gradcam_last(A, W, cls, out_dims):
    """Grad-CAM ("explainable block") at the last
    convolutional layer, written as its definition (Selvaraju et al.):
      dy_c/dA_k  — the gradient of the class score y_c = FC(GAP(A))_c; the head is
                   GAP + FC, so its backward gives W[c, k] / V at every voxel
      alpha_k    = mean over voxels of dy_c / dA_k
      cam        = ReLU(sum_k alpha_k A_k)
      map        = trilinear(cam, out_dims), align_corners=False (reading X11)
    A: (N, d, h, w, C) float64 (NDHWC, as the rest of the oracle); W: (2, C);
    cls: int or per-sample ints.  Returns (N, D, H, W) float64."""
    N, C = A.shape[0], A.shape[4]
    V = A.shape[1] * A.shape[2] * A.shape[3]
    cls = np.broadcast_to(np.asarray(cls), (N,))
    out = []
    for n in range(N):
        grad = np.broadcast_to(W[cls[n]] / V, A.shape[1:])          # GAP + FC backward, every voxel
        alpha = grad.reshape(-1, C).mean(axis=0)
        cam = relu(A[n] @ alpha)                                     # (d, h, w)
        out.append(upsample_trilinear(cam[None, :, :, :, None], out_dims)[0, :, :, :, 0])
    return np.stack(out)


def softmax_ce(z, y):
    """Mean softmax cross-entropy over the batch (reading X12) and dL/dz."""
    zmax = z.max(axis=1, keepdims=True)
    e = np.exp(z - zmax)
    p = e / e.sum(axis=1, keepdims=True)
    n = z.shape[0]
    loss = -np.mean(np.log(p[np.arange(n), y]))
    dz = p.copy()
    dz[np.arange(n), y] -= 1.0
    return loss, dz / n


# ----------------------------------------------------------------------------
# The training step (P:156 update, Eqs. 9-11 combination)
# ----------------------------------------------------------------------------

class Net:
    def __init__(self, depth: int, base_width: int, in_dims, store: str = "f64"):
        assert store in ("f64", "bf16")
        self.store = store
        self.depth, self.base_width, self.in_dims = depth, base_width, tuple(in_dims)
        self.units = build_units(depth, base_width, in_dims)
        self.tensors = param_tensors(self.units)
        self.n_params = int(sum(np.prod(s) for _, s, _ in self.tensors))
        self.bn_names = bn_layers(self.units)
        shapes = {n: s for n, s, _ in self.tensors}
        self.bn_channels = [shapes[n + ".gamma"][0] for n in self.bn_names]

    def forward_backward(self, P: Params, x, y, loss_scale=1.0, bnstate: BNState | None = None,
                         units=None):
        """One micro-batch: forward with train-mode BN, loss, backward.
        x float [N,D,H,W] (single input channel), y int [N].
        Returns (loss, grads dict scaled by loss_scale)."""
        global Q, QW
        Q = QW = (_bf16_round if self.store == "bf16" else _identity)
        try:
            return self._forward_backward(P, x, y, loss_scale, bnstate)
        finally:
            Q = QW = _identity

    def _forward_backward(self, P, x, y, loss_scale, bnstate):
        h = np.asarray(x, dtype=np.float64)[..., None]
        caches = []
        bns = []
        for ui, u in enumerate(self.units):
            h, c = unit_forward(P, ui, u, h, bns)
            caches.append(c)
        loss, dz = softmax_ce(h, np.asarray(y))
        G = {}
        g = dz * loss_scale
        for ui in reversed(range(len(self.units))):
            g = unit_backward(P, ui, self.units[ui], g, caches[ui], G)
        if bnstate is not None:
            for name, cache in bns:
                bnstate.update(name, cache)
        return loss, G, h

    def unit_step(self, P: Params, ui: int, x, dout=None, y=None):
        """Teacher-forced single unit (test infrastructure for per-unit parity):
        unit ui's forward from the given input x (NDHWC; the stem takes the raw
        [N,D,H,W] volume) and its backward from the given output gradient dout —
        the same unit_forward / unit_backward the whole step chains, in
        this Net's storage mode.  For the head, dout is None and y the labels:
        its incoming gradient is dz of the cross-entropy; dout None for
        any other unit runs the forward only.
        Returns dict(out, dx, G, bns, cache, loss)."""
        global Q, QW
        Q = QW = (_bf16_round if self.store == "bf16" else _identity)
        try:
            u = self.units[ui]
            h = np.asarray(x, dtype=np.float64)
            if u.kind == "stem":
                h = h[..., None]
            bns = []
            out, c = unit_forward(P, ui, u, h, bns)
            loss = None
            if u.kind == "head":
                loss, dout = softmax_ce(out, np.asarray(y))
            G, dx = {}, None
            if dout is not None:             # dout None (not the head): forward only
                dx = unit_backward(P, ui, u, np.asarray(dout, dtype=np.float64), c, G)
            return dict(out=out, dx=dx, G=G, bns=bns, cache=c, loss=loss)
        finally:
            Q = QW = _identity

    def flat(self, G) -> np.ndarray:
        return np.concatenate([np.asarray(G[n], dtype=np.float64).ravel() for n, _, _ in self.tensors])

    def train_step(self, arrays, x, y, lr: float, m: int = 1, Mb: int = 1, bnstate: BNState | None = None):
        """Synchronous hybrid/data-parallel step:
        G = (1/m) sum_r (1/Mb) sum_k grad mean_{n in (r,k)} loss_n  (Eq. 11 with
        micro-batches), delta = -lr * G, loss = mean over (r,k).
        x holds the global batch m*b samples, replica r owns samples [r*b, (r+1)*b)
        (equal sharding) and micro-batch k of replica r the k-th b/Mb slice.
        Running stats are updated sequentially over k, per replica; the returned
        state is replica 0's (every replica sees its own data)."""
        P = Params(self.tensors, arrays)
        Ntot = x.shape[0]
        assert Ntot % m == 0 and (Ntot // m) % Mb == 0
        b = Ntot // m
        mb = b // Mb
        Gsum = np.zeros(self.n_params)
        losses = []
        states = []
        for r in range(m):
            st = BNState(self.bn_names, self.bn_channels)
            if bnstate is not None and r == 0:
                st = bnstate
            for k in range(Mb):
                sl = slice(r * b + k * mb, r * b + (k + 1) * mb)
                loss, G, _ = self.forward_backward(P, x[sl], y[sl], 1.0, st)
                Gsum += self.flat(G) / (m * Mb)
                losses.append(loss)
            states.append(st)
        flat_w = np.concatenate([np.asarray(a, dtype=np.float64).ravel() for a in arrays])
        delta = -lr * Gsum
        return dict(loss=float(np.mean(losses)), grad=Gsum, delta=delta, new_params=flat_w + delta,
                    bn_state=states[0], losses=losses)


def delayed_pipeline_train(net, arrays, batches, lr, unit_stage):
    """Delayed-gradient pipelined training (PAPER.md:156
    "all partitions are computed simultaneously", Eqs. 1-2; reading F1 in
    DESIGN.md).  unit_stage[u] = pipeline stage (0..S-1) of unit u, non-decreasing
    along the chain; stage s is S-1-s iterations from the loss.  Iteration t
    (batches[t] = (x, y)):
      1. forward of batch t through every stage with its CURRENT weights, saving
         each stage's forward state and a copy of the weights it used (w^{(t)});
         loss of batch t and dl/dz at the head;
      2. every stage s backpropagates batch b = t - (S-1-s) (if b >= 0): the last
         stage the batch just forwarded (delay 0), stage s < S-1 the gradient of
         its output that stage s+1 produced in iteration t-1 -- through its saved
         forward state and the weights of that forward (Eq. 1: the Jacobian at
         w^{t-i+1}, the version that produced a^{t-i+1}), giving its weight
         gradient and the gradient of its input (sent to stage s-1, used there in
         iteration t+1);
      3. every stage that backpropagated updates its CURRENT weights,
         w <- w - lr * g (Eq. 2 with the delayed gradient).
    S = 1 is plain SGD.  Returns dict(losses, params (flat, float64), bn_state)."""
    global Q, QW
    Q = QW = (_bf16_round if net.store == "bf16" else _identity)
    try:
        S = max(unit_stage) + 1
        assert all(unit_stage[i] <= unit_stage[i + 1] for i in range(len(unit_stage) - 1))
        P = Params(net.tensors, [np.asarray(a, dtype=np.float64).copy() for a in arrays])
        st = BNState(net.bn_names, net.bn_channels)
        stage_units = [[u for u in range(len(net.units)) if unit_stage[u] == s] for s in range(S)]
        saved = {}      # (stage, batch) -> (weights dict used, [(ui, cache)], input of the stage)
        pending = {}    # (stage, batch) -> gradient of the stage's output
        losses = []
        for t, (x, y) in enumerate(batches):
            h = np.asarray(x, dtype=np.float64)[..., None]
            for s in range(S):                                  # 1. forward of batch t
                used = Params(net.tensors, [P[n].copy() for n in P.names])
                caches = []
                bns = []
                for ui in stage_units[s]:
                    h, c = unit_forward(used, ui, net.units[ui], h, bns)
                    caches.append((ui, c))
                for name, cache in bns:
                    st.update(name, cache)
                saved[(s, t)] = (used, caches)
            loss, dz = softmax_ce(h, np.asarray(y))
            losses.append(loss)
            pending[(S - 1, t)] = dz
            updates = []
            for s in reversed(range(S)):                        # 2. delayed backward
                b = t - (S - 1 - s)
                if b < 0:
                    continue
                used, caches = saved.pop((s, b))
                g = pending.pop((s, b))
                G = {}
                for ui, c in reversed(caches):
                    g = unit_backward(used, ui, net.units[ui], g, c, G)
                if s > 0:
                    pending[(s - 1, b)] = g
                updates.append(G)
            for G in updates:                                   # 3. update current weights
                for n, v in G.items():
                    P.d[n] = P.d[n] - lr * np.asarray(v, dtype=np.float64)
        flat = np.concatenate([P[n].ravel() for n in P.names])
        return dict(losses=losses, params=flat, bn_state=st)
    finally:
        Q = QW = _identity


def async_allreduce_train(net, arrays, batches, lr, m):
    """ASGD with ring all-reduce ("ASGD ... no need of
    waiting for the slowest GPU in every iteration"; reading F4 in DESIGN.md):
    the all-reduce of iteration t's gradients runs while iteration t+1 computes, so
    the update of iteration t uses the replica-averaged gradient of iteration t-1:
        G^t = (1/m) sum_r grad of replica r's mean loss on its shard at w^t (Eq. 11)
        w^{t+1} = w^t - lr G^{t-1},   G^{-1} = 0
    Every replica applies the same G^{t-1}, so the replicas stay identical.
    batches[t] = (x, y) of the global batch of iteration t (replica r owns its r-th
    equal shard).  Returns dict(losses [t][r], params (flat float64))."""
    cur = [np.asarray(a, dtype=np.float64).copy() for a in arrays]
    sizes = [int(np.prod(s)) for _, s, _ in net.tensors]
    offs = np.cumsum([0] + sizes)
    g_prev = np.zeros(net.n_params)
    losses = []
    for x, y in batches:
        res = net.train_step(cur, x, y, 0.0, m=m)          # G^t at w^t (no update)
        losses.append(res["losses"])
        flat = np.concatenate([c.ravel() for c in cur]) - lr * g_prev
        cur = [flat[offs[i]:offs[i + 1]].reshape(s) for i, (_, s, _) in enumerate(net.tensors)]
        g_prev = res["grad"]
    return dict(losses=losses, params=np.concatenate([c.ravel() for c in cur]))


def unit_costs(units) -> list:
    """Per-sample MAC cost of each top-level unit (a1; P:366 conv complexity
    O(Co*Ci*T*H*W*Kt*Kh*Kw); light-layer constants BN 2, ReLU/pool/add/mul/
    sigmoid/upsample 1 per output element, GAP 1 per input element, FC in*out,
    softmax 2 per class: SPEC S:87 design decision)."""
    def vol(d):
        return d[0] * d[1] * d[2]

    def block_cost(cin, cout, stride, din):
        do = tuple(conv_out(v, 3, stride, 1) for v in din)
        e = cout * vol(do)
        c = cout * cin * vol(do) * 27 + 2 * e + e + cout * cout * vol(do) * 27 + 2 * e
        if stride != 1 or cin != cout:
            c += cout * cin * vol(do) + 2 * e
        c += e + e      # add + relu
        return c

    out = []
    for u in units:
        if u.kind == "stem":
            d1 = u.extra["conv_dims"]
            e = u.cout * vol(d1)
            c = u.cout * 1 * vol(d1) * 27 + 2 * e + e
            if u.extra["pool"]:
                c += u.cout * vol(u.out_dims)
            out.append(c)
        elif u.kind == "block":
            out.append(block_cost(u.cin, u.cout, u.stride, u.in_dims))
        elif u.kind == "att":
            ch = u.cout
            d, dm = u.in_dims, u.extra["mask_dims"]
            e = ch * vol(d)
            c = block_cost(ch, ch, 1, d)              # trunk
            c += ch * vol(dm)                          # maxpool
            c += block_cost(ch, ch, 1, dm)             # mask residual block
            c += e                                     # upsample
            c += ch * ch * vol(d) + 2 * e + e          # mconv1 + BN + ReLU
            c += ch * ch * vol(d)                      # mconv2
            c += e + e                                 # sigmoid + multiply
            out.append(c)
        elif u.kind == "head":
            out.append(u.cin * vol(u.in_dims) + u.cin * u.cout + 2 * u.cout)
    return out
