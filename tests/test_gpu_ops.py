"""Op-level teacher-forced parity of the RN_BF16 step.

Every operation of the step is checked ELEMENT BY ELEMENT on the GPU's own inputs:
the step runs once on the GPU, every tensor it keeps is read back (rn_get_saved /
rn_get_activation / rn_get_unit_grad / rn_get_grads), and each op's GPU output is
compared with the oracle's primitive (oracle/net.py: conv3d, conv3d_backward,
bn_forward, bn_backward, maxpool3(_backward), upsample_trilinear(_backward),
sigmoid, softmax_ce) applied in float64 to the GPU's inputs of that op.  So the
comparison carries ONE op's arithmetic difference (fp32 accumulation order and
one bf16 rounding of the stored result), never the bf16 chaos of a chain of BN
layers (reading X23), and a tight element-wise bound applies everywhere:

  bf16-stored tensors : |a - b| <= 2^-7 |b| + 2^-9 max|b|   (<= 2 bf16 ulps, plus
                         fp32 cancellation headroom relative to the tensor's scale)
  fp32 weight / BN-parameter gradients, BN statistics:
                        |a - b| <= 1e-3 |b| + 1e-4 max|b|  and rel-L2 <= 1e-4
  max-pool argmax     : bit-exact (first maximum, reading X10)

Each row reports rel-L2 and the worst element's bound ratio; the table is printed
(pytest -s) and written to gpurun_out/ when that directory exists.  Op order and
formulas: P:364 (blocks, attention module), P:156 (chain rule), P:486 (CE, SGD);
readings X6-X12 in DESIGN.md."""
import os

import numpy as np
import pytest
import torch

import synthetic
from oracle import net as O

from paper_2104_05035_b200 import rn

pytestmark = pytest.mark.gpu

Qb = O._bf16_round          # the rounding the GPU applies when it stores bf16
BF16 = (2.0 ** -7, 2.0 ** -9)
F32 = (1e-3, 1e-4)


class Table:
    def __init__(self):
        self.rows = []

    def chk(self, unit, name, got, ref, kind="bf16"):
        got = np.asarray(got, dtype=np.float64).reshape(-1)
        ref = np.asarray(ref, dtype=np.float64).reshape(-1)
        assert got.shape == ref.shape, (unit, name, got.shape, ref.shape)
        d = np.abs(got - ref)
        r = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
        if kind == "exact":
            ratio = float(np.count_nonzero(d))        # number of mismatches (must be 0)
            ok = ratio == 0
        else:
            rt, at = BF16 if kind == "bf16" else F32
            bound = rt * np.abs(ref) + at * max(np.abs(ref).max(), 1e-30)
            ratio = float((d / bound).max())
            ok = ratio <= 1.0 and (kind == "bf16" or r <= 1e-4)
        self.rows.append((unit, name, kind, r, ratio, ok))

    def report(self, tag):
        lines = [f"{'unit':>4}  {'tensor':<28} {'kind':<5} {'rel-L2':>9} {'ratio':>8}"]
        for u, n, k, r, q, ok in self.rows:
            lines.append(f"{u:>4}  {n:<28} {k:<5} {r:9.2e} {q:8.3f}{'' if ok else '  <-- FAIL'}")
        bad = [x for x in self.rows if not x[5]]
        lines.append(f"{len(self.rows)} tensors, {len(bad)} over; worst bf16 ratio "
                     f"{max([x[4] for x in self.rows if x[2] == 'bf16'] or [0]):.3f}, worst f32 ratio "
                     f"{max([x[4] for x in self.rows if x[2] == 'f32'] or [0]):.3f}")
        txt = "\n".join(lines)
        print(txt)
        if os.path.isdir("gpurun_out"):
            with open(f"gpurun_out/op_parity_{tag}.txt", "w") as f:
                f.write(txt + "\n")
        return bad, txt


def bn_ref(h, gamma, beta):
    """oracle bn_forward on h + the [4][C] statistics rn_get_saved reports."""
    y, c = O.bn_forward(h, gamma, beta)
    scale = gamma * c["invstd"]
    return y, c, np.stack([c["mu"], c["invstd"], scale, beta - c["mu"] * scale])


def check_block(T, plan, P, ui, pre, sname, x, dout, G, k_gpu, stride, dx_acc=None):
    """One residual block on the GPU's tensors.  sname: rn_get_saved prefix.
    Returns the reference dx (before comparing it, the caller decides where the GPU
    stored it)."""
    shp = dout.shape
    C = shp[-1]
    get = lambda n, s=shp: plan.get_saved(ui, sname + n, s).astype(np.float64)
    W = lambda n: O._bf16_round(P[pre + n])                       # the bf16 copies the kernels read
    h1, a1, h2, out = get("h1"), get("a1"), get("h2"), get("out")
    proj = (pre + ".proj") in P.d
    # forward
    T.chk(ui, sname + "h1", h1, Qb(O.conv3d(x, W(".conv1"), stride, 1)))
    y1, c1, st1 = bn_ref(h1, P[pre + ".bn1.gamma"], P[pre + ".bn1.beta"])
    T.chk(ui, sname + "bn1.stats", get("bn1.stats", (4, C)), st1, "f32")
    T.chk(ui, sname + "a1", a1, Qb(O.relu(y1)))
    T.chk(ui, sname + "h2", h2, Qb(O.conv3d(a1, W(".conv2"), 1, 1)))
    y2, c2, st2 = bn_ref(h2, P[pre + ".bn2.gamma"], P[pre + ".bn2.beta"])
    T.chk(ui, sname + "bn2.stats", get("bn2.stats", (4, C)), st2, "f32")
    if proj:
        hp = get("hp")
        T.chk(ui, sname + "hp", hp, Qb(O.conv3d(x, W(".proj"), stride, 0)))
        yp, cp, stp = bn_ref(hp, P[pre + ".projbn.gamma"], P[pre + ".projbn.beta"])
        T.chk(ui, sname + "projbn.stats", get("projbn.stats", (4, C)), stp, "f32")
        skip = yp
    else:
        skip = x
    T.chk(ui, sname + "out", out, Qb(O.relu(y2 + skip)))
    # backward, every op from the GPU's own inputs
    dz = dout * (out > 0)
    dh2_ref, dg2, db2 = O.bn_backward(dz, c2, P[pre + ".bn2.gamma"])
    dh2 = get("dh2")
    T.chk(ui, sname + "dh2", dh2, Qb(dh2_ref))
    T.chk(ui, pre + ".bn2.gamma", G(pre + ".bn2.gamma"), dg2, "f32")
    T.chk(ui, pre + ".bn2.beta", G(pre + ".bn2.beta"), db2, "f32")
    da1_ref, dW2 = O.conv3d_backward(a1, W(".conv2"), dh2, 1, 1)
    T.chk(ui, pre + ".conv2", G(pre + ".conv2"), dW2, "f32")
    da1 = get("da1")
    T.chk(ui, sname + "da1", da1, Qb(da1_ref))
    dh1_ref, dg1, db1 = O.bn_backward(da1 * (a1 > 0), c1, P[pre + ".bn1.gamma"])
    dh1 = get("dh1")
    T.chk(ui, sname + "dh1", dh1, Qb(dh1_ref))
    T.chk(ui, pre + ".bn1.gamma", G(pre + ".bn1.gamma"), dg1, "f32")
    T.chk(ui, pre + ".bn1.beta", G(pre + ".bn1.beta"), db1, "f32")
    dx1, dW1 = O.conv3d_backward(x, W(".conv1"), dh1, stride, 1)
    T.chk(ui, pre + ".conv1", G(pre + ".conv1"), dW1, "f32")
    if proj:
        dhp_ref, dgp, dbp = O.bn_backward(dz, cp, P[pre + ".projbn.gamma"])
        dhp = get("dhp")
        T.chk(ui, sname + "dhp", dhp, Qb(dhp_ref))
        T.chk(ui, pre + ".projbn.gamma", G(pre + ".projbn.gamma"), dgp, "f32")
        T.chk(ui, pre + ".projbn.beta", G(pre + ".projbn.beta"), dbp, "f32")
        dxp, dWp = O.conv3d_backward(x, W(".proj"), dhp, stride, 0)
        T.chk(ui, pre + ".proj", G(pre + ".proj"), dWp, "f32")
        return Qb(dx1 + dxp)
    acc = 0.0 if dx_acc is None else dx_acc
    return Qb(acc + dx1 + dz)


def op_parity(depth, w, dims, N):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan = rn.Plan(rn.net_desc(depth, w, dims), N, rn.RN_BF16, stream=st)
        arrays = synthetic.perturb_params(plan.tensors, synthetic.init_params(plan.tensors, seed=0))
        flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
        plan.set_params(flat)
        x, y = synthetic.make_batch(N, *dims, seed=1)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        loss = plan.forward(xd, yd)
        plan.backward()
        g_gpu = plan.get_grads().astype(np.float64)
        st.synchronize()
    net = O.Net(depth, w, dims)
    P = O.Params(net.tensors, arrays)
    offs, o = {}, 0
    for name, shape, _ in net.tensors:
        n = int(np.prod(shape))
        offs[name] = (o, shape)
        o += n
    G = lambda n: g_gpu[offs[n][0]:offs[n][0] + int(np.prod(offs[n][1]))].reshape(offs[n][1])
    T = Table()
    units = net.units
    acts, douts = [], []
    for ui, u in enumerate(units):
        if u.kind == "head":
            acts.append(plan.get_activation(ui, 0, (N, u.cin)).astype(np.float64))
            douts.append(None)
        else:
            shp = (N,) + tuple(u.out_dims) + (u.cout,)
            acts.append(plan.get_activation(ui, 0, shp).astype(np.float64))
            douts.append(plan.get_unit_grad(ui, shp).astype(np.float64))
    for ui, u in enumerate(units):
        pre = f"u{ui}"
        xin = x.astype(np.float64)[..., None] if ui == 0 else acts[ui - 1].astype(np.float64)
        dx_gpu = douts[ui - 1] if ui > 0 else None
        if u.kind == "stem":
            cd = tuple(u.extra["conv_dims"])
            C = u.cout
            h = plan.get_saved(ui, "h", (N,) + cd + (C,)).astype(np.float64)
            T.chk(ui, "h", h, Qb(O.conv3d(xin, P[pre + ".conv"], u.stride, 1)))   # fp32 master weights
            yb, cb, stb = bn_ref(h, P[pre + ".bn.gamma"], P[pre + ".bn.beta"])
            T.chk(ui, "bn.stats", plan.get_saved(ui, "bn.stats", (4, C)), stb, "f32")
            a = O.relu(yb)
            if u.extra["pool"]:
                pooled, am = O.maxpool3(a)
                T.chk(ui, "out", acts[ui], Qb(pooled))
                am_gpu = plan.get_saved(ui, "am", acts[ui].shape)
                T.chk(ui, "am", am_gpu, am, "exact")
            else:
                T.chk(ui, "out", acts[ui], Qb(a))
            if u.extra["pool"] and C in O.STEM_POOLED_BWD_WIDTHS:
                # reading X23c: pooled-resolution backward, nothing rounded at the conv
                # resolution, the h-term of dh with the conv's unrounded output
                dy = O.maxpool3_backward(douts[ui], am_gpu.astype(np.int64), a.shape) * (a > 0)
                h_raw = O.conv3d(xin, P[pre + ".conv"], u.stride, 1)
                A, B, Cc, dgb, dbb = O.bn_backward_coefs(dy, cb, P[pre + ".bn.gamma"], h=h_raw)
                dh = A * dy + B * h_raw + Cc
            else:
                if u.extra["pool"]:
                    d1 = plan.get_saved(ui, "d1", (N,) + cd + (C,)).astype(np.float64)
                    T.chk(ui, "d1 (pool adjoint*mask)", d1,
                          Qb(O.maxpool3_backward(douts[ui], am_gpu.astype(np.int64), a.shape)) * (a > 0))
                    dy = d1
                else:
                    dy = douts[ui] * (acts[ui] > 0)
                dh, dgb, dbb = O.bn_backward(dy, cb, P[pre + ".bn.gamma"])
                dh = Qb(dh)
            T.chk(ui, pre + ".bn.gamma", G(pre + ".bn.gamma"), dgb, "f32")
            T.chk(ui, pre + ".bn.beta", G(pre + ".bn.beta"), dbb, "f32")
            _, dW = O.conv3d_backward(xin, P[pre + ".conv"], dh, u.stride, 1, need_dx=False)
            T.chk(ui, pre + ".conv", G(pre + ".conv"), dW, "f32")
        elif u.kind == "block":
            ref_dx = check_block(T, plan, P, ui, pre, "", xin, douts[ui].astype(np.float64), G, 0, u.stride)
            T.chk(ui, "dx", dx_gpu, ref_dx)
        elif u.kind == "att":
            C = u.cout
            shp = (N,) + tuple(u.out_dims) + (C,)
            mshp = (N,) + tuple(u.extra["mask_dims"]) + (C,)
            W = lambda n: O._bf16_round(P[pre + n])
            g = lambda n, s=shp: plan.get_saved(ui, n, s).astype(np.float64)
            u0, am = g("u0", mshp), plan.get_saved(ui, "am", mshp)
            u0_ref, am_ref = O.maxpool3(xin)
            T.chk(ui, "u0", u0, u0_ref, "exact")
            T.chk(ui, "am", am, am_ref, "exact")
            mout = g("mask.out", mshp)
            up = g("up")
            T.chk(ui, "up", up, Qb(O.upsample_trilinear(mout, tuple(u.out_dims))))
            mh = g("mh")
            T.chk(ui, "mh", mh, Qb(O.conv3d(up, W(".mconv1"), 1, 0)))
            ym, cm, stm = bn_ref(mh, P[pre + ".mbn.gamma"], P[pre + ".mbn.beta"])
            T.chk(ui, "mbn.stats", plan.get_saved(ui, "mbn.stats", (4, C)), stm, "f32")
            r = g("r")
            T.chk(ui, "r", r, Qb(O.relu(ym)))
            m = g("m")
            T.chk(ui, "m", m, Qb(O.conv3d(r, W(".mconv2"), 1, 0) + P[pre + ".mconv2.bias"]))
            Tt = g("trunk.out")
            sg = O.sigmoid(m)
            T.chk(ui, "out", acts[ui], Qb((1.0 + sg) * Tt))
            # backward
            dout = douts[ui].astype(np.float64)
            dT = g("dT")
            T.chk(ui, "dT", dT, Qb(dout * (1.0 + sg)))
            dm_raw = dout * Tt * sg * (1.0 - sg)
            T.chk(ui, pre + ".mconv2.bias", G(pre + ".mconv2.bias"), dm_raw.sum(axis=(0, 1, 2, 3)), "f32")
            dm = g("dm")
            T.chk(ui, "dm", dm, Qb(dm_raw))
            dr_ref, dWm2 = O.conv3d_backward(r, W(".mconv2"), dm, 1, 0)
            T.chk(ui, pre + ".mconv2", G(pre + ".mconv2"), dWm2, "f32")
            dr = g("dr")
            T.chk(ui, "dr", dr, Qb(dr_ref))
            dmh_ref, dgm, dbm = O.bn_backward(dr * (r > 0), cm, P[pre + ".mbn.gamma"])
            T.chk(ui, pre + ".mbn.gamma", G(pre + ".mbn.gamma"), dgm, "f32")
            T.chk(ui, pre + ".mbn.beta", G(pre + ".mbn.beta"), dbm, "f32")
            dmh = g("dmh")
            T.chk(ui, "dmh", dmh, Qb(dmh_ref))
            dup_ref, dWm1 = O.conv3d_backward(up, W(".mconv1"), dmh, 1, 0)
            T.chk(ui, pre + ".mconv1", G(pre + ".mconv1"), dWm1, "f32")
            dup = g("dup")
            T.chk(ui, "dup", dup, Qb(dup_ref))
            dum = g("dum", mshp)
            T.chk(ui, "dum", dum, Qb(O.upsample_trilinear_backward(dup, tuple(u.extra["mask_dims"]))))
            du0_ref = check_block(T, plan, P, ui, pre + ".mask", "mask.", u0, dum, G, 0, 1)
            du0 = g("du0", mshp)
            T.chk(ui, "du0", du0, du0_ref)
            dx_mask = Qb(O.maxpool3_backward(du0, am.astype(np.int64), xin.shape))
            ref_dx = check_block(T, plan, P, ui, pre + ".trunk", "trunk.", xin, dT, G, 0, 1, dx_acc=dx_mask)
            T.chk(ui, "dx", dx_gpu, ref_dx)
        else:  # head: GAP + FC + softmax-CE
            gvec = xin.mean(axis=(1, 2, 3))
            T.chk(ui, "gap", acts[ui], gvec, "f32")
            gg = acts[ui].astype(np.float64)
            z = gg @ P[pre + ".fc.weight"].T + P[pre + ".fc.bias"]
            l_ref, dz = O.softmax_ce(z, y)
            T.chk(ui, "loss", np.array([loss]), np.array([l_ref]), "f32")
            T.chk(ui, "dz", plan.get_saved(ui, "dz", (N, 2)), dz, "f32")
            T.chk(ui, pre + ".fc.weight", G(pre + ".fc.weight"), dz.T @ gg, "f32")
            T.chk(ui, pre + ".fc.bias", G(pre + ".fc.bias"), dz.sum(axis=0), "f32")
            V = int(np.prod(u.in_dims))
            T.chk(ui, "dx", dx_gpu, Qb(np.broadcast_to((dz @ P[pre + ".fc.weight"])[:, None, None, None, :] / V,
                                                      xin.shape)))
    return T


@pytest.mark.parametrize("depth,w,dims,N,tag", [
    (0, 24, (16, 16, 16), 2, "tiny_w24"),           # SIMT convs, C = 24 (channel groups of 3)
    (18, 64, (40, 48, 40), 2, "r18_small"),
    (18, 64, (91, 109, 91), 8, "bench"),           # bench.py's configuration (BASELINE configs[1])
])
def test_bf16_op_parity(depth, w, dims, N, tag):
    T = op_parity(depth, w, dims, N)
    bad, txt = T.report(tag)
    assert not bad, "\n" + txt
