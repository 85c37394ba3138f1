"""Whole-step pins for the oracle (CPU only):
* PyTorch CPU float64 autograd of an independently written 3D-ResAttNet
  (library routine; shares nothing with oracle/net.py beyond the parameter
  order contract) — loss, every gradient, running statistics;
* the data-parallel objective Eq. 9 with per-replica BN (reading X9) and the
  micro-batch mean (X18) through autograd;
* central finite differences of the oracle's own loss;
* parameter counts and unit costs hand-derived in DESIGN.md."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthetic
from oracle import net as O


def torch_resattnet_loss(net, arrays, x, y, running=None):
    """Independent torch definition of the network (NCDHW, library ops)."""
    P = {n: torch.tensor(a, dtype=torch.float64, requires_grad=True) for (n, _, _), a in zip(net.tensors, arrays)}

    def bn(h, name):
        rm = torch.zeros(h.shape[1], dtype=torch.float64)
        rv = torch.ones(h.shape[1], dtype=torch.float64)
        out = F.batch_norm(h, rm, rv, P[name + ".gamma"], P[name + ".beta"], training=True, momentum=0.1, eps=1e-5)
        if running is not None:
            running[name] = (rm, rv)
        return out

    def block(h, pre, stride):
        o = F.relu(bn(F.conv3d(h, P[pre + ".conv1"], stride=stride, padding=1), pre + ".bn1"))
        o = bn(F.conv3d(o, P[pre + ".conv2"], padding=1), pre + ".bn2")
        if pre + ".proj" in P:
            s = bn(F.conv3d(h, P[pre + ".proj"], stride=stride), pre + ".projbn")
        else:
            s = h
        return F.relu(o + s)

    h = torch.tensor(x, dtype=torch.float64)[:, None]
    for ui, u in enumerate(net.units):
        pre = f"u{ui}"
        if u.kind == "stem":
            h = F.relu(bn(F.conv3d(h, P[pre + ".conv"], stride=u.stride, padding=1), pre + ".bn"))
            if u.extra["pool"]:
                h = F.max_pool3d(h, 3, 2, 1)
        elif u.kind == "block":
            h = block(h, pre, u.stride)
        elif u.kind == "att":
            T = block(h, pre + ".trunk", 1)
            mm = block(F.max_pool3d(h, 3, 2, 1), pre + ".mask", 1)
            mm = F.interpolate(mm, size=T.shape[2:], mode="trilinear", align_corners=False)
            mm = F.relu(bn(F.conv3d(mm, P[pre + ".mconv1"]), pre + ".mbn"))
            mm = F.conv3d(mm, P[pre + ".mconv2"], P[pre + ".mconv2.bias"])
            h = (1 + torch.sigmoid(mm)) * T
        else:
            g = h.mean(dim=(2, 3, 4))
            h = F.linear(g, P[pre + ".fc.weight"], P[pre + ".fc.bias"])
    loss = F.cross_entropy(h, torch.tensor(y, dtype=torch.long))
    return loss, P


def test_param_counts_and_costs():
    # hand derivations in DESIGN.md §"Network": tiny 10 866, r18 42 607 490, r34 72 917 122
    assert O.Net(0, 8, (16, 16, 16)).n_params == 10866
    assert O.Net(18, 64, (91, 109, 91)).n_params == 42607490
    assert O.Net(34, 64, (91, 109, 91)).n_params == 72917122
    tiny = O.Net(0, 8, (16, 16, 16))
    # stem: conv 8*1*16^3*27 = 884736, BN 2*32768, ReLU 32768 (per sample)
    assert O.unit_costs(tiny.units) == [983040, 14385152, 16908288, 32788]
    r18 = O.Net(18, 64, (91, 109, 91))
    assert [u.out_dims for u in r18.units][:1] == [(23, 28, 23)]
    assert r18.units[-1].in_dims == (3, 4, 3)
    assert sum(O.unit_costs(r18.units)) == 19385019908


@pytest.mark.parametrize("perturb", [False, True])
def test_tiny_step_vs_torch_autograd(perturb):
    net = O.Net(0, 8, (16, 16, 16))
    arrays = synthetic.init_params(net.tensors, seed=0)
    if perturb:
        arrays = synthetic.perturb_params(net.tensors, arrays)
    x, y = synthetic.make_batch(2, 16, 16, 16, seed=1)
    res = net.train_step(arrays, x, y, lr=1e-4)
    running = {}
    loss_t, P = torch_resattnet_loss(net, arrays, x, y, running)
    loss_t.backward()
    assert abs(res["loss"] - loss_t.item()) < 1e-12 * abs(loss_t.item())
    gt = np.concatenate([P[n].grad.numpy().ravel() for n, _, _ in net.tensors])
    np.testing.assert_allclose(res["grad"], gt, rtol=1e-9, atol=1e-12 * np.abs(gt).max())
    np.testing.assert_allclose(res["delta"], -1e-4 * gt, rtol=1e-9, atol=1e-16)
    st = res["bn_state"]
    for name in net.bn_names:
        np.testing.assert_allclose(st.mean[name], running[name][0].numpy(), rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(st.var[name], running[name][1].numpy(), rtol=1e-10)


def test_data_parallel_objective_eq9():
    """m=2 replicas x Mb=2 micro-batches: G must be the gradient of
    (1/(m*Mb)) sum_(r,k) mean-loss_(r,k) with BN per (r,k) — Eq. 9-11 + X9/X18."""
    net = O.Net(0, 8, (16, 16, 16))
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(8, 16, 16, 16, seed=3)
    res = net.train_step(arrays, x, y, lr=1e-4, m=2, Mb=2)
    tot = None
    grads = None
    for k in range(4):
        sl = slice(2 * k, 2 * k + 2)
        lt, P = torch_resattnet_loss(net, arrays, x[sl], y[sl])
        lt.backward()
        g = np.concatenate([P[n].grad.numpy().ravel() for n, _, _ in net.tensors])
        grads = g if grads is None else grads + g
        tot = lt.item() if tot is None else tot + lt.item()
    np.testing.assert_allclose(res["grad"], grads / 4, rtol=1e-9, atol=1e-13)
    assert abs(res["loss"] - tot / 4) < 1e-12


def test_finite_differences_tiny():
    net = O.Net(0, 8, (8, 8, 8))
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(2, 8, 8, 8, seed=1)
    P = O.Params(net.tensors, arrays)
    _, G, _ = net.forward_backward(P, x, y)
    g = net.flat(G)
    flat = np.concatenate([a.astype(np.float64).ravel() for a in arrays])
    sizes = [int(np.prod(s)) for _, s, _ in net.tensors]
    offs = np.cumsum([0] + sizes)

    def loss_at(v):
        arr = [v[offs[i]:offs[i + 1]].reshape(s) for i, (_, s, _) in enumerate(net.tensors)]
        loss, _, _ = net.forward_backward(O.Params(net.tensors, arr), x, y)
        return loss

    r = np.random.default_rng(5)
    idx = r.choice(flat.size, 120, replace=False)
    eps = 1e-6
    ok = 0
    checked = 0
    for i in idx:
        vp, vm = flat.copy(), flat.copy()
        vp[i] += eps
        vm[i] -= eps
        l0, lp, lm = loss_at(flat), loss_at(vp), loss_at(vm)
        fwd, bwd = (lp - l0) / eps, (l0 - lm) / eps
        if abs(fwd - bwd) > 1e-3 * max(abs(fwd), abs(bwd), 1e-6):
            continue                                      # kink (ReLU/max) — excluded per SPEC S:365-373
        fd = (lp - lm) / (2 * eps)
        checked += 1
        if abs(fd - g[i]) <= 1e-5 * max(abs(fd), 1e-3):
            ok += 1
    assert checked >= 100
    assert ok >= 0.99 * checked


def test_bf16_storage_gap():
    """Evidence for reading X23: rounding the stored activations/gradients to
    bf16 (what any bf16 tensor-core path does) moves the early-layer gradients of
    this network far more than 2e-2 from the float64 definition, while the loss
    moves by < 1e-3.  Hence the bf16 gradient parity is checked against the
    bf16-storage oracle (tests/test_gpu_parity.py::test_bf16_step)."""
    net64 = O.Net(0, 8, (16, 16, 16))
    net16 = O.Net(0, 8, (16, 16, 16), store="bf16")
    arrays = synthetic.perturb_params(net64.tensors, synthetic.init_params(net64.tensors, seed=0))
    x, y = synthetic.make_batch(2, 16, 16, 16, seed=1)
    a = net64.train_step(arrays, x, y, 1e-4)
    b = net16.train_step(arrays, x, y, 1e-4)
    assert abs(a["loss"] - b["loss"]) < 1e-3 * a["loss"]
    gap = np.linalg.norm(a["grad"] - b["grad"]) / np.linalg.norm(a["grad"])
    assert gap > 2e-2
    # the rounding itself: bf16 RNE of fp32 (pins the helper against torch's cast)
    v = np.random.default_rng(0).standard_normal(1000) * 100
    t = torch.tensor(v, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(O._bf16_round(v), t)


@pytest.mark.parametrize("depth", [18, 34])
def test_deep_step_vs_torch_autograd(depth):
    """Pins the r18 / r34 COMPOSITION of the oracle: stride-2
    stage-entry blocks with the 1x1x1 projection branch (block_backward's dz ->
    projection BN backward -> dxp path), the stem max-pool and its adjoint, three
    attention modules at three resolutions, and r34's 3/4/6/3 block counts —
    against the independently written torch float64 autograd model.  Width 4 and a
    40x48x40 volume keep it CPU-cheap while every stage keeps >= 2x2x2 voxels."""
    dims = (40, 48, 40)
    net = O.Net(depth, 4, dims)
    kinds = [u.kind for u in net.units]
    assert kinds.count("att") == 3 and sum(1 for u in net.units if u.kind == "block" and u.stride == 2) == 3
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(2, *dims, seed=1)
    res = net.train_step(arrays, x, y, lr=1e-4)
    running = {}
    loss_t, P = torch_resattnet_loss(net, arrays, x, y, running)
    loss_t.backward()
    assert abs(res["loss"] - loss_t.item()) < 1e-11 * abs(loss_t.item())
    off = 0
    for name, shape, _ in net.tensors:
        n = int(np.prod(shape))
        gt = P[name].grad.numpy().ravel()
        np.testing.assert_allclose(res["grad"][off:off + n], gt, rtol=1e-7, atol=1e-9 * np.abs(gt).max() + 1e-300,
                                   err_msg=name)
        off += n
    st = res["bn_state"]
    for name in net.bn_names:
        np.testing.assert_allclose(st.mean[name], running[name][0].numpy(), rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(st.var[name], running[name][1].numpy(), rtol=1e-9)


def test_deep_finite_differences_proj_and_stem():
    """Central finite differences of the r18 oracle's own loss at coordinates of
    the stem conv (pool adjoint on the path), a stage-entry projection conv and its
    BN, and the stage-3 attention mask conv — the branches only the deep network
    has (SPEC S:365-373 kink rule)."""
    dims = (24, 28, 24)
    net = O.Net(18, 4, dims)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(2, *dims, seed=1)
    _, G, _ = net.forward_backward(O.Params(net.tensors, arrays), x, y)
    names = [t[0] for t in net.tensors]
    r = np.random.default_rng(11)
    checked = ok = 0
    for tname in ("u0.conv", "u4.proj", "u4.projbn.gamma", "u7.proj", "u9.mconv1"):
        ti = names.index(tname)
        for _ in range(6):
            j = int(r.integers(arrays[ti].size))
            vals = []
            for e in (1e-6, 0.0, -1e-6):
                arr = [a.copy() for a in arrays]
                arr[ti] = arr[ti].astype(np.float64)
                arr[ti].reshape(-1)[j] += e
                vals.append(net.forward_backward(O.Params(net.tensors, arr), x, y)[0])
            lp, l0, lm = vals
            fwd, bwd = (lp - l0) / 1e-6, (l0 - lm) / 1e-6
            if abs(fwd - bwd) > 1e-3 * max(abs(fwd), abs(bwd), 1e-6):
                continue
            fd = (lp - lm) / 2e-6
            g = np.asarray(G[tname]).reshape(-1)[j]
            checked += 1
            ok += abs(fd - g) <= 1e-5 * max(abs(fd), 1e-3)
    assert checked >= 15 and ok >= checked - 1, (checked, ok)


def test_unit_step_composes_to_whole_step():
    """Net.unit_step (teacher-forced single unit, used by the per-unit GPU parity
    test) chained over all units with the oracle's own outputs reproduces
    forward_backward exactly (r18 composition, both storage modes)."""
    dims = (24, 28, 24)
    for store in ("f64", "bf16"):
        net = O.Net(18, 4, dims, store=store)
        arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
        x, y = synthetic.make_batch(2, *dims, seed=1)
        P = O.Params(net.tensors, arrays)
        loss, Gw, _ = net.forward_backward(P, x, y)
        outs, h = [], x
        for ui in range(len(net.units)):
            r = net.unit_step(P, ui, h, None, y)
            outs.append(r)
            h = r["out"]
        assert outs[-1]["loss"] == loss
        g = None
        G = {}
        for ui in reversed(range(len(net.units))):
            xin = x if ui == 0 else outs[ui - 1]["out"]
            r = net.unit_step(P, ui, xin, g, y)
            G.update(r["G"])
            g = r["dx"]
        for n, _, _ in net.tensors:
            assert np.array_equal(np.asarray(G[n]), np.asarray(Gw[n])), n
