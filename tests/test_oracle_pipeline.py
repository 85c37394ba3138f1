"""Pins for the oracle's delayed-gradient pipelined training (
PAPER.md:156, Eqs. 1-2; reading F1): CPU only.
* S = 1 reduces to plain SGD ("delay-zero equivalence");
* lr = 0 leaves the weights unchanged;
* S = 2 against an independently written torch float64 emulation of the same
  schedule (explicit autograd graphs kept per in-flight batch, functional weight
  versions: the Jacobian at the forward's weights, the update on the current ones);
* the delay is real: S = 2 differs from plain SGD after the pipeline fills."""
import numpy as np
import torch
import torch.nn.functional as F

import synthetic
from oracle import net as O

DIMS = (16, 16, 16)


def batches(T, N=2, seed0=10):
    return [synthetic.make_batch(N, *DIMS, seed=seed0 + t) for t in range(T)]


def setup():
    net = O.Net(0, 8, DIMS)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    return net, arrays


def test_single_stage_is_plain_sgd():
    net, arrays = setup()
    bs = batches(3)
    res = O.delayed_pipeline_train(net, arrays, bs, 1e-2, [0] * len(net.units))
    cur = [a.astype(np.float64) for a in arrays]
    for t, (x, y) in enumerate(bs):
        r = net.train_step(cur, x, y, 1e-2)
        assert abs(r["loss"] - res["losses"][t]) <= 1e-13 * abs(r["loss"])
        flat = r["new_params"]
        offs = np.cumsum([0] + [int(np.prod(s)) for _, s, _ in net.tensors])
        cur = [flat[offs[i]:offs[i + 1]].reshape(s) for i, (_, s, _) in enumerate(net.tensors)]
    np.testing.assert_allclose(res["params"], np.concatenate([c.ravel() for c in cur]), rtol=1e-12, atol=1e-15)


def test_zero_learning_rate_keeps_weights():
    net, arrays = setup()
    res = O.delayed_pipeline_train(net, arrays, batches(3), 0.0, [0, 0, 1, 1])
    assert np.array_equal(res["params"], np.concatenate([a.astype(np.float64).ravel() for a in arrays]))


def _torch_units(net):
    """Independent torch definition of each top-level unit (NCDHW library ops)."""
    def bn(h, P, name):
        return F.batch_norm(h, None, None, P[name + ".gamma"], P[name + ".beta"], training=True, eps=1e-5)

    def block(h, P, pre, stride):
        o = F.relu(bn(F.conv3d(h, P[pre + ".conv1"], stride=stride, padding=1), P, pre + ".bn1"))
        o = bn(F.conv3d(o, P[pre + ".conv2"], padding=1), P, pre + ".bn2")
        s = bn(F.conv3d(h, P[pre + ".proj"], stride=stride), P, pre + ".projbn") if pre + ".proj" in P else h
        return F.relu(o + s)

    def unit(ui, h, P):
        u, pre = net.units[ui], f"u{ui}"
        if u.kind == "stem":
            h = F.relu(bn(F.conv3d(h, P[pre + ".conv"], stride=u.stride, padding=1), P, pre + ".bn"))
            return F.max_pool3d(h, 3, 2, 1) if u.extra["pool"] else h
        if u.kind == "block":
            return block(h, P, pre, u.stride)
        if u.kind == "att":
            T = block(h, P, pre + ".trunk", 1)
            m = block(F.max_pool3d(h, 3, 2, 1), P, pre + ".mask", 1)
            m = F.interpolate(m, size=T.shape[2:], mode="trilinear", align_corners=False)
            m = F.relu(bn(F.conv3d(m, P[pre + ".mconv1"]), P, pre + ".mbn"))
            m = F.conv3d(m, P[pre + ".mconv2"], P[pre + ".mconv2.bias"])
            return (1 + torch.sigmoid(m)) * T
        return F.linear(h.mean(dim=(2, 3, 4)), P[pre + ".fc.weight"], P[pre + ".fc.bias"])
    return unit


def test_two_stages_vs_torch_emulation():
    net, arrays = setup()
    stage = [0, 0, 1, 1]                       # stem + block | attention + head
    bs = batches(4)
    lr = 1e-2
    res = O.delayed_pipeline_train(net, arrays, bs, lr, stage)
    unit = _torch_units(net)
    names = [n for n, _, _ in net.tensors]
    cur = {n: torch.tensor(a, dtype=torch.float64) for n, a in zip(names, arrays)}
    owner = {n: stage[int(n.split(".")[0][1:])] for n in names}
    graphs = {}                                # batch -> (stage-0 output, stage-0 params used)
    pend = {}
    losses = []
    for t, (x, y) in enumerate(bs):
        P0 = {n: v.clone().requires_grad_(True) for n, v in cur.items() if owner[n] == 0}
        P1 = {n: v.clone().requires_grad_(True) for n, v in cur.items() if owner[n] == 1}
        h = torch.tensor(x, dtype=torch.float64)[:, None]
        for ui in (0, 1):
            h = unit(ui, h, P0)
        graphs[t] = (h, P0)
        a = h.detach().requires_grad_(True)
        z = unit(3, unit(2, a, P1), P1)
        loss = F.cross_entropy(z, torch.tensor(y, dtype=torch.long))
        losses.append(loss.item())
        loss.backward()                        # stage 1: delay 0
        upd = {n: p.grad for n, p in P1.items()}
        pend[t] = a.grad
        if t - 1 >= 0:                         # stage 0: batch t-1, its output gradient from iteration t-1
            h0, P0o = graphs.pop(t - 1)
            h0.backward(pend.pop(t - 1))
            upd.update({n: p.grad for n, p in P0o.items()})
        for n, g in upd.items():
            cur[n] = cur[n] - lr * g
    np.testing.assert_allclose(res["losses"], losses, rtol=1e-10)
    ref = np.concatenate([cur[n].numpy().ravel() for n in names])
    np.testing.assert_allclose(res["params"], ref, rtol=1e-9, atol=1e-12)
    # the delay matters: plain SGD (S = 1) ends elsewhere
    sgd = O.delayed_pipeline_train(net, arrays, bs, lr, [0] * 4)
    assert np.linalg.norm(sgd["params"] - res["params"]) > 1e-6 * np.linalg.norm(res["params"])


def test_async_allreduce_oracle():
    """f4 (reading F4): lr = 0 keeps the weights; the first iteration applies no
    update (G^{-1} = 0); against an independent torch emulation (autograd per
    replica shard, the averaged gradient applied one iteration late)."""
    net, arrays = setup()
    bs = [synthetic.make_batch(4, *DIMS, seed=20 + t) for t in range(3)]
    res0 = O.async_allreduce_train(net, arrays, bs, 0.0, 2)
    assert np.array_equal(res0["params"], np.concatenate([a.astype(np.float64).ravel() for a in arrays]))
    res = O.async_allreduce_train(net, arrays, bs[:1], 1e-2, 2)
    assert np.array_equal(res["params"], res0["params"])            # one iteration: nothing applied yet
    lr = 1e-2
    res = O.async_allreduce_train(net, arrays, bs, lr, 2)
    unit = _torch_units(net)
    names = [n for n, _, _ in net.tensors]
    cur = {n: torch.tensor(a, dtype=torch.float64) for n, a in zip(names, arrays)}
    g_prev = None
    for x, y in bs:
        grads = {n: torch.zeros_like(v) for n, v in cur.items()}
        for r in range(2):
            P = {n: v.clone().requires_grad_(True) for n, v in cur.items()}
            h = torch.tensor(x[2 * r:2 * r + 2], dtype=torch.float64)[:, None]
            for ui in range(len(net.units)):
                h = unit(ui, h, P)
            F.cross_entropy(h, torch.tensor(y[2 * r:2 * r + 2], dtype=torch.long)).backward()
            for n in names:
                grads[n] += P[n].grad / 2
        if g_prev is not None:
            cur = {n: cur[n] - lr * g_prev[n] for n in names}
        g_prev = grads
    ref = np.concatenate([cur[n].numpy().ravel() for n in names])
    np.testing.assert_allclose(res["params"], ref, rtol=1e-9, atol=1e-12)
