"""GPU parity: librn.so (through the C ABI) against the float64 oracle on the
same seeded inputs and weights.  Tolerances:
* RN_F32: per-tensor relative L2 error <= 1e-4 for loss, every gradient tensor
  and the BN running statistics; the update dw = w' - w within 1e-4 relative
  plus the fp32 rounding bound of storing w' (ulp(w')/2 per element).
* RN_BF16: the same quantities within 2e-2 relative (north_star)."""
import numpy as np
import pytest
import torch

import synthetic
from oracle import net as O
from paper_2104_05035_b200 import rn

pytestmark = pytest.mark.gpu

LR = 1e-4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def run_both(depth, w, dims, N, dtype, perturb=True, Mb=1, seed=1):
    desc = rn.net_desc(depth, w, dims)
    net = O.Net(depth, w, dims)
    plan = rn.Plan(desc, N, dtype, micro_batches=Mb)
    assert [t[0] for t in plan.tensors] == [t[0] for t in net.tensors]
    arrays = synthetic.init_params(net.tensors, seed=0)
    if perturb:
        arrays = synthetic.perturb_params(net.tensors, arrays)
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    plan.set_params(flat)
    x, y = synthetic.make_batch(N, *dims, seed=seed)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    loss = plan.forward(xd, yd)
    plan.backward()
    g = plan.get_grads()
    plan.step(LR)
    w1 = plan.get_params()
    rm, rv = plan.get_bn_running()
    ref = net.train_step(arrays, x, y, LR, m=1, Mb=Mb)
    return dict(net=net, flat=flat, loss=loss, g=g, w1=w1, rm=rm, rv=rv, ref=ref, plan=plan)


def check(res, tol, check_running=True):
    net, ref = res["net"], res["ref"]
    assert abs(res["loss"] - ref["loss"]) <= tol * abs(ref["loss"]), (res["loss"], ref["loss"])
    off = 0
    worst = []
    for name, shape, kind in net.tensors:
        n = int(np.prod(shape))
        e = rel(res["g"][off:off + n], ref["grad"][off:off + n])
        worst.append((e, name))
        off += n
    worst.sort(reverse=True)
    assert worst[0][0] <= tol, worst[:5]
    # update: dw = w' - w (exact in float64), bound = tol*|dw_ref| + ulp(w')/2
    dw = res["w1"].astype(np.float64) - res["flat"].astype(np.float64)
    ulp = np.spacing(np.abs(res["w1"]).astype(np.float32)).astype(np.float64)
    err = np.linalg.norm(dw - ref["delta"])
    assert err <= tol * np.linalg.norm(ref["delta"]) + np.linalg.norm(ulp / 2), (err, np.linalg.norm(ref["delta"]))
    if check_running:
        st = ref["bn_state"]
        m_ref = np.concatenate([st.mean[n] for n in net.bn_names])
        v_ref = np.concatenate([st.var[n] for n in net.bn_names])
        assert rel(res["rm"], m_ref) <= tol
        assert rel(res["rv"], v_ref) <= tol
    return worst


def test_tiny_f32_parity():
    """configs[0]: tiny 3D-ResAttNet, 2 x 1 x 16^3, one fp32 step."""
    res = run_both(0, 8, (16, 16, 16), 2, rn.RN_F32)
    check(res, 1e-4)


def test_tiny_f32_parity_ragged_microbatches():
    """odd volume (ragged tiles, odd upsampling 8->15 etc.), 3 micro-batches of 1."""
    res = run_both(0, 8, (15, 13, 11), 3, rn.RN_F32, Mb=3)
    check(res, 1e-4)


def test_r18_small_volume_f32_parity():
    """r18 structure (all stages, projections, 3 attention modules) on a small volume."""
    res = run_both(18, 8, (24, 28, 20), 2, rn.RN_F32)
    check(res, 1e-4)


def test_r18_small_volume_bf16_parity():
    res = run_both(18, 16, (32, 36, 30), 2, rn.RN_BF16)
    check(res, 2e-2)


def test_tiny_bf16_parity():
    res = run_both(0, 8, (16, 16, 16), 2, rn.RN_BF16)
    check(res, 2e-2)


def test_gpu_deterministic():
    a = run_both(0, 8, (16, 16, 16), 2, rn.RN_F32)
    b = run_both(0, 8, (16, 16, 16), 2, rn.RN_F32)
    assert np.array_equal(a["g"], b["g"]) and a["loss"] == b["loss"]
