"""rn_train_step (forward + backward + SGD in one call, each unit's SGD issued on
the weight-gradient stream right after the unit's backward: DESIGN.md "early SGD")
against the three separate calls rn_forward / rn_backward / rn_step: the same
kernels and per-element arithmetic, so every weight, gradient and loss is equal
bit for bit after several steps, with CUDA graphs on (the captured path) and off."""
import numpy as np
import pytest
import torch

import synthetic
from paper_2104_05035_b200 import rn

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("depth,w,dims,dtype,graphs", [
    (18, 64, (40, 48, 40), rn.RN_BF16, 1),
    (18, 64, (40, 48, 40), rn.RN_BF16, 0),
    (0, 8, (16, 16, 16), rn.RN_F32, 1),
])
def test_train_step_equals_separate_calls(depth, w, dims, dtype, graphs):
    desc = rn.net_desc(depth, w, dims)
    tensors = rn.net_params(desc)[0]
    arrays = synthetic.perturb_params(tensors, synthetic.init_params(tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    bs = [synthetic.make_batch(2, *dims, seed=20 + t) for t in range(4)]
    lrs = [1e-3, 1e-3, 5e-4, 5e-4]  # a changed learning rate re-captures the fused phase
    res = []
    for fused in (False, True):
        st = torch.cuda.Stream()
        plan = rn.Plan(desc, 2, dtype, stream=st)
        plan.set_option("graphs", graphs)
        plan.set_params(flat)
        losses = []
        with torch.cuda.stream(st):
            for (x, y), lr in zip(bs, lrs):
                xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
                if fused:
                    losses.append(plan.train_step(xd, yd, lr, want_loss=True))
                else:
                    losses.append(plan.forward(xd, yd))
                    plan.backward()
                    plan.step(lr)
            st.synchronize()
        res.append(dict(losses=losses, w=plan.get_params(), g=plan.get_grads()))
    a, b = res
    assert a["losses"] == b["losses"]
    assert np.array_equal(a["g"], b["g"])
    assert np.array_equal(a["w"], b["w"])
    assert not np.array_equal(a["w"], flat)  # the steps did update


def test_train_step_direct_inputs():
    """rn_train_step called with the SAME device buffers (new batch contents copied
    in each step): from the third call on the fused step runs straight on them —
    its graphs re-captured for those pointers, no staging copy — and must still
    equal the separate calls bit for bit; a different buffer afterwards falls back
    to the staged path (graphs re-captured again)."""
    depth, w, dims, dtype = 18, 64, (40, 48, 40), rn.RN_BF16
    desc = rn.net_desc(depth, w, dims)
    tensors = rn.net_params(desc)[0]
    arrays = synthetic.perturb_params(tensors, synthetic.init_params(tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    bs = [synthetic.make_batch(2, *dims, seed=40 + t) for t in range(6)]
    res = []
    for fused in (False, True):
        st = torch.cuda.Stream()
        plan = rn.Plan(desc, 2, dtype, stream=st)
        plan.set_params(flat)
        losses = []
        with torch.cuda.stream(st):
            xd = torch.empty((2,) + dims, dtype=torch.float32, device="cuda")
            yd = torch.empty((2,), dtype=torch.int32, device="cuda")
            for t, (x, y) in enumerate(bs):
                if t == 5:  # a new buffer: back to the staged path
                    xd = torch.empty((2,) + dims, dtype=torch.float32, device="cuda")
                xd.copy_(torch.from_numpy(x))
                yd.copy_(torch.from_numpy(y))
                if fused:
                    losses.append(plan.train_step(xd, yd, 1e-3, want_loss=True))
                else:
                    losses.append(plan.forward(xd, yd))
                    plan.backward()
                    plan.step(1e-3)
            st.synchronize()
        res.append(dict(losses=losses, w=plan.get_params(), g=plan.get_grads()))
    a, b = res
    assert a["losses"] == b["losses"]
    assert np.array_equal(a["g"], b["g"])
    assert np.array_equal(a["w"], b["w"])
