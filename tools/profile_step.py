"""Run a few r18 bf16 training steps through librn (for ncu launch lists).
Usage: python tools/profile_step.py [steps] [batch]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (91, 109, 91)
desc = rn.net_desc(18, 64, dims)
plan = rn.Plan(desc, batch, rn.RN_BF16)
arrays = synthetic.init_params(plan.tensors, seed=0)
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(batch, *dims, seed=1)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(steps):
    plan.forward(xd, yd, want_loss=False)
    plan.backward()
    plan.step(1e-4)
torch.cuda.synchronize()
print("launches", rn.kernel_launches())
