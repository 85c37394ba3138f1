"""Tiny steps for compute-sanitizer (initcheck / racecheck / synccheck / memcheck).
Usage: python tools/san_tiny.py <depth> <width> <D> <H> <W> <batch> <micro_batches> <dtype f32|bf16> [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

depth, w, D, H, W, N, Mb = (int(v) for v in sys.argv[1:8])
dt = rn.RN_BF16 if sys.argv[8] == "bf16" else rn.RN_F32
steps = int(sys.argv[9]) if len(sys.argv) > 9 else 2
plan = rn.Plan(rn.net_desc(depth, w, (D, H, W)), N, dt, micro_batches=Mb)
plan.set_option("graphs", 0)
arrays = synthetic.perturb_params(plan.tensors, synthetic.init_params(plan.tensors, seed=0))
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(N, D, H, W, seed=1)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(steps):
    loss = plan.forward(xd, yd)
    plan.backward()
    plan.step(1e-4)
torch.cuda.synchronize()
print("loss", loss)
