"""Device time of rn_gradcam after a forward of the r18 bench configuration
(batch 8, 91x109x91): CUDA events on the plan stream.  Usage: python tools/time_gradcam.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

dims, N = (91, 109, 91), 8
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    plan = rn.Plan(rn.net_desc(18, 64, dims), N, rn.RN_BF16, stream=st)
    arrays = synthetic.init_params(plan.tensors, seed=0)
    plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
    x, y = synthetic.make_batch(N, *dims, seed=1)
    plan.forward(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), want_loss=False)
    m = torch.empty((N,) + dims, dtype=torch.float32, device="cuda")
    for _ in range(3):
        plan.gradcam(1, m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    R = 20
    for _ in range(R):
        plan.gradcam(1, m)
    e1.record(st)
    st.synchronize()
us = e0.elapsed_time(e1) * 1000 / R
print(f"rn_gradcam r18 batch 8 -> 8 x 91x109x91 fp32 map: {us:.1f} us per call "
      f"(map write {N * 91 * 109 * 91 * 4 / 1e6:.1f} MB -> {N * 91 * 109 * 91 * 4 / us / 1e3:.0f} GB/s)")
