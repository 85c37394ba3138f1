"""Per-phase device time of the r18 batch-8 bf16 step (forward / backward / step),
CUDA graphs on, events on the plan stream.  Usage: python tools/phase_time.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dims = (91, 109, 91)
st = torch.cuda.Stream()
plan = rn.Plan(rn.net_desc(18, 64, dims), 8, rn.RN_BF16, stream=st)
arrays = synthetic.init_params(plan.tensors, seed=0)
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(8, *dims, seed=1)
with torch.cuda.stream(st):
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(5):
        plan.forward(xd, yd, want_loss=False)
        plan.backward()
        plan.step(1e-4)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tot = np.zeros(3)
    for _ in range(reps):
        ev[0].record(st)
        plan.forward(xd, yd, want_loss=False)
        ev[1].record(st)
        plan.backward()
        ev[2].record(st)
        plan.step(1e-4)
        ev[3].record(st)
        st.synchronize()
        tot += [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
tot /= reps
print(f"forward {tot[0]:.3f} ms  backward {tot[1]:.3f} ms  step {tot[2]:.3f} ms  total {tot.sum():.3f} ms")
