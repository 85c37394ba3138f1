import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synthetic
from paper_2104_05035_b200 import rn
dims, N = (91, 109, 91), 8
for side in (1, 0, 1, 0):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan = rn.Plan(rn.net_desc(18, 64, dims), N, rn.RN_BF16, stream=st)
        plan.set_option("wgrad_stream", side)
        arrays = synthetic.init_params(plan.tensors, seed=0)
        plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
        x, y = synthetic.make_batch(N, *dims, seed=1)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        def step():
            plan.forward(xd, yd, want_loss=False); plan.backward(); plan.step(1e-4)
        for _ in range(5): step()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(30): step()
        e1.record(st)
        st.synchronize()
    ms = e0.elapsed_time(e1) / 30
    print(f"wgrad_stream={side}: {ms:.4f} ms/step, {N / ms * 1000:.1f} samples/s")
    del plan
