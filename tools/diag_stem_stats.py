"""Diagnostic: stem BN statistics (GPU, from rn_get_saved) vs float64 on the GPU's own h,
after the forward and after the backward."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synthetic
from paper_2104_05035_b200 import rn

dims = (91, 109, 91)
for N in (8,):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan = rn.Plan(rn.net_desc(18, 64, dims), N, rn.RN_BF16, stream=st)
        arrays = synthetic.perturb_params(plan.tensors, synthetic.init_params(plan.tensors, seed=0))
        plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
        x, y = synthetic.make_batch(N, *dims, seed=1)
        plan.forward(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        st.synchronize()
    cd = (46, 55, 46)
    g, b = arrays[1].astype(np.float64), arrays[2].astype(np.float64)
    for phase in ("fwd", "bwd"):
        if phase == "bwd":
            plan.backward()
            st.synchronize()
        h = plan.get_saved(0, "h", (N,) + cd + (64,)).astype(np.float64)
        s = plan.get_saved(0, "bn.stats", (4, 64)).astype(np.float64)
        mu = h.mean(axis=(0, 1, 2, 3))
        var = ((h - mu) ** 2).mean(axis=(0, 1, 2, 3))
        inv = 1 / np.sqrt(var + 1e-5)
        ref = np.stack([mu, inv, g * inv, b - mu * g * inv])
        for r in range(4):
            e = np.abs(s[r] - ref[r])
            print(f"{phase} row {r}: rel-L2 {np.linalg.norm(s[r]-ref[r])/np.linalg.norm(ref[r]):.2e} "
                  f"worst ch {np.argmax(e)} gpu {s[r][np.argmax(e)]:.6e} ref {ref[r][np.argmax(e)]:.6e}")
