"""Per-CTA phase timeline of every conv_tc launch of one r18 batch-8 bf16 step
(RN_TC_TRACE %globaltimer stamps in k_conv_tc.cu): launch span, and the median
CTA's entry -> dependency wait -> first TMA -> first MMA -> last MMA -> first
epilogue -> epilogue end -> exit.  Usage: python tools/tc_trace.py [graphs 0|1]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

dims = (91, 109, 91)
st = torch.cuda.Stream()
plan = rn.Plan(rn.net_desc(18, 64, dims), 8, rn.RN_BF16, stream=st)
plan.set_option("graphs", 0)
arrays = synthetic.init_params(plan.tensors, seed=0)
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(8, *dims, seed=1)
with torch.cuda.stream(st):
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(3):
        plan.forward(xd, yd, want_loss=False)
        plan.backward()
        plan.step(1e-4)
    st.synchronize()
    os.environ["RN_TC_TRACE"] = "1"
    plan.forward(xd, yd, want_loss=False)
    plan.backward()
    plan.step(1e-4)
    st.synchronize()
L = rn.lib()
L.rn_dbg_tc_trace.restype = C.c_int
buf = np.zeros(256 * 296 * 8, dtype=np.uint64)
meta = np.zeros(256 * 8, dtype=np.int32)
n = L.rn_dbg_tc_trace(buf.ctypes.data_as(C.c_void_p), 256, meta.ctypes.data_as(C.c_void_p))
buf = buf.reshape(256, 296, 8).astype(np.int64)
meta = meta.reshape(256, 8)
names = ["entry", "deps", "tma0", "mma0", "mmaN", "epi0", "epiN", "exit"]
print(f"{n} conv_tc launches; times in us relative to the launch's first CTA entry (median CTA)")
print(f"{'#':>3} {'BN':>3} {'S':>2} {'grid':>4} {'items':>5} {'ks':>3} {'kb':>4}  {'span':>6} " +
      " ".join(f"{x:>6}" for x in names[1:]))
tot = 0.0
for i in range(n):
    g = meta[i][2]
    t = buf[i, :g, :]
    t0 = t[:, 0].min()
    span = (t[:, 7].max() - t0) / 1000
    tot += span
    rel = (t - t0) / 1000.0
    med = np.median(rel, axis=0)
    if meta[i][1] < 0:  # CTA pairs: the MMA stamps come from the leaders (even CTAs)
        med[3:5] = np.median(rel[0::2, 3:5], axis=0)
    print(f"{i:>3} {meta[i][0]:>3} {meta[i][1]:>2} {g:>4} {meta[i][3]:>5} {meta[i][4]:>3} {meta[i][7]:>4}  {span:6.1f} " +
          " ".join(f"{v:6.1f}" for v in med[1:]))
print(f"sum of launch spans {tot:.1f} us")
