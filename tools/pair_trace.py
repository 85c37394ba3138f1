"""Per-CTA phase timeline of the CTA-pair stage-1 convolutions of one r18 batch-8
bf16 step (RN_PAIR_TRACE %globaltimer stamps in k_conv_pair.cu).  Per launch, the
median CTA (us from the launch's first CTA entry): setup+dependency wait, weights
resident, and for every item the first / last MMA issue and the epilogue window.
Usage: python tools/pair_trace.py"""
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
        plan.train_step(xd, yd, 1e-4)
    st.synchronize()
    os.environ["RN_PAIR_TRACE"] = "1"
    plan.train_step(xd, yd, 1e-4)
    st.synchronize()
L = rn.lib()
L.rn_dbg_pair_trace.restype = C.c_int
buf = np.zeros(64 * 148 * 32, dtype=np.uint64)
meta = np.zeros(64 * 4, dtype=np.int32)
n = L.rn_dbg_pair_trace(buf.ctypes.data_as(C.c_void_p), 64, meta.ctypes.data_as(C.c_void_p))
buf = buf.reshape(64, 148, 32).astype(np.int64)
meta = meta.reshape(64, 4)
print(f"{n} conv_pair launches; us from the launch's first CTA entry; median over CTAs (leader CTAs for MMA stamps)")
for i in range(n):
    t = buf[i]
    t0 = t[:, 0][t[:, 0] > 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    span = np.nanmax(rel[:, 31])
    med = np.nanmedian(rel, axis=0)
    items = []
    for k in range(6):
        if not np.isnan(med[4 + 2 * k]):
            items.append(f"i{k}: mma {med[4 + 2 * k]:.1f}-{med[5 + 2 * k]:.1f} epi {med[16 + 2 * k]:.1f}-{med[17 + 2 * k]:.1f}")
    kind = ("dgrad" if meta[i][0] else "fprop") + ("+res" if meta[i][1] else "") + f" st{meta[i][2]}"
    print(f"{i:2d} {kind:14s} pairs-items {meta[i][3]:4d} span {span:5.1f} ready {med[1]:.1f} w {med[2]:.1f} | " +
          " | ".join(items) + f" | exit {med[31]:.1f}")
