"""Per-kernel device time of the r18 bf16 training step under CUPTI (torch.profiler),
with the CUDA graphs as bench.py runs them (warm, back-to-back, real clocks).
Usage: python tools/kprof.py [steps=5] [batch=8] [out.txt]"""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = sys.argv[3] if len(sys.argv) > 3 else None
dims = (91, 109, 91)
desc = rn.net_desc(18, 64, dims)
stream = torch.cuda.Stream()
plan = rn.Plan(desc, batch, rn.RN_BF16, stream=stream)
if os.environ.get("KPROF_NOGRAPH"):
    plan.set_option("graphs", 0)
if os.environ.get("KPROF_NOSIDE"):
    plan.set_option("wgrad_stream", 0)
for kv in filter(None, os.environ.get("KPROF_OPTS", "").split(",")):  # e.g. KPROF_OPTS=fused_stats=0
    k, v = kv.split("=")
    plan.set_option(k, int(v))
arrays = synthetic.init_params(plan.tensors, seed=0)
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(batch, *dims, seed=1)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()


def step():
    plan.forward(xd, yd, want_loss=False)
    plan.backward()
    plan.step(1e-4)


with torch.cuda.stream(stream):
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / steps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
seq = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.replace("(anonymous namespace)::", "").replace("rn::", "").split("(")[0]
        name = name.replace("void ", "")[:80]
        dur = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        tot[name] += dur
        cnt[name] += 1
        seq.append((ev.time_range.start if hasattr(ev, "time_range") else 0, name, dur))
s = sum(tot.values())
lines = [f"step {step_ms:.3f} ms (events, no profiler); kernel sum per step {s / steps / 1e3:.3f} ms (CUPTI)"]
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    lines.append(f"{v / steps:9.1f} us {100 * v / s:5.1f}% {cnt[k] // steps:4d}/step  {k}")
seq.sort()
n1 = len(seq) // steps
lines.append("--- launches of one step, in order (us) ---")
for i, (t0, name, dur) in enumerate(seq[:n1]):
    lines.append(f"{i:4d} {dur:8.1f}  {name}")
txt = "\n".join(lines)
print(txt)
if out:
    open(out, "w").write(txt + "\n")
