"""Stream timeline of the r18 bf16 training step (rn_train_step, CUDA graphs, as
bench.py runs it) under CUPTI: per stream busy time, the main stream's idle gaps
(dependency waits / launch latency on the critical path) and the kernels around
the largest gaps.  Usage: python tools/timeline.py [out.txt]"""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
dims = (91, 109, 91)
stream = torch.cuda.Stream()
plan = rn.Plan(rn.net_desc(18, 64, dims), 8, rn.RN_BF16, stream=stream)
for kv in filter(None, os.environ.get("KPROF_OPTS", "").split(",")):
    k, v = kv.split("=")
    plan.set_option(k, int(v))
arrays = synthetic.init_params(plan.tensors, seed=0)
plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
x, y = synthetic.make_batch(8, *dims, seed=1)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
with torch.cuda.stream(stream):
    for _ in range(6):
        plan.train_step(xd, yd, 1e-4)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            plan.train_step(xd, yd, 1e-4)
        torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        ev.append((e.time_range.start, e.time_range.end, e.device_resource_id, e.name))
ev.sort()
# the last full step: from the last memset of the gradient array ... use the middle third
t0, t1 = ev[0][0], ev[-1][1]
span = (t1 - t0) / 3
lo, hi = t0 + span, t0 + 2 * span
step = [e for e in ev if lo <= e[0] < hi]
byst = collections.defaultdict(list)
for e in step:
    byst[e[2]].append(e)
main = max(byst, key=lambda s: sum(b - a for a, b, _, _ in byst[s]))
print(f"window {span:.1f} us (one step); streams: " + ", ".join(
    f"{s}: {len(v)} kernels, busy {sum(b - a for a, b, _, _ in v):.1f} us" for s, v in byst.items()), file=out)
m = byst[main]
gaps = []
for (a0, b0, _, n0), (a1, b1, _, n1) in zip(m, m[1:]):
    if a1 > b0:
        gaps.append((a1 - b0, n0, n1))
print(f"main stream {main}: busy {sum(b - a for a, b, _, _ in m):.1f} us, idle gaps {sum(g[0] for g in gaps):.1f} us "
      f"over {len(gaps)} gaps", file=out)
hist = collections.Counter()
for g in gaps:
    hist[min(int(g[0]), 20)] += 1
print("gap histogram (us: count): " + ", ".join(f"{k}{'+' if k == 20 else ''}: {v}" for k, v in sorted(hist.items())),
      file=out)
print("largest gaps:", file=out)
for g, n0, n1 in sorted(gaps, reverse=True)[:25]:
    print(f"  {g:7.1f} us  after {n0[:60]}  before {n1[:60]}", file=out)
# side-stream activity overlapping main-stream kernels
# union of all streams: time with no kernel running (the graph maps branches to several streams)
iv = sorted((a, b) for a, b, _, _ in step)
cover, cur_a, cur_b = 0.0, None, None
idle = []
for a, b in iv:
    if cur_b is None or a > cur_b:
        if cur_b is not None:
            cover += cur_b - cur_a
            idle.append((a - cur_b, cur_b))
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
cover += cur_b - cur_a
print(f"any-kernel-running {cover:.1f} us of {span:.1f}; fully idle {sum(g for g, _ in idle):.1f} us in {len(idle)} gaps",
      file=out)
# concurrency: time with exactly k kernels running
pts = sorted([(a, 1) for a, b in iv] + [(b, -1) for a, b in iv])
conc = collections.Counter()
k, last = 0, pts[0][0]
for t, d in pts:
    conc[k] += t - last
    k += d
    last = t
print("time by number of concurrent kernels: " + ", ".join(f"{k}: {v:.0f} us" for k, v in sorted(conc.items())), file=out)
# per kernel family: total time, and time overlapped with another kernel
fam = collections.defaultdict(lambda: [0.0, 0.0, 0])
for a, b, s, n in step:
    key = n.split("(")[0].replace("void ", "").replace("rn::", "").replace("(anonymous namespace)::", "")[:48]
    ov = 0.0
    for a2, b2, s2, n2 in step:
        if (a2, b2, s2) != (a, b, s):
            ov = max(ov, min(b, b2) - max(a, a2))
    fam[key][0] += b - a
    fam[key][1] += max(0.0, min(ov, b - a))
    fam[key][2] += 1
print("kernel family: total us, launches (overlap: max single-partner overlap, indicative)", file=out)
for key, (t, o, c) in sorted(fam.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {t:8.1f} {c:4d}  ov {o:7.1f}  {key}", file=out)
# critical-path increments on the main stream: with PDL a kernel starts early and waits,
# so its CUPTI duration overstates; end_i - end_{i-1} is what it adds to the stream's span
inc = collections.defaultdict(lambda: [0.0, 0])
prev_end = None
rows = []
for a, b, s, n in m:
    key = n.split("(")[0].replace("void ", "").replace("rn::", "").replace("(anonymous namespace)::", "")[:48]
    d = b - (prev_end if prev_end is not None else a)
    prev_end = b if prev_end is None else max(prev_end, b)
    inc[key][0] += d
    inc[key][1] += 1
    rows.append((d, key))
print(f"main-stream end-to-end increments (sum {sum(v[0] for v in inc.values()):.1f} us):", file=out)
for key, (t, c) in sorted(inc.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {t:8.1f} {c:4d}  {key}", file=out)
print("main-stream sequence (increment us, kernel):", file=out)
for d, key in rows:
    print(f"  {d:7.1f}  {key}", file=out)
