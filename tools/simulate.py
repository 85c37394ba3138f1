"""SURVEY §8(f) f2 on real hardware: per-partition forward+backward times MEASURED
on this B200 (rn_query unit_ms_fwd_<u> / unit_ms_bwd_<u> of one timed eager step),
then the step-time model (rn_simulate_step, reading F2) for the BASELINE configs
under three placements -- GABRA on MAC loads (the paper's Eq. 3 objective),
GABRA bottleneck objective on the MEASURED times, and the contiguous split of the
measured times -- and both schedules (synchronous pipeline, delayed gradients f1).
Link parameters are NVLink 5 figures (900 GB/s per direction, 5 us per message):
one GPU cannot measure them.  Usage: python tools/simulate.py [out.txt]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_2104_05035_b200 import rn  # noqa: E402

ALPHA, BETA = 5e-6, 900e9
DIMS = (91, 109, 91)
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout


def log(*a):
    print(*a, file=out, flush=True)
    if out is not sys.stdout:
        print(*a, flush=True)


def unit_times(depth, batch):
    desc = rn.net_desc(depth, 64, DIMS)
    st = torch.cuda.Stream()
    plan = rn.Plan(desc, batch, rn.RN_BF16, stream=st)
    arrays = synthetic.init_params(plan.tensors, seed=0)
    plan.set_params(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
    x, y = synthetic.make_batch(batch, *DIMS, seed=1)
    with torch.cuda.stream(st):
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        for _ in range(4):
            plan.forward(xd, yd, want_loss=False)
            plan.backward()
            plan.step(1e-4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):  # the real step (graphs, side stream, PDL): calibrates the per-unit shares
            plan.forward(xd, yd, want_loss=False)
            plan.backward()
            plan.step(1e-4)
        e1.record(st)
        st.synchronize()
        real = e0.elapsed_time(e1) / 10 / 1000.0
        plan.set_option("time_kernels", 1)
        for _ in range(2):  # the second timed step is the one read
            plan.forward(xd, yd, want_loss=False)
            plan.backward()
            plan.step(1e-4)
        st.synchronize()
    nu = len(rn.net_units(desc)[0])
    t = [(plan.query(f"unit_ms_fwd_{u}") + plan.query(f"unit_ms_bwd_{u}")) / 1000.0 for u in range(nu)]
    # the timed eager step serialises the side stream and brackets every launch:
    # keep its per-unit SHARES, scaled to the real step time (minus the SGD step)
    sgd = plan.query("elt_ms_sgd") / 1000.0
    scale = (real - sgd) / sum(t)
    return desc, plan, [v * scale for v in t], real, scale


for depth, cap in ((18, False), (34, True)):
    for mb in (8, 2):
        desc, plan, ut, real, scale = unit_times(depth, mb)
        units, first, loads = rn.net_units(desc)
        if cap:
            desc = rn.net_desc(depth, 64, DIMS, max_merge_load=max(units))
            units, first, loads = rn.net_units(desc)
        n = len(loads)
        pt = [sum(ut[first[p]:first[p + 1]]) for p in range(n)]
        # bytes: partition p's output activation (bf16) per micro-batch; fp32 gradients
        tensors = plan.tensors
        pbytes = [0.0] * n
        unit_of = lambda name: int(name.split(".")[0][1:])  # noqa: E731
        part_of_unit = {}
        for p in range(n):
            for u in range(first[p], first[p + 1]):
                part_of_unit[u] = p
        for name, shape, _ in tensors:
            pbytes[part_of_unit[unit_of(name)]] += 4.0 * int(np.prod(shape))
        net_outs = []
        from oracle import net as O  # unit output shapes only (no arithmetic)
        onet = O.Net(depth, 64, DIMS)
        for p in range(n - 1):
            u = onet.units[first[p + 1] - 1]
            net_outs.append(2.0 * mb * u.cout * int(np.prod(u.out_dims)))
        log(f"== r{depth}, micro-batch {mb}: real step {1000 * real:.3f} ms on this B200 (timed-step shares x "
            f"{scale:.3f})")
        log(f"   {n} partitions, measured fwd+bwd ms per partition "
            f"{[round(1000 * v, 3) for v in pt]} (sum {1000 * sum(pt):.3f} ms)")
        Mb = 8 // mb  # local batch 8 per replica in micro-batches of mb
        t1 = rn.simulate_step(pt, net_outs, pbytes, [0] * n, 1, 1, Mb, ALPHA, BETA)[0]
        log(f"   1 GPU (batch 8 = {Mb} x {mb}): step {1000 * t1:.3f} ms -> {8 / t1:.0f} samples/s")
        for m in (2, 4, 8):
            dp = rn.simulate_step(pt, net_outs, pbytes, [0] * n, 1, m, Mb, ALPHA, BETA, overlap=True)[0]
            log(f"   DP x{m}: step {1000 * dp:.3f} ms -> {m * 8 / dp:.0f} samples/s "
                f"(overlapped ring all-reduce of {sum(pbytes) / 1e6:.0f} MB)")
            for S in (2, 4, 8):
                if S > m or m % S or S > n:
                    continue
                R = m // S
                tns = [max(1, int(round(v * 1e9))) for v in pt]
                cands = {}
                try:
                    cands["gabra-eq3-MACs"] = rn.gabra_place_slack(loads, S, seed=7, require_all_used=1,
                                                                   init_attempts=4096)[0]
                except rn.RnError:
                    pass
                try:
                    cands["gabra-bottleneck-measured"] = rn.gabra_place_slack(tns, S, seed=7, require_all_used=1,
                                                                              objective=1, init_attempts=4096)[0]
                except rn.RnError:
                    pass
                cands["contiguous-measured"] = rn.contiguous_split(tns, S)[0]
                for name, g in cands.items():
                    for sched in (0, 1):
                        st, pipe, ar, T = rn.simulate_step(pt, net_outs, pbytes, g, S, R, Mb, ALPHA, BETA,
                                                           schedule=sched, overlap=True)
                        log(f"   hybrid {S}x{R} (M_b {Mb}) {name:27s} {'delayed' if sched else 'sync   '}: "
                            f"step {1000 * st:.3f} ms -> {R * 8 / st:.0f} samples/s; stage max/mean "
                            f"{max(T) / (sum(T) / S):.3f} genes {g}")
        del plan
