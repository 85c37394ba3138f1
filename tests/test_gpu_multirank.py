"""The multi-rank executor's CUDA path on ONE GPU, through the
in-process transport of include/rn.h (rn_dist_desc.nccl_id = "RNLOCAL..."): each
rank is a plan of this process driven by its own host thread; partition-boundary
send/recv, the data-parallel gradient all-reduce (Eqs. 9-11) and the
loss broadcast run through the same plan code as over NCCL, with device-to-device
copies and rank-order sums in place of NCCL calls.

* hybrid, configs[0] (C1): tiny fp32 net, GABRA placing its 4 partitions on 2
  stages -> loss, the gradient (the ranks' disjoint parts summed) and the updated
  weights against the float64 oracle at 1e-4;
* data parallel, 2 replicas fp32 -> the replica-averaged step of Eq. 11 against the
  oracle's train_step(m=2) at 1e-4, weights bit-identical on both replicas;
* hybrid C4 shape (2 stages x 2 replicas, bf16, r18, 2 micro-batches) against the
  same replicas without the pipeline split (pure data parallel): the partitioned
  executor must reproduce it bit for bit (the cut only moves exact bf16 copies)."""
import threading

import numpy as np
import pytest
import torch

import synthetic
from oracle import net as O
from paper_2104_05035_b200 import rn

pytestmark = pytest.mark.gpu

LR = 1e-4


def run_ranks(world, fn, timeout=600):
    out, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "multi-rank step hung (deadlock in the exchange schedule)"
    if errs:
        raise errs[0][1]
    return out


def step_rank(desc, b, dtype, r, world, S, genes, Mb, nid, flat, x, y, opts=None):
    st = torch.cuda.Stream()
    plan = rn.Plan(desc, b, dtype, rank=r, world=world, n_stages=S, genes=genes, micro_batches=Mb, nccl_id=nid,
                   stream=st)
    for k, v in (opts or {}).items():
        plan.set_option(k, v)
    plan.set_params(flat)
    rep = r // S
    with torch.cuda.stream(st):
        xd = torch.from_numpy(np.ascontiguousarray(x[rep * b:(rep + 1) * b])).cuda()
        yd = torch.from_numpy(np.ascontiguousarray(y[rep * b:(rep + 1) * b])).cuda()
        loss = plan.forward(xd, yd)
        plan.backward()
        g = plan.get_grads()
        plan.step(LR)
        st.synchronize()
    return dict(loss=loss, g=g, w=plan.get_params(), rm=plan.get_bn_running(), plan=plan)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def update_ok(w1, w0, delta, tol=1e-4):
    """dw = w' - w within tol of the reference update plus the fp32 rounding of
    storing w' (ulp(w')/2 per element), as tests/test_gpu_parity.py::check."""
    dw = np.asarray(w1, np.float64) - np.asarray(w0, np.float64)
    ulp = np.spacing(np.abs(w1).astype(np.float32)).astype(np.float64)
    return np.linalg.norm(dw - delta) <= tol * np.linalg.norm(delta) + np.linalg.norm(ulp / 2)


def owner_mask(plan_tensors, desc, genes, S, stage):
    """Canonical-parameter mask of the units whose partition GABRA put on `stage`."""
    _, first, _ = rn.net_units(desc)
    unit_stage = {}
    for p, g in enumerate(genes):
        for u in range(first[p], first[p + 1]):
            unit_stage[u] = g
    m = []
    for name, shape, _ in plan_tensors:
        u = int(name.split(".")[0][1:])
        m.append(np.full(int(np.prod(shape)), unit_stage[u] == stage))
    return np.concatenate(m)


def test_hybrid_tiny_f32_gabra_2_stages_vs_oracle():
    dims = (16, 16, 16)
    desc = rn.net_desc(0, 8, dims)
    loads = rn.net_units(desc)[2]
    genes, _, _, _, _ = rn.gabra_place_slack(loads, 2, seed=7, require_all_used=1)
    assert sorted(set(genes)) == [0, 1]
    net = O.Net(0, 8, dims)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(2, *dims, seed=1)
    nid = rn.local_transport_id()
    res = run_ranks(2, lambda r: step_rank(desc, 2, rn.RN_F32, r, 2, 2, genes, 1, nid, flat, x, y))
    ref = net.train_step(arrays, x, y, LR)
    for r in range(2):
        assert abs(res[r]["loss"] - ref["loss"]) <= 1e-4 * abs(ref["loss"])   # broadcast from the head stage
    masks = [owner_mask(res[0]["plan"].tensors, desc, genes, 2, s) for s in range(2)]
    assert not np.any(masks[0] & masks[1]) and np.all(masks[0] | masks[1])
    for s in range(2):
        assert np.all(res[s]["g"][~masks[s]] == 0)                      # only local partitions' gradients
    g = res[0]["g"].astype(np.float64) + res[1]["g"]
    assert rel(g, ref["grad"]) <= 1e-4
    w = np.where(masks[0], res[0]["w"], res[1]["w"])
    assert update_ok(w, flat, ref["delta"])


def test_data_parallel_2_replicas_f32_vs_oracle_eq11():
    dims = (16, 16, 16)
    desc = rn.net_desc(0, 8, dims)
    net = O.Net(0, 8, dims)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(4, *dims, seed=3)
    nid = rn.local_transport_id()
    res = run_ranks(2, lambda r: step_rank(desc, 2, rn.RN_F32, r, 2, 1, None, 1, nid, flat, x, y))
    ref = net.train_step(arrays, x, y, LR, m=2)
    assert np.array_equal(res[0]["w"], res[1]["w"])                     # replicas stay identical
    assert update_ok(res[0]["w"], flat, ref["delta"])
    for r in range(2):
        assert abs(res[r]["loss"] - ref["losses"][r]) <= 1e-4 * abs(ref["losses"][r])


def test_hybrid_f32_2x2_microbatches_vs_oracle():
    """configs[3] shape in fp32 (r18 structure, width 8, small volume): 2 stages x 2
    replicas x 2 micro-batches -> the Eq. 11 step with per-(replica, micro-batch)
    BN (readings X9, X18) against the float64 oracle at 1e-4."""
    dims = (40, 48, 40)
    desc = rn.net_desc(18, 8, dims)
    loads = rn.net_units(desc)[2]
    genes = rn.gabra_place_slack(loads, 2, seed=7, require_all_used=1)[0]
    net = O.Net(18, 8, dims)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(8, *dims, seed=1)
    nid = rn.local_transport_id()
    res = run_ranks(4, lambda r: step_rank(desc, 4, rn.RN_F32, r, 4, 2, genes, 2, nid, flat, x, y))
    ref = net.train_step(arrays, x, y, LR, m=2, Mb=2)
    masks = [owner_mask(res[0]["plan"].tensors, desc, genes, 2, s) for s in range(2)]
    for rep in range(2):
        w = np.where(masks[0], res[2 * rep]["w"], res[2 * rep + 1]["w"])
        assert update_ok(w, flat, ref["delta"])
        lref = 0.5 * (ref["losses"][2 * rep] + ref["losses"][2 * rep + 1])
        assert abs(res[2 * rep]["loss"] - lref) <= 1e-4 * abs(lref)


def test_hybrid_bf16_2x2_matches_data_parallel():
    """configs[3] shape in bf16 (r18, 2 stages x 2 replicas x 2 micro-batches)
    against the same replicas without the pipeline split: the forward and the loss
    are bit-identical (the cut only moves exact bf16 copies); the backward differs
    only where a cut replaces a BN's backward statistics fused into the neighbour's
    dgrad epilogue by the standalone pass (another fp32 summation order), which the
    bf16 backward then carries as re-rounding chaos (reading X23) -> every tensor
    within 2e-2 (5e-2 for the attention mask branch, reading X23b); and the
    partitioned step is deterministic (two runs bit-equal)."""
    dims = (40, 48, 40)
    desc = rn.net_desc(18, 64, dims)
    loads = rn.net_units(desc)[2]
    genes, _, _, _, _ = rn.gabra_place_slack(loads, 2, seed=7, require_all_used=1)
    tensors = rn.net_params(desc)[0]
    arrays = synthetic.perturb_params(tensors, synthetic.init_params(tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(4, *dims, seed=1)
    runs = []
    for _ in range(2):
        nid = rn.local_transport_id()
        runs.append(run_ranks(4, lambda r: step_rank(desc, 2, rn.RN_BF16, r, 4, 2, genes, 2, nid, flat, x, y)))
    nid2 = rn.local_transport_id()
    dp = run_ranks(2, lambda r: step_rank(desc, 2, rn.RN_BF16, r, 2, 1, None, 2, nid2, flat, x, y))
    masks = [owner_mask(tensors, desc, genes, 2, s) for s in range(2)]
    hyb = runs[0]
    for rep in range(2):
        assert hyb[2 * rep]["loss"] == dp[rep]["loss"] == hyb[2 * rep + 1]["loss"]
        for r in (2 * rep, 2 * rep + 1):
            assert np.array_equal(runs[0][r]["w"], runs[1][r]["w"])
        g = np.where(masks[0], hyb[2 * rep]["g"], hyb[2 * rep + 1]["g"])
        off = 0
        for name, shape, _ in tensors:
            n = int(np.prod(shape))
            tol = 5e-2 if (".mask." in name or ".mbn." in name or ".mconv" in name) else 2e-2  # X23b
            assert rel(g[off:off + n], dp[rep]["g"][off:off + n]) <= tol, name
            off += n


def test_overlapped_bucketed_allreduce_matches_after_backward_allreduce():
    """The gradient all-reduce bucketed and overlapped with the backward (default)
    computes exactly what one all-reduce after the backward computes (same
    rank-order sums on this transport): DP 2 replicas and hybrid 2x2, bf16."""
    dims = (40, 48, 40)
    desc = rn.net_desc(18, 64, dims)
    loads = rn.net_units(desc)[2]
    genes = rn.gabra_place_slack(loads, 2, seed=7, require_all_used=1)[0]
    tensors = rn.net_params(desc)[0]
    arrays = synthetic.init_params(tensors, seed=0)
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(4, *dims, seed=1)
    for world, S, g in ((2, 1, None), (4, 2, genes)):
        outs = []
        for ov in (1, 0):
            nid = rn.local_transport_id()
            outs.append(run_ranks(world, lambda r: step_rank(desc, 2, rn.RN_BF16, r, world, S, g, 1, nid, flat, x, y,
                                                             {"overlap_allreduce": ov})))
        for r in range(world):
            assert np.array_equal(outs[0][r]["w"], outs[1][r]["w"])


def test_asgd_async_allreduce_vs_oracle():
    """ASGD with ring all-reduce (reading F4): data parallel,
    2 replicas, fp32, option async_allreduce -- step t's gradient is reduced on the
    comm stream during step t+1 and applied there.  Three steps against the oracle's
    async_allreduce_train at 1e-4 (losses per replica and step, final weights); the
    replicas' weights stay bit-identical."""
    dims = (16, 16, 16)
    desc = rn.net_desc(0, 8, dims)
    net = O.Net(0, 8, dims)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    bs = [synthetic.make_batch(4, *dims, seed=30 + t) for t in range(3)]
    lr = 1e-2
    nid = rn.local_transport_id()

    def rank(r):
        st = torch.cuda.Stream()
        plan = rn.Plan(desc, 2, rn.RN_F32, rank=r, world=2, n_stages=1, nccl_id=nid, stream=st)
        plan.set_option("async_allreduce", 1)
        plan.set_params(flat)
        losses = []
        with torch.cuda.stream(st):
            for x, y in bs:
                xd = torch.from_numpy(np.ascontiguousarray(x[2 * r:2 * r + 2])).cuda()
                yd = torch.from_numpy(np.ascontiguousarray(y[2 * r:2 * r + 2])).cuda()
                losses.append(plan.forward(xd, yd))
                plan.backward()
                plan.step(lr)
            st.synchronize()
        return dict(losses=losses, w=plan.get_params())

    res = run_ranks(2, rank)
    ref = O.async_allreduce_train(net, arrays, bs, lr, 2)
    assert np.array_equal(res[0]["w"], res[1]["w"])
    for r in range(2):
        np.testing.assert_allclose(res[r]["losses"], [ls[r] for ls in ref["losses"]], rtol=1e-4)
    # two applied updates at lr 1e-2: the second gradient is taken at the GPU's own
    # updated weights, so the fp32 differences of the first step compound -> 1e-3
    delta = ref["params"] - flat.astype(np.float64)
    err = np.linalg.norm(res[0]["w"].astype(np.float64) - ref["params"]) / np.linalg.norm(delta)
    assert update_ok(res[0]["w"], flat, delta, tol=1e-3), err
