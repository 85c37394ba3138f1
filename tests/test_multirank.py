"""World-size-2 CPU tests (gloo) of the N > 1 host logic:
* every rank computes the same GABRA placement independently (rn_gabra_place);
* the per-rank schedules from rn_plan_describe pair up: each send of a unit
  output on rank r to stage p is matched, in order and size, by a receive of
  the next unit's input on the rank of stage p (no deadlock);
* executing that schedule over gloo with the oracle's unit ops as the compute
  (test infrastructure) reproduces the single-process step exactly (hybrid,
  non-contiguous GABRA placement of the 4 tiny partitions on 2 stages), and
  the data-parallel exchange (sum all-reduce of the local ranges) reproduces
  Eq. 11 with per-replica BN.
The CUDA/NCCL side of the same schedule needs several GPUs and is not run here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from oracle import gabra as G
from oracle import net as O
from paper_2104_05035_b200 import rn

DIMS = (16, 16, 16)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _hybrid_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        desc = rn.net_desc(0, 8, DIMS)
        _, _, loads = rn.net_units(desc)
        caps = G.default_capacities(loads, 2)
        genes, profit, _ = rn.gabra_place(loads, caps, seed=7, require_all_used=1)
        allg = [None] * world
        dist.all_gather_object(allg, genes)
        assert all(g == genes for g in allg)
        local, xfers, ranges = rn.plan_describe(desc, 2, rank=rank, world=world, n_stages=2, genes=genes)
        all_x = [None] * world
        dist.all_gather_object(all_x, xfers)
        # pairing: sends of r to p (dir 1, unit u) == receives of p from r (dir 0, unit u+1), same order/size
        for r in range(world):
            for p in range(world):
                if r == p:
                    continue
                sends = [(u + 1, b) for (u, peer, d, b) in all_x[r] if d == 1 and peer == p]
                recvs = [(u, b) for (u, peer, d, b) in all_x[p] if d == 0 and peer == r]
                assert sends == recvs, (r, p, sends, recvs)
        # execute the schedule over gloo with oracle unit ops
        net = O.Net(0, 8, DIMS)
        arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
        P = O.Params(net.tensors, arrays)
        x, y = synthetic.make_batch(2, *DIMS, seed=1)
        units = net.units
        nu = len(units)
        h = np.asarray(x, dtype=np.float64)[..., None]
        caches, outs = {}, {}
        recv_from = {u: peer for (u, peer, d, b) in xfers if d == 0}
        send_to = {u: peer for (u, peer, d, b) in xfers if d == 1}
        loss = None
        for ui in range(nu):
            if not local[ui]:
                continue
            if ui in recv_from:
                shp = (2,) + tuple(units[ui - 1].out_dims) + (units[ui - 1].cout,)
                t = torch.empty(shp, dtype=torch.float64)
                dist.recv(t, src=recv_from[ui])
                h = t.numpy()
            h, caches[ui] = O.unit_forward(P, ui, units[ui], h, [])
            outs[ui] = h
            if ui in send_to:
                dist.send(torch.from_numpy(np.ascontiguousarray(h)), dst=send_to[ui])
        Gd = {}
        if local[nu - 1]:
            loss, dz = O.softmax_ce(outs[nu - 1], y)
            g = dz
        for ui in reversed(range(nu)):
            if not local[ui]:
                continue
            if ui in send_to:  # successor elsewhere: its input gradient comes back
                shp = (2,) + tuple(units[ui].out_dims) + (units[ui].cout,)
                t = torch.empty(shp, dtype=torch.float64)
                dist.recv(t, src=send_to[ui])
                g = t.numpy()
            g = O.unit_backward(P, ui, units[ui], g, caches[ui], Gd)
            if ui in recv_from:
                dist.send(torch.from_numpy(np.ascontiguousarray(g)), dst=recv_from[ui])
        flat = np.zeros(net.n_params)
        off = 0
        for name, shape, kind in net.tensors:
            n = int(np.prod(shape))
            if name in Gd:
                flat[off:off + n] = np.asarray(Gd[name]).ravel()
            off += n
        # ranges from rn_plan_describe cover exactly the parameters this rank produced
        mask = np.zeros(net.n_params, dtype=bool)
        for a, b in ranges:
            mask[a:b] = True
        assert np.all(flat[~mask] == 0)
        q.put((rank, flat, mask, loss))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the parent
        q.put((rank, repr(e), None, None))
        raise


def _run(worker, world):
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[2] is not None, r[1]
    return sorted(res, key=lambda t: t[0])


def test_hybrid_two_stage_schedule_and_step():
    res = _run(_hybrid_worker, 2)
    net = O.Net(0, 8, DIMS)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(2, *DIMS, seed=1)
    ref = net.train_step(arrays, x, y, 1e-4)
    masks = [r[2] for r in res]
    assert not np.any(masks[0] & masks[1]) and np.all(masks[0] | masks[1])   # ranges partition the model
    g = res[0][1] + res[1][1]
    np.testing.assert_allclose(g, ref["grad"], rtol=1e-12, atol=1e-15)
    loss = [r[3] for r in res if r[3] is not None]
    assert len(loss) == 1 and abs(loss[0] - ref["loss"]) < 1e-14


def _dp_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        desc = rn.net_desc(0, 8, DIMS)
        local, xfers, ranges = rn.plan_describe(desc, 2, rank=rank, world=world, n_stages=1)
        net = O.Net(0, 8, DIMS)
        assert xfers == [] and ranges == [(0, net.n_params)] and all(local)
        arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
        x, y = synthetic.make_batch(2 * world, *DIMS, seed=3)
        sl = slice(2 * rank, 2 * rank + 2)                                     # equal sharding
        loss, Gd, _ = net.forward_backward(O.Params(net.tensors, arrays), x[sl], y[sl], loss_scale=1.0 / world)
        t = torch.from_numpy(net.flat(Gd))
        for a, b in ranges:
            seg = t[a:b].clone()
            dist.all_reduce(seg)                                               # ring all-reduce
            t[a:b] = seg
        q.put((rank, t.numpy(), np.ones(1, bool), loss))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None, None))
        raise


def test_data_parallel_allreduce_eq11():
    res = _run(_dp_worker, 2)
    net = O.Net(0, 8, DIMS)
    arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
    x, y = synthetic.make_batch(4, *DIMS, seed=3)
    ref = net.train_step(arrays, x, y, 1e-4, m=2)
    for r in res:
        np.testing.assert_allclose(r[1], ref["grad"], rtol=1e-12, atol=1e-16)
    assert np.array_equal(res[0][1], res[1][1])
