"""bench.py — 3D-ResAttNet training throughput (samples/s) on B200 through librn.so.

Contract:
  python bench.py --gpus N --steps K --warmup W              (our arm)
  python bench.py --impl reference --gpus N --steps K ...    (the CPU float64 oracle)
N = 1: BASELINE configs[1] (r18-style 3D-ResAttNet, batch 8, 1x91x109x91, bf16).
N > 1 (torchrun, one rank per GPU): configs[2], pure data parallel, 8 samples per
rank (weak scaling), gradient all-reduce over NCCL inside rn_step.
Prints ONE JSON line on rank 0."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D-ResAttNet train samples/s at 1/2/4/8 B200; conv tensor-pipe util %"
DIMS = (91, 109, 91)


ELT_FAMILIES = ("bn_apply", "bn_bwd_apply", "bn_partials", "stem_pool_fwd", "stem_pool_bwd", "maxpool_fwd",
                "maxpool_bwd", "upsample_fwd", "upsample_bwd", "att_fwd", "att_bwd", "sgd")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--depth", type=int, default=18)
    ap.add_argument("--batch", type=int, default=8, help="samples per replica")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--stages", type=int, default=1, help="pipeline stages per replica (hybrid)")
    ap.add_argument("--micro-batches", type=int, default=1)
    ap.add_argument("--ga-objective", type=int, default=0, choices=[0, 1],
                    help="GABRA objective for --stages > 1: 0 = the paper's Eq. 3, 1 = bottleneck (SURVEY f2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--f32-steps", type=int, default=5,
                    help="also time the RN_F32 path (the paper's implicit fp32 precision) at N=1; 0 = skip")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


def cpu_baseline(depth, batch_dims, n_samples=2):
    """The oracle as it stands, timed on this host's cores on a bounded sample."""
    import synthetic
    from oracle import net as O
    net = O.Net(depth, 64 if depth else 8, batch_dims)
    arrays = synthetic.init_params(net.tensors, seed=0)
    x, y = synthetic.make_batch(n_samples, *batch_dims, seed=1)
    t0 = time.perf_counter()
    net.train_step(arrays, x, y, 1e-4)
    dt = time.perf_counter() - t0
    return {"value": n_samples / dt, "unit": "samples/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"one float64 NumPy train step of {n_samples} samples of 1x{batch_dims[0]}x{batch_dims[1]}x"
                      f"{batch_dims[2]} (same recipe/weights), {dt:.1f} s"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthetic
    from oracle import net as O
    net = O.Net(a.depth, 64 if a.depth else 8, DIMS)
    arrays = synthetic.init_params(net.tensors, seed=0)
    x, y = synthetic.make_batch(1, *DIMS, seed=1)
    for _ in range(a.warmup):
        net.train_step(arrays, x, y, 1e-4)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        net.train_step(arrays, x, y, 1e-4)
    dt = time.perf_counter() - t0
    v = a.steps / dt
    out = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": a.gpus, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": 1000 * dt / a.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"3D-ResAttNet-{a.depth} train step, 1x91x109x91 volumes (oracle sample: 1 "
                                  f"sample/step)", "global_batch": 1, "parallelism": "cpu"},
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": "samples/s", "cores": os.cpu_count(), "kind": "oracle",
                            "sample": "1 sample per step, float64 NumPy oracle"},
           "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    from paper_2104_05035_b200 import rn
    import synthetic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    S = a.stages
    replicas = world // S
    dtype = rn.RN_BF16 if a.dtype == "bf16" else rn.RN_F32
    desc = rn.net_desc(a.depth, 64 if a.depth else 8, DIMS)
    genes = None
    if S > 1:
        loads = rn.net_units(desc)[2]
        # reading G4b: smallest capacity slack (1.1, 1.2, ...) with a feasible placement
        genes = rn.gabra_place_slack(loads, S, seed=7, require_all_used=1, objective=a.ga_objective,
                                     init_attempts=4096)[0]
    nid = None
    if world > 1:
        obj = [rn.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    stream = torch.cuda.Stream(dev)
    plan = rn.Plan(desc, a.batch, dtype, rank=rank, world=world, n_stages=S, genes=genes,
                   micro_batches=a.micro_batches, nccl_id=nid, stream=stream, device=dev)
    arrays = synthetic.init_params(plan.tensors, seed=0)
    plan.set_params(np.concatenate([x.ravel() for x in arrays]).astype(np.float32))
    x, y = synthetic.make_batch(a.batch * replicas, *DIMS, seed=1)
    r = rank // S
    xs, ys = x[r * a.batch:(r + 1) * a.batch], y[r * a.batch:(r + 1) * a.batch]
    xd = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
    yd = torch.from_numpy(np.ascontiguousarray(ys)).to(dev)
    lr = 1e-4

    def step():  # rn_train_step: forward + backward + SGD (per-unit early SGD when it applies)
        plan.train_step(xd, yd, lr)

    with torch.cuda.stream(stream):
        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        clocks = ClockSampler(local_rank)
        clocks.start()
        n0 = rn.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        launches = rn.kernel_launches() - n0
        ms = e0.elapsed_time(e1)
        ck = clocks.stop()
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        # conv kernels timed live with CUDA events on the launching stream, one eager
        # step with an event pair around every conv launch; a spin kernel queued first
        # holds the GPU until the whole step is enqueued, so no host gap is timed
        plan.set_option("time_kernels", 1)
        step()  # warm (kernel attributes, event pool)
        torch.cuda.synchronize(dev)
        torch.cuda._sleep(int(2e9 * 0.05))  # ~50 ms of device spin on the plan stream
        step()
        torch.cuda.synchronize(dev)
        conv_ms, conv_fl = plan.query("conv_ms"), plan.query("conv_flops")
        pair_ms, pair_fl = plan.query("conv_ms_pair"), plan.query("conv_flops_pair")
        pair_n = plan.query("conv_launches_pair")
        # per conv class / kernel family ("reported per layer class")
        classes = {}
        for key in ("fprop", "dgrad", "wgrad", "pair", "tcconv", "tcwgrad", "stem"):
            cms, cfl = plan.query("conv_ms_" + key), plan.query("conv_flops_" + key)
            classes[key] = {"ms_per_step": cms, "tflops": (cfl / (cms / 1000.0) / 1e12) if cms > 0 else None,
                            "launches": plan.query("conv_launches_" + key)}
        # HBM-bound (elementwise) launches, same live timing: algorithmic bytes / duration
        elt = {}
        for fam in ELT_FAMILIES:
            ems, eby = plan.query("elt_ms_" + fam), plan.query("elt_bytes_" + fam)
            if ems > 0:
                elt[fam] = {"ms_per_step": ems, "gbs": eby / (ems / 1000.0) / 1e9, "bytes_per_step": eby,
                            "launches": plan.query("elt_launches_" + fam)}
        elt_ms, elt_by = plan.query("elt_ms"), plan.query("elt_bytes")
        plan.set_option("time_kernels", 0)
        torch.cuda.synchronize(dev)
        # end-to-end through the public C ABI with pinned host buffers
        xh = torch.from_numpy(np.ascontiguousarray(xs)).pin_memory().numpy()
        yh = torch.from_numpy(np.ascontiguousarray(ys)).pin_memory().numpy()
        if world > 1:
            dist.barrier()
        # the public pipelined host-input loop: each step's batch crosses PCIe inside
        # the timed call (step i+1's copy overlaps step i's compute)
        plan.train_steps_host([xh] * 4, [yh] * 4, lr)  # warm the side stream / staging slots (graphs per slot)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        plan.train_steps_host([xh] * a.e2e_steps, [yh] * a.e2e_steps, lr)
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())

        f32 = None
        if world == 1 and a.f32_steps > 0 and dtype == rn.RN_BF16:
            p32 = rn.Plan(desc, a.batch, rn.RN_F32, stream=stream, device=dev)
            p32.set_params(np.concatenate([v.ravel() for v in arrays]).astype(np.float32))

            def step32():
                p32.forward(xd, yd, want_loss=False)
                p32.backward()
                p32.step(lr)
            for _ in range(2):
                step32()
            torch.cuda.synchronize(dev)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(a.f32_steps):
                step32()
            f1.record(stream)
            torch.cuda.synchronize(dev)
            fms = f0.elapsed_time(f1) / a.f32_steps
            f32 = {"value": a.batch / (fms / 1000.0), "unit": "samples/s", "ms_per_step": fms, "steps": a.f32_steps,
                   "dtype": "f32", "note": "RN_F32: fp32 storage, fp32 SIMT FFMA convolutions (no TF32), same "
                                           "workload; parity 1e-4 vs float64 (tests/test_gpu_parity.py)"}
            del p32

    step_ms = ms / a.steps
    samples_per_step = a.batch * replicas
    value = samples_per_step * a.steps / (ms / 1000.0)
    pk = peaks()
    # the kernels run inside a ~4 ms step: at full clock (no power cap seen) the burst
    # peak applies, the sustained (power-capped) figure only when the run was capped
    full_clock = (ck.get("sm_mhz") is not None and ck.get("sm_max_mhz") and
                  ck["sm_mhz"] >= 0.95 * ck["sm_max_mhz"] and "sw_power_cap" not in ck.get("reasons", []))
    peak_key = "bf16_tflops" if full_clock else "bf16_tflops_sustained"
    peak_tf = pk.get(peak_key, 1400.0) if dtype == rn.RN_BF16 else 0.0
    hbm = pk.get("hbm_gbs", 6550.0)
    tf = lambda fl, ms: fl / (ms / 1000.0) / 1e12 if ms > 0 else 0.0  # noqa: E731
    pair_tf, conv_tf = tf(pair_fl, pair_ms), tf(conv_fl, conv_ms)
    traffic = None
    try:  # dram bytes of one conv_pair_kernel launch from the committed ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["conv_pair_kernel"]["dram_bytes"]
    except Exception:
        pass
    roof = {"bound": "tensor",
            "kernel": "conv_pair_kernel (stage-1 3x3x3 64->64 fprop+dgrad, tcgen05 cta_group::2; the dominant kernel)",
            "achieved": pair_tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": (pair_tf / peak_tf) if peak_tf else None,
            "traffic": traffic, "launches_per_step": pair_n,
            "kernel_ms_per_step": pair_ms, "kernel_share_of_step": pair_ms / step_ms,
            "flops_per_launch": pair_fl / pair_n if pair_n else None,
            "all_convs": {"achieved": conv_tf, "frac": (conv_tf / peak_tf) if peak_tf else None,
                          "ms_per_step": conv_ms, "share_of_step": conv_ms / step_ms,
                          "note": "every fprop/dgrad/wgrad launch, algorithmic 2*M*N*K FLOPs",
                          "by_class": classes},
            "all_convs_frac": (conv_tf / peak_tf) if peak_tf else None,
            "class_frac": {k: (c["tflops"] / peak_tf if (c["tflops"] and peak_tf) else None) for k, c in classes.items()},
            "elementwise": {"bound": "hbm", "peak_gbs": hbm, "ms_per_step": elt_ms,
                            "gbs": elt_by / (elt_ms / 1000.0) / 1e9 if elt_ms > 0 else None,
                            "frac": (elt_by / (elt_ms / 1000.0) / 1e9 / hbm) if elt_ms > 0 else None,
                            "note": "every BN / pool / upsample / attention / SGD launch; algorithmic bytes = each "
                                    "tensor element read + written once (DESIGN.md 7)",
                            "by_family": {k: dict(v, frac=v["gbs"] / hbm) for k, v in elt.items()}},
            "peak_source": ("MEASURED_PEAKS.json " + peak_key + (" (full clock during the run: burst peak)"
                                                                  if full_clock else " (clock below max: sustained)"))
            if "_fallback" not in pk else "fallback"}
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
               "config": {"workload": f"3D-ResAttNet-{a.depth} train step (fwd+bwd+SGD), {a.batch} x 1x91x109x91 "
                                      f"per replica, random-init weights",
                          "global_batch": samples_per_step, "per_replica_batch": a.batch, "stages": S,
                          "micro_batches": a.micro_batches, "parallelism": f"dp{replicas}" + (f"xpp{S}" if S > 1 else ""),
                          "l2": "working set per step >> 126 MB L2 (activations ~1 GB), no flush needed"},
               "clocks": ck, "gpu_launches": launches,
               "e2e": {"value": samples_per_step * a.e2e_steps / e2e_s, "unit": "samples/s",
                       "h2d_bytes_per_step": int(xs.nbytes + ys.nbytes), "d2h_bytes_per_step": 4},
               "roofline": roof}
        if f32 is not None:
            out["f32_path"] = f32
        if world == 1 and not a.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(a.depth, DIMS)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
