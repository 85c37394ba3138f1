"""Thin ctypes binding of librn.so (include/rn.h).  Argument marshalling only:
every step of the training path runs in librn's CUDA kernels; torch provides
device memory (the plan workspace), streams and process groups.  There is no
CPU fallback: if librn.so is missing or the CUDA call fails, this raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librn.so")

RN_F32, RN_BF16 = 0, 1
STATUS = {0: "RN_OK", 1: "RN_ERR_ARG", 2: "RN_ERR_SCHEMA", 3: "RN_ERR_INFEASIBLE", 4: "RN_ERR_NUMERIC",
          5: "RN_ERR_CUDA", 6: "RN_ERR_NCCL", 7: "RN_ERR_STATE", 8: "RN_ERR_SIZE"}
EXPORTS = ["rn_ga_default", "rn_gabra_place", "rn_gabra_place_slack", "rn_simulate_step", "rn_contiguous_split", "rn_net_units", "rn_net_param_count", "rn_net_param_info",
           "rn_nccl_unique_id", "rn_plan", "rn_plan_delayed", "rn_delayed_step", "rn_plan_describe", "rn_plan_bind", "rn_set_params", "rn_get_params", "rn_get_grads",
           "rn_get_bn_running", "rn_get_activation", "rn_get_unit_grad", "rn_get_saved", "rn_forward", "rn_backward", "rn_step", "rn_train_step", "rn_train_step_host",
           "rn_train_steps_host", "rn_gradcam",
           "rn_kernel_launches", "rn_set_option", "rn_query", "rn_op_conv3d", "rn_plan_destroy", "rn_last_error"]


class RnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class GaParams(C.Structure):
    _fields_ = [("pop_size", C.c_int32), ("t_max", C.c_int32), ("p_cross", C.c_double), ("p_mut", C.c_double),
                ("seed", C.c_uint64), ("dup_retries", C.c_int32), ("init_attempts", C.c_int32),
                ("require_all_used", C.c_int32), ("early_stop_at_ub", C.c_int32), ("objective", C.c_int32)]


class NetDesc(C.Structure):
    _fields_ = [("depth", C.c_int32), ("base_width", C.c_int32), ("in_d", C.c_int32), ("in_h", C.c_int32),
                ("in_w", C.c_int32), ("n_classes", C.c_int32), ("alpha", C.c_double),
                ("max_merge_load", C.c_int64)]


class DistDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("n_stages", C.c_int32),
                ("genes", C.POINTER(C.c_int32)), ("micro_batches", C.c_int32), ("nccl_id", C.c_uint8 * 128)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RnError(7, f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        L.rn_last_error.restype = C.c_char_p
        L.rn_kernel_launches.restype = C.c_int64
        L.rn_plan_destroy.restype = None
        L.rn_ga_default.restype = None
        for name in EXPORTS:
            f = getattr(L, name)
            if name not in ("rn_last_error", "rn_kernel_launches", "rn_plan_destroy", "rn_ga_default"):
                f.restype = C.c_int
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise RnError(st, lib().rn_last_error().decode(errors="replace"))


def net_desc(depth=0, base_width=8, in_dims=(16, 16, 16), alpha=1.0, max_merge_load=0):
    return NetDesc(depth, base_width, in_dims[0], in_dims[1], in_dims[2], 2, alpha, max_merge_load)


def ga_params(**kw):
    g = GaParams()
    lib().rn_ga_default(C.byref(g))
    for k, v in kw.items():
        setattr(g, k, v)
    return g


def gabra_place(loads, caps, **kw):
    """rn_gabra_place: returns (genes 0-based list, profit, per-GPU loads)."""
    n, m = len(loads), len(caps)
    L = (C.c_int64 * n)(*loads)
    D = (C.c_int64 * m)(*caps)
    genes = (C.c_int32 * n)()
    profit = C.c_double()
    gl = (C.c_int64 * m)()
    gp = ga_params(**kw)
    _check(lib().rn_gabra_place(n, L, m, D, C.byref(gp), genes, C.byref(profit), gl))
    return list(genes), profit.value, list(gl)


def gabra_place_slack(loads, m, **kw):
    """rn_gabra_place_slack: (genes, profit, per-GPU loads, capacities, slack)."""
    n = len(loads)
    L = (C.c_int64 * n)(*loads)
    genes = (C.c_int32 * n)()
    profit = C.c_double()
    gl = (C.c_int64 * m)()
    caps = (C.c_int64 * m)()
    slack = C.c_double()
    gp = ga_params(**kw)
    _check(lib().rn_gabra_place_slack(n, L, m, C.byref(gp), genes, C.byref(profit), gl, caps, C.byref(slack)))
    return list(genes), profit.value, list(gl), list(caps), slack.value


class SimDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_stages", C.c_int32), ("replicas", C.c_int32), ("micro_batches", C.c_int32),
                ("schedule", C.c_int32), ("overlap", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
                ("part_time", C.POINTER(C.c_double)), ("cut_bytes", C.POINTER(C.c_double)),
                ("param_bytes", C.POINTER(C.c_double)), ("genes", C.POINTER(C.c_int32))]


def simulate_step(part_time, cut_bytes, param_bytes, genes, S, R, Mb, alpha, beta, schedule=0, overlap=False):
    """rn_simulate_step: (step, pipeline, allreduce, per-stage T_s)."""
    n = len(part_time)
    pt = (C.c_double * n)(*part_time)
    cb = (C.c_double * max(n - 1, 1))(*(list(cut_bytes) or [0.0]))
    pb = (C.c_double * n)(*param_bytes)
    gn = (C.c_int32 * n)(*genes)
    d = SimDesc(n, S, R, Mb, schedule, 1 if overlap else 0, alpha, beta, pt, cb, pb, gn)
    st, pp, ar = C.c_double(), C.c_double(), C.c_double()
    ts = (C.c_double * S)()
    _check(lib().rn_simulate_step(C.byref(d), C.byref(st), C.byref(pp), C.byref(ar), ts))
    return st.value, pp.value, ar.value, list(ts)


def contiguous_split(loads, S):
    """rn_contiguous_split: (genes, max stage load)."""
    n = len(loads)
    L = (C.c_int64 * n)(*loads)
    g = (C.c_int32 * n)()
    mx = C.c_int64()
    _check(lib().rn_contiguous_split(n, L, S, g, C.byref(mx)))
    return list(g), mx.value


def net_units(desc: NetDesc):
    nu, npart = C.c_int32(), C.c_int32()
    ul = (C.c_int64 * 64)()
    pf = (C.c_int32 * 65)()
    pl = (C.c_int64 * 64)()
    _check(lib().rn_net_units(C.byref(desc), C.byref(nu), ul, C.byref(npart), pf, pl))
    return list(ul[:nu.value]), list(pf[:npart.value + 1]), list(pl[:npart.value])


KIND = {0: "conv", 1: "bn_gamma", 2: "bn_beta", 3: "fc_w", 4: "bias"}


def net_params(desc: NetDesc):
    """[(name, shape, kind)] in canonical order, from the library."""
    n, nt, nb = C.c_int64(), C.c_int32(), C.c_int32()
    _check(lib().rn_net_param_count(C.byref(desc), C.byref(n), C.byref(nt), C.byref(nb)))
    out = []
    for i in range(nt.value):
        nd, kind, unit = C.c_int32(), C.c_int32(), C.c_int32()
        shp = (C.c_int64 * 5)()
        name = C.create_string_buffer(128)
        _check(lib().rn_net_param_info(C.byref(desc), i, C.byref(nd), shp, C.byref(kind), C.byref(unit), name, 128))
        out.append((name.value.decode(), tuple(shp[:nd.value]), KIND[kind.value]))
    return out, n.value, nb.value


def local_transport_id() -> bytes:
    """An id selecting the in-process transport (include/rn.h rn_dist_desc):
    ranks = plans of this process on one device, one host thread per rank."""
    return b"RNLOCAL\0" + os.urandom(120)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().rn_nccl_unique_id(buf))
    return bytes(buf)


class Plan:
    """One rank's plan.  torch provides the workspace and the stream."""

    def __init__(self, desc: NetDesc, local_batch: int, dtype=RN_F32, rank=0, world=1, n_stages=1, genes=None,
                 micro_batches=1, nccl_id: bytes | None = None, stream=None, device=None, delayed=False):
        import torch
        self.torch = torch
        self.desc = desc
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        dd = DistDesc()
        dd.rank, dd.world, dd.n_stages, dd.micro_batches = rank, world, n_stages, micro_batches
        self._genes = None
        if genes is not None:
            self._genes = (C.c_int32 * len(genes))(*genes)
            dd.genes = C.cast(self._genes, C.POINTER(C.c_int32))
        if nccl_id is not None:
            C.memmove(dd.nccl_id, nccl_id, 128)
        self.h = C.c_void_p()
        ws = C.c_size_t()
        make = lib().rn_plan_delayed if delayed else lib().rn_plan
        _check(make(C.byref(desc), C.byref(dd), local_batch, dtype, C.c_void_p(self.stream.cuda_stream),
                    C.byref(self.h), C.byref(ws)))
        self.ws_bytes = ws.value
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        ptr = self.workspace.data_ptr()
        aligned = (ptr + 255) // 256 * 256
        _check(lib().rn_plan_bind(self.h, C.c_void_p(aligned), C.c_size_t(self.ws_bytes)))
        self.tensors, self.n_params, self.n_bn = net_params(desc)
        self.local_batch = local_batch

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                lib().rn_plan_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    # --- parameters ---
    def set_params(self, flat: np.ndarray):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check(lib().rn_set_params(self.h, a.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(a.size)))

    def get_params(self) -> np.ndarray:
        a = np.empty(self.n_params, dtype=np.float32)
        _check(lib().rn_get_params(self.h, a.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(a.size)))
        return a

    def get_grads(self) -> np.ndarray:
        a = np.empty(self.n_params, dtype=np.float32)
        _check(lib().rn_get_grads(self.h, a.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(a.size)))
        return a

    def get_bn_running(self):
        m = np.empty(self.n_bn, dtype=np.float32)
        v = np.empty(self.n_bn, dtype=np.float32)
        _check(lib().rn_get_bn_running(self.h, m.ctypes.data_as(C.POINTER(C.c_float)),
                                       v.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(self.n_bn)))
        return m, v

    def get_activation(self, unit: int, micro_batch: int, shape) -> np.ndarray:
        n = int(np.prod(shape))
        a = np.empty(n, dtype=np.float32)
        _check(lib().rn_get_activation(self.h, unit, micro_batch, a.ctypes.data_as(C.POINTER(C.c_float)),
                                       C.c_int64(n)))
        return a.reshape(shape)

    def get_unit_grad(self, unit: int, shape) -> np.ndarray:
        """dl/d(output of `unit`) of the last micro-batch of the last backward."""
        n = int(np.prod(shape))
        a = np.empty(n, dtype=np.float32)
        _check(lib().rn_get_unit_grad(self.h, unit, a.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(n)))
        return a.reshape(shape)

    def get_saved(self, unit: int, name: str, shape, micro_batch: int = 0) -> np.ndarray:
        """A saved forward tensor / backward temporary / BN statistics of `unit` (rn_get_saved)."""
        n = int(np.prod(shape))
        a = np.empty(n, dtype=np.float32)
        _check(lib().rn_get_saved(self.h, unit, name.encode(), micro_batch, a.ctypes.data_as(C.POINTER(C.c_float)),
                                  C.c_int64(n)))
        return a.reshape(shape)

    def gradcam(self, cls: int, map_dev):
        """rn_gradcam into a float32 device tensor of b x D x H x W (stream-ordered)."""
        _check(lib().rn_gradcam(self.h, C.c_int32(cls), C.c_void_p(map_dev.data_ptr()), C.c_int64(map_dev.numel())))

    # --- step ---
    def delayed_step(self, x_dev, y_dev, lr: float, want_loss=True):
        """rn_delayed_step (x_dev / y_dev may be None on stages that do not read them)."""
        loss = C.c_float()
        _check(lib().rn_delayed_step(self.h, C.c_void_p(x_dev.data_ptr() if x_dev is not None else 0),
                                     C.c_void_p(y_dev.data_ptr() if y_dev is not None else 0), C.c_float(lr),
                                     C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def forward(self, x_dev, y_dev, want_loss=True):
        loss = C.c_float()
        _check(lib().rn_forward(self.h, C.c_void_p(x_dev.data_ptr()), C.c_void_p(y_dev.data_ptr()),
                                C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def backward(self):
        _check(lib().rn_backward(self.h))

    def step(self, lr: float):
        _check(lib().rn_step(self.h, C.c_float(lr)))

    def train_step(self, x_dev, y_dev, lr: float, want_loss=False):
        """rn_train_step: forward + backward + SGD from device inputs (early per-unit SGD)."""
        loss = C.c_float()
        _check(lib().rn_train_step(self.h, C.c_void_p(x_dev.data_ptr()), C.c_void_p(y_dev.data_ptr()),
                                   C.c_float(lr), C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def train_step_host(self, x_host: np.ndarray, y_host: np.ndarray, lr: float) -> float:
        loss = C.c_float()
        _check(lib().rn_train_step_host(self.h, C.c_void_p(x_host.ctypes.data), C.c_void_p(y_host.ctypes.data),
                                        C.c_float(lr), C.byref(loss)))
        return loss.value

    def train_steps_host(self, xs, ys, lr: float) -> np.ndarray:
        """len(xs) steps from host batches (pinned numpy views recommended); the
        copy of batch i+1 overlaps step i.  Returns the per-step losses."""
        n = len(xs)
        assert len(ys) == n
        xp = (C.c_void_p * n)(*[C.c_void_p(x.ctypes.data) for x in xs])
        yp = (C.c_void_p * n)(*[C.c_void_p(y.ctypes.data) for y in ys])
        out = np.empty(n, dtype=np.float32)
        _check(lib().rn_train_steps_host(self.h, xp, yp, C.c_int32(n), C.c_float(lr),
                                         out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def set_option(self, key: str, value: int):
        _check(lib().rn_set_option(self.h, key.encode(), C.c_int64(value)))

    def query(self, key: str) -> float:
        v = C.c_double()
        _check(lib().rn_query(self.h, key.encode(), C.byref(v)))
        return v.value


def kernel_launches() -> int:
    return lib().rn_kernel_launches(None)


def op_conv3d(dtype, op, geom, a, b, out, impl=0, stream=None):
    """rn_op_conv3d on torch CUDA tensors (see include/rn.h)."""
    import torch
    g = (C.c_int32 * 12)(*[int(v) for v in geom])
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().rn_op_conv3d(dtype, op, g, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                              C.c_void_p(out.data_ptr()), impl, C.c_void_p(s.cuda_stream)))


def plan_describe(desc: NetDesc, local_batch, dtype=RN_F32, rank=0, world=1, n_stages=1, genes=None,
                  micro_batches=1):
    """rn_plan_describe: (local unit mask, [(unit, peer_stage, dir, bytes)], [(begin, end)])."""
    dd = DistDesc()
    dd.rank, dd.world, dd.n_stages, dd.micro_batches = rank, world, n_stages, micro_batches
    keep = None
    if genes is not None:
        keep = (C.c_int32 * len(genes))(*genes)
        dd.genes = C.cast(keep, C.POINTER(C.c_int32))
    cap = 256
    lu = (C.c_int32 * 64)()
    nx, nr = C.c_int32(), C.c_int32()
    xf = (C.c_int64 * (4 * cap))()
    rg = (C.c_int64 * (2 * cap))()
    _check(lib().rn_plan_describe(C.byref(desc), C.byref(dd), local_batch, dtype, lu, cap, C.byref(nx), xf,
                                  C.byref(nr), rg))
    nu = len(net_units(desc)[0])
    xfers = [tuple(xf[4 * i:4 * i + 4]) for i in range(nx.value)]
    return [bool(v) for v in lu[:nu]], xfers, [tuple(rg[2 * i:2 * i + 2]) for i in range(nr.value)]
