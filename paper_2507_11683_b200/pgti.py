"""ctypes binding of libpgti (include/pgti.h): argument marshalling only.

Every entry point keeps the C name without the ``pgti_`` prefix.  Device buffers are torch
tensors (PyTorch is used for device memory, streams and process groups only); every step of
the path runs in libpgti's kernels.  There is no CPU fallback: if libpgti.so is missing or
fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpgti.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing -- build it with `python -m "
                      "paper_2507_11683_b200.build` (there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "TOO_FEW_ENTRIES", 3: "ZERO_VARIANCE", 4: "NONFINITE",
          5: "OUT_OF_RANGE", 6: "SHAPE", 7: "TOO_FEW_WINDOWS", 8: "ALIGNMENT", 9: "WORKSPACE",
          10: "CUDA", 11: "NCCL", 12: "UNSUPPORTED"}


class PgtiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pgti {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


_vp, _i32, _i64, _u64, _f32, _f64, _sz = (C.c_void_p, C.c_int32, C.c_int64, C.c_uint64,
                                          C.c_float, C.c_double, C.c_size_t)


class DcrnnDesc(C.Structure):
    _fields_ = [("N", _i32), ("F", _i32), ("F_out", _i32), ("L", _i32), ("H", _i32), ("K", _i32),
                ("T_in", _i32), ("T_out", _i32), ("B", _i32), ("precision", _i32),
                ("ld", _i64), ("nnz", _i64),
                ("a_rowptr", _vp), ("a_col", _vp), ("Pf_val", _vp), ("PbT_val", _vp),
                ("at_rowptr", _vp), ("at_col", _vp), ("Pb_val", _vp), ("PfT_val", _vp),
                ("win_rows", _i32), ("win_max", _i32),
                ("a_win_ptr", _vp), ("a_win_nodes", _vp), ("a_lcol", _vp),
                ("at_win_ptr", _vp), ("at_win_nodes", _vp), ("at_lcol", _vp),
                ("model", _i32), ("teacher_forcing", _i32), ("cheb", _i32)]


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_lib_last_error = _sig("pgti_last_error", C.c_char_p)
version = lambda: _sig("pgti_version", C.c_char_p)().decode()  # noqa: E731
_check_dev = _sig("pgti_check_device_error", C.c_int, _vp)
_graph_build = _sig("pgti_graph_build", C.c_int, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                    _vp, _vp, _vp, _vp)
_graph_windows = _sig("pgti_graph_windows", C.c_int, _i32, _vp, _vp, _i32, _vp, _vp, _vp,
                      C.POINTER(_i32))
_load = _sig("pgti_load_series", C.c_int, C.POINTER(_vp), _vp, _i64, _i64, _i64, _i64, _vp, _i64,
             _vp)
_stats = _sig("pgti_series_stats", C.c_int, _vp, _i64, C.c_int, _i64, _i64, _f64, _vp, _vp)
_normalize = _sig("pgti_series_normalize", C.c_int, _vp, _f64, _f64, _vp)
_stats_fin = _sig("pgti_stats_finalize", C.c_int, _vp, _f64, C.POINTER(_f64), C.POINTER(_f64))
_moments = _sig("pgti_series_moments", C.c_int, _vp, _i64, C.c_int, _i64, _i64, _vp, _vp,
                C.POINTER(_f64), C.POINTER(_f64), _vp)
_mean_losses = _sig("pgti_mean_losses", C.c_int, _vp, _vp, _i64, _vp, C.POINTER(_f64), _vp)
_info = _sig("pgti_series_info", C.c_int, _vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
             C.POINTER(_i64), C.POINTER(_i64))
_destroy = _sig("pgti_series_destroy", C.c_int, _vp)
_make_index = _sig("pgti_make_index", C.c_int, _vp, _i64, _i64, C.c_int, C.c_int, C.c_int, _u64,
                   _u64, C.c_int, C.c_int, _vp, C.POINTER(_i64), _vp)
_gather = _sig("pgti_gather_batch", C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp)
_num_params = _sig("pgti_dcrnn_num_params", _sz, C.POINTER(DcrnnDesc))
_desc_size = _sig("pgti_dcrnn_desc_size", _sz)()
if _desc_size != C.sizeof(DcrnnDesc):
    raise ImportError(f"libpgti's pgti_dcrnn_desc is {_desc_size} bytes, the binding's "
                      f"{C.sizeof(DcrnnDesc)}: rebuild the extension")
_ws_bytes = _sig("pgti_dcrnn_workspace_bytes", _sz, C.POINTER(DcrnnDesc))
_step = _sig("pgti_dcrnn_step", C.c_int, C.POINTER(DcrnnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _sz,
             _vp, _vp)
_step_idx = _sig("pgti_dcrnn_step_indexed", C.c_int, C.POINTER(DcrnnDesc), _vp, _vp, _vp, _vp,
                 _vp, _vp, _sz, _vp, _vp)
_loss = _sig("pgti_dcrnn_loss", C.c_int, C.POINTER(DcrnnDesc), _vp, _vp, _vp, _vp, _vp, _sz, _vp)
_diffuse = _sig("pgti_diffuse", C.c_int, C.POINTER(DcrnnDesc), _vp, _i64, _vp, _vp)
_diffuse_adj = _sig("pgti_diffuse_adjoint", C.c_int, C.POINTER(DcrnnDesc), _vp, _i64, _vp, _vp)
_uid = _sig("pgti_comm_unique_id", C.c_int, _vp)
_comm_init = _sig("pgti_comm_init", C.c_int, C.POINTER(_vp), _vp, C.c_int, C.c_int, C.c_int)
_allreduce = _sig("pgti_allreduce_grads", C.c_int, _vp, _vp, _sz, _vp)
_allreduce64 = _sig("pgti_allreduce_f64", C.c_int, _vp, _vp, _sz, _vp)
_comm_destroy = _sig("pgti_comm_destroy", C.c_int, _vp)
_adam = _sig("pgti_adam_step", C.c_int, _vp, _vp, _vp, _vp, _sz, _i64, _vp, _f32, _f32, _f32,
             _f32, _f32, _vp)


_prof_enable = _sig("pgti_profile_enable", C.c_int, C.c_int)
_prof_n = _sig("pgti_profile_num_classes", C.c_int)
_prof_name = _sig("pgti_profile_class_name", C.c_char_p, C.c_int)
_prof_read = _sig("pgti_profile_read", C.c_int, _vp, _vp, _vp, _vp, C.c_int)
_launch_count = _sig("pgti_launch_count", C.c_uint64)
_prof_timeline = _sig("pgti_profile_timeline", C.c_int, _vp, _vp, _vp, _vp, C.c_int,
                      C.POINTER(C.c_int))


def profile_timeline() -> list:
    """[(class, start_ms, end_ms, stream)] of the recorded eager launches (before profile_read)."""
    cnt = C.c_int(0)
    _ok(_prof_timeline(None, None, None, None, 0, C.byref(cnt)))
    n = cnt.value
    cls, st, en = np.zeros(n, np.int32), np.zeros(n), np.zeros(n)
    sid = np.zeros(n, np.int64)
    if n:
        _ok(_prof_timeline(cls.ctypes.data, st.ctypes.data, en.ctypes.data, sid.ctypes.data, n,
                           C.byref(cnt)))
    names = [_prof_name(i).decode() for i in range(_prof_n())]
    return [(names[c], float(a), float(b), int(s)) for c, a, b, s in zip(cls, st, en, sid)]


def profile_enable(on: bool = True):
    _ok(_prof_enable(int(on)))


def profile_read() -> dict:
    """{class: dict(ms, bytes, flops, launches)} of eager launches since the last read."""
    n = _prof_n()
    ms, by, fl = (np.zeros(n) for _ in range(3))
    la = np.zeros(n, np.int64)
    _ok(_prof_read(ms.ctypes.data, by.ctypes.data, fl.ctypes.data, la.ctypes.data, n))
    return {_prof_name(i).decode(): dict(ms=float(ms[i]), bytes=float(by[i]), flops=float(fl[i]),
                                         launches=int(la[i])) for i in range(n)}


def launch_count() -> int:
    return int(_launch_count())


def last_error() -> str:
    return _lib_last_error().decode()


def _ok(status: int):
    if status != 0:
        raise PgtiError(status, last_error())


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def set_gather_mode(mode: str):
    """K1 variant: "ldg" (LDG/STG.128) or "tma" (cp.async.bulk staging)."""
    assert mode in ("ldg", "tma")
    os.environ["PGTI_GATHER"] = mode


def check_device_error(stream=None):
    _ok(_check_dev(_stream(stream)))


# ------------------------------------------------------------------------------ graph
def graph_build(N: int, src, dst, w) -> dict:
    """Host CSR build of P_f, P_b^T (pattern A) and P_b, P_f^T (pattern A^T)."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    w = np.ascontiguousarray(w, np.float32)
    nnz = src.size
    out = dict(a_rowptr=np.zeros(N + 1, np.int32), a_col=np.zeros(nnz, np.int32),
               Pf_val=np.zeros(nnz, np.float32), PbT_val=np.zeros(nnz, np.float32),
               at_rowptr=np.zeros(N + 1, np.int32), at_col=np.zeros(nnz, np.int32),
               Pb_val=np.zeros(nnz, np.float32), PfT_val=np.zeros(nnz, np.float32))
    _ok(_graph_build(N, nnz, _ptr(src), _ptr(dst), _ptr(w), *(_ptr(out[k]) for k in (
        "a_rowptr", "a_col", "Pf_val", "PbT_val", "at_rowptr", "at_col", "Pb_val", "PfT_val"))))
    return out


def default_win_rows(N: int) -> int:
    """Rows per SpMM staging window (0 = gather neighbour rows straight from L2).  Round 2 (two
    vectors per lane, entry lists, 3 CTAs per SM at 16 rows): 16 rows beat 32 in the bf16 step,
    full PeMS 897 vs 870 and METR-LA 39.8 K vs 37.2 K samples/s (same box).  Round 1 (samples/s,
    no plan / 16 / 32 / 64 rows): METR-LA 30.8 K / 31.2 K / 31.7 K; PeMS-Bay 22.0 K / 22.6 K /
    22.6 K; PeMS-All-LA 2.74 K / 2.96 K / 3.01 K / 2.11 K; full PeMS 662 / 725 / 740 / 515.
    PGTI_WIN_ROWS overrides (A/B measurements)."""
    env = os.environ.get("PGTI_WIN_ROWS")
    if env is not None:
        return int(env)
    return 16


def graph_windows(N: int, rowptr, col, rows: int) -> dict:
    """pgti_graph_windows on one CSR pattern -> win_ptr, win_nodes, lcol (int16 bits), max."""
    rowptr = np.ascontiguousarray(rowptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    nnz = int(rowptr[N])
    nwin = (N + rows - 1) // rows if rows > 0 else 0
    win_ptr = np.zeros(nwin + 1, np.int32)
    win_nodes = np.zeros(max(nnz, 1), np.int32)
    lcol = np.zeros(max(nnz, 1), np.uint16)
    mx = _i32(0)
    _ok(_graph_windows(N, _ptr(rowptr), _ptr(col), rows, _ptr(win_ptr), _ptr(win_nodes),
                       _ptr(lcol), C.byref(mx)))
    return dict(win_ptr=win_ptr, win_nodes=win_nodes[:max(int(win_ptr[-1]), 1)].copy(),
                lcol=lcol.view(np.int16), max_union=int(mx.value))


def add_windows(csr: dict, N: int, rows: int | None = None) -> dict:
    """Adds the SpMM staging plans of both patterns to a graph_build dict (rows=0: none)."""
    rows = default_win_rows(N) if rows is None else rows
    out = dict(csr)
    if rows <= 0 or csr["a_col"].size == 0:
        out["win_rows"], out["win_max"] = 0, 0
        return out
    mx = 0
    for pat in ("a", "at"):
        w = graph_windows(N, csr[pat + "_rowptr"], csr[pat + "_col"], rows)
        out[pat + "_win_ptr"], out[pat + "_win_nodes"] = w["win_ptr"], w["win_nodes"]
        out[pat + "_lcol"] = w["lcol"]
        mx = max(mx, w["max_union"])
    out["win_rows"], out["win_max"] = rows, mx
    return out


# ------------------------------------------------------------------------------ series
class Series:
    """Handle over a caller-owned device buffer [nrows][ld] (kept alive here)."""

    def __init__(self, host_rows, row0: int, N: int, F: int, dev_buf, ld: int, stream=None):
        h = _vp()
        nrows = host_rows.shape[0]
        self._host = host_rows  # keep the source alive until the async copy completes
        self.buf = dev_buf
        _ok(_load(C.byref(h), _ptr(host_rows), row0, nrows, N, F, _ptr(dev_buf), ld,
                  _stream(stream)))
        self.h = h
        self.row0, self.nrows, self.N, self.F, self.ld = row0, nrows, N, F, ld

    def stats(self, S_tr: int, T_in: int, row_lo: int, row_hi: int, shift: float, dev_sums,
              stream=None):
        _ok(_stats(self.h, S_tr, T_in, row_lo, row_hi, shift, _ptr(dev_sums), _stream(stream)))

    def moments(self, S_tr: int, T_in: int, row_lo: int, row_hi: int, dev_sums, comm=None,
                stream=None):
        """pgti_series_moments: Alg. 1's (mu, sigma), summed over the ranks of `comm`."""
        mu, sigma = _f64(), _f64()
        _ok(_moments(self.h, S_tr, T_in, row_lo, row_hi, comm.h if comm is not None else None,
                     _ptr(dev_sums), C.byref(mu), C.byref(sigma), _stream(stream)))
        return mu.value, sigma.value

    def normalize(self, mu: float, sigma: float, stream=None):
        _ok(_normalize(self.h, mu, sigma, _stream(stream)))

    def info(self):
        v = [_i64() for _ in range(5)]
        _ok(_info(self.h, *(C.byref(x) for x in v)))
        return tuple(x.value for x in v)

    def make_index(self, win_lo, win_hi, T_in, T_out, B, seed, epoch, rank, shuffle, dev_idx,
                   stream=None) -> int:
        n = _i64()
        _ok(_make_index(self.h, win_lo, win_hi, T_in, T_out, B, seed, epoch, rank, int(shuffle),
                        _ptr(dev_idx), C.byref(n), _stream(stream)))
        return n.value

    def gather(self, dev_idx, B, T_in, T_out, x, y, stream=None):
        _ok(_gather(self.h, _ptr(dev_idx), B, T_in, T_out, _ptr(x), _ptr(y), _stream(stream)))

    def close(self):
        if self.h:
            _ok(_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------ model
class DCRNN:
    """pgti_dcrnn_desc + the device CSR arrays it points to."""

    def __init__(self, N, F, F_out, L, H, K, T_in, T_out, B, ld, csr_dev: dict | None,
                 precision: int = 0, model: int = 0, teacher_forcing: int = 0, cheb: bool = False):
        """model 0: stepwise stacked PGT-DCRNN; 1: Li et al. encoder-decoder (teacher_forcing:
        decoder fed the previous target instead of its own prediction).  cheb: diffusion blocks
        by the Chebyshev recurrence T_k = 2 P T_{k-1} - T_{k-2} (reading c25)."""
        self.csr = csr_dev or {}
        g = lambda k: _ptr(self.csr.get(k))  # noqa: E731
        nnz = int(self.csr["a_col"].numel()) if csr_dev else 0
        self.desc = DcrnnDesc(N, F, F_out, L, H, K, T_in, T_out, B, precision, ld, nnz,
                              g("a_rowptr"), g("a_col"), g("Pf_val"), g("PbT_val"),
                              g("at_rowptr"), g("at_col"), g("Pb_val"), g("PfT_val"),
                              int(self.csr.get("win_rows", 0)), int(self.csr.get("win_max", 0)),
                              g("a_win_ptr"), g("a_win_nodes"), g("a_lcol"),
                              g("at_win_ptr"), g("at_win_nodes"), g("at_lcol"),
                              int(model), self._tf_mask(teacher_forcing, T_out), int(bool(cheb)))
        self.model = int(model)
        self.N, self.F, self.F_out, self.L, self.H, self.K = N, F, F_out, L, H, K
        self.T_in, self.T_out, self.B, self.ld = T_in, T_out, B, ld

    @staticmethod
    def _tf_mask(tf, T_out: int) -> int:
        """True: every decoder step fed the target; False: none; an int: the step bit mask."""
        if tf is True:
            return (1 << max(T_out - 1, 0)) - 1
        return int(tf)

    def set_teacher_forcing(self, tf):
        """Per-step mask for the next steps (scheduled sampling draws one per training step)."""
        self.desc.teacher_forcing = self._tf_mask(tf, self.T_out)

    @property
    def M(self):
        return 2 * self.K + 1

    def num_params(self) -> int:
        n = _num_params(C.byref(self.desc))
        if n == 0:
            raise PgtiError(6, "invalid pgti_dcrnn_desc")
        return n

    def workspace_bytes(self) -> int:
        n = _ws_bytes(C.byref(self.desc))
        if n == 0:
            raise PgtiError(6, "invalid pgti_dcrnn_desc")
        return n

    def act_dump_floats(self) -> int:
        R = self.N * self.B
        steps = self.T_in + (self.T_out if self.model else 0)
        return steps * self.L * 4 * R * self.H + self.T_out * R * self.F_out

    def step(self, params, grads, x, y, loss_dev, workspace, act_dump=None, stream=None):
        _ok(_step(C.byref(self.desc), _ptr(params), _ptr(grads), _ptr(x), _ptr(y),
                  _ptr(loss_dev), _ptr(workspace), workspace.numel() * workspace.element_size(),
                  _ptr(act_dump), _stream(stream)))

    def step_indexed(self, params, grads, series, dev_idx, loss_dev, workspace, act_dump=None,
                     stream=None):
        """pgti_dcrnn_step_indexed: zero-copy step reading windows from `series` (a Series)."""
        _ok(_step_idx(C.byref(self.desc), _ptr(params), _ptr(grads), series.h, _ptr(dev_idx),
                      _ptr(loss_dev), _ptr(workspace),
                      workspace.numel() * workspace.element_size(), _ptr(act_dump),
                      _stream(stream)))

    def loss(self, params, x, y, loss_dev, workspace, stream=None):
        """pgti_dcrnn_loss: forward + loss only (validation)."""
        _ok(_loss(C.byref(self.desc), _ptr(params), _ptr(x), _ptr(y), _ptr(loss_dev),
                  _ptr(workspace), workspace.numel() * workspace.element_size(),
                  _stream(stream)))

    def diffuse(self, X, W, out, stream=None):
        _ok(_diffuse(C.byref(self.desc), _ptr(X), W, _ptr(out), _stream(stream)))

    def diffuse_adjoint(self, dT, W, dZ, stream=None):
        _ok(_diffuse_adj(C.byref(self.desc), _ptr(dT), W, _ptr(dZ), _stream(stream)))


def csr_to_device(csr: dict, device):
    import torch
    return {k: torch.from_numpy(v).to(device) if isinstance(v, np.ndarray) else v
            for k, v in csr.items()}


# ------------------------------------------------------------------------------ comm / adam
def stats_finalize(sums, shift: float):
    """pgti_stats_finalize: host sums (s0, s1, s2) about `shift` -> (mean, population var)."""
    a = (_f64 * 3)(*[float(v) for v in sums])
    mean, var = _f64(), _f64()
    _ok(_stats_fin(C.cast(a, _vp), shift, C.byref(mean), C.byref(var)))
    return mean.value, var.value


def mean_losses(dev_losses, n: int, dev_scratch, comm=None, stream=None) -> float:
    """pgti_mean_losses: mean of n device per-batch losses over every rank of `comm`."""
    out = _f64()
    _ok(_mean_losses(comm.h if comm is not None else None, _ptr(dev_losses), n,
                     _ptr(dev_scratch), C.byref(out), _stream(stream)))
    return out.value


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _ok(_uid(C.cast(buf, _vp)))
    return bytes(buf)


class Comm:
    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = _vp()
        _ok(_comm_init(C.byref(h), C.cast(buf, _vp), rank, world, device))
        self.h = h

    def allreduce_grads(self, grads, stream=None):
        _ok(_allreduce(self.h, _ptr(grads), grads.numel(), _stream(stream)))

    def allreduce_f64(self, buf, stream=None):
        _ok(_allreduce64(self.h, _ptr(buf), buf.numel(), _stream(stream)))

    def close(self):
        if self.h:
            _ok(_comm_destroy(self.h))
            self.h = None


def adam_step(params, grads, m, v, step: int, lr: float, beta1=0.9, beta2=0.999, eps=1e-8,
              grad_scale=1.0, dev_step=None, stream=None):
    _ok(_adam(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), params.numel(), step, _ptr(dev_step),
              lr, beta1, beta2, eps, grad_scale, _stream(stream)))
