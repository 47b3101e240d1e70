"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import synth


def scale_rel(a, ref) -> float:
    """Scale-relative error max|a - ref| / max|ref| (DESIGN reading c19)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(a - ref)) / (den if den > 0 else 1.0))


def ld_of(cfg) -> int:
    return (cfg.N * cfg.F + 3) // 4 * 4


def load_series(pgti, torch, v_rows, row0, cfg, mu=None, sigma=None):
    """Raw rows -> device series (+ normalise with the given stats)."""
    ld = ld_of(cfg)
    host = np.ascontiguousarray(v_rows, np.float32)
    buf = torch.empty(host.shape[0] * ld, dtype=torch.float32, device="cuda")
    s = pgti.Series(host, row0, cfg.N, cfg.F, buf, ld)
    if mu is not None:
        s.normalize(mu, sigma)
    return s


def model_for(pgti, torch, cfg, graph, precision=0, win_rows=None):
    """win_rows: SpMM staging window (None = the library default, 0 = no staging plan)."""
    csr = pgti.graph_build(cfg.N, *graph)
    csr = pgti.add_windows(csr, cfg.N, win_rows)
    csr = pgti.csr_to_device(csr, "cuda")
    return pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out, cfg.B,
                      ld_of(cfg), csr, precision, cheb=getattr(cfg, "cheb", False))


def run_step(pgti, torch, model, theta, x, y, dump=True):
    n = model.num_params()
    params = torch.from_numpy(np.ascontiguousarray(theta, np.float32)).cuda()
    grads = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
    loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    act = torch.empty(model.act_dump_floats(), dtype=torch.float32, device="cuda") if dump else None
    model.step(params, grads, x, y, loss, ws, act)
    pgti.check_device_error()
    return (float(loss.item()), grads.cpu().numpy(),
            act.cpu().numpy() if dump else None)


def split_dump(act, cfg, B):
    """act_dump -> (acts[T_in][L][4][N][B][H], yhat[T_out][N][B][F_out])."""
    R = cfg.N * B
    n1 = cfg.T_in * cfg.L * 4 * R * cfg.H
    acts = act[:n1].reshape(cfg.T_in, cfg.L, 4, cfg.N, B, cfg.H)
    yhat = act[n1:].reshape(cfg.T_out, cfg.N, B, cfg.F_out)
    return acts, yhat


SMALL_CONFIGS = {
    # ragged: N*B not a multiple of the 64-row tile, N*F not a multiple of 4
    "tiny2": synth.Config("tiny2", N=12, E=60, F=2, T_in=3, T_out=2, L=2, H=16, K=2, B=3),
    "cp": synth.CONFIGS["chickenpox"],
    "odd": synth.Config("odd", N=33, E=80, F=3, T_in=5, T_out=5, L=2, H=64, K=1, B=5, F_out=2),
    "k0": synth.Config("k0", N=9, E=40, F=1, T_in=4, T_out=3, L=3, H=16, K=0, B=2),
    "k3": synth.Config("k3", N=17, E=50, F=2, T_in=4, T_out=2, L=1, H=32, K=3, B=7),
}
