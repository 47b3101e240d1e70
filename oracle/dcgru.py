"""Stepwise stacked DCGRU (PGT-DCRNN), MAE loss and its reverse mode, float64.

Model (readings c1-c7):
* PGT-DCRNN feeds "one temporal slice at a time", "maintains
  and updates a hidden state across time steps, producing an output at each
  step"; it implements Li et al.'s diffusion convolution.  P:168 -- each layer
  aggregates spatial neighbours inside "gated mechanisms of recurrent networks".
* Li et al. Eq. 2-3 [ext]: diffusion features of Z are
  T(Z) = [Z, P_f Z, ..., P_f^K Z, P_b Z, ..., P_b^K Z] (M = 2K+1 blocks, plain
  matrix powers, K = hops -- readings c2, c3); the DCGRU is
      r = sigma(T([in, H]) W_r + b_r),  u = sigma(T([in, H]) W_u + b_u)
      c = tanh(T([in, r*H]) W_c + b_c),  H' = u*H + (1-u)*c.
* L layers are stacked; layer l > 0 takes H^{l-1}_t as input.  H starts at 0.
  The readout y_hat = H^L W_out + b_out is taken on the last T_out steps
  (reading c6), predicting channel 0 .. F_out-1 (reading c7).
* Loss = mean |y_hat - y[..., :F_out]| over B T_out N F_out (P:347 MAE),
  subgradient 0 at ties (reading c20).
* Parameter layout (flat): per layer W_ru[M][C_in][2H], b_ru[2H],
  W_c[M][C_in][H], b_c[H]; then W_out[H][F_out], b_out[F_out].  Block m = 0 is
  the identity, 1..K are P_f^k, K+1..2K are P_b^k; C_in lists input channels
  then hidden; gate columns r = [0,H), u = [H,2H).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class Dims:
    N: int
    F: int
    F_out: int
    L: int
    H: int
    K: int
    T_in: int
    T_out: int
    cheb: bool = False  # reading c25: blocks by the Chebyshev recurrence instead of powers

    @property
    def M(self) -> int:
        return 2 * self.K + 1

    def c_in(self, l: int) -> int:
        return (self.F if l == 0 else self.H) + self.H

    def f_in(self, l: int) -> int:
        return self.F if l == 0 else self.H

    @staticmethod
    def of(cfg) -> "Dims":
        return Dims(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out,
                    bool(getattr(cfg, "cheb", False)))


def unpack(theta: np.ndarray, d: Dims):
    """Views of the flat parameter vector in the layout of the module docstring."""
    theta = np.asarray(theta, dtype=np.float64)
    off = 0

    def take(*shape):
        nonlocal off
        n = int(np.prod(shape))
        out = theta[off:off + n].reshape(shape)
        off += n
        return out

    layers = []
    for l in range(d.L):
        c = d.c_in(l)
        layers.append(dict(W_ru=take(d.M, c, 2 * d.H), b_ru=take(2 * d.H),
                           W_c=take(d.M, c, d.H), b_c=take(d.H)))
    W_out, b_out = take(d.H, d.F_out), take(d.F_out)
    assert off == theta.size, f"theta has {theta.size} entries, layout needs {off}"
    return layers, W_out, b_out


def num_params(d: Dims) -> int:
    n = 0
    for l in range(d.L):
        n += d.M * d.c_in(l) * 3 * d.H + 3 * d.H
    return n + d.H * d.F_out + d.F_out


def diffusion_features(Pf, Pb, Z: np.ndarray, K: int, cheb: bool = False) -> np.ndarray:
    """T(Z) for Z[N][W]: [Z, P_f Z, ..., P_f^K Z, P_b Z, ..., P_b^K Z] -> [M][N][W].
    P^k Z is evaluated as k successive products (the definition of the power).
    cheb (reading c25, Li et al.'s DCRNN code [ext]): block k of each direction is instead the
    Chebyshev recurrence T_0 = Z, T_1 = P Z, T_k = 2 P T_{k-1} - T_{k-2}, restarted from Z for
    each direction."""
    out = [Z]
    for P in (Pf, Pb):
        prev, T = Z, Z
        for k in range(K):
            if cheb and k >= 1:
                T, prev = 2.0 * np.asarray(P @ T) - prev, T
            else:
                T, prev = np.asarray(P @ T), T
            out.append(np.asarray(T))
    return np.stack(out)


def diffusion_adjoint(Pf, Pb, dT: np.ndarray, K: int, cheb: bool = False) -> np.ndarray:
    """Transpose of diffusion_features: dZ = dT_0 + sum_k (P_f^k)^T dT_k
    + sum_k (P_b^k)^T dT_{K+k}, with (P^k)^T = (P^T)^k applied k times.
    cheb: dZ = dT_0 + sum_k C_k(P_f^T) dT_k + sum_k C_k(P_b^T) dT_{K+k}, the transpose of a
    polynomial in P being the same polynomial in P^T; C_k(A) X is evaluated by the forward
    recurrence C_0 X = X, C_1 X = A X, C_k X = 2 A C_{k-1} X - C_{k-2} X."""
    PfT, PbT = Pf.T, Pb.T
    if cheb:
        dZ = np.array(dT[0], dtype=np.float64, copy=True)
        for A, base in ((PfT, 0), (PbT, K)):
            for k in range(1, K + 1):
                prev, cur = np.asarray(dT[base + k]), np.asarray(A @ dT[base + k])
                for _ in range(k - 1):
                    cur, prev = 2.0 * np.asarray(A @ cur) - prev, cur
                dZ += cur
        return dZ
    dZ = np.array(dT[0], dtype=np.float64, copy=True)
    for k in range(1, K + 1):
        a = dT[k]
        for _ in range(k):
            a = PfT @ a
        dZ += np.asarray(a)
        b = dT[K + k]
        for _ in range(k):
            b = PbT @ b
        dZ += np.asarray(b)
    return dZ


def _feats_batched(Pf, Pb, Z: np.ndarray, K: int, cheb: bool = False) -> np.ndarray:
    """T(Z) for a batch Z[B][N][C] -> [B][N][M*C] (column m*C + c = block m, channel c)."""
    B, N, C = Z.shape
    T = diffusion_features(Pf, Pb, Z.transpose(1, 0, 2).reshape(N, B * C), K, cheb)
    M = T.shape[0]
    return T.reshape(M, N, B, C).transpose(2, 1, 0, 3).reshape(B, N, M * C)


def _adjoint_batched(Pf, Pb, dT: np.ndarray, K: int, C: int, cheb: bool = False) -> np.ndarray:
    """Transpose of _feats_batched: dT[B][N][M*C] -> dZ[B][N][C]."""
    B, N, MC = dT.shape
    M = MC // C
    d = dT.reshape(B, N, M, C).transpose(2, 1, 0, 3).reshape(M, N, B * C)
    return diffusion_adjoint(Pf, Pb, d, K, cheb).reshape(N, B, C).transpose(1, 0, 2)


def _sigmoid(a):
    return 1.0 / (1.0 + np.exp(-a))


def forward(theta, d: Dims, Pf, Pb, x: np.ndarray, y: np.ndarray | None = None):
    """x[B][T_in][N][F], y[B][T_out][N][F] (float64 of the standardised float32
    snapshots).  Returns dict(loss, yhat[B][T_out][N][F_out], acts, cache)."""
    layers, W_out, b_out = unpack(theta, d)
    x = np.asarray(x, np.float64)
    B = x.shape[0]
    assert x.shape == (B, d.T_in, d.N, d.F), x.shape
    H = [np.zeros((B, d.N, d.H)) for _ in range(d.L)]
    yhat = np.zeros((B, d.T_out, d.N, d.F_out))
    cache = []
    for t in range(d.T_in):
        inp = x[:, t]
        step = []
        for l in range(d.L):
            p = layers[l]
            c_in = d.c_in(l)
            Hprev = H[l]
            TZ = _feats_batched(Pf, Pb, np.concatenate([inp, Hprev], axis=-1), d.K, d.cheb)
            G = TZ @ p["W_ru"].reshape(d.M * c_in, 2 * d.H) + p["b_ru"]
            r, u = _sigmoid(G[..., :d.H]), _sigmoid(G[..., d.H:])
            TZ2 = _feats_batched(Pf, Pb, np.concatenate([inp, r * Hprev], axis=-1), d.K, d.cheb)
            c = np.tanh(TZ2 @ p["W_c"].reshape(d.M * c_in, d.H) + p["b_c"])
            Hn = u * Hprev + (1.0 - u) * c
            step.append(dict(Hprev=Hprev, TZ=TZ, TZ2=TZ2, r=r, u=u, c=c, H=Hn))
            H[l] = Hn
            inp = Hn
        cache.append(step)
        if t >= d.T_in - d.T_out:
            yhat[:, t - (d.T_in - d.T_out)] = H[d.L - 1] @ W_out + b_out
    out = dict(yhat=yhat, cache=cache)
    if y is not None:
        y = np.asarray(y, np.float64)
        assert y.shape == (B, d.T_out, d.N, d.F), y.shape
        out["loss"] = float(np.mean(np.abs(yhat - y[..., :d.F_out])))
    return out


def backward(theta, d: Dims, Pf, Pb, x, y, fwd=None):
    """Reverse mode of forward() + MAE (BPTT over t = T_in-1..0, l = L-1..0).
    Returns (loss, grad[theta.size] float64, fwd)."""
    if fwd is None:
        fwd = forward(theta, d, Pf, Pb, x, y)
    layers, W_out, b_out = unpack(theta, d)
    y = np.asarray(y, np.float64)
    B = y.shape[0]
    grads_l = [dict(W_ru=np.zeros_like(p["W_ru"]), b_ru=np.zeros_like(p["b_ru"]),
                    W_c=np.zeros_like(p["W_c"]), b_c=np.zeros_like(p["b_c"])) for p in layers]
    resid = fwd["yhat"] - y[..., :d.F_out]
    count = resid.size
    dyhat = np.sign(resid) / count                        # d mean|.| ; 0 at ties
    dW_out = np.zeros_like(W_out)
    db_out = dyhat.sum(axis=(0, 1, 2))
    dH = [np.zeros((B, d.N, d.H)) for _ in range(d.L)]
    for t in reversed(range(d.T_in)):
        if t >= d.T_in - d.T_out:
            tt = t - (d.T_in - d.T_out)
            HL = fwd["cache"][t][d.L - 1]["H"]
            dW_out += np.einsum("bnh,bno->ho", HL, dyhat[:, tt])
            dH[d.L - 1] = dH[d.L - 1] + dyhat[:, tt] @ W_out.T
        for l in reversed(range(d.L)):
            cc = fwd["cache"][t][l]
            p, g = layers[l], grads_l[l]
            c_in, f_in = d.c_in(l), d.f_in(l)
            Hprev, r, u, c = cc["Hprev"], cc["r"], cc["u"], cc["c"]
            dHn = dH[l]
            dU = dHn * (Hprev - c)
            dHprev = dHn * u
            dCpre = dHn * (1.0 - u) * (1.0 - c * c)
            g["W_c"] += np.einsum("bnk,bnj->kj", cc["TZ2"], dCpre).reshape(g["W_c"].shape)
            g["b_c"] += dCpre.sum(axis=(0, 1))
            dTZ2 = dCpre @ p["W_c"].reshape(d.M * c_in, d.H).T
            dZ2 = _adjoint_batched(Pf, Pb, dTZ2, d.K, c_in, d.cheb)
            dinp = dZ2[..., :f_in].copy()
            drH = dZ2[..., f_in:]
            dHprev += drH * r
            dG = np.concatenate([drH * Hprev * r * (1.0 - r), dU * u * (1.0 - u)], axis=-1)
            g["W_ru"] += np.einsum("bnk,bnj->kj", cc["TZ"], dG).reshape(g["W_ru"].shape)
            g["b_ru"] += dG.sum(axis=(0, 1))
            dTZ = dG @ p["W_ru"].reshape(d.M * c_in, 2 * d.H).T
            dZ = _adjoint_batched(Pf, Pb, dTZ, d.K, c_in, d.cheb)
            dinp += dZ[..., :f_in]
            dHprev += dZ[..., f_in:]
            dH[l] = dHprev
            if l > 0:
                dH[l - 1] = dH[l - 1] + dinp
    flat = []
    for g in grads_l:
        flat += [g["W_ru"].ravel(), g["b_ru"], g["W_c"].ravel(), g["b_c"]]
    flat += [dW_out.ravel(), db_out]
    return fwd["loss"], np.concatenate(flat), fwd


def activations(fwd, d: Dims):
    """Per (t, l) H, r, u, c as arrays [T_in][L][4][B][N][H], and yhat."""
    acts = np.stack([np.stack([np.stack([s["H"], s["r"], s["u"], s["c"]]) for s in step])
                     for step in fwd["cache"]])
    return acts, fwd["yhat"]
