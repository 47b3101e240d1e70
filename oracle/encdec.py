"""Li et al. DCRNN encoder-decoder ("the PyTorch
implementation of DCRNN" that the paper's optimisations also apply to), float64.

Model (reading c24; Li et al. 2018 [ext]):
* Encoder: the L-layer DCGRU stack of oracle.dcgru (same cell, same per-layer parameter layout,
  C_in = F + H at layer 0, 2H above) run over x_0 .. x_{T_in-1}, hidden states from 0.  No
  readout on the encoder.
* Decoder: a second L-layer DCGRU stack (own parameters; layer 0 has C_in = F_out + H) that
  starts from the encoder's final hidden states and runs T_out steps.  Its layer-0 input is the
  GO symbol (zeros, F_out channels) at step 0 and the previous step's prediction at step s > 0
  ("fed its own predictions"); with teacher forcing it is the previous ground truth
  y_{s-1}[..., :F_out] instead.  teacher_forcing is per step (reading c24): True = every step,
  False = none, an int = a bit mask (bit s-1 set: step s >= 1 is fed the target) -- the per-step
  coin flips of Li et al.'s scheduled sampling, drawn by the caller.
* Output projection on every decoder step: yhat_s = H^L_s W_out + b_out (F_out channels).
* Loss = mean |yhat - y[..., :F_out]|, subgradient 0 at ties (reading c20).
* Flat parameter layout: encoder layers (W_ru[M][C_in][2H], b_ru, W_c[M][C_in][H], b_c), then
  decoder layers (same, decoder C_in), then W_out[H][F_out], b_out[F_out].  For the METR-LA
  configuration (L 2, H 64, K 2, F 2, F_out 1) that is 372,353 values, Li et al.'s count [ext].

`forward` is written out with numpy; `loss_and_grad` differentiates a torch float64 transcription
of the same forward with torch.autograd (a library primitive for the reverse mode; pinned by
central finite differences and by agreement with the numpy forward in tests).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from .dcgru import Dims, _feats_batched, _sigmoid


def layer_shapes(d: Dims):
    """[(name, shape)] of the flat parameter vector, in order."""
    out = []
    for part, f0 in (("enc", d.F), ("dec", d.F_out)):
        for l in range(d.L):
            c = (f0 if l == 0 else d.H) + d.H
            out += [(f"{part}{l}.W_ru", (d.M, c, 2 * d.H)), (f"{part}{l}.b_ru", (2 * d.H,)),
                    (f"{part}{l}.W_c", (d.M, c, d.H)), (f"{part}{l}.b_c", (d.H,))]
    out += [("W_out", (d.H, d.F_out)), ("b_out", (d.F_out,))]
    return out


def num_params(d: Dims) -> int:
    return sum(int(np.prod(s)) for _, s in layer_shapes(d))


def unpack(theta, d: Dims) -> dict:
    theta = np.asarray(theta, np.float64)
    out, off = {}, 0
    for name, shape in layer_shapes(d):
        n = int(np.prod(shape))
        out[name] = theta[off:off + n].reshape(shape)
        off += n
    assert off == theta.size, (off, theta.size)
    return out


def _cell(p: dict, pre: str, d: Dims, Pf, Pb, inp, Hprev):
    """One DCGRU cell (Li et al. Eq. 2-3 [ext]; oracle.dcgru's reading c1)."""
    c_in = inp.shape[-1] + d.H
    TZ = _feats_batched(Pf, Pb, np.concatenate([inp, Hprev], axis=-1), d.K, d.cheb)
    G = TZ @ p[pre + ".W_ru"].reshape(d.M * c_in, 2 * d.H) + p[pre + ".b_ru"]
    r, u = _sigmoid(G[..., :d.H]), _sigmoid(G[..., d.H:])
    TZ2 = _feats_batched(Pf, Pb, np.concatenate([inp, r * Hprev], axis=-1), d.K, d.cheb)
    c = np.tanh(TZ2 @ p[pre + ".W_c"].reshape(d.M * c_in, d.H) + p[pre + ".b_c"])
    return u * Hprev + (1.0 - u) * c


def fed_truth(teacher_forcing, s: int) -> bool:
    """Whether decoder step s (>= 1) is fed the previous target (see the module docstring)."""
    if isinstance(teacher_forcing, (bool, np.bool_)):
        return bool(teacher_forcing)
    return bool((int(teacher_forcing) >> (s - 1)) & 1)


def forward(theta, d: Dims, Pf, Pb, x, y=None, teacher_forcing=False) -> dict:
    """x[B][T_in][N][F], y[B][T_out][N][F].  Returns dict(yhat[B][T_out][N][F_out], loss,
    H_enc = the encoder's final hidden states [L][B][N][H])."""
    p = unpack(theta, d)
    x = np.asarray(x, np.float64)
    B = x.shape[0]
    H = [np.zeros((B, d.N, d.H)) for _ in range(d.L)]
    for t in range(d.T_in):
        inp = x[:, t]
        for l in range(d.L):
            H[l] = _cell(p, f"enc{l}", d, Pf, Pb, inp, H[l])
            inp = H[l]
    H_enc = [h.copy() for h in H]
    yhat = np.zeros((B, d.T_out, d.N, d.F_out))
    prev = np.zeros((B, d.N, d.F_out))                  # GO symbol
    for s in range(d.T_out):
        inp = prev
        for l in range(d.L):
            H[l] = _cell(p, f"dec{l}", d, Pf, Pb, inp, H[l])
            inp = H[l]
        yhat[:, s] = H[d.L - 1] @ p["W_out"] + p["b_out"]
        prev = (np.asarray(y, np.float64)[:, s, :, :d.F_out] if fed_truth(teacher_forcing, s + 1)
                else yhat[:, s])
    out = dict(yhat=yhat, H_enc=H_enc)
    if y is not None:
        y = np.asarray(y, np.float64)
        out["loss"] = float(np.mean(np.abs(yhat - y[..., :d.F_out])))
    return out


def loss_and_grad(theta, d: Dims, Pf, Pb, x, y, teacher_forcing=False):
    """(loss, d loss / d theta) by torch float64 autograd of the same forward."""
    import torch
    th = torch.tensor(np.asarray(theta, np.float64), requires_grad=True)
    Pft = torch.tensor(np.asarray(Pf.toarray() if hasattr(Pf, "toarray") else Pf, np.float64))
    Pbt = torch.tensor(np.asarray(Pb.toarray() if hasattr(Pb, "toarray") else Pb, np.float64))
    xt = torch.tensor(np.asarray(x, np.float64))
    yt = torch.tensor(np.asarray(y, np.float64))
    p, off = {}, 0
    for name, shape in layer_shapes(d):
        n = int(np.prod(shape))
        p[name] = th[off:off + n].reshape(shape)
        off += n

    def feats(Z):                                       # [B][N][C] -> [B][N][M][C]
        out = [Z]
        for P in (Pft, Pbt):
            prev, T = Z, Z
            for k in range(d.K):
                PT = torch.einsum("ij,bjc->bic", P, T)
                T, prev = (2.0 * PT - prev if d.cheb and k >= 1 else PT), T
                out.append(T)
        return torch.stack(out, 2)

    def cell(pre, inp, Hprev):
        TZ = feats(torch.cat([inp, Hprev], -1))
        G = torch.einsum("bnmc,mcj->bnj", TZ, p[pre + ".W_ru"]) + p[pre + ".b_ru"]
        r, u = torch.sigmoid(G[..., :d.H]), torch.sigmoid(G[..., d.H:])
        TZ2 = feats(torch.cat([inp, r * Hprev], -1))
        c = torch.tanh(torch.einsum("bnmc,mcj->bnj", TZ2, p[pre + ".W_c"]) + p[pre + ".b_c"])
        return u * Hprev + (1.0 - u) * c

    B = xt.shape[0]
    H = [torch.zeros(B, d.N, d.H, dtype=torch.float64) for _ in range(d.L)]
    for t in range(d.T_in):
        inp = xt[:, t]
        for l in range(d.L):
            H[l] = cell(f"enc{l}", inp, H[l])
            inp = H[l]
    prev = torch.zeros(B, d.N, d.F_out, dtype=torch.float64)
    outs = []
    for s in range(d.T_out):
        inp = prev
        for l in range(d.L):
            H[l] = cell(f"dec{l}", inp, H[l])
            inp = H[l]
        yh = H[d.L - 1] @ p["W_out"] + p["b_out"]
        outs.append(yh)
        prev = yt[:, s, :, :d.F_out] if fed_truth(teacher_forcing, s + 1) else yh
    yhat = torch.stack(outs, 1)
    loss = torch.mean(torch.abs(yhat - yt[..., :d.F_out]))
    (g,) = torch.autograd.grad(loss, th)
    return float(loss.detach()), g.numpy(), yhat.detach().numpy()
