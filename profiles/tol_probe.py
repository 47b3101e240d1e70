"""Per-tensor gradient error of the CUDA step against the oracle (diagnostic for reading c19's
near-zero floor): for each parameter tensor prints max|ref|, max|ref|/gscale, max|delta| and the
scale-relative error with and without the floor, plus the oracle's near-tie residual count.

    python profiles/tol_probe.py [--bimodal]   (GPU box; writes one JSON line per config)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import dcgru  # noqa: E402
from paper_2507_11683_b200 import pgti  # noqa: E402
import test_gpu_parity as T  # noqa: E402


def probe(cfg, precision, B=None):
    env = (pgti, torch)
    c = (T._step_case_tc(env, cfg, B=B) if precision else T._step_case(env, cfg, B=B))
    g, gr = c["g"].astype(np.float64), c["g_ref"]
    gscale = float(np.max(np.abs(gr)))
    out, off = [], 0
    for name, shp in synth.param_shapes(c["cfg"]):
        n = int(np.prod(shp))
        d = np.abs(g[off:off + n] - gr[off:off + n])
        mref = float(np.max(np.abs(gr[off:off + n])))
        out.append(dict(t=name, ref=mref, ref_over_gscale=mref / gscale, dmax=float(d.max()),
                        e_plain=float(d.max() / mref) if mref else None,
                        e_floor1e3=float(d.max() / max(mref, 1e-3 * gscale))))
        off += n
    yref = c["fwd"]["yhat"]
    xo, yo = c["ref"].batch(c["ref"].plan(1, 0, epoch=0)[:c["B"]])
    resid = np.abs(yref - yo[..., :c["cfg"].F_out])
    near = {f"{t:g}": int((resid < t).sum()) for t in (1e-4, 1e-3, 1e-2)}
    return dict(cfg=c["cfg"].name, B=c["B"], precision=precision, gscale=gscale,
                loss_rel=abs(c["loss"] - c["loss_ref"]) / abs(c["loss_ref"]),
                residuals=int(resid.size), near_ties=near, tensors=out)


if __name__ == "__main__":
    cases = [(T.TC_CONFIGS[k], 1, None) for k in T.TC_CONFIGS] + \
        [(synth.CONFIGS["metr_la"], 1, 64), (synth.CONFIGS["pems_bay"], 1, 16)] + \
        [(T.SMALL_CONFIGS[k], 0, None) for k in T.SMALL_CONFIGS] + \
        [(synth.CONFIGS["metr_la"], 0, 64)]
    for cfg, prec, B in cases:
        print(json.dumps(probe(cfg, prec, B)), flush=True)
