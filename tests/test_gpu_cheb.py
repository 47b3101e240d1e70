"""Chebyshev-recurrence diffusion blocks (desc.cheb = 1, reading c25) through the
C ABI against the float64 oracle: the diffusion and its adjoint (Clenshaw in the fp32 path), the
stepwise training step in fp32 (1e-5) and on the bf16 tcgen05 path (2e-2), and the Li et al.
encoder-decoder."""
import numpy as np
import pytest

import synth
from gpu_util import ld_of, load_series, model_for, run_step, scale_rel
from oracle import dcgru, encdec, pipeline, transitions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_11683_b200 import build
    build.build()
    from paper_2507_11683_b200 import pgti
    return pgti, torch


def _graph(N, kind):
    return {"er": lambda: synth.random_graph(N, 0.15, seed=N),
            "knn": lambda: synth.make_graph(N, 8),
            "ring": lambda: synth.ring_graph(N)}[kind]()


@pytest.mark.parametrize("N,W,K,graph,rows", [(37, 24, 3, "er", 7), (207, 4096, 2, "knn", None),
                                               (64, 128, 4, "ring", 0), (100, 40, 5, "knn", 32),
                                               (30, 8, 2, "er", 0)])
def test_cheb_diffusion_and_adjoint_vs_oracle(env, N, W, K, graph, rows):
    pgti, torch = env
    g = _graph(N, graph)
    cfg = synth.Config("d", N=N, E=10, F=1, T_in=1, T_out=1, L=1, H=16, K=K, B=1, cheb=True)
    model = model_for(pgti, torch, cfg, g, win_rows=rows)
    assert model.desc.cheb == 1
    Pf, Pb = transitions.transition_matrices(N, *g)
    rng = np.random.default_rng(K)
    Z = rng.normal(size=(N, W)).astype(np.float32)
    M = 2 * K + 1
    out = torch.empty(M * N * W, device="cuda")
    model.diffuse(torch.from_numpy(Z).cuda(), W, out)
    want = dcgru.diffusion_features(Pf, Pb, Z.astype(np.float64), K, cheb=True)
    got = out.cpu().numpy().reshape(M, N, W)
    for m in range(M):  # Chebyshev blocks grow like 2^k: relative to each block's own scale
        assert scale_rel(got[m], want[m]) <= 1e-6, m
    dT = rng.normal(size=(M, N, W)).astype(np.float32)
    dZ = torch.empty(N * W, device="cuda")
    model.diffuse_adjoint(torch.from_numpy(dT).cuda(), W, dZ)
    want = dcgru.diffusion_adjoint(Pf, Pb, dT.astype(np.float64), K, cheb=True)
    assert scale_rel(dZ.cpu().numpy().reshape(N, W), want) <= 1e-6


def test_cheb_k1_is_the_power_series(env):
    """With K = 1 the two bases coincide (T_1 = P Z): identical bits."""
    pgti, torch = env
    N, W = 50, 64
    g = _graph(N, "knn")
    res = []
    for cheb in (False, True):
        cfg = synth.Config("d", N=N, E=10, F=1, T_in=1, T_out=1, L=1, H=16, K=1, B=1, cheb=cheb)
        m = model_for(pgti, torch, cfg, g)
        Z = torch.from_numpy(np.random.default_rng(0).normal(size=(N, W)).astype(np.float32))
        out = torch.empty(3 * N * W, device="cuda")
        m.diffuse(Z.cuda(), W, out)
        dZ = torch.empty(N * W, device="cuda")
        m.diffuse_adjoint(out, W, dZ)
        res.append((out.cpu().numpy(), dZ.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def _step(env, cfg, precision, seed=0):
    pgti, torch = env
    ref = pipeline.Reference(cfg)
    assert ref.d.cheb
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0, epoch=seed)[:cfg.B]
    idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(idx, cfg.B, cfg.T_in, cfg.T_out, x, y)
    model = model_for(pgti, torch, cfg, ref.graph, precision=precision)
    theta = synth.make_params(cfg, seed=synth.SEED_PARAMS + seed, kind="random")
    loss, g, _ = run_step(pgti, torch, model, theta, x, y, dump=False)
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    assert np.min(np.abs(fwd["yhat"] - yo[..., :cfg.F_out])) > 1e-5
    return loss, g, loss_ref, g_ref


def _check(cfg, loss, g, loss_ref, g_ref, tol):
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    gscale = np.max(np.abs(g_ref))
    off = 0
    for name, shp in synth.param_shapes(cfg):
        n = int(np.prod(shp))
        den = max(np.max(np.abs(g_ref[off:off + n])), 1e-3 * gscale)
        e = np.max(np.abs(g[off:off + n].astype(np.float64) - g_ref[off:off + n])) / den
        assert e <= tol, (name, e)
        off += n


FP32 = {
    "ch_k2": synth.Config("ch_k2", N=23, E=60, F=2, T_in=3, T_out=2, L=2, H=16, K=2, B=3,
                          cheb=True),
    "ch_k3": synth.Config("ch_k3", N=31, E=60, F=3, F_out=2, T_in=4, T_out=3, L=1, H=16, K=3,
                          B=5, cheb=True),
}
TC = {
    "ch_tc_k2": synth.Config("ch_tc_k2", N=40, E=60, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=6,
                             cheb=True),
    "ch_tc_k3": synth.Config("ch_tc_k3", N=20, E=60, F=1, T_in=3, T_out=2, L=2, H=64, K=3, B=4,
                             cheb=True),
}


@pytest.mark.parametrize("name", list(FP32))
def test_cheb_step_fp32_vs_oracle(env, name):
    cfg = FP32[name]
    _check(cfg, *_step(env, cfg, 0), tol=1e-5)


@pytest.mark.parametrize("name", list(TC))
def test_cheb_step_bf16_vs_oracle(env, name):
    cfg = TC[name]
    _check(cfg, *_step(env, cfg, 1), tol=2e-2)


def test_cheb_step_metr_la_bf16(env):
    """METR-LA shape with Chebyshev blocks on the tcgen05 path (B = 16)."""
    cfg = synth.CONFIGS["metr_la"].replace(B=16, cheb=True)
    _check(cfg, *_step(env, cfg, 1), tol=2e-2)


@pytest.mark.parametrize("name", ["ch_tc_k2", "ch_tc_k3", "metr_la"])
def test_cheb_step_bf16_mma_vs_oracle(env, name, monkeypatch):
    """The tensor-core window SpMM's Chebyshev epilogue (alpha acc + beta T_{k-2} on the fp32
    fragments) forced on every bf16 hop (PGTI_SPMM_MMA=1): K = 2 and 3, and METR-LA B = 16,
    against the oracle at 2e-2."""
    cfg = TC.get(name) or synth.CONFIGS["metr_la"].replace(B=16, cheb=True)
    monkeypatch.setenv("PGTI_SPMM_MMA", "1")
    _check(cfg, *_step(env, cfg, 1), tol=2e-2)


@pytest.mark.parametrize("precision,tol", [(0, 1e-5), (1, 2e-2)])
def test_cheb_encdec_vs_oracle(env, precision, tol):
    pgti, torch = env
    cfg = synth.Config("ch_ed", N=24, E=60, F=2, T_in=3, T_out=3, L=2,
                       H=16 if precision == 0 else 64, K=2, B=4, cheb=True)
    ref = pipeline.Reference(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0, epoch=0)[:cfg.B]
    idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(idx, cfg.B, cfg.T_in, cfg.T_out, x, y)
    csr = pgti.csr_to_device(pgti.add_windows(pgti.graph_build(cfg.N, *ref.graph), cfg.N), "cuda")
    model = pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out, cfg.B,
                       ld, csr, precision, model=1, teacher_forcing=0b1, cheb=True)
    d = dcgru.Dims.of(cfg)
    theta = synth.make_params(cfg, seed=synth.SEED_PARAMS, kind="random", model="encdec")
    n = model.num_params()
    assert n == theta.size == encdec.num_params(d)
    params = torch.from_numpy(theta).cuda()
    grads = torch.full((n,), float("nan"), device="cuda")
    loss = torch.zeros(1, device="cuda")
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    model.step(params, grads, x, y, loss, ws)
    pgti.check_device_error()
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, yhat_ref = encdec.loss_and_grad(theta.astype(np.float64), d, ref.Pf, ref.Pb,
                                                     xo.astype(np.float64), yo.astype(np.float64),
                                                     teacher_forcing=0b1)
    assert np.min(np.abs(yhat_ref - yo[..., :cfg.F_out])) > 1e-5
    assert abs(loss.item() - loss_ref) <= tol * abs(loss_ref)
    g = grads.cpu().numpy().astype(np.float64)
    gscale = np.max(np.abs(g_ref))
    off = 0
    for nm, shp in encdec.layer_shapes(d):
        k = int(np.prod(shp))
        den = max(np.max(np.abs(g_ref[off:off + k])), 1e-3 * gscale)
        assert np.max(np.abs(g[off:off + k] - g_ref[off:off + k])) / den <= tol, nm
        off += k


def test_cheb_trainer_graph_zero_copy_first_loss(env):
    """Trainer(cheb=True) on the bf16 path under CUDA-graph replay with zero-copy windows: the
    first step's loss equals the oracle's Chebyshev loss on the same sampled windows (2e-2), and
    zero-copy and gather give the same parameters after 3 steps (bitwise)."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer
    cfg = TC["ch_tc_k2"]
    ref = pipeline.Reference(cfg)
    theta = synth.make_params(cfg, kind="random")
    res = []
    for zc in (False, True):
        tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, precision=1,
                     use_cuda_graph=True, zero_copy=zc)
        assert tr.cheb and tr.model.desc.cheb == 1
        tr.start_epoch(0)
        tr.step(0)
        idx = tr.epoch_plan()[:cfg.B].cpu().numpy()
        xo, yo = ref.batch(idx)
        want = dcgru.forward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                             xo.astype(np.float64), yo.astype(np.float64))["loss"]
        assert abs(tr.loss.item() - want) <= 2e-2 * abs(want)
        for j in (1, 2):
            tr.step(j)
        tr.check()
        res.append(tr.params.cpu().numpy())
    assert np.array_equal(res[0], res[1])
