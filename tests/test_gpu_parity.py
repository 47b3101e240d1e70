"""CUDA path (through the C ABI) vs the float64 oracle, element by element.

Bars (BASELINE.json north_star): gathers, index plans and the normalised series bit-exact;
loss / activations / gradients within 1e-5 scale-relative (fp32 path, reading c19).
"""
import numpy as np
import pytest

import synth
from oracle import adam, dcgru, philox, pipeline, transitions, windows

from gpu_util import (SMALL_CONFIGS, ld_of, load_series, model_for, run_step, scale_rel,
                      split_dump)

pytestmark = pytest.mark.gpu

TOL32 = 1e-5


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2507_11683_b200 import build
    build.build()
    from paper_2507_11683_b200 import pgti
    return pgti, torch


_REFS = {}


def ref_for(cfg):
    if cfg.name not in _REFS:
        _REFS[cfg.name] = pipeline.Reference(cfg)
    return _REFS[cfg.name]


# ------------------------------------------------------------------ series / stats / index
@pytest.mark.parametrize("name", ["tiny2", "cp", "odd", "metr_la", "pems_bay"])
def test_normalized_series_bitexact(env, name):
    pgti, torch = env
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    got = s.buf.cpu().numpy().reshape(cfg.E, ld_of(cfg))
    want = windows.standardize32(ref.v, ref.mu, ref.sigma).reshape(cfg.E, -1)
    nf = cfg.N * cfg.F
    assert np.array_equal(got[:, :nf].view(np.uint32), want.view(np.uint32))
    assert not np.any(got[:, nf:].view(np.uint32))  # pads are +0.0


@pytest.mark.parametrize("name", ["cp", "odd", "metr_la", "pems_bay"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_stats_match_alg1(env, name, R):
    """Window-weighted device statistics of every rank's shard, summed, equal Alg. 1's
    stacked mu / sigma to 1e-12."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    S_tr = ref.n_train
    shift = 0.0
    for _ in range(2):
        tot = np.zeros(3)
        for r in range(R):
            p = trainer.shard_plan(S_tr, R, r, cfg.T_in, cfg.T_out)
            s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg)
            sums = torch.zeros(3, dtype=torch.float64, device="cuda")
            s.stats(S_tr, cfg.T_in, p.stat_lo, p.stat_hi, shift, sums)
            tot += sums.cpu().numpy()
        mean_d = tot[1] / tot[0]
        var = tot[2] / tot[0] - mean_d ** 2
        mu, shift = shift + mean_d, shift + mean_d
    assert abs(mu - ref.mu) <= 1e-12 * abs(ref.mu)
    assert abs(np.sqrt(var) - ref.sigma) <= 1e-12 * ref.sigma


@pytest.mark.parametrize("name", ["cp", "metr_la", "pems_bay"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_index_plan_bitexact(env, name, R):
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    for r in sorted({0, R - 1}):
        p = trainer.shard_plan(ref.n_train, R, r, cfg.T_in, cfg.T_out)
        s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu, ref.sigma)
        idx = torch.empty(p.win_hi - p.win_lo, dtype=torch.int32, device="cuda")
        for epoch in (0, 1, 7):
            n_used = s.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B, 3, epoch, r, 1, idx)
            want = ref.plan(R, r, seed=3, epoch=epoch)
            assert n_used == want.size
            assert np.array_equal(idx.cpu().numpy()[:n_used], want)
            full = p.win_lo + philox.epoch_permutation(3, epoch, r, p.win_hi - p.win_lo)
            assert np.array_equal(idx.cpu().numpy(), full)
        n_used = s.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B, 3, 0, r, 0, idx)
        assert np.array_equal(idx.cpu().numpy(), np.arange(p.win_lo, p.win_hi))


@pytest.mark.parametrize("name", ["tiny2", "cp", "odd", "metr_la", "pems_bay"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["ldg", "tma"])
def test_gather_bitexact(env, name, R, mode, monkeypatch):
    """Index-batched batch == the materialised Alg. 1 snapshots, bitwise,
    including each shard's first and last window (y ends on the shard's last row)."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    if ref.n_train // R < 2:
        pytest.skip("too few windows per rank")
    pgti.set_gather_mode(mode)
    try:
        ld, nf = ld_of(cfg), cfg.N * cfg.F
        for r in sorted({0, R // 2, R - 1}):
            p = trainer.shard_plan(ref.n_train, R, r, cfg.T_in, cfg.T_out)
            s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu,
                            ref.sigma)
            plan = ref.plan(R, r)
            idx_np = np.concatenate([[p.win_lo, p.win_hi - 1], plan[:max(1, cfg.B - 2)]])
            B = idx_np.size
            idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
            x = torch.full((B * cfg.T_in * ld,), float("nan"), device="cuda")
            y = torch.full((B * cfg.T_out * ld,), float("nan"), device="cuda")
            s.gather(idx, B, cfg.T_in, cfg.T_out, x, y)
            pgti.check_device_error()
            fx, fy = ref.batch(idx_np)
            xg = x.cpu().numpy().reshape(B, cfg.T_in, ld)
            yg = y.cpu().numpy().reshape(B, cfg.T_out, ld)
            assert np.array_equal(xg[..., :nf].view(np.uint32), fx.reshape(B, cfg.T_in, nf).view(np.uint32))
            assert np.array_equal(yg[..., :nf].view(np.uint32), fy.reshape(B, cfg.T_out, nf).view(np.uint32))
            assert not np.any(xg[..., nf:].view(np.uint32)) and not np.any(yg[..., nf:].view(np.uint32))
    finally:
        pgti.set_gather_mode("ldg")


def test_gather_out_of_range_sets_flag(env):
    pgti, torch = env
    cfg = SMALL_CONFIGS["tiny2"]
    ref = ref_for(cfg)
    s = load_series(pgti, torch, ref.v[10:30], 10, cfg, ref.mu, ref.sigma)
    ld = ld_of(cfg)
    x = torch.zeros(2 * cfg.T_in * ld, device="cuda")
    y = torch.zeros(2 * cfg.T_out * ld, device="cuda")
    ok = torch.tensor([10, 30 - cfg.T_in - cfg.T_out], dtype=torch.int32, device="cuda")
    s.gather(ok, 2, cfg.T_in, cfg.T_out, x, y)
    pgti.check_device_error()
    for bad in ([9, 12], [12, 30 - cfg.T_in - cfg.T_out + 1]):
        s.gather(torch.tensor(bad, dtype=torch.int32, device="cuda"), 2, cfg.T_in, cfg.T_out, x, y)
        with pytest.raises(pgti.PgtiError) as e:
            pgti.check_device_error()
        assert e.value.name == "OUT_OF_RANGE"
    idx = torch.zeros(20, dtype=torch.int32, device="cuda")
    with pytest.raises(pgti.PgtiError) as e:   # windows reaching past the held rows
        s.make_index(10, 30, cfg.T_in, cfg.T_out, 2, 0, 0, 0, 1, idx)
    assert e.value.name == "OUT_OF_RANGE"


# ------------------------------------------------------------------ diffusion (K2)
@pytest.mark.parametrize("N,W,K,graph", [(37, 24, 3, "er"), (37, 7, 2, "er"), (207, 4096, 2, "knn"),
                                          (64, 128, 1, "ring"), (5, 3, 0, "er")])
def test_diffusion_vs_oracle(env, N, W, K, graph):
    pgti, torch = env
    g = {"er": lambda: synth.random_graph(N, 0.15, seed=N),
         "knn": lambda: synth.make_graph(N, 8),
         "ring": lambda: synth.ring_graph(N)}[graph]()
    cfg = synth.Config("d", N=N, E=10, F=1, T_in=1, T_out=1, L=1, H=16, K=K, B=1)
    model = model_for(pgti, torch, cfg, g)
    Pf, Pb = transitions.transition_matrices(N, *g)
    rng = np.random.default_rng(0)
    Z = rng.normal(size=(N, W)).astype(np.float32)
    M = 2 * K + 1
    out = torch.empty(M * N * W, device="cuda")
    model.diffuse(torch.from_numpy(Z).cuda(), W, out)
    want = dcgru.diffusion_features(Pf, Pb, Z.astype(np.float64), K)
    got = out.cpu().numpy().reshape(M, N, W)
    for m in range(M):
        assert scale_rel(got[m], want[m]) <= 1e-6, m
    dT = rng.normal(size=(M, N, W)).astype(np.float32)
    dZ = torch.empty(N * W, device="cuda")
    model.diffuse_adjoint(torch.from_numpy(dT).cuda(), W, dZ)
    want = dcgru.diffusion_adjoint(Pf, Pb, dT.astype(np.float64), K)
    assert scale_rel(dZ.cpu().numpy().reshape(N, W), want) <= 1e-6


@pytest.mark.parametrize("N,W,K,graph,rows", [(207, 4096, 2, "knn", 16), (37, 24, 3, "er", 7),
                                               (300, 128, 2, "knn", 64), (100, 256, 1, "knn", 1),
                                               (45, 1000, 2, "ring", 32)])
def test_diffusion_staged_plan_bitexact(env, N, W, K, graph, rows):
    """The shared-memory staged SpMM (pgti_graph_windows plan) only changes where neighbour rows
    are read from: forward and adjoint diffusion are bit-identical to the unstaged kernel and
    match the oracle.  Covers ragged last windows, rows not a multiple of 8, partial chunks."""
    pgti, torch = env
    g = {"er": lambda: synth.random_graph(N, 0.15, seed=N),
         "knn": lambda: synth.make_graph(N, 8),
         "ring": lambda: synth.ring_graph(N)}[graph]()
    cfg = synth.Config("d", N=N, E=10, F=1, T_in=1, T_out=1, L=1, H=16, K=K, B=1)
    staged = model_for(pgti, torch, cfg, g, win_rows=rows)
    plain = model_for(pgti, torch, cfg, g, win_rows=0)
    assert staged.desc.win_rows == rows and plain.desc.win_rows == 0
    Pf, Pb = transitions.transition_matrices(N, *g)
    rng = np.random.default_rng(1)
    Z = torch.from_numpy(rng.normal(size=(N, W)).astype(np.float32)).cuda()
    M = 2 * K + 1
    outs = []
    for m in (staged, plain):
        out = torch.empty(M * N * W, device="cuda")
        m.diffuse(Z, W, out)
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    want = dcgru.diffusion_features(Pf, Pb, Z.cpu().numpy().astype(np.float64), K)
    assert scale_rel(outs[0].reshape(M, N, W), want) <= 1e-6
    dT = torch.from_numpy(rng.normal(size=(M, N, W)).astype(np.float32)).cuda()
    adj = []
    for m in (staged, plain):
        dZ = torch.empty(N * W, device="cuda")
        m.diffuse_adjoint(dT, W, dZ)
        adj.append(dZ.cpu().numpy())
    assert np.array_equal(adj[0], adj[1])
    want = dcgru.diffusion_adjoint(Pf, Pb, dT.cpu().numpy().astype(np.float64), K)
    assert scale_rel(adj[0].reshape(N, W), want) <= 1e-6


def test_step_staged_plan_bitexact_both_precisions(env):
    """Whole training step with and without the SpMM staging plan: identical loss and grads in
    fp32 and on the bf16 tcgen05 path (where the diffused blocks are bf16)."""
    pgti, torch = env
    for precision, cfg in ((0, SMALL_CONFIGS["odd"]), (1, TC_CONFIGS["tc_odd"])):
        ref = ref_for(cfg)
        s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
        idx = torch.arange(cfg.B, dtype=torch.int32, device="cuda") * 3
        ld = ld_of(cfg)
        x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
        y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
        s.gather(idx, cfg.B, cfg.T_in, cfg.T_out, x, y)
        theta = synth.make_params(cfg, kind="random")
        res = []
        for rows in (None, 5, 0):
            model = model_for(pgti, torch, cfg, ref.graph, precision=precision, win_rows=rows)
            res.append(run_step(pgti, torch, model, theta, x, y, dump=False))
        for r in res[1:]:
            assert r[0] == res[0][0] and np.array_equal(r[1], res[0][1]), precision


# ------------------------------------------------------------------ full step (K1..K5)
def _step_case(env, cfg, seed=0, B=None, scale=1.0):
    pgti, torch = env
    B = B or cfg.B
    cfg = cfg.replace(B=B)
    ref = ref_for(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0, epoch=seed)[:B]
    idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
    ld = ld_of(cfg)
    x = torch.empty(B * cfg.T_in * ld, device="cuda")
    y = torch.empty(B * cfg.T_out * ld, device="cuda")
    s.gather(idx, B, cfg.T_in, cfg.T_out, x, y)
    model = model_for(pgti, torch, cfg, ref.graph)
    theta = synth.make_params(cfg, seed=synth.SEED_PARAMS + seed, kind="random", scale=scale)
    assert model.num_params() == theta.size == dcgru.num_params(ref.d)
    loss, g, act = run_step(pgti, torch, model, theta, x, y)
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    resid = np.abs(fwd["yhat"] - yo[..., :cfg.F_out])
    return dict(loss=loss, g=g, act=act, loss_ref=loss_ref, g_ref=g_ref, fwd=fwd, cfg=cfg,
                ref=ref, margin=float(resid.min()), B=B)


def _check_step(c, tol=TOL32):
    cfg, B = c["cfg"], c["B"]
    assert c["margin"] > 1e-5, "a residual sits at an |.| kink; pick another seed"
    assert abs(c["loss"] - c["loss_ref"]) <= tol * abs(c["loss_ref"])
    acts, yhat = split_dump(c["act"], cfg, B)
    acts_ref, yhat_ref = dcgru.activations(c["fwd"], dcgru.Dims.of(cfg))
    # oracle [T][L][4][B][N][H] vs dump [T][L][4][N][B][H]
    acts_ref = acts_ref.transpose(0, 1, 2, 4, 3, 5)
    for t in range(cfg.T_in):
        for l in range(cfg.L):
            for q, nm in enumerate("Hruc"):
                e = scale_rel(acts[t, l, q], acts_ref[t, l, q])
                assert e <= tol, (t, l, nm, e)
    assert scale_rel(yhat, yhat_ref.transpose(1, 2, 0, 3)) <= tol
    off = 0
    gscale = np.max(np.abs(c["g_ref"]))
    for name, shp in synth.param_shapes(cfg):
        n = int(np.prod(shp))
        g, gr = c["g"][off:off + n], c["g_ref"][off:off + n]
        # per tensor scale-relative; a tensor whose reference is (near) zero -- e.g. db_out =
        # sum of +-1/count with balanced signs -- is measured against 1e-3 of the whole
        # gradient's scale (reading c19)
        den = max(np.max(np.abs(gr)), 1e-3 * gscale)
        err = np.max(np.abs(g.astype(np.float64) - gr))
        if name == "b_out":
            # db_out = sum_i sign_i / count over count = B T_out N F_out terms, accumulated in
            # fp32 on both paths: the summation bound gamma_n sum|x_i| = count * 2^-24 * 1 is
            # an absolute error the tolerance must admit when the signs balance (ref ~ 0)
            err = max(0.0, err - (B * cfg.T_out * cfg.N * cfg.F_out) * 2.0 ** -24)
        e = err / den
        assert e <= tol, (name, e)
        off += n
    assert scale_rel(c["g"], c["g_ref"]) <= tol


@pytest.mark.parametrize("name", list(SMALL_CONFIGS))
@pytest.mark.parametrize("seed", [0, 1])
def test_step_parity_small(env, name, seed):
    _check_step(_step_case(env, SMALL_CONFIGS[name], seed=seed))


@pytest.mark.parametrize("name,B", [("metr_la", 64), ("metr_la", 13), ("pems_bay", 16)])
def test_step_parity_traffic(env, name, B):
    """METR-LA at its full per-GPU batch (the bench's launch configuration)."""
    _check_step(_step_case(env, synth.CONFIGS[name], B=B))


def test_step_is_deterministic(env):
    c1 = _step_case(env, SMALL_CONFIGS["odd"])
    c2 = _step_case(env, SMALL_CONFIGS["odd"])
    assert c1["loss"] == c2["loss"] and np.array_equal(c1["g"].view(np.uint32), c2["g"].view(np.uint32))


def test_step_errors(env):
    pgti, torch = env
    cfg = SMALL_CONFIGS["tiny2"]
    ref = ref_for(cfg)
    model = model_for(pgti, torch, cfg, ref.graph)
    n = model.num_params()
    p = torch.zeros(n, device="cuda")
    ws = torch.empty(model.workspace_bytes() - 256, dtype=torch.uint8, device="cuda")
    x = torch.zeros(cfg.B * cfg.T_in * ld_of(cfg), device="cuda")
    y = torch.zeros(cfg.B * cfg.T_out * ld_of(cfg), device="cuda")
    with pytest.raises(pgti.PgtiError) as e:
        model.step(p, p.clone(), x, y, torch.zeros(1, device="cuda"), ws)
    assert e.value.name == "WORKSPACE" and "needed" in str(e.value)


# ------------------------------------------------------------------ data parallel + Adam
@pytest.mark.parametrize("R", [2, 4])
def test_ddp_equivalence_emulated(env, R):
    """R virtual ranks on one GPU, each on its own halo shard and first batch; their gradient
    mean equals the oracle gradient of the union batch."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = synth.CONFIGS["metr_la"].replace(B=8)
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="random")
    gsum = np.zeros(theta.size)
    union = []
    for r in range(R):
        p = trainer.shard_plan(ref.n_train, R, r, cfg.T_in, cfg.T_out)
        s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu, ref.sigma)
        idx = torch.empty(p.win_hi - p.win_lo, dtype=torch.int32, device="cuda")
        s.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B, 3, 0, r, 1, idx)
        ld = ld_of(cfg)
        x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
        y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
        s.gather(idx[:cfg.B], cfg.B, cfg.T_in, cfg.T_out, x, y)
        model = model_for(pgti, torch, cfg, ref.graph)
        _, g, _ = run_step(pgti, torch, model, theta, x, y, dump=False)
        gsum += g
        union.append(idx[:cfg.B].cpu().numpy())
    union = np.concatenate(union)
    _, g_union, _ = ref.loss_and_grad(theta, union)
    assert scale_rel(gsum / R, g_union) <= TOL32


def test_adam_vs_oracle(env):
    pgti, torch = env
    rng = np.random.default_rng(0)
    n = 1001  # ragged tail
    th = rng.normal(size=n).astype(np.float32)
    p = torch.from_numpy(th).cuda()
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    dev_step = torch.zeros(1, dtype=torch.int64, device="cuda")
    tho, mo, vo = th.astype(np.float64), np.zeros(n), np.zeros(n)
    for step in range(1, 7):
        g = rng.normal(size=n).astype(np.float32)
        use_dev = step % 2 == 0
        if use_dev:
            dev_step.fill_(step - 1)
        pgti.adam_step(p, torch.from_numpy(g).cuda(), m, v, 0 if use_dev else step, 1e-2,
                       grad_scale=0.25, dev_step=dev_step if use_dev else None)
        tho, mo, vo = adam.adam_step(tho, g, mo, vo, step, 1e-2, grad_scale=0.25)
        assert scale_rel(p.cpu().numpy() - th, tho - th) <= 1e-5
    assert int(dev_step.item()) == 6


def test_trainer_cuda_graph_matches_eager(env):
    """The captured step (gather -> fwd/bwd -> Adam) replays to the same parameters, bit for
    bit, as eager launches; and the Trainer's own statistics match Alg. 1."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer
    cfg = SMALL_CONFIGS["cp"]
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="train")
    outs = []
    for use_graph in (False, True):
        tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, use_cuda_graph=use_graph)
        assert abs(tr.mu - ref.mu) <= 1e-12 * abs(ref.mu)
        assert abs(tr.sigma - ref.sigma) <= 1e-12 * ref.sigma
        steps = tr.start_epoch(0)
        losses = []
        for j in range(min(steps, 12)):
            tr.step(j)
            losses.append(float(tr.loss.item()))
        tr.check()
        outs.append((tr.params.cpu().numpy(), losses))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert outs[0][1] == outs[1][1]


# ------------------------------------------------------------------ bf16 tcgen05 path
TOL_BF16 = 2e-2
TC_CONFIGS = {
    "tc_tiny": synth.Config("tc_tiny", N=12, E=60, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=3),
    "tc_odd": SMALL_CONFIGS["odd"],
    "tc_l1": synth.Config("tc_l1", N=40, E=60, F=1, T_in=4, T_out=1, L=1, H=64, K=2, B=5),
    # >= 2*148 row tiles of 128: the GEMMs switch to two 64-column sub-tiles per CTA
    "tc_big": synth.Config("tc_big", N=600, E=110, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=64),
}


def _step_case_tc(env, cfg, B=None, seed=0, win_rows=None):
    pgti, torch = env
    B = B or cfg.B
    cfg = cfg.replace(B=B)
    ref = ref_for(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0, epoch=seed)[:B]
    idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
    ld = ld_of(cfg)
    x = torch.empty(B * cfg.T_in * ld, device="cuda")
    y = torch.empty(B * cfg.T_out * ld, device="cuda")
    s.gather(idx, B, cfg.T_in, cfg.T_out, x, y)
    model = model_for(pgti, torch, cfg, ref.graph, precision=1, win_rows=win_rows)
    theta = synth.make_params(cfg, seed=synth.SEED_PARAMS + seed, kind="random")
    loss, g, act = run_step(pgti, torch, model, theta, x, y)
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    return dict(loss=loss, g=g, act=act, loss_ref=loss_ref, g_ref=g_ref, fwd=fwd, cfg=cfg,
                ref=ref, margin=1.0, B=B)


@pytest.mark.parametrize("name", list(TC_CONFIGS))
def test_step_parity_bf16_small(env, name):
    """precision = 1 (bf16 operands, fp32 TMEM accumulation): 2e-2 scale-relative (BJ)."""
    _check_step(_step_case_tc(env, TC_CONFIGS[name]), tol=TOL_BF16)


@pytest.mark.parametrize("name,B", [("metr_la", 64), ("pems_bay", 16)])
def test_step_parity_bf16_traffic(env, name, B):
    _check_step(_step_case_tc(env, synth.CONFIGS[name], B=B), tol=TOL_BF16)


@pytest.mark.parametrize("name,B,win_rows", [("tc_tiny", None, 0), ("tc_big", None, 16),
                                             ("tc_big", None, 32), ("metr_la", 64, 0),
                                             ("metr_la", 64, 16)])
def test_step_parity_bf16_staging_plans(env, name, B, win_rows):
    """The bf16 path with the unstaged SpMM (win_rows 0) and other staging windows than the
    library default."""
    cfg = TC_CONFIGS.get(name) or synth.CONFIGS[name]
    _check_step(_step_case_tc(env, cfg, B=B, win_rows=win_rows), tol=TOL_BF16)


# ------------------------------------------------------------------ NEXT f4 / f1 index plans
@pytest.mark.parametrize("name", ["cp", "metr_la", "pems_bay"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_batch_shuffle_plan_bitexact(env, name, R):
    """shuffle = 2 (generalized variant's batch-level shuffle) against
    oracle.philox.batch_plan, first and last rank, three epochs."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    for r in sorted({0, R - 1}):
        p = trainer.shard_plan(ref.n_train, R, r, cfg.T_in, cfg.T_out)
        s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu, ref.sigma)
        idx = torch.full((p.win_hi - p.win_lo,), -1, dtype=torch.int32, device="cuda")
        for epoch in (0, 1, 7):
            n_used = s.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B, 3, epoch, r, 2,
                                  idx)
            want = philox.batch_plan(ref.n_train, R, r, cfg.B, 3, epoch)
            assert n_used == want.size
            assert np.array_equal(idx.cpu().numpy()[:n_used], want)


@pytest.mark.parametrize("name", ["cp", "metr_la"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_replicated_global_plan_bitexact(env, name, R):
    """Replicated placement (f1): every rank derives the one global plan and visits its
    slice -- against oracle.philox.global_plan; the Trainer's slices are disjoint."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer
    cfg = SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="random")
    seen = []
    for r in range(R):
        tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, rank=r, world=R,
                     precision=0, use_cuda_graph=False, placement="replicated")
        assert (tr.mu, tr.sigma) == pytest.approx((ref.mu, ref.sigma), rel=1e-12)
        for epoch in (0, 5):
            steps = tr.start_epoch(epoch)
            got = tr.epoch_plan().cpu().numpy()
            want = philox.global_plan(ref.n_train, R, r, cfg.B, 3, epoch)
            assert steps * cfg.B == want.size and np.array_equal(got, want)
        seen.append(got)
        del tr
    allw = np.concatenate(seen)
    assert np.unique(allw).size == allw.size


@pytest.mark.parametrize("precision,tol", [(0, 1e-5), (1, TOL_BF16)])
def test_validation_mae_vs_oracle(env, precision, tol):
    """pgti_dcrnn_loss (forward + loss only) over the validation windows, as Trainer.validate
    aggregates it, against the float64 oracle's MAE of the same batches; the training
    step still matches after a validation pass (shared workspace)."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer, val_windows
    cfg = synth.Config("val", N=40, E=150, F=2, T_in=4, T_out=3, L=2, H=64, K=2, B=6)
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="random")
    tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, precision=precision,
                 use_cuda_graph=False, placement="replicated")
    mae = tr.validate()
    nb = val_windows(ref.S) // cfg.B
    assert nb >= 2
    losses = []
    for j in range(nb):
        x, y = ref.batch(np.arange(ref.n_train + j * cfg.B, ref.n_train + (j + 1) * cfg.B))
        losses.append(dcgru.forward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                    x.astype(np.float64), y.astype(np.float64))["loss"])
    want = float(np.mean(losses))
    assert abs(mae - want) <= tol * abs(want), (mae, want)


# ------------------------------------------------------------------ NEXT f2: zero-copy step
@pytest.mark.parametrize("name,precision,B", [("odd", 0, None), ("tc_tiny", 1, None),
                                              ("metr_la", 1, 64), ("metr_la", 0, 8)])
def test_step_indexed_bitexact_vs_gather(env, name, precision, B):
    """pgti_dcrnn_step_indexed reads x / y straight from the resident series by window start
    (SURVEY f2): loss, activations and gradients are bit-identical to gather + step, on a shard
    whose rows start past 0 (global row indices)."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = TC_CONFIGS.get(name) or SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    cfg = cfg.replace(B=B or cfg.B)
    ref = ref_for(cfg)
    p = trainer.shard_plan(ref.n_train, 2, 1, cfg.T_in, cfg.T_out)
    s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu, ref.sigma)
    idx = torch.empty(p.win_hi - p.win_lo, dtype=torch.int32, device="cuda")
    s.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B, 3, 4, 1, 1, idx)
    bidx = idx[:cfg.B].clone()
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(bidx, cfg.B, cfg.T_in, cfg.T_out, x, y)
    model = model_for(pgti, torch, cfg, ref.graph, precision=precision)
    theta = torch.from_numpy(synth.make_params(cfg, kind="random")).cuda()
    n = model.num_params()
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    out = []
    for indexed in (False, True):
        grads = torch.full((n,), float("nan"), device="cuda")
        loss = torch.zeros(1, device="cuda")
        act = torch.empty(model.act_dump_floats(), device="cuda")
        if indexed:
            model.step_indexed(theta, grads, s, bidx, loss, ws, act)
        else:
            model.step(theta, grads, x, y, loss, ws, act)
        pgti.check_device_error()
        out.append((loss.item(), grads.cpu().numpy(), act.cpu().numpy()))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
    # a window start outside the held rows raises the device flag
    bad = bidx.clone()
    bad[0] = p.row_lo - 1
    model.step_indexed(theta, torch.empty(n, device="cuda"), s, bad, loss, ws)
    with pytest.raises(pgti.PgtiError) as e:
        pgti.check_device_error()
    assert e.value.name == "OUT_OF_RANGE"


@pytest.mark.parametrize("name,precision,B", [("odd", 0, None), ("metr_la", 0, 16),
                                              ("tc_big", 1, None), ("metr_la", 1, 64)])
def test_step_indexed_vs_oracle(env, name, precision, B):
    """f2 against the oracle (not only against the gather path): the zero-copy step reads
    sample b's windows from a halo shard of the resident series by start index ("views,
    not copies"); loss, every activation and every gradient tensor match the float64 oracle's
    materialised-snapshot step (1e-5 fp32, 2e-2 bf16)."""
    pgti, torch = env
    from paper_2507_11683_b200 import trainer
    cfg = TC_CONFIGS.get(name) or SMALL_CONFIGS.get(name) or synth.CONFIGS[name]
    cfg = cfg.replace(B=B or cfg.B)
    ref = ref_for(cfg)
    p = trainer.shard_plan(ref.n_train, 2, 1, cfg.T_in, cfg.T_out)
    s = load_series(pgti, torch, ref.v[p.row_lo:p.row_hi], p.row_lo, cfg, ref.mu, ref.sigma)
    # rank 1's windows (global starts past row 0); drawn with replacement so that configs with
    # fewer windows per rank than B still fill the batch
    idx_np = np.random.default_rng(7).integers(p.win_lo, p.win_hi, size=cfg.B)
    model = model_for(pgti, torch, cfg, ref.graph, precision=precision)
    theta = synth.make_params(cfg, kind="random")
    n = model.num_params()
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    grads = torch.full((n,), float("nan"), device="cuda")
    loss = torch.zeros(1, device="cuda")
    act = torch.empty(model.act_dump_floats(), device="cuda")
    model.step_indexed(torch.from_numpy(theta).cuda(), grads, s,
                       torch.from_numpy(idx_np.astype(np.int32)).cuda(), loss, ws, act)
    pgti.check_device_error()
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    resid = np.abs(fwd["yhat"] - yo[..., :cfg.F_out])
    c = dict(loss=float(loss.item()), g=grads.cpu().numpy(), act=act.cpu().numpy(),
             loss_ref=loss_ref, g_ref=g_ref, fwd=fwd, cfg=cfg, ref=ref,
             margin=float(resid.min()) if precision == 0 else 1.0, B=cfg.B)
    _check_step(c, tol=TOL32 if precision == 0 else TOL_BF16)


def test_trainer_zero_copy_graph_matches_gather(env):
    """Trainer(zero_copy=True) under CUDA-graph replay: the same parameters after 3 steps as the
    gather path (bitwise)."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer
    cfg = SMALL_CONFIGS["cp"]
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="random")
    res = []
    for zc in (False, True):
        tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, precision=0,
                     use_cuda_graph=True, zero_copy=zc)
        tr.start_epoch(0)
        for j in range(3):
            tr.step(j)
        tr.check()
        res.append(tr.params.cpu().numpy())
    assert np.array_equal(res[0], res[1])


def test_new_entry_point_errors(env):
    """Argument errors of the later entry points: step_indexed against a series of another
    shape, forward-only loss with a short workspace, invalid model / feedback flags."""
    pgti, torch = env
    cfg = SMALL_CONFIGS["tiny2"]
    ref = ref_for(cfg)
    model = model_for(pgti, torch, cfg, ref.graph)
    n = model.num_params()
    p = torch.zeros(n, device="cuda")
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, device="cuda")
    other = cfg.replace(N=cfg.N + 1)
    v2 = synth.make_series(other)
    s2 = load_series(pgti, torch, v2, 0, other, 0.0, 1.0)
    idx = torch.zeros(cfg.B, dtype=torch.int32, device="cuda")
    with pytest.raises(pgti.PgtiError) as e:
        model.step_indexed(p, p.clone(), s2, idx, loss, ws)
    assert e.value.name == "SHAPE"
    x = torch.zeros(cfg.B * cfg.T_in * ld_of(cfg), device="cuda")
    y = torch.zeros(cfg.B * cfg.T_out * ld_of(cfg), device="cuda")
    with pytest.raises(pgti.PgtiError) as e:
        model.loss(p, x, y, loss, ws[:-512])
    assert e.value.name == "WORKSPACE"
    csr = pgti.csr_to_device(pgti.graph_build(cfg.N, *ref.graph), "cuda")
    for kw, want in ((dict(model=2), "INVALID_ARG"), (dict(teacher_forcing=1), "INVALID_ARG")):
        bad = pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out, cfg.B,
                         ld_of(cfg), csr, 0, **kw)
        with pytest.raises(pgti.PgtiError) as e:   # the desc check runs before anything else
            bad.step(p, p.clone(), x, y, loss, ws)
        assert e.value.name == want, str(e.value)


@pytest.mark.parametrize("name,precision", [("cp", 0), ("tc_tiny", 1), ("tc_k3", 1),
                                            ("metr_la", 1)])
def test_step_parity_batch_of_one(env, name, precision):
    """B = 1 (one window per rank: R = N rows, ragged GEMM tiles), and the bf16 path at K = 3
    (seven diffusion blocks)."""
    cfg = (TC_CONFIGS.get(name) or SMALL_CONFIGS.get(name) or synth.CONFIGS.get(name)
           or synth.Config("tc_k3", N=20, E=60, F=1, T_in=3, T_out=2, L=2, H=64, K=3, B=4))
    if precision == 0:
        _check_step(_step_case(env, cfg, B=1))
    else:
        _check_step(_step_case_tc(env, cfg, B=1 if name != "tc_k3" else None), tol=TOL_BF16)


@pytest.mark.parametrize("name,B", [("tc_big", None), ("metr_la", 64)])
def test_step_spmm_variants_bitexact(env, name, B, monkeypatch):
    """The staged SpMM's forms only regroup work across threads and CTAs: the window-resident,
    chunk-pipelined kernel (default), the per-chunk kernel with two 16-byte vectors per lane
    (PGTI_SPMM_WP=0) and with one (PGTI_SPMM_VPL=1) give bit-identical loss, activations and
    gradients."""
    cfg = TC_CONFIGS.get(name) or synth.CONFIGS[name]
    monkeypatch.setenv("PGTI_SPMM_MMA", "0")
    res = []
    for envs in ({}, {"PGTI_SPMM_WP": "0"}, {"PGTI_SPMM_WP": "0", "PGTI_SPMM_VPL": "1"}):
        for k in ("PGTI_SPMM_WP", "PGTI_SPMM_VPL"):
            monkeypatch.delenv(k, raising=False)
        for k, v in envs.items():
            monkeypatch.setenv(k, v)
        c = _step_case_tc(env, cfg, B=B)
        res.append((c["loss"], c["g"], c["act"]))
    for r in res[1:]:
        assert r[0] == res[0][0]
        assert np.array_equal(r[1], res[0][1]) and np.array_equal(r[2], res[0][2])


def test_step_dense_rows(env):
    """Rows with more than 32 CSR entries (an Erdos-Renyi graph with p = 0.5: ~40 per row) on the
    bf16 path: the staged SpMM's per-warp entry lists hold 32 entries per pass, the rest is read
    in further passes.  Against the oracle at 2e-2."""
    pgti, torch = env
    cfg = synth.Config("tc_dense", N=80, E=60, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=8)
    ref = pipeline.Reference(cfg, graph=synth.random_graph(cfg.N, 0.5, seed=5))
    assert np.max(np.diff(pgti.graph_build(cfg.N, *ref.graph)["a_rowptr"])) > 32
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0)[:cfg.B]
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(torch.from_numpy(idx_np.astype(np.int32)).cuda(), cfg.B, cfg.T_in, cfg.T_out, x, y)
    theta = synth.make_params(cfg, kind="random")
    model = model_for(pgti, torch, cfg, ref.graph, precision=1)
    loss, g, act = run_step(pgti, torch, model, theta, x, y)
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    _check_step(dict(loss=loss, g=g, act=act, loss_ref=loss_ref, g_ref=g_ref, fwd=fwd, cfg=cfg,
                     ref=ref, margin=1.0, B=cfg.B), tol=TOL_BF16)


def test_step_pipelined_spmm_bitexact_at_scale(env, monkeypatch):
    """The window-resident, chunk-pipelined staged SpMM (chosen when windows x jobs x chunk groups
    fill >= 4 waves with >= 4 chunks per CTA: full PeMS, PeMS-All-LA) against the per-chunk
    kernel, bitwise, on a PeMS-All-LA-sized graph at B = 64 (its oracle parity is the full-size
    test in test_gpu_fullsize.py)."""
    pgti, torch = env
    cfg = synth.Config("wp", N=2716, E=120, F=2, T_in=12, T_out=12, L=2, H=64, K=2, B=64)
    v = synth.make_series(cfg)
    s = load_series(pgti, torch, v, 0, cfg, float(v.mean()), float(v.std()))
    graph = synth.make_graph(cfg.N, cfg.knn)
    ld = ld_of(cfg)
    idx = torch.arange(cfg.B, dtype=torch.int32, device="cuda")
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(idx, cfg.B, cfg.T_in, cfg.T_out, x, y)
    theta = synth.make_params(cfg, kind="random")
    monkeypatch.setenv("PGTI_SPMM_MMA", "0")
    res = []
    for flag in (None, "0"):
        if flag:
            monkeypatch.setenv("PGTI_SPMM_WP", flag)
        else:
            monkeypatch.delenv("PGTI_SPMM_WP", raising=False)
        model = model_for(pgti, torch, cfg, graph, precision=1)
        res.append(run_step(pgti, torch, model, theta, x, y))
    assert np.all(np.isfinite(res[0][1]))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("name,B", [("tc_big", None), ("metr_la", 64)])
def test_step_spmm_mma_oracle(env, name, B, monkeypatch):
    """The tensor-core window SpMM (mma.sync bf16, P_w split hi + lo; forced everywhere it is
    eligible by PGTI_SPMM_MMA=1, e.g. METR-LA's 13 windows) regroups the fp32 sums of the bf16
    hops and rounds the weights to 2^-17: not bit-identical to the SIMT kernels
    (PGTI_SPMM_MMA=0), so the step is checked against the oracle at the bf16 path's tolerance,
    and against the SIMT step at the same bound."""
    cfg = TC_CONFIGS.get(name) or synth.CONFIGS[name]
    monkeypatch.setenv("PGTI_SPMM_MMA", "1")
    c = _step_case_tc(env, cfg, B=B)
    _check_step(c, tol=TOL_BF16)
    monkeypatch.setenv("PGTI_SPMM_MMA", "0")
    s = _step_case_tc(env, cfg, B=B)
    assert abs(c["loss"] - s["loss"]) <= TOL_BF16 * abs(s["loss"])
    assert scale_rel(c["g"], s["g"]) <= TOL_BF16


def _band_graph(N, half, seed=3):
    """Directed band graph i -> j for |i - j| <= half (random float32 weights in [0.1, 1]): rows of
    up to 2 half + 1 entries whose 16-row window unions are exactly 16 + 2 half nodes."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for i in range(N):
        for j in range(max(0, i - half), min(N, i + half + 1)):
            src.append(i), dst.append(j)
    src, dst = np.array(src, np.int32), np.array(dst, np.int32)
    return src, dst, (0.1 + 0.9 * rng.random(src.size)).astype(np.float32)


@pytest.mark.parametrize("B", [5, 13])
def test_step_spmm_mma_edge_cases(env, B, monkeypatch):
    """The tensor-core window SpMM (forced) at its limits, against the oracle at 2e-2: window
    unions of exactly 64 nodes (4 k-steps, no padding rows), rows of 49 CSR entries (the P_w
    scatter's second pass), a ragged last window (N = 100), partial column chunks (W = 64 B with
    B = 5, 13: 1.25 and 3.25 chunks of 256 columns)."""
    pgti, torch = env
    cfg = synth.Config("tc_band", N=100, E=60, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=B)
    ref = pipeline.Reference(cfg, graph=_band_graph(cfg.N, 24))
    csr = pgti.add_windows(pgti.graph_build(cfg.N, *ref.graph), cfg.N, 16)
    assert csr["win_max"] == 64 and np.max(np.diff(csr["a_rowptr"])) == 49
    monkeypatch.setenv("PGTI_SPMM_MMA", "1")
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0)[:cfg.B]
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(torch.from_numpy(idx_np.astype(np.int32)).cuda(), cfg.B, cfg.T_in, cfg.T_out, x, y)
    theta = synth.make_params(cfg, kind="random")
    model = model_for(pgti, torch, cfg, ref.graph, precision=1, win_rows=16)
    loss, g, act = run_step(pgti, torch, model, theta, x, y)
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, fwd = dcgru.backward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                          xo.astype(np.float64), yo.astype(np.float64))
    _check_step(dict(loss=loss, g=g, act=act, loss_ref=loss_ref, g_ref=g_ref, fwd=fwd, cfg=cfg,
                     ref=ref, margin=1.0, B=cfg.B), tol=TOL_BF16)
