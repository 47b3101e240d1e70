"""The Trainer's captured step on the bench's path, and the collectives at world 1.

* Alg. 1's statistics finished inside libpgti (pgti_series_moments) equal the
  oracle's stacked mu / sigma to 1e-12, with and without a (1-rank) NCCL communicator.
* The gradient all-reduce (a8) runs in the 1-GPU suite: a Trainer given a 1-rank
  communicator calls pgti_allreduce_grads inside the captured CUDA graph, and the R = 1 identity
  (the mean over one rank is that rank's gradient) holds bit for bit against the same
  Trainer without a communicator.
* The bf16 tcgen05 step (per-layer streams, aux weight-gradient streams, PDL edges) replayed as
  a CUDA graph gives the same parameters, bit for bit, as eager launches after several Adam
  steps -- stepwise model and encoder-decoder, L = 2 -- and its first loss matches the oracle.
* The validation MAE mean (pgti_mean_losses) equals the mean of the per-batch losses.
"""
import numpy as np
import pytest

import synth
from oracle import dcgru, pipeline

pytestmark = pytest.mark.gpu

TC2 = synth.Config("tc2", N=40, E=120, F=2, T_in=4, T_out=3, L=2, H=64, K=2, B=6)


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2507_11683_b200 import build
    build.build()
    from paper_2507_11683_b200 import pgti
    return pgti, torch


@pytest.fixture(scope="module")
def comm1(env):
    """A 1-rank NCCL communicator on cuda:0."""
    pgti, _ = env
    c = pgti.Comm(pgti.comm_unique_id(), 0, 1, 0)
    yield c
    c.close()


_REFS = {}


def ref_for(cfg):
    if cfg.name not in _REFS:
        _REFS[cfg.name] = pipeline.Reference(cfg)
    return _REFS[cfg.name]


@pytest.mark.parametrize("name", ["chickenpox", "metr_la", "pems_bay"])
@pytest.mark.parametrize("use_comm", [False, True])
def test_series_moments_match_alg1(env, comm1, name, use_comm):
    pgti, torch = env
    from gpu_util import load_series
    cfg = synth.CONFIGS[name]
    ref = ref_for(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg)
    sums = torch.zeros(3, dtype=torch.float64, device="cuda")
    mu, sigma = s.moments(ref.n_train, cfg.T_in, 0, ref.n_train + cfg.T_in - 1, sums,
                          comm1 if use_comm else None)
    assert abs(mu - ref.mu) <= 1e-12 * abs(ref.mu), (mu, ref.mu)
    assert abs(sigma - ref.sigma) <= 1e-12 * ref.sigma, (sigma, ref.sigma)
    # rows that no training window reads contribute nothing (TOO_FEW_ENTRIES when alone)
    with pytest.raises(pgti.PgtiError) as e:
        s.moments(ref.n_train, cfg.T_in, ref.n_train + cfg.T_in, cfg.E, sums)
    assert e.value.name == "TOO_FEW_ENTRIES"


def _train(env, cfg, ref, theta, steps, **kw):
    from paper_2507_11683_b200.trainer import Trainer
    tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, **kw)
    n = tr.start_epoch(0)
    losses = []
    for j in range(min(steps, n)):
        tr.step(j)
        losses.append(float(tr.loss.item()))
    tr.check()
    return tr, losses


@pytest.mark.parametrize("precision", [0, 1])
def test_one_rank_allreduce_in_captured_step_is_identity(env, comm1, precision):
    """a8 at world 1: pgti_allreduce_grads (ncclAllReduce SUM, in place) inside the captured
    graph; grad_scale 1/R = 1; parameters after 5 Adam steps bitwise equal to no all-reduce."""
    pgti, torch = env
    cfg = TC2
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="train")
    out = []
    for comm in (None, comm1):
        tr, losses = _train(env, cfg, ref, theta, 5, comm=comm, precision=precision,
                            use_cuda_graph=True)
        assert tr.graph is not None
        out.append((tr.params.cpu().numpy().view(np.uint32), losses))
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    # (NCCL short-circuits an in-place SUM over one rank: the captured call enqueues no kernel,
    # which is exactly the R = 1 identity; the 2-rank data path is tests/test_gpu_multi.py)


@pytest.mark.parametrize("model", [0, 1])
def test_bf16_graph_replay_matches_eager(env, model):
    """the bench's configuration (precision 1, L = 2, CUDA graph with the per-layer
    and aux streams and PDL edges) against eager launches, bitwise after 6 steps; the first
    step's loss against the float64 oracle (2e-2, BJ)."""
    pgti, torch = env
    cfg = TC2
    ref = ref_for(cfg)
    theta = synth.make_params(cfg, kind="train", model="encdec" if model else "stepwise")
    if model:
        theta = theta * 0.5   # fan-in-scaled init keeps the fed-back decoder well conditioned
    res = []
    for use_graph in (False, True):
        tr, losses = _train(env, cfg, ref, theta.astype(np.float32), 6, precision=1,
                            use_cuda_graph=use_graph, model=model)
        res.append((tr.params.cpu().numpy(), losses, tr.epoch_plan()[:cfg.B].cpu().numpy()))
    assert res[0][1] == res[1][1], (res[0][1], res[1][1])
    assert np.array_equal(res[0][0].view(np.uint32), res[1][0].view(np.uint32))
    idx = res[0][2]
    x, y = ref.batch(idx)
    if model:
        from oracle import encdec
        loss_ref = encdec.forward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                  x.astype(np.float64), y.astype(np.float64))["loss"]
    else:
        loss_ref = dcgru.forward(theta.astype(np.float64), ref.d, ref.Pf, ref.Pb,
                                 x.astype(np.float64), y.astype(np.float64))["loss"]
    assert abs(res[0][1][0] - loss_ref) <= 2e-2 * abs(loss_ref), (res[0][1][0], loss_ref)


@pytest.mark.parametrize("use_comm", [False, True])
def test_mean_losses(env, comm1, use_comm):
    pgti, torch = env
    rng = np.random.default_rng(5)
    v = rng.uniform(0.1, 2.0, size=1237).astype(np.float32)
    scratch = torch.zeros(2, dtype=torch.float64, device="cuda")
    got = pgti.mean_losses(torch.from_numpy(v).cuda(), v.size, scratch,
                           comm1 if use_comm else None)
    assert abs(got - v.astype(np.float64).mean()) <= 1e-13 * v.mean()
    assert np.isnan(pgti.mean_losses(torch.zeros(1, device="cuda"), 0, scratch))
