"""Li et al. DCRNN encoder-decoder (desc.model = 1, reading c24) through the C ABI
against oracle.encdec (float64): loss, predictions, every gradient tensor (1e-5 scale-relative,
reading c19), in both decoder feedback modes; and the bit-exact zero-copy variant."""
import numpy as np
import pytest

import synth
from gpu_util import ld_of, load_series, scale_rel
from oracle import dcgru, encdec, pipeline

pytestmark = pytest.mark.gpu
TOL32 = 1e-5

CFGS = {
    "ed_small": synth.Config("ed_small", N=12, E=60, F=2, T_in=3, T_out=4, L=2, H=16, K=2, B=3),
    "ed_odd": synth.Config("ed_odd", N=33, E=70, F=3, F_out=2, T_in=4, T_out=2, L=1, H=32, K=1,
                           B=5),
    "ed_k0": synth.Config("ed_k0", N=9, E=50, F=2, T_in=2, T_out=3, L=3, H=16, K=0, B=2),
}
_REFS = {}


def _ref(cfg):
    if cfg.name not in _REFS:
        _REFS[cfg.name] = pipeline.Reference(cfg)
    return _REFS[cfg.name]


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_11683_b200 import build
    build.build()
    from paper_2507_11683_b200 import pgti
    return pgti, torch


def _model(pgti, torch, cfg, graph, tf, precision=0):
    csr = pgti.csr_to_device(pgti.graph_build(cfg.N, *graph), "cuda")
    return pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out, cfg.B,
                      ld_of(cfg), csr, precision, model=1, teacher_forcing=tf,
                      cheb=cfg.cheb)


MODES = {"own": 0, "tf": True, "mixed": 0b1}  # mixed: only decoder step 1 fed the target


def _case(env, cfg, tf, seed=0, precision=0):
    pgti, torch = env
    tf = MODES.get(tf, tf)
    ref = _ref(cfg)
    s = load_series(pgti, torch, ref.v, 0, cfg, ref.mu, ref.sigma)
    idx_np = ref.plan(1, 0, epoch=seed)[:cfg.B]
    idx = torch.from_numpy(idx_np.astype(np.int32)).cuda()
    ld = ld_of(cfg)
    x = torch.empty(cfg.B * cfg.T_in * ld, device="cuda")
    y = torch.empty(cfg.B * cfg.T_out * ld, device="cuda")
    s.gather(idx, cfg.B, cfg.T_in, cfg.T_out, x, y)
    model = _model(pgti, torch, cfg, ref.graph, tf, precision)
    d = dcgru.Dims.of(cfg)
    n = model.num_params()
    assert n == encdec.num_params(d)
    if precision == 0:
        theta = np.random.default_rng(seed + 11).uniform(-0.4, 0.4, n).astype(np.float32)
    else:  # the bf16 path at the fan-in scaled init (as the stepwise bf16 parity tests)
        theta = synth.make_params(cfg, seed=synth.SEED_PARAMS + seed, kind="random",
                                  model="encdec")
    params = torch.from_numpy(theta).cuda()
    grads = torch.full((n,), float("nan"), device="cuda")
    loss = torch.zeros(1, device="cuda")
    ws = torch.empty(model.workspace_bytes(), dtype=torch.uint8, device="cuda")
    act = torch.empty(model.act_dump_floats(), device="cuda")
    model.step(params, grads, x, y, loss, ws, act)
    pgti.check_device_error()
    xo, yo = ref.batch(idx_np)
    loss_ref, g_ref, yhat_ref = encdec.loss_and_grad(theta.astype(np.float64), d, ref.Pf, ref.Pb,
                                                     xo.astype(np.float64),
                                                     yo.astype(np.float64), teacher_forcing=tf)
    margin = np.min(np.abs(yhat_ref - yo[..., :cfg.F_out].astype(np.float64)))
    return dict(loss=loss.item(), g=grads.cpu().numpy(), act=act.cpu().numpy(), loss_ref=loss_ref,
                g_ref=g_ref, yhat_ref=yhat_ref, margin=margin, d=d, model=model, s=s, idx=idx,
                params=params, ws=ws)


@pytest.mark.parametrize("tf", list(MODES))
@pytest.mark.parametrize("name", list(CFGS))
def test_encdec_step_vs_oracle(env, name, tf):
    cfg = CFGS[name]
    c = _case(env, cfg, tf)
    assert c["margin"] > 1e-5, "a residual sits at an |.| kink; pick another seed"
    assert abs(c["loss"] - c["loss_ref"]) <= TOL32 * abs(c["loss_ref"])
    R = cfg.N * cfg.B
    steps = cfg.T_in + cfg.T_out
    yhat = c["act"][steps * cfg.L * 4 * R * cfg.H:].reshape(cfg.T_out, cfg.N, cfg.B, cfg.F_out)
    assert scale_rel(yhat, c["yhat_ref"].transpose(1, 2, 0, 3)) <= TOL32
    gscale = np.max(np.abs(c["g_ref"]))
    off = 0
    for nm, shp in encdec.layer_shapes(c["d"]):
        n = int(np.prod(shp))
        g, gr = c["g"][off:off + n].astype(np.float64), c["g_ref"][off:off + n]
        den = max(np.max(np.abs(gr)), 1e-3 * gscale)
        assert np.max(np.abs(g - gr)) / den <= TOL32, (nm, np.max(np.abs(g - gr)) / den)
        off += n
    assert off == c["g"].size


def test_encdec_zero_copy_bitexact(env):
    pgti, torch = env
    cfg = CFGS["ed_small"]
    c = _case(env, cfg, "own")
    grads = torch.full_like(c["params"], float("nan"))
    loss = torch.zeros(1, device="cuda")
    c["model"].step_indexed(c["params"], grads, c["s"], c["idx"], loss, c["ws"])
    pgti.check_device_error()
    assert loss.item() == c["loss"] and np.array_equal(grads.cpu().numpy(), c["g"])


def test_encdec_metr_la_shape(env):
    """METR-LA-shaped encoder-decoder (372,353 parameters, 12 + 12 steps) at B = 8."""
    cfg = synth.CONFIGS["metr_la"].replace(B=8)
    c = _case(env, cfg, "mixed")
    assert c["model"].num_params() == 372353
    assert c["margin"] > 1e-5
    assert abs(c["loss"] - c["loss_ref"]) <= TOL32 * abs(c["loss_ref"])
    assert scale_rel(c["g"], c["g_ref"]) <= TOL32


TOL_BF16 = 2e-2
TC_CFGS = {
    "ed_tc": synth.Config("ed_tc", N=12, E=60, F=2, T_in=3, T_out=4, L=2, H=64, K=2, B=3),
    "ed_tc_odd": synth.Config("ed_tc_odd", N=33, E=70, F=3, F_out=2, T_in=4, T_out=2, L=1,
                              H=64, K=1, B=5),
    "ed_tc_l3": synth.Config("ed_tc_l3", N=20, E=60, F=2, T_in=2, T_out=3, L=3, H=64, K=2, B=4),
}


def _check(c, tol):
    assert c["margin"] > 1e-5, "a residual sits at an |.| kink; pick another seed"
    assert abs(c["loss"] - c["loss_ref"]) <= tol * abs(c["loss_ref"])
    gscale = np.max(np.abs(c["g_ref"]))
    off = 0
    for nm, shp in encdec.layer_shapes(c["d"]):
        n = int(np.prod(shp))
        g, gr = c["g"][off:off + n].astype(np.float64), c["g_ref"][off:off + n]
        den = max(np.max(np.abs(gr)), 1e-3 * gscale)
        assert np.max(np.abs(g - gr)) / den <= tol, (nm, np.max(np.abs(g - gr)) / den)
        off += n


@pytest.mark.parametrize("tf", list(MODES))
@pytest.mark.parametrize("name", list(TC_CFGS))
def test_encdec_bf16_vs_oracle(env, name, tf):
    """The encoder-decoder on the bf16 tcgen05 path (decoder input diffused per step, its layer-0
    input gradient by the skinny x-part dgrad) at the 2e-2 bf16 tolerance."""
    _check(_case(env, TC_CFGS[name], tf, precision=1), TOL_BF16)


@pytest.mark.parametrize("tf", list(MODES))
def test_encdec_bf16_metr_la(env, tf):
    cfg = synth.CONFIGS["metr_la"].replace(B=16)
    _check(_case(env, cfg, tf, precision=1), TOL_BF16)


def test_scheduled_sampling_trainer_matches_oracle_masks(env):
    """Trainer(scheduled_sampling=k): each step draws the decoder's per-step feeding mask; the
    step's loss equals the oracle's for that mask (fp32, 1e-5)."""
    pgti, torch = env
    from paper_2507_11683_b200.trainer import Trainer
    cfg = CFGS["ed_small"]
    ref = _ref(cfg)
    d = dcgru.Dims.of(cfg)
    theta = np.random.default_rng(3).uniform(-0.4, 0.4, encdec.num_params(d)).astype(np.float32)
    tr = Trainer(cfg, ref.graph, lambda a, b: ref.v[a:b], theta, precision=0, use_cuda_graph=False,
                 model=1, scheduled_sampling=2.0, lr=0.0)
    tr.start_epoch(0)
    masks = set()
    for j in range(6):
        tr.step(j)
        mask = tr.model.desc.teacher_forcing
        masks.add(mask)
        idx = tr.epoch_plan()[j * cfg.B:(j + 1) * cfg.B].cpu().numpy()
        xo, yo = ref.batch(idx)
        want = encdec.forward(theta.astype(np.float64), d, ref.Pf, ref.Pb, xo.astype(np.float64),
                              yo.astype(np.float64), teacher_forcing=mask)["loss"]
        assert abs(tr.loss.item() - want) <= TOL32 * abs(want), (j, mask)
    assert len(masks) > 1  # the curriculum actually varies the feeding
