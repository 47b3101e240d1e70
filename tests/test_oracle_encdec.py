"""Pins for oracle.encdec (Li et al. DCRNN encoder-decoder, reading c24)."""
import numpy as np
import pytest

import synth
from oracle import dcgru, encdec, transitions


def _dims(**kw):
    base = dict(N=5, F=2, F_out=1, L=2, H=3, K=2, T_in=3, T_out=2)
    base.update(kw)
    return dcgru.Dims(**base)


def _problem(d, B=2, seed=0):
    rng = np.random.default_rng(seed)
    g = synth.random_graph(d.N, 0.4, seed=seed + 100)
    Pf, Pb = transitions.transition_matrices(d.N, *g)
    x = rng.normal(size=(B, d.T_in, d.N, d.F))
    y = rng.normal(size=(B, d.T_out, d.N, d.F))
    theta = rng.uniform(-0.5, 0.5, encdec.num_params(d))
    return theta, Pf, Pb, x, y


def test_param_count_is_li_et_al():
    # Li et al.'s DCRNN on METR-LA (2 layers, 64 units, K = 2, 2 input channels, 1 output):
    # 372,353 trainable parameters [ext]
    assert encdec.num_params(dcgru.Dims.of(synth.CONFIGS["metr_la"])) == 372353


def test_encoder_is_the_stepwise_stack():
    """The encoder's final states equal oracle.dcgru's (independently pinned) stepwise stack run
    with the encoder's parameters."""
    d = _dims()
    theta, Pf, Pb, x, y = _problem(d)
    out = encdec.forward(theta, d, Pf, Pb, x, y)
    n_enc = sum(int(np.prod(s)) for name, s in encdec.layer_shapes(d) if name.startswith("enc"))
    step_theta = np.concatenate([theta[:n_enc], np.zeros(d.H * d.F_out + d.F_out)])
    ref = dcgru.forward(step_theta, d.__class__(d.N, d.F, d.F_out, d.L, d.H, d.K, d.T_in, 1),
                        Pf, Pb, x)
    for l in range(d.L):
        assert np.allclose(out["H_enc"][l], ref["cache"][d.T_in - 1][l]["H"], rtol=0, atol=1e-14)


def test_numpy_and_torch_transcriptions_agree():
    d = _dims()
    theta, Pf, Pb, x, y = _problem(d, seed=3)
    for tf in (False, True):
        out = encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=tf)
        loss, _, yhat = encdec.loss_and_grad(theta, d, Pf, Pb, x, y, teacher_forcing=tf)
        assert np.allclose(yhat, out["yhat"], rtol=0, atol=1e-13)
        assert abs(loss - out["loss"]) < 1e-14


def test_single_step_decoder_ignores_the_feedback_mode():
    # with T_out = 1 the decoder only ever sees the GO symbol
    d = _dims(T_out=1)
    theta, Pf, Pb, x, y = _problem(d, seed=4)
    a = encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=False)["yhat"]
    b = encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=True)["yhat"]
    assert np.array_equal(a, b)


def test_teacher_forcing_feeds_the_truth():
    # feeding y_{s-1} and feeding the model's own yhat_{s-1} coincide when y is set to the
    # model's own predictions
    d = _dims(T_out=3)
    theta, Pf, Pb, x, y = _problem(d, seed=5)
    own = encdec.forward(theta, d, Pf, Pb, x, y)["yhat"]
    y2 = y.copy()
    y2[..., :d.F_out] = own
    tf = encdec.forward(theta, d, Pf, Pb, x, y2, teacher_forcing=True)["yhat"]
    assert np.allclose(tf, own, rtol=0, atol=1e-14)


def test_step_mask_selects_the_fed_inputs():
    """A per-step mask (scheduled sampling's coin flips): mask 0 == own predictions, the full mask
    == teacher forcing, and any mask is exact when y equals the model's own predictions."""
    d = _dims(T_out=4)
    theta, Pf, Pb, x, y = _problem(d, seed=6)
    own = encdec.forward(theta, d, Pf, Pb, x, y)["yhat"]
    assert np.array_equal(encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=0)["yhat"], own)
    full = encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=True)["yhat"]
    assert np.array_equal(encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=0b111)["yhat"],
                          full)
    mixed = encdec.forward(theta, d, Pf, Pb, x, y, teacher_forcing=0b010)["yhat"]
    assert np.array_equal(mixed[:, :2], own[:, :2])        # steps 0, 1 fed GO / own prediction
    assert not np.allclose(mixed[:, 2], own[:, 2])          # step 2 fed the target y_1
    y2 = y.copy()
    y2[..., :d.F_out] = own
    for m in (0b001, 0b010, 0b101):
        assert np.allclose(encdec.forward(theta, d, Pf, Pb, x, y2, teacher_forcing=m)["yhat"], own,
                           rtol=0, atol=1e-14)


@pytest.mark.parametrize("tf,L,K", [(False, 2, 2), (True, 1, 1), (False, 1, 0), (0b10, 2, 1)])
def test_gradient_finite_differences(tf, L, K):
    d = _dims(N=4, H=2, L=L, K=K, T_in=2, T_out=3)
    theta, Pf, Pb, x, y = _problem(d, seed=L * 7 + K)
    loss, grad, yhat = encdec.loss_and_grad(theta, d, Pf, Pb, x, y, teacher_forcing=tf)
    assert np.min(np.abs(yhat - y[..., :1])) > 1e-4  # away from |.| kinks
    h = 1e-6
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (encdec.forward(tp, d, Pf, Pb, x, y, teacher_forcing=tf)["loss"] -
              encdec.forward(tm, d, Pf, Pb, x, y, teacher_forcing=tf)["loss"]) / (2 * h)
        if abs(grad[i]) > 1e-8 or abs(fd) > 1e-8:
            assert abs(fd - grad[i]) <= 1e-5 * max(abs(grad[i]), abs(fd)) + 1e-9, (i, fd, grad[i])


def test_chebyshev_encdec_transcriptions_and_gradient():
    d = _dims(N=4, H=2, L=2, K=2, T_in=2, T_out=3, cheb=True)
    theta, Pf, Pb, x, y = _problem(d, seed=12)
    out = encdec.forward(theta, d, Pf, Pb, x, y)
    loss, grad, yhat = encdec.loss_and_grad(theta, d, Pf, Pb, x, y)
    assert np.allclose(yhat, out["yhat"], rtol=0, atol=1e-13)
    assert np.min(np.abs(yhat - y[..., :1])) > 1e-4
    h = 1e-6
    for i in range(0, theta.size, 7):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (encdec.forward(tp, d, Pf, Pb, x, y)["loss"] -
              encdec.forward(tm, d, Pf, Pb, x, y)["loss"]) / (2 * h)
        if abs(grad[i]) > 1e-8 or abs(fd) > 1e-8:
            assert abs(fd - grad[i]) <= 1e-5 * max(abs(grad[i]), abs(fd)) + 1e-9, (i, fd, grad[i])
