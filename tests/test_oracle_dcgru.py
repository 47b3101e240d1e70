"""Pins for oracle.transitions and oracle.dcgru (diffusion, DCGRU, MAE, BPTT, Adam, DDP)."""
import math

import numpy as np
import pytest

import synth
from oracle import adam, dcgru, transitions


def _sig(a):
    return 1.0 / (1.0 + math.exp(-a))


# ----------------------------------------------------------------- transitions
def test_transition_matrices_hand_example():
    # A = [[1,2,0],[0,1,3],[4,0,1]] (A[i][j] = weight of i -> j)
    src = [0, 0, 1, 1, 2, 2]
    dst = [0, 1, 1, 2, 0, 2]
    w = [1, 2, 1, 3, 4, 1]
    Pf, Pb = transitions.transition_matrices(3, src, dst, w, dense=True)
    assert np.allclose(Pf, [[1 / 3, 2 / 3, 0], [0, 1 / 4, 3 / 4], [4 / 5, 0, 1 / 5]], rtol=0, atol=1e-15)
    assert np.allclose(Pb, [[1 / 5, 0, 4 / 5], [2 / 3, 1 / 3, 0], [0, 3 / 4, 1 / 4]], rtol=0, atol=1e-15)


def test_zero_degree_rows_are_zero():
    Pf, Pb = transitions.transition_matrices(3, [0], [1], [2.0], dense=True)
    assert np.array_equal(Pf, [[0, 1, 0], [0, 0, 0], [0, 0, 0]])
    assert np.array_equal(Pb, [[0, 0, 0], [1, 0, 0], [0, 0, 0]])


def test_row_stochastic():
    src, dst, w = synth.make_graph(50, 8, seed=4)
    Pf, Pb = transitions.transition_matrices(50, src, dst, w, dense=True)
    assert np.allclose(Pf.sum(1), 1, atol=1e-14) and np.allclose(Pb.sum(1), 1, atol=1e-14)


# ------------------------------------------------------------------- diffusion
def test_diffusion_vs_matrix_power():
    src, dst, w = synth.random_graph(9, 0.3, seed=5)
    Pf, Pb = transitions.transition_matrices(9, src, dst, w, dense=True)
    Pfs, Pbs = transitions.transition_matrices(9, src, dst, w)
    Z = np.random.default_rng(0).normal(size=(9, 7))
    K = 3
    T = dcgru.diffusion_features(Pfs, Pbs, Z, K)
    assert T.shape == (2 * K + 1, 9, 7)
    assert np.array_equal(T[0], Z)
    for k in range(1, K + 1):
        assert np.allclose(T[k], np.linalg.matrix_power(Pf, k) @ Z, rtol=1e-12, atol=1e-14)
        assert np.allclose(T[K + k], np.linalg.matrix_power(Pb, k) @ Z, rtol=1e-12, atol=1e-14)


def test_diffusion_ring_is_roll():
    N = 7
    Pf, Pb = transitions.transition_matrices(N, *synth.ring_graph(N))
    Z = np.random.default_rng(1).normal(size=(N, 3))
    K = 3
    T = dcgru.diffusion_features(Pf, Pb, Z, K)
    for k in range(1, K + 1):
        assert np.array_equal(T[k], np.roll(Z, -k, axis=0))      # (P_f Z)[i] = Z[i+1]
        assert np.array_equal(T[K + k], np.roll(Z, k, axis=0))   # (P_b Z)[i] = Z[i-1]


def test_diffusion_complete_graph_and_self_loops():
    N = 6
    src, dst = np.nonzero(np.ones((N, N)))
    Pf, Pb = transitions.transition_matrices(N, src, dst, np.ones(src.size))
    Z = np.random.default_rng(2).normal(size=(N, 4))
    T = dcgru.diffusion_features(Pf, Pb, Z, 2)
    for m in range(1, 5):
        assert np.allclose(T[m], np.broadcast_to(Z.mean(0), Z.shape), atol=1e-14)
    Pf, Pb = transitions.transition_matrices(N, np.arange(N), np.arange(N), np.full(N, 2.5))
    T = dcgru.diffusion_features(Pf, Pb, Z, 2)
    assert all(np.array_equal(T[m], Z) for m in range(5))


def test_diffusion_adjoint_dot_product():
    src, dst, w = synth.random_graph(11, 0.25, seed=6)
    Pf, Pb = transitions.transition_matrices(11, src, dst, w)
    rng = np.random.default_rng(3)
    Z = rng.normal(size=(11, 5))
    dT = rng.normal(size=(5, 11, 5))
    lhs = np.sum(dcgru.diffusion_features(Pf, Pb, Z, 2) * dT)
    rhs = np.sum(Z * dcgru.diffusion_adjoint(Pf, Pb, dT, 2))
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


# ----------------------------------------------------------------------- DCGRU
def _dims(**kw):
    base = dict(N=5, F=2, F_out=1, L=2, H=3, K=2, T_in=3, T_out=2)
    base.update(kw)
    return dcgru.Dims(**base)


def _blocks(theta, d):
    return dcgru.unpack(theta, d)  # views into theta: writes go through


def _rand_problem(d, B=2, seed=0, graph=None):
    rng = np.random.default_rng(seed)
    g = graph if graph is not None else synth.random_graph(d.N, 0.4, seed=seed + 100)
    Pf, Pb = transitions.transition_matrices(d.N, *g)
    x = rng.normal(size=(B, d.T_in, d.N, d.F))
    y = rng.normal(size=(B, d.T_out, d.N, d.F))
    theta = rng.uniform(-0.5, 0.5, dcgru.num_params(d))
    return theta, Pf, Pb, x, y, g


def test_num_params_matches_layout():
    cfg = synth.CONFIGS["metr_la"]
    assert dcgru.num_params(dcgru.Dims.of(cfg)) == synth.num_params(cfg) == 186689
    assert dcgru.num_params(dcgru.Dims.of(synth.CONFIGS["chickenpox"])) == 15969


def test_zero_params_give_bout():
    # theta = 0 -> gates 0.5, c = 0, H stays 0 -> yhat = b_out
    d = _dims()
    _, Pf, Pb, x, y, _ = _rand_problem(d)
    theta = np.zeros(dcgru.num_params(d))
    theta[-1] = 0.7
    out = dcgru.forward(theta, d, Pf, Pb, x, y)
    assert np.array_equal(out["yhat"], np.full_like(out["yhat"], 0.7))


def test_bias_only_closed_form():
    # all weights 0: r, u, c constant per unit, H_t = c (1 - u^(t+1)) in every layer
    d = _dims(T_in=4, T_out=3)
    _, Pf, Pb, x, y, _ = _rand_problem(d)
    rng = np.random.default_rng(9)
    theta = np.zeros(dcgru.num_params(d))
    layers, W_out, b_out = _blocks(theta, d)
    for p in layers:
        p["b_ru"][:] = rng.normal(size=2 * d.H)
        p["b_c"][:] = rng.normal(size=d.H)
    W_out[:] = rng.normal(size=W_out.shape)
    b_out[:] = 0.3
    out = dcgru.forward(theta, d, Pf, Pb, x, y)
    acts, yhat = dcgru.activations(out, d)
    for t in range(d.T_in):
        for l, p in enumerate(layers):
            u = np.array([_sig(b) for b in p["b_ru"][d.H:]])
            c = np.tanh(p["b_c"])
            Ht = c * (1 - u ** (t + 1))
            assert np.allclose(acts[t, l, 0], np.broadcast_to(Ht, acts[t, l, 0].shape), atol=1e-15)
        if t >= d.T_in - d.T_out:
            pL = layers[-1]
            u = np.array([_sig(b) for b in pL["b_ru"][d.H:]])
            Ht = np.tanh(pL["b_c"]) * (1 - u ** (t + 1))
            assert np.allclose(yhat[:, t - 1], Ht @ W_out + 0.3, atol=1e-14)


def test_ring_block_order_and_orientation():
    # ring i -> i+1; a weight on block m of the input channel makes c read
    # x[n+k] (P_f^k) or x[n-k] (P_b^k)
    N, K = 6, 2
    g = synth.ring_graph(N)
    Pf, Pb = transitions.transition_matrices(N, *g)
    d = dcgru.Dims(N=N, F=1, F_out=1, L=1, H=1, K=K, T_in=1, T_out=1)
    x = np.random.default_rng(0).normal(size=(1, 1, N, 1))
    for m, shift in [(0, 0), (1, 1), (2, 2), (3, -1), (4, -2)]:
        theta = np.zeros(dcgru.num_params(d))
        layers, W_out, _ = _blocks(theta, d)
        layers[0]["W_c"][m, 0, 0] = 0.8
        W_out[:] = 1.0
        yhat = dcgru.forward(theta, d, Pf, Pb, x)["yhat"][0, 0, :, 0]
        want = 0.5 * np.tanh(0.8 * np.roll(x[0, 0, :, 0], -shift))
        assert np.allclose(yhat, want, atol=1e-15), m


def test_ring_hidden_channel_and_gate_columns():
    # C_in order (input first, hidden second), gate columns (r first, u second)
    N, K = 5, 1
    Pf, Pb = transitions.transition_matrices(N, *synth.ring_graph(N))
    d = dcgru.Dims(N=N, F=1, F_out=1, L=1, H=1, K=K, T_in=2, T_out=1)
    x = np.random.default_rng(1).normal(size=(1, 2, N, 1))
    theta = np.zeros(dcgru.num_params(d))
    layers, W_out, _ = _blocks(theta, d)
    a, w, br, bu = 0.9, -1.3, 0.4, -0.7
    layers[0]["W_c"][0, 0, 0] = a      # block 0, input channel
    layers[0]["W_c"][1, 1, 0] = w      # block 1 (P_f), hidden channel
    layers[0]["b_ru"][:] = [br, bu]
    W_out[:] = 1.0
    yhat = dcgru.forward(theta, d, Pf, Pb, x)["yhat"][0, 0, :, 0]
    r, u = _sig(br), _sig(bu)
    x0, x1 = x[0, 0, :, 0], x[0, 1, :, 0]
    H0 = (1 - u) * np.tanh(a * x0)
    H1 = u * H0 + (1 - u) * np.tanh(a * x1 + w * r * np.roll(H0, -1))
    assert np.allclose(yhat, H1, atol=1e-15)


def test_self_loop_graph_equals_k0_with_summed_blocks():
    # P = I: every diffusion block equals Z, so the K=2 model equals the K=0
    # model (a per-node GRU) whose weights are the block sums
    d2 = _dims(K=2)
    d0 = _dims(K=0)
    N = d2.N
    g = (np.arange(N, dtype=np.int32), np.arange(N, dtype=np.int32), np.ones(N, np.float32))
    theta, Pf, Pb, x, y, _ = _rand_problem(d2, graph=g)
    l2, W2, b2 = _blocks(theta, d2)
    theta0 = np.zeros(dcgru.num_params(d0))
    l0, W0, b0 = _blocks(theta0, d0)
    for p2, p0 in zip(l2, l0):
        p0["W_ru"][0] = p2["W_ru"].sum(0)
        p0["W_c"][0] = p2["W_c"].sum(0)
        p0["b_ru"][:], p0["b_c"][:] = p2["b_ru"], p2["b_c"]
    W0[:], b0[:] = W2, b2
    o2 = dcgru.forward(theta, d2, Pf, Pb, x, y)
    o0 = dcgru.forward(theta0, d0, Pf, Pb, x, y)
    assert np.allclose(o2["yhat"], o0["yhat"], atol=1e-13)


def test_node_permutation_equivariance():
    d = _dims()
    theta, _, _, x, y, g = _rand_problem(d, seed=4)
    perm = np.random.default_rng(5).permutation(d.N)
    inv = np.argsort(perm)
    Pf, Pb = transitions.transition_matrices(d.N, *g)
    Pf2, Pb2 = transitions.transition_matrices(d.N, inv[g[0]], inv[g[1]], g[2])
    l1, g1, f1 = dcgru.backward(theta, d, Pf, Pb, x, y)
    l2, g2, f2 = dcgru.backward(theta, d, Pf2, Pb2, x[:, :, perm], y[:, :, perm])
    assert np.allclose(f2["yhat"], f1["yhat"][:, :, perm], atol=1e-13)
    assert abs(l1 - l2) < 1e-13 and np.allclose(g1, g2, atol=1e-12)


def test_loss_closed_forms():
    # yhat == y -> 0; yhat = y + 1 -> 1 (yhat = b_out via theta = 0)
    d = _dims()
    _, Pf, Pb, x, y, _ = _rand_problem(d)
    theta = np.zeros(dcgru.num_params(d))
    theta[-1] = 0.25
    y = y.copy()
    y[..., 0] = 0.25
    assert dcgru.forward(theta, d, Pf, Pb, x, y)["loss"] == 0.0
    y[..., 0] = -0.75
    assert dcgru.forward(theta, d, Pf, Pb, x, y)["loss"] == 1.0


@pytest.mark.parametrize("L,K,T_in,T_out", [(2, 2, 3, 2), (1, 1, 2, 1), (2, 0, 2, 2)])
def test_backward_finite_differences(L, K, T_in, T_out):
    # central differences, relative error < 1e-5 on every coordinate
    d = _dims(L=L, K=K, T_in=T_in, T_out=T_out, N=4, H=2)
    theta, Pf, Pb, x, y, _ = _rand_problem(d, seed=L * 10 + K)
    loss, grad, fwd = dcgru.backward(theta, d, Pf, Pb, x, y)
    assert np.min(np.abs(fwd["yhat"] - y[..., :1])) > 1e-4  # away from |.| kinks
    h = 1e-6
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (dcgru.forward(tp, d, Pf, Pb, x, y)["loss"] -
              dcgru.forward(tm, d, Pf, Pb, x, y)["loss"]) / (2 * h)
        if abs(grad[i]) > 1e-8 or abs(fd) > 1e-8:
            assert abs(fd - grad[i]) <= 1e-5 * max(abs(grad[i]), abs(fd)) + 1e-9, (i, fd, grad[i])


def test_backward_vs_torch_autograd():
    # an independent float64 autograd (torch, CPU) of the same model
    torch = pytest.importorskip("torch")
    d = _dims(N=7, H=4, T_in=4, T_out=3)
    theta, Pf, Pb, x, y, _ = _rand_problem(d, B=3, seed=11)
    loss, grad, _ = dcgru.backward(theta, d, Pf, Pb, x, y)
    th = torch.tensor(theta, dtype=torch.float64, requires_grad=True)
    Pft = torch.tensor(Pf.toarray())
    Pbt = torch.tensor(Pb.toarray())
    xt, yt = torch.tensor(x), torch.tensor(y)
    off = [0]

    def take(*shape):
        n = int(np.prod(shape))
        out = th[off[0]:off[0] + n].reshape(shape)
        off[0] += n
        return out

    layers = []
    for l in range(d.L):
        c = d.c_in(l)
        layers.append((take(d.M, c, 2 * d.H), take(2 * d.H), take(d.M, c, d.H), take(d.H)))
    W_out, b_out = take(d.H, d.F_out), take(d.F_out)

    def feats(Z):  # Z [B,N,C] -> [B,N,M,C]
        out, T = [Z], Z
        for _ in range(d.K):
            T = torch.einsum("ij,bjc->bic", Pft, T)
            out.append(T)
        T = Z
        for _ in range(d.K):
            T = torch.einsum("ij,bjc->bic", Pbt, T)
            out.append(T)
        return torch.stack(out, 2)

    B = x.shape[0]
    Hs = [torch.zeros(B, d.N, d.H, dtype=torch.float64) for _ in range(d.L)]
    preds = []
    for t in range(d.T_in):
        inp = xt[:, t]
        for l, (Wru, bru, Wc, bc) in enumerate(layers):
            G = torch.einsum("bnmc,mcj->bnj", feats(torch.cat([inp, Hs[l]], -1)), Wru) + bru
            r, u = torch.sigmoid(G[..., :d.H]), torch.sigmoid(G[..., d.H:])
            cc = torch.tanh(torch.einsum("bnmc,mcj->bnj", feats(torch.cat([inp, r * Hs[l]], -1)), Wc) + bc)
            Hs[l] = u * Hs[l] + (1 - u) * cc
            inp = Hs[l]
        if t >= d.T_in - d.T_out:
            preds.append(Hs[-1] @ W_out + b_out)
    lt = (torch.stack(preds, 1) - yt[..., :d.F_out]).abs().mean()
    lt.backward()
    assert abs(lt.item() - loss) < 1e-13
    assert np.allclose(th.grad.numpy(), grad, rtol=1e-10, atol=1e-13)


def test_ddp_equivalence_union_batch():
    # mean of R per-rank gradients on B windows each == gradient of the
    # union batch of R*B windows (equal B per rank)
    d = _dims()
    theta, Pf, Pb, x, y, _ = _rand_problem(d, B=8, seed=21)
    l_all, g_all, _ = dcgru.backward(theta, d, Pf, Pb, x, y)
    for R in (2, 4, 8):
        parts = [dcgru.backward(theta, d, Pf, Pb, x[r::R], y[r::R])[1] for r in range(R)]
        assert np.allclose(adam.allreduce_mean(parts), g_all, rtol=1e-12, atol=1e-15)
    assert np.array_equal(adam.allreduce_mean([g_all]), g_all)          # R = 1 identity
    assert adam.allreduce_mean([np.array([1.0]), np.array([3.0])])[0] == 2.0


def test_adam_hand_step_and_torch():
    # theta 0, g 1, lr 0.1, step 1 -> -0.1 (m_hat = v_hat = 1)
    th, m, v = adam.adam_step(np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 1, 0.1)
    assert abs(th[0] + 0.1 / (1 + 1e-8)) < 1e-17
    th, _, _ = adam.adam_step(np.ones(3), np.zeros(3), np.zeros(3), np.zeros(3), 1, 0.1)
    assert np.array_equal(th, np.ones(3))  # zero grad at step 1 -> unchanged
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    p0 = rng.normal(size=20)
    p = torch.tensor(p0, requires_grad=True)
    opt = torch.optim.Adam([p], lr=1e-2)
    th, m, v = p0.copy(), np.zeros(20), np.zeros(20)
    for step in range(1, 6):
        g = rng.normal(size=20)
        p.grad = torch.tensor(g * 0.5)
        opt.step()
        th, m, v = adam.adam_step(th, g, m, v, step, 1e-2, grad_scale=0.5)
        assert np.allclose(p.detach().numpy(), th, rtol=1e-14, atol=1e-15)


# --------------------------------------------------------- Chebyshev variant (reading c25)
@pytest.mark.parametrize("a", [0.3, -0.7, 1.0])
def test_chebyshev_blocks_on_scaled_identity(a):
    """With P = a I the recurrence gives the Chebyshev polynomials of the first kind:
    T_0 = 1, T_1 = a, T_2 = 2a^2 - 1, T_3 = 4a^3 - 3a."""
    N, W, K = 4, 3, 3
    P = a * np.eye(N)
    Z = np.random.default_rng(0).normal(size=(N, W))
    T = dcgru.diffusion_features(P, P, Z, K, cheb=True)
    want = [1.0, a, 2 * a * a - 1, 4 * a ** 3 - 3 * a]
    for k in range(K + 1):
        assert np.allclose(T[k], want[k] * Z, rtol=0, atol=1e-14)
        if k:
            assert np.allclose(T[K + k], want[k] * Z, rtol=0, atol=1e-14)


def test_chebyshev_k1_equals_powers_and_adjoint_identity():
    src, dst, w = synth.random_graph(9, 0.3, seed=8)
    Pf, Pb = transitions.transition_matrices(9, src, dst, w, dense=True)
    rng = np.random.default_rng(1)
    Z = rng.normal(size=(9, 5))
    assert np.array_equal(dcgru.diffusion_features(Pf, Pb, Z, 1, cheb=True),
                          dcgru.diffusion_features(Pf, Pb, Z, 1))
    for K in (2, 3):
        T = dcgru.diffusion_features(Pf, Pb, Z, K, cheb=True)
        dT = rng.normal(size=T.shape)
        lhs = np.sum(T * dT)
        rhs = np.sum(Z * dcgru.diffusion_adjoint(Pf, Pb, dT, K, cheb=True))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_chebyshev_backward_finite_differences():
    d = dcgru.Dims(N=4, F=2, F_out=1, L=2, H=2, K=2, T_in=3, T_out=2, cheb=True)
    theta, Pf, Pb, x, y, _ = _rand_problem(d, seed=9)
    loss, grad, fwd = dcgru.backward(theta, d, Pf, Pb, x, y)
    assert np.min(np.abs(fwd["yhat"] - y[..., :1])) > 1e-4
    h = 1e-6
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (dcgru.forward(tp, d, Pf, Pb, x, y)["loss"] -
              dcgru.forward(tm, d, Pf, Pb, x, y)["loss"]) / (2 * h)
        if abs(grad[i]) > 1e-8 or abs(fd) > 1e-8:
            assert abs(fd - grad[i]) <= 1e-5 * max(abs(grad[i]), abs(fd)) + 1e-9, (i, fd, grad[i])
