"""The oracle's end-to-end reference pipeline for one configuration (SURVEY
8(c) rows O1-O13): synthetic inputs -> Alg. 1 materialisation -> index plan ->
batch -> DCGRU forward/backward -> (DDP mean) -> Adam.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

import synth

from . import dcgru, philox, transitions, windows


class Reference:
    """Everything the oracle derives for a config, built lazily.

    ``materialize_all``: stack every snapshot (Alg. 1) -- the default for the
    small configs; for large ones only the requested windows are stacked
    (same definition on fewer windows).
    """

    def __init__(self, cfg, data_seed=synth.SEED_DATA, graph_seed=synth.SEED_GRAPH,
                 materialize_all=None, graph=None, v=None):
        self.cfg = cfg
        self.d = dcgru.Dims.of(cfg)
        self.graph = graph if graph is not None else synth.make_graph(cfg.N, cfg.knn, graph_seed)
        self.v = v if v is not None else synth.make_series(cfg, data_seed, graph_seed=graph_seed)
        self.S = windows.num_windows(cfg.E, cfg.T_in, cfg.T_out)
        self.n_train, self.n_val, self.n_test = windows.split_counts(self.S)
        self.mu, self.sigma = windows.alg1_stats(self.v, cfg.T_in, cfg.T_out)
        self.Pf, self.Pb = transitions.transition_matrices(cfg.N, *self.graph)
        if materialize_all is None:
            materialize_all = self.S * (cfg.T_in + cfg.T_out) * cfg.N * cfg.F * 4 < (1 << 30)
        self.features = self.targets = None
        if materialize_all:
            self.features, self.targets = windows.materialize(self.v, cfg.T_in, cfg.T_out,
                                                              self.mu, self.sigma)

    def batch(self, idx):
        """x[B][T_in][N][F], y[B][T_out][N][F] float32 snapshots of windows idx."""
        idx = np.asarray(idx, dtype=np.int64)
        if self.features is not None:
            return self.features[idx], self.targets[idx]
        return windows.materialize(self.v, self.cfg.T_in, self.cfg.T_out, self.mu, self.sigma,
                                   starts=idx)

    def plan(self, R, r, seed=synth.SEED_SHUFFLE, epoch=0, shuffle=True, B=None):
        return philox.index_plan(self.n_train, R, r, B or self.cfg.B, seed, epoch, shuffle)

    def loss_and_grad(self, theta, idx):
        x, y = self.batch(idx)
        return dcgru.backward(theta, self.d, self.Pf, self.Pb, x.astype(np.float64),
                              y.astype(np.float64))
