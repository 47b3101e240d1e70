"""Host driver of the index-batched training step (distributed-index-batching).

Host-side arithmetic here is bookkeeping only (window counts, shard ranges, Adam step count);
every value the model sees is produced by libpgti kernels:

  load (one H2D copy) -> stats (window-weighted Alg. 1) -> normalise
   -> per-epoch index plan -> per step: gather -> DCGRU
  forward/backward -> NCCL all-reduce -> Adam.

Halo sharding (BASELINE.json north_star, the default): rank r of R owns window starts
[r S_r, (r+1) S_r), S_r = floor(S_tr / R), and holds series rows [r S_r, (r+1) S_r + T_in +
T_out - 1).  The last rank additionally holds the rows the statistics need up to S_tr + T_in - 1.

Replicated placement (the paper's distributed-index-batching): every rank
holds the whole series, derives the same global permutation of all training windows with no
exchange and visits its slice of it; validation MAE is all-reduced each epoch.
Batch-level shuffle (generalized variant): shuffle="batch" keeps each batch's
membership and permutes the batch order.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import pgti


def window_count(E: int, T_in: int, T_out: int) -> int:
    """S = E - T_in - T_out + 1 windows (Eq. 2; DESIGN reading c11)."""
    return max(0, E - T_in - T_out + 1)


def train_windows(S: int) -> int:
    """round(S * 0.70) (Alg. 1)."""
    return round(S * 0.70)


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    win_lo: int     # first global window start of this rank
    win_hi: int     # one past the last
    row_lo: int     # first global series row held
    row_hi: int     # one past the last row held
    stat_lo: int    # rows whose Alg. 1 statistics this rank contributes
    stat_hi: int


def shard_plan(S_tr: int, R: int, r: int, T_in: int, T_out: int) -> ShardPlan:
    S_r = S_tr // R
    win_lo, win_hi = r * S_r, (r + 1) * S_r
    row_lo, row_hi = win_lo, win_hi + T_in + T_out - 1
    stat_lo = win_lo
    stat_hi = win_hi if r < R - 1 else S_tr + T_in - 1
    row_hi = max(row_hi, stat_hi)
    return ShardPlan(win_lo, win_hi, row_lo, row_hi, stat_lo, stat_hi)


def replicated_plan(S_tr: int, E: int, T_in: int) -> ShardPlan:
    """Replicated placement: all rows [0, E) held, all training windows in the (global) plan,
    statistics computed locally over the rows training windows read (no exchange)."""
    return ShardPlan(0, S_tr, 0, E, 0, S_tr + T_in - 1)


def val_windows(S: int) -> int:
    """Validation windows after the training ones: S - round(0.7 S) - round(0.2 S) (the 70/10/20
    split of P:243, Alg. 1 line 200 with Python round)."""
    return S - round(S * 0.70) - round(S * 0.20)


def row_pitch(N: int, F: int) -> int:
    """ld = roundup(N F, 4) floats: 16-byte aligned time rows (SURVEY decision 5)."""
    return (N * F + 3) // 4 * 4


class Trainer:
    """One rank of distributed-index-batching.

    cfg: any object with N, E, F, F_out, T_in, T_out, L, H, K, B.
    graph: (src, dst, w) edge list.  series_fn(row_lo, row_hi) -> float32 [rows][N][F] raw
    values of those global rows.  params0: float32 [num_params] initial parameters.
    """

    def __init__(self, cfg, graph, series_fn, params0, rank=0, world=1, device=0, comm=None,
                 seed=3, lr=1e-2, precision=0, shuffle=True, use_cuda_graph=True,
                 placement="halo", zero_copy=False, model=0, teacher_forcing=0,
                 scheduled_sampling=None, cheb=None):
        import torch

        self.torch = torch
        self.cfg, self.rank, self.world, self.comm = cfg, rank, world, comm
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        self.seed, self.lr, self.shuffle = seed, lr, shuffle
        self.S = window_count(cfg.E, cfg.T_in, cfg.T_out)
        self.S_tr = train_windows(self.S)
        assert placement in ("halo", "replicated"), placement
        assert shuffle in (True, False, "batch"), shuffle
        assert not (placement == "replicated" and shuffle == "batch"), "batch shuffle is per shard"
        self.placement = placement
        self.zero_copy = zero_copy  # f2: windows read from the series by index, no x/y gather
        # Li et al.'s curriculum (encoder-decoder): decoder step s >= 1 is fed the target with
        # probability k / (k + exp(step / k)), one coin per step and batch; the mask lives in the
        # descriptor, so this runs eager (no captured graph)
        assert scheduled_sampling is None or (model == 1 and not use_cuda_graph), \
            "scheduled sampling needs the encoder-decoder and eager steps"
        self.ss_k = scheduled_sampling
        self.ss_rng = np.random.default_rng(seed * 1000003 + rank)
        self.steps_done = 0
        self.S_r = self.S_tr // world
        self.idx_off = 0
        self.plan = (shard_plan(self.S_tr, world, rank, cfg.T_in, cfg.T_out)
                     if placement == "halo" else replicated_plan(self.S_tr, cfg.E, cfg.T_in))
        self.ld = row_pitch(cfg.N, cfg.F)
        p = self.plan
        rows = np.ascontiguousarray(series_fn(p.row_lo, p.row_hi), dtype=np.float32)
        assert rows.shape == (p.row_hi - p.row_lo, cfg.N, cfg.F), rows.shape
        self.host_rows = torch.from_numpy(rows).pin_memory()
        self.series_buf = torch.empty((p.row_hi - p.row_lo) * self.ld, dtype=torch.float32,
                                      device=self.dev)
        self.series = pgti.Series(self.host_rows, p.row_lo, cfg.N, cfg.F, self.series_buf,
                                  self.ld)
        self.mu, self.sigma = self._stats()
        self.series.normalize(self.mu, self.sigma)

        csr = pgti.graph_build(cfg.N, *graph)
        self.cheb = bool(getattr(cfg, "cheb", False) if cheb is None else cheb)
        csr = pgti.add_windows(csr, cfg.N)
        self.csr = pgti.csr_to_device(csr, self.dev)
        self.model = pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in,
                                cfg.T_out, cfg.B, self.ld, self.csr, precision, model=model,
                                teacher_forcing=teacher_forcing, cheb=self.cheb)
        n = self.model.num_params()
        assert params0.size == n, (params0.size, n)
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.params = torch.from_numpy(np.ascontiguousarray(params0, np.float32)).to(self.dev)
        self.grads = torch.zeros(n, **f32)
        self.m = torch.zeros(n, **f32)
        self.v = torch.zeros(n, **f32)
        self.ws = torch.empty(self.model.workspace_bytes(), dtype=torch.uint8, device=self.dev)
        self.loss = torch.zeros(1, **f32)
        B, T_in, T_out = cfg.B, cfg.T_in, cfg.T_out
        self.x = torch.empty(B * T_in * self.ld, **f32)
        self.y = torch.empty(B * T_out * self.ld, **f32)
        self.idx = torch.empty(max(1, p.win_hi - p.win_lo), dtype=torch.int32, device=self.dev)
        self.idx_cur = torch.empty(B, dtype=torch.int32, device=self.dev)
        self.dev_step = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.n_used = 0
        self.use_cuda_graph = use_cuda_graph
        self.graph = None

    # ------------------------------------------------------------------ setup
    def _stats(self):
        """Alg. 1's mu, sigma over the training windows: both passes, the cross-rank
        sum of the halo shards' partial sums and the finalisation run inside libpgti
        (pgti_series_moments); the replicated placement holds every row and sums locally."""
        p = self.plan
        sums = self.torch.zeros(3, dtype=self.torch.float64, device=self.dev)
        comm = self.comm if self.placement == "halo" else None
        return self.series.moments(self.S_tr, self.cfg.T_in, p.stat_lo, p.stat_hi, sums, comm)

    def steps_per_epoch(self) -> int:
        return self.S_r // self.cfg.B

    def start_epoch(self, epoch: int) -> int:
        p, cfg = self.plan, self.cfg
        code = {False: 0, True: 1, "batch": 2}[self.shuffle]
        if self.placement == "halo":
            self.n_used = self.series.make_index(p.win_lo, p.win_hi, cfg.T_in, cfg.T_out, cfg.B,
                                                 self.seed, epoch, self.rank, code, self.idx)
            return self.n_used // cfg.B
        # one global plan, identical on every rank (Philox rank word 0); this rank's slice
        self.series.make_index(0, self.S_tr, cfg.T_in, cfg.T_out, cfg.B, self.seed, epoch, 0,
                               code, self.idx)
        self.idx_off = self.rank * self.S_r
        self.n_used = (self.S_r // cfg.B) * cfg.B
        return self.n_used // cfg.B

    def epoch_plan(self):
        """This rank's window starts of the current epoch, in visiting order (device int32)."""
        return self.idx[self.idx_off:self.idx_off + self.n_used]

    def validate(self) -> float:
        """Validation MAE (normalised units) over the validation windows [S_tr, S_tr + S_val),
        split evenly over the ranks (whole batches), forward + loss only (pgti_dcrnn_loss),
        per-rank sums all-reduced.  Needs the replicated placement (every rank holds the
        validation rows)."""
        assert self.placement == "replicated", "validation rows are held by the replicated placement"
        torch, cfg = self.torch, self.cfg
        B = cfg.B
        V_r = val_windows(self.S) // self.world
        nb = V_r // B
        lo = self.S_tr + self.rank * V_r
        vidx = torch.empty(max(1, V_r), dtype=torch.int32, device=self.dev)
        losses = torch.zeros(max(1, nb), dtype=torch.float32, device=self.dev)
        if nb:
            self.series.make_index(lo, lo + V_r, cfg.T_in, cfg.T_out, B, self.seed, 0, 0, 0, vidx)
        for j in range(nb):
            self.series.gather(vidx[j * B:(j + 1) * B], B, cfg.T_in, cfg.T_out, self.x, self.y)
            self.model.loss(self.params, self.x, self.y, losses[j:j + 1], self.ws)
        scratch = torch.zeros(2, dtype=torch.float64, device=self.dev)
        return pgti.mean_losses(losses, nb, scratch,
                                self.comm)

    # ------------------------------------------------------------------ one step
    def _body(self, idx):
        cfg = self.cfg
        if self.ss_k:
            k = float(self.ss_k)
            p = k / (k + math.exp(min(self.steps_done / k, 700.0)))
            coins = self.ss_rng.uniform(size=max(cfg.T_out - 1, 0)) < p
            self.model.set_teacher_forcing(sum(1 << i for i, c in enumerate(coins) if c))
            self.steps_done += 1
        if self.zero_copy:
            self.model.step_indexed(self.params, self.grads, self.series, idx, self.loss, self.ws)
        else:
            self.series.gather(idx, cfg.B, cfg.T_in, cfg.T_out, self.x, self.y)
            self.model.step(self.params, self.grads, self.x, self.y, self.loss, self.ws)
        if self.comm is not None:   # a 1-rank communicator (world 1) runs the same identity SUM
            self.comm.allreduce_grads(self.grads)
        pgti.adam_step(self.params, self.grads, self.m, self.v, 0, self.lr,
                       grad_scale=1.0 / self.world, dev_step=self.dev_step)

    def step(self, j: int):
        """Batch j of the current epoch (gather -> fwd/bwd -> all-reduce -> Adam)."""
        B = self.cfg.B
        sl = self.idx[self.idx_off + j * B:self.idx_off + (j + 1) * B]
        if not self.use_cuda_graph:
            self._body(sl)
            return
        self.idx_cur.copy_(sl)
        self._replay()

    def step_from_host(self, idx_host):
        """End-to-end form: this step's B window starts come from (pinned) host memory."""
        self.idx_cur.copy_(idx_host, non_blocking=True)
        if not self.use_cuda_graph:
            self._body(self.idx_cur)
            return
        self._replay()

    def _replay(self):
        if self.graph is None:
            torch = self.torch
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):      # warm-up outside capture (loads every kernel)
                snap = [t.clone() for t in (self.params, self.m, self.v, self.dev_step)]
                self._body(self.idx_cur)
                for t, c in zip((self.params, self.m, self.v, self.dev_step), snap):
                    t.copy_(c)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._body(self.idx_cur)
            self.graph = g
        self.graph.replay()

    def check(self):
        pgti.check_device_error()
