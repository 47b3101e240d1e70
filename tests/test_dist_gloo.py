"""world_size-2 CPU (gloo) coverage of the N>1 host logic of distributed-index-batching:
shard plans, the statistics row partition (every rank sums only rows it holds) and the
gradient mean (ranks all-reduce their gradients)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

CFG = synth.Config("gloo", N=10, E=70, F=2, T_in=4, T_out=3, L=2, H=16, K=2, B=3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import philox, pipeline, windows
        from paper_2507_11683_b200 import trainer
        ref = pipeline.Reference(CFG)
        S_tr = ref.n_train
        p = trainer.shard_plan(S_tr, world, rank, CFG.T_in, CFG.T_out)
        assert (p.win_lo, p.win_hi - p.win_lo) == philox.shard(S_tr, world, rank)
        # only the rows this rank holds
        held = ref.v[p.row_lo:p.row_hi].astype(np.float64).reshape(p.row_hi - p.row_lo, -1)
        t = np.arange(p.stat_lo, p.stat_hi)
        w = np.clip(np.minimum(t, S_tr - 1) - np.maximum(0, t - CFG.T_in + 1) + 1, 0, None)
        rows = held[t - p.row_lo]
        part = torch.tensor([w.sum() * rows.shape[1], (w[:, None] * rows).sum(),
                             (w[:, None] * rows ** 2).sum()], dtype=torch.float64)
        dist.all_reduce(part)
        mu = part[1].item() / part[0].item()
        sigma = np.sqrt(part[2].item() / part[0].item() - mu * mu)
        assert abs(mu - ref.mu) <= 1e-12 * abs(ref.mu)
        assert abs(sigma - ref.sigma) <= 1e-10 * ref.sigma
        # gradient of this rank's first batch, all-reduced (SUM) then / R == union batch
        theta = synth.make_params(CFG, kind="random")
        idx = ref.plan(world, rank)[:CFG.B]
        assert idx.min() >= p.win_lo and idx.max() < p.win_hi
        assert idx.max() + CFG.T_in + CFG.T_out <= p.row_hi
        _, g, _ = ref.loss_and_grad(theta, idx)
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)
        all_idx = [torch.zeros(CFG.B, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_idx, torch.from_numpy(idx))
        if rank == 0:
            union = np.concatenate([a.numpy() for a in all_idx])
            _, g_union, _ = ref.loss_and_grad(theta, union)
            err = np.max(np.abs(gt.numpy() / world - g_union)) / np.max(np.abs(g_union))
            assert err < 1e-12, err
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.slow
def test_two_rank_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
