"""Real multi-GPU check of distributed-index-batching (launched by torchrun, one rank per GPU):
each rank loads only its halo shard, computes the gradient of its first batch with libpgti, the
ranks SUM the gradients with pgti_allreduce_grads (NCCL), and rank 0 compares the mean with the
oracle gradient of the union batch.  Also checks the all-reduced statistics.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
        tests/dist_step_check.py [precision]
Exit code 0 = pass.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402


def main():
    precision = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2507_11683_b200 import pgti
    from paper_2507_11683_b200.trainer import Trainer, shard_plan, train_windows, window_count

    cfg = synth.CONFIGS["metr_la"].replace(B=8)
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(pgti.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = pgti.Comm(bytes(uid.cpu().numpy().tolist()), rank, world, local)
    graph = synth.make_graph(cfg.N, cfg.knn)
    theta = synth.make_params(cfg, kind="random")
    p = shard_plan(train_windows(window_count(cfg.E, cfg.T_in, cfg.T_out)), world, rank,
                   cfg.T_in, cfg.T_out)
    rows = synth.make_series(cfg, row_lo=p.row_lo, row_hi=p.row_hi)
    tr = Trainer(cfg, graph, lambda a, b: rows, theta, rank, world, local, comm,
                 precision=precision, use_cuda_graph=False)
    tr.start_epoch(0)
    idx = tr.idx[:cfg.B].clone()
    tr.series.gather(idx, cfg.B, cfg.T_in, cfg.T_out, tr.x, tr.y)
    tr.model.step(tr.params, tr.grads, tr.x, tr.y, tr.loss, tr.ws)
    comm.allreduce_grads(tr.grads)
    pgti.check_device_error()
    g_mean = (tr.grads.double() / world).cpu().numpy()
    all_idx = [torch.zeros(cfg.B, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(all_idx, idx)
    stats = torch.tensor([tr.mu, tr.sigma], dtype=torch.float64, device=dev)
    ok = torch.ones(1, device=dev)
    if rank == 0:
        from oracle import pipeline
        ref = pipeline.Reference(cfg, materialize_all=False)
        union = np.concatenate([a.cpu().numpy() for a in all_idx]).astype(np.int64)
        _, g_ref, _ = ref.loss_and_grad(theta, union)
        err = np.max(np.abs(g_mean - g_ref)) / np.max(np.abs(g_ref))
        tol = 1e-5 if precision == 0 else 2e-2
        e_mu = abs(tr.mu - ref.mu) / abs(ref.mu)
        e_sd = abs(tr.sigma - ref.sigma) / ref.sigma
        print(f"world={world} precision={precision} grad rel err {err:.3e} (tol {tol}); "
              f"mu rel {e_mu:.1e} sigma rel {e_sd:.1e}", flush=True)
        if not (err <= tol and e_mu <= 1e-12 and e_sd <= 1e-12):
            ok.zero_()
    # the bench's captured step (gather -> fwd/bwd -> NCCL all-reduce -> Adam, per-layer and aux
    # streams, PDL) against eager launches on every rank: parameters after 3 steps bitwise equal
    params = []
    for use_graph in (False, True):
        t2 = Trainer(cfg, graph, lambda a, b: rows, theta, rank, world, local, comm,
                     precision=precision, use_cuda_graph=use_graph)
        t2.start_epoch(0)
        for j in range(3):
            t2.step(j)
        t2.check()
        params.append(t2.params.cpu().numpy().view(np.uint32))
        t2.graph = None
        del t2
    torch.cuda.synchronize()
    same = np.array_equal(params[0], params[1])
    print(f"rank {rank}: captured step == eager after 3 steps: {same}", flush=True)
    if not same:
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    dist.broadcast(ok, 0)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
