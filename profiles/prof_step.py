"""Eager training steps of a workload's shape for ncu / compute-sanitizer (one GPU).

Kernel shapes depend on N, B, F, H, K, L, T_in, T_out -- not on the series length -- so the
series is cut to --rows rows (fast setup); every kernel the bench's step launches runs with the
bench's shapes, launched eagerly (no CUDA graph) so each launch is a separate ncu result.

    python profiles/prof_step.py --config pems --steps 2 [--rows 2000] [--precision 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="pems")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--rows", type=int, default=2000)
    ap.add_argument("--precision", type=int, default=1)
    ap.add_argument("--graph", action="store_true", help="replay a captured step instead")
    ap.add_argument("--tiny", action="store_true",
                    help="the tc_tiny shape (N 12, B 3, L 2, H 64, K 2): sanitizer runs")
    ap.add_argument("--B", type=int, default=0, help="override the per-GPU batch")
    a = ap.parse_args()
    import torch

    import synth
    from paper_2507_11683_b200.trainer import Trainer
    cfg = (synth.Config("tc_tiny", N=12, E=60, F=2, T_in=3, T_out=2, L=2, H=64, K=2, B=3)
           if a.tiny else synth.CONFIGS[a.config])
    if a.B:
        cfg = cfg.replace(B=a.B)
    cfg = cfg.replace(E=min(cfg.E, max(a.rows, 4 * cfg.B + cfg.T_in + cfg.T_out)))
    graph = synth.make_graph(cfg.N, cfg.knn)
    params = synth.make_params(cfg, kind="train")
    tr = Trainer(cfg, graph, lambda lo, hi: synth.make_series(cfg, row_lo=lo, row_hi=hi), params,
                 precision=a.precision, use_cuda_graph=a.graph)
    tr.start_epoch(0)
    for j in range(a.steps):
        tr.step(j)
    torch.cuda.synchronize()
    tr.check()
    print(f"{cfg.name}: {a.steps} steps ok, loss {float(tr.loss.item()):.6f}")


if __name__ == "__main__":
    main()
