"""Probe: does splitting one step's batch into independent micro-batches on separate streams
raise throughput on a latency-bound workload?  Times (CUDA graphs, device events):
  a) one B-row step;  b) S micro-steps of B/S rows each on S streams concurrently;
  c) one B/S-row step alone.
    python profiles/split_probe.py [--config metr_la] [--splits 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="metr_la")
    ap.add_argument("--splits", type=int, default=2)
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    from paper_2507_11683_b200 import pgti
    cfg = synth.CONFIGS[args.config]
    ld = (cfg.N * cfg.F + 3) // 4 * 4
    csr = pgti.csr_to_device(pgti.add_windows(pgti.graph_build(cfg.N, *synth.make_graph(
        cfg.N, cfg.knn)), cfg.N), "cuda")
    theta = torch.from_numpy(synth.make_params(cfg, kind="train")).cuda()

    def make(B):
        m = pgti.DCRNN(cfg.N, cfg.F, cfg.F_out, cfg.L, cfg.H, cfg.K, cfg.T_in, cfg.T_out, B, ld,
                       csr, 1)
        g = torch.empty(m.num_params(), device="cuda")
        x = torch.randn(B * cfg.T_in * ld, device="cuda")
        y = torch.randn(B * cfg.T_out * ld, device="cuda")
        loss = torch.zeros(1, device="cuda")
        ws = torch.empty(m.workspace_bytes(), dtype=torch.uint8, device="cuda")
        return lambda s: m.step(theta, g, x, y, loss, ws, stream=s.cuda_stream)

    def timeit(fns):
        streams = [torch.cuda.Stream() for _ in fns]
        main_s = torch.cuda.Stream()
        for _ in range(3):  # warm-up outside capture
            for f, s in zip(fns, streams):
                f(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=main_s):
            for s in streams:
                s.wait_stream(main_s)
            for f, s in zip(fns, streams):
                f(s)
            for s in streams:
                main_s.wait_stream(s)
        for _ in range(5):
            graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            graph.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.iters

    B, S = cfg.B, args.splits
    full = timeit([make(B)])
    split = timeit([make(B // S) for _ in range(S)])
    one = timeit([make(B // S)])
    print(f"{cfg.name}: B={B} step {full:.3f} ms ({B / full * 1e3:.0f} samples/s); "
          f"{S} x B={B // S} concurrent {split:.3f} ms ({B / split * 1e3:.0f} samples/s); "
          f"one B={B // S} {one:.3f} ms")
    np.random.seed(0)


if __name__ == "__main__":
    main()
