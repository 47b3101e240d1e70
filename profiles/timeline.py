"""Per-launch timeline of one eager training step (CUDA events around every libpgti launch,
pgti_profile_timeline): how long each stream is busy, how much of the step runs 0 / 1 / 2+
kernels at once, and the share of each kernel class.  Event brackets add a little time per
launch, so absolute times are upper bounds; the structure is what this is for.

    python profiles/timeline.py [--config metr_la] [--precision 1] [--json out.json]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="metr_la")
    ap.add_argument("--precision", type=int, default=1)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch

    import synth
    from paper_2507_11683_b200 import pgti
    from paper_2507_11683_b200.trainer import Trainer, shard_plan, train_windows, window_count
    cfg = synth.CONFIGS[args.config]
    p = shard_plan(train_windows(window_count(cfg.E, cfg.T_in, cfg.T_out)), 1, 0, cfg.T_in,
                   cfg.T_out)
    rows = synth.make_series(cfg, row_lo=p.row_lo, row_hi=p.row_hi)
    tr = Trainer(cfg, synth.make_graph(cfg.N, cfg.knn), lambda a, b: rows,
                 synth.make_params(cfg, kind="train"), precision=args.precision,
                 use_cuda_graph=False)
    tr.start_epoch(0)
    for j in range(3):
        tr.step(j)
    torch.cuda.synchronize()
    pgti.profile_read()
    pgti.profile_enable(True)
    tr.step(3)
    torch.cuda.synchronize()
    tl = pgti.profile_timeline()
    pgti.profile_read()
    pgti.profile_enable(False)

    t0 = min(a for _, a, _, _ in tl)
    t1 = max(b for _, _, b, _ in tl)
    span = t1 - t0
    streams = collections.defaultdict(float)
    cls_ms = collections.defaultdict(float)
    for c, a, b, s in tl:
        streams[s] += b - a
        cls_ms[c] += b - a
    # concurrency profile over the step
    edges = sorted([(a, 1) for _, a, _, _ in tl] + [(b, -1) for _, _, b, _ in tl])
    conc = collections.defaultdict(float)
    level, last = 0, t0
    for t, d in edges:
        conc[level] += t - last
        level += d
        last = t
    out = {"config": cfg.name, "precision": args.precision, "launches": len(tl),
           "step_ms": span,
           "stream_busy_ms": {f"stream{i}": v for i, v in enumerate(sorted(streams.values(),
                                                                            reverse=True))},
           "concurrency_ms": {f"{k}": v for k, v in sorted(conc.items())},
           "class_ms": dict(sorted(cls_ms.items(), key=lambda kv: -kv[1]))}
    print(json.dumps(out, indent=1))
    if args.json:
        json.dump({"summary": out, "launches": tl}, open(args.json, "w"))


if __name__ == "__main__":
    main()
