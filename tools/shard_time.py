"""Single-rank share of a strong-scaling run, measured on one GPU: the time of
one FWI gradient over the first `count` shots of the config's survey -- what
rank 0 of an N-rank run owns (contiguous blocks, shards.shard_bounds) -- for
the shot counts of N = 1, 2, 4, 8.  No collective is involved (the all-reduce
of one gradient is microseconds, DESIGN s7), so t(count_N) bounds the N-GPU
gradient time from below and t(30) / (N t(count_N)) is the efficiency the
kernels allow.  This is NOT a multi-GPU measurement.

    python tools/shard_time.py [--config c3] [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nt", type=int, default=None)
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import shards, synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case(a.config, nt=a.nt)
    geom = case["geometry"]
    S = geom.n_sources
    prop = Propagator(case["grid"], geom, case["wavelet"], case["config"], dtype="float32")
    prop.set_model(case["true"].m)
    obs = prop.synthetic().clone()
    prop.set_model(case["init"].m)
    base = None
    for world in (1, 2, 4, 8):
        s0, cnt = shards.shard_bounds(S, world, 0)
        prop.gradient(obs[s0:s0 + cnt], shots=(s0, cnt))
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prop.gradient(obs[s0:s0 + cnt], shots=(s0, cnt))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        base = base or t
        print(f"N={world}: rank 0 owns {cnt} of {S} shots: {t:8.2f} ms per gradient; "
              f"speed-up bound {base / t:5.2f}x, efficiency bound {base / (world * t):5.2f}")
    prop.close()


if __name__ == "__main__":
    main()
