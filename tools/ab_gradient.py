"""Interleaved A/B timing of full FWI gradients between handle variants that
differ in an environment knob read at sg_create (e.g. SG_L2_PERSIST), so
clock / power-cap drift hits both arms alike.

    python tools/ab_gradient.py --env SG_L2_PERSIST=1 [--config c3] [--reps 6]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", action="append", default=[], help="KEY=VALUE for arm B")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--misfit", action="store_true", help="time misfit (forward) too")
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case(a.config)
    args = (case["grid"], case["geometry"], case["wavelet"], case["config"])
    ref = Propagator(*args, dtype="float32", recon="full")
    ref.set_model(case["true"].m)
    obs = ref.synthetic().clone()
    ref.close()
    times = {"A": [], "B": []}
    vals = {}

    def make(envs):
        saved = {}
        for kv in envs:
            k, v = kv.split("=", 1)
            saved[k] = os.environ.get(k)
            os.environ[k] = v
        p = Propagator(*args, dtype="float32", recon="full")
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
        p.set_model(case["init"].m)
        p.gradient(obs)
        return p

    # blocks A B B A A B ... (one handle alive at a time: each holds the full
    # C3 history), `per` timed gradients per block
    per = 2
    order = ["A", "B", "B", "A"] * max(1, a.reps // (2 * per))
    for name in order:
        p = make([] if name == "A" else a.env)
        for _ in range(per):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            v, g = p.gradient(obs)
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1))
        vals[name] = (v, g.clone())
        p.close()
        del p
        torch.cuda.empty_cache()
    for name in ("A", "B"):
        t = sorted(times[name])
        print(f"arm {name} {'(' + ' '.join(a.env) + ')' if name == 'B' else '(default)'}: "
              f"min {t[0]:.2f} ms median {t[len(t) // 2]:.2f} ms all {[round(x, 2) for x in times[name]]}")
    ga, gb = vals["A"][1], vals["B"][1]
    print("value equal", vals["A"][0] == vals["B"][0], "gradient bitwise", torch.equal(ga, gb))


if __name__ == "__main__":
    main()
