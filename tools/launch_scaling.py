"""Step-kernel time vs shots per launch (C3 grid): separates the fixed
per-launch cost from the per-shot cost.  python tools/launch_scaling.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
    case = synthetic.layered_case(cfgname)
    prop = Propagator(case["grid"], case["geometry"], case["wavelet"], case["config"],
                      dtype="float32", recon="full", use_graphs=False)
    prop.set_model(case["init"].m)
    for cnt in (1, 2, 4, 8, 15, 30):
        f = prop.time_step_kernel(0, cnt, 40)
        b = prop.time_step_kernel(1, cnt, 40)
        fp = prop.time_step_kernel(2, cnt, 40)
        print(f"shots {cnt:3d}: forward(hist) {f*1e3:6.1f} us  adjoint {b*1e3:6.1f} us  "
              f"forward(plain) {fp*1e3:6.1f} us", flush=True)


if __name__ == "__main__":
    main()
