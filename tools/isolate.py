"""Run one (dtype, order, direction) combination of the step kernel in a
fresh process so a device fault is attributed to exactly one kernel."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from cases import small_case
from paper_2008_11778_b200 import wavesim
dtype, order, top, graphs, what = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1", sys.argv[4] == "1", sys.argv[5]
case = small_case(order, top)
g = case["gold"]
p = wavesim.Propagator(case["grid"], case["geometry"], case["wavelet"], case["config"], dtype=dtype, use_graphs=graphs)
p.set_model(g["m"])
if what == "fwd":
    out = p.synthetic(); torch.cuda.synchronize()
    err = np.linalg.norm(out.double().cpu().numpy() - g["syn"]) / np.linalg.norm(g["syn"])
else:
    v, gr = p.gradient(g["obs"]); torch.cuda.synchronize()
    err = np.linalg.norm(gr.double().cpu().numpy() - g["grad"]) / np.linalg.norm(g["grad"])
print("OK", err)
'''.replace("ROOT", repr(ROOT))

for dtype in ("float64", "float32"):
    for order in (2, 8):
        for what in ("fwd", "grad"):
            r = subprocess.run([sys.executable, "-c", CHILD, dtype, str(order), "1", "0", what],
                               capture_output=True, text=True, timeout=300,
                               env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
            tail = (r.stdout.strip().splitlines() or [""])[-1]
            err = [l for l in r.stderr.splitlines() if "rror" in l][-1:]
            print(dtype, order, what, "rc", r.returncode, tail, err, flush=True)
