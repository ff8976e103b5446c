import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2008_11778_b200 import synthetic, gradients
case = synthetic.layered_case("c3")
geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
from paper_2008_11778_b200.wavesim import Propagator
tmp = Propagator(grid, geom, wav, cfg, dtype="float32"); tmp.set_model(case["true"].m)
obs = tmp.synthetic(); tmp.close()
obj = gradients.FwiObjective(grid, obs, wav, geom, cfg, dtype="float32")
p_host = np.ascontiguousarray(case["init"].m.ravel())
p_dev = torch.as_tensor(p_host, device="cuda", dtype=torch.float32)
for _ in range(3): obj.value_and_grad(p_dev)
torch.cuda.synchronize()
for label, p in (("dev", p_dev), ("host", p_host), ("dev", p_dev), ("host", p_host)):
    t0 = time.perf_counter()
    for _ in range(5): obj.value_and_grad(p)
    torch.cuda.synchronize()
    print(label, (time.perf_counter() - t0) / 5 * 1e3, "ms")
# pieces
t0 = time.perf_counter()
for _ in range(20): obj.prop.set_model(p_host)
torch.cuda.synchronize(); print("set_model host", (time.perf_counter()-t0)/20*1e3)
t0 = time.perf_counter()
for _ in range(20): obj.prop.set_model(p_dev)
torch.cuda.synchronize(); print("set_model dev", (time.perf_counter()-t0)/20*1e3)
g = torch.empty((grid.nz, grid.nx), device="cuda")
t0 = time.perf_counter()
for _ in range(20): x = g.double().cpu().numpy()
print("grad d2h", (time.perf_counter()-t0)/20*1e3)
