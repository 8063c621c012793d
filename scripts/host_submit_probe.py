import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2104_06069_b200 import bitlamb as bl, layouts
sizes = layouts.CONFIG1
d = sum(sizes)
torch.cuda.set_device(0)
st = torch.cuda.Stream()
cl = bl.SimCluster(1, d, device=0, stream=st.cuda_stream)
opt = bl.Optimizer("onebit_lamb", [(f"l{i}", s) for i, s in enumerate(sizes)], bl.HyperParams(total_steps=1000, warmup_steps=2), cl)
g = torch.randn((1, d), device="cuda") * 1e-3
t = 0
for _ in range(5):
    opt.step(g, t, 1e-3); t += 1
cl.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(50):
        opt.step_resident(t, 1e-3); t += 1
    t1 = time.perf_counter()
    cl.synchronize()
    t2 = time.perf_counter()
    print("host submit us/step", (t1 - t0) / 50 * 1e6, "total us/step", (t2 - t0) / 50 * 1e6)
