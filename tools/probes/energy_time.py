"""Time one config-5 energy sample (irk_energy, N = 8,192) and print its bits."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2511_03655_b200 import irk, workloads as wl
w = wl.plummer()
with irk.Integrator(w.problem, w.dim, w.h, 1, 1, w.params) as ig:
    y = torch.tensor(w.y, dtype=torch.float64, device='cuda')
    for _ in range(2): ig.energy(y)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): out = ig.energy(y)
    e1.record(); torch.cuda.synchronize()
    print('energy N=8192 ms per call', e0.elapsed_time(e1) / 10, out.item().hex())
