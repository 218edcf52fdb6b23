"""Small invocations of every kernel family, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

cases = [
    (wl.kepler_ensemble(batch=300, nsteps=40), {}),                              # g8 (auto)
    (wl.kepler_ensemble(batch=300, nsteps=40), {"mapping": 1}),                  # g1q
    (wl.kepler_ensemble(batch=9000, nsteps=16), {"balance": 4, "mapping": 1}),   # g1q, many units
    (wl.kepler_ensemble(batch=9000, nsteps=16), {"balance": 4, "schedule": 1, "mapping": 1}),  # chunked
    (wl.kepler_ensemble(batch=70, nsteps=20), {"mode": irk.FIRST_ORDER}),       # fo8
    (wl.kepler_ensemble(batch=70, nsteps=20), {"mode": irk.FIRST_ORDER, "mapping": 1}),  # fo_q
    (wl.henon_heiles(batch=33, nsteps=30), {}),
    (wl.schwarzschild(batch=20, nsteps=30), {}),
    (wl.six_body_ensemble(batch=23, nsteps=30), {}),                            # nbody8 (auto)
    (wl.six_body_ensemble(batch=23, nsteps=30), {"mapping": 1, "balance": 7}),  # nbody_q
    (wl.fpu_ensemble(batch=5, nsteps=30), {}),
    (wl.plummer(N=512, nsteps=3), {}),
    (wl.plummer(N=512, nsteps=3), {"vshards": 4, "device_loop": 0}),
]
for w, kw in cases:
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=5, **kw) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it)
        ig.energy(Y)
        torch.cuda.synchronize()
        print(w.name, kw, ig.stats(ws)[0], flush=True)
print("done")
