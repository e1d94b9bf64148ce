"""Relative errors of the fused GPU RK2 against the reference's full-size
trajectory goldens (tests/golden/c5traj.npz, c3traj.npz)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1905_09071_b200 as g  # noqa: E402
from paper_1905_09071_b200.workloads import CONFIGS, initial_state  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class Cfg:
    def __init__(self, n0, dt, steps, record_every):
        self.n_classes = n0.size
        self.initial = g.InitialCondition.from_vector(n0)
        self.time = g.TimeGrid(0.0, dt, steps)
        self.record_every = record_every


for name, kind, rec in (("C5", "c5", 10), ("C3", "exp256", 20)):
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}traj.npz")
    if not os.path.exists(path):
        continue
    c = np.load(path)
    cfg = CONFIGS[name]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    final, series = g.integrate(Cfg(initial_state(kind, cfg.n_classes, normalised=True), cfg.dt, cfg.steps, rec),
                                kernels=ks)
    v = final.n
    k = np.arange(1, v.size + 1, dtype=np.float64)
    sums = np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])
    e_n = np.abs(v[c["idx"]] - c["n_final"]).max() / np.abs(c["n_final"]).max()
    e_s = (np.abs(sums - c["n_sums"]) / np.abs(c["n_sums"])).max()
    rows = np.array(series.rows())
    e_r = (np.abs(rows[:, 1:4] - c["rows"][:, 1:4]) / np.abs(c["rows"][:, 1:4])).max()
    print(f"{name} N={cfg.n_classes} steps={cfg.steps}: final-state rel max-norm {e_n:.2e}, "
          f"checksums {e_s:.2e}, moment rows {e_r:.2e}")
