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

path = os.path.join(ROOT, "tests", "golden", "c4traj.npz")
if os.path.exists(path):
    from paper_1905_09071_b200 import construct

    c = np.load(path)
    N = 1 << 20
    cores3 = construct.c4_d3_from_skeleton(N, [c["I0"], c["I1"], c["I2"]], [None, c["J1"], c["J2"], c["J3"]])
    ks = g.KernelSet({2: g.TTKernel(construct.c4_d2_cores(N)), 3: g.TTKernel(cores3)})
    final, series = g.integrate(Cfg(initial_state("mono", N), 0.01, 2, 1), kernels=ks)
    v = final.n
    k = np.arange(1, v.size + 1, dtype=np.float64)
    sums = np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])
    e_n = np.abs(v[c["idx"]] - c["n2_final"]).max() / np.abs(c["n2_final"]).max()
    sel = [0, 1, 4]  # M2-weighted sums are roundoff-dominated here (see the test)
    e_s = (np.abs(sums[sel] - c["n2_sums"][sel]) / np.abs(c["n2_sums"][sel])).max()
    rows = np.array(series.rows())
    e_r = (np.abs(rows[:, 1:3] - c["n2_rows"][:, 1:3]) / np.abs(c["n2_rows"][:, 1:3])).max()
    print(f"C4 N={N} first 2 steps (TT ranks {[x.shape[2] for x in cores3]}; the literal 100-step run diverges "
          f"at step {int(c['lit_fail_step'])} in the reference): final-state rel max-norm {e_n:.2e}, "
          f"checksums (M0, M1, max) {e_s:.2e}, moment rows (M0, M1) {e_r:.2e}")
