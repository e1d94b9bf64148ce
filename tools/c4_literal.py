"""Config C4 as literally specified (N = 2^20, dt = 0.01, monodisperse) on the
GPU, with the TT-cross kernel rebuilt from the stored skeleton: per-step
moment rows and the failure step, to compare with the reference's own run
(tests/golden/c4traj.npz)."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1905_09071_b200 as g  # noqa: E402
from paper_1905_09071_b200 import construct  # noqa: E402
from paper_1905_09071_b200.workloads import initial_state  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
c = np.load(os.path.join(ROOT, "tests", "golden", "c4traj.npz"))
N = 1 << 20
cores3 = construct.c4_d3_from_skeleton(N, [c["I0"], c["I1"], c["I2"]], [None, c["J1"], c["J2"], c["J3"]])
ks = g.KernelSet({2: g.TTKernel(construct.c4_d2_cores(N)), 3: g.TTKernel(cores3)})
print("reference: fail_step", int(c["lit_fail_step"]), "warned", bool(c["lit_warned"]), "rows", c["lit_rows"].tolist())


class Cfg:
    def __init__(self, n0, dt, steps, record_every):
        self.n_classes = n0.size
        self.initial = g.InitialCondition.from_vector(n0)
        self.time = g.TimeGrid(0.0, dt, steps)
        self.record_every = record_every


for rec in (10, 1):
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        try:
            final, series = g.integrate(Cfg(initial_state("mono", N), 0.01, 100, rec), kernels=ks)
            print("gpu: no failure; rows", np.array(series.rows()).tolist()[:3])
        except g.StepFailureError as e:
            rows = np.array(e.series.rows())
            print(f"gpu (record_every={rec}): fail_step {e.step_index}, warned {any('Step' in type(x.message).__name__ for x in w)}")
            for r in rows:
                print("   ", " ".join(f"{x:.6e}" for x in r))
