"""B200-native right-hand-side evaluator for the multi-particle Smoluchowski
equations (arXiv 1905.09071), a drop-in for the hot path of the reference
package ``ttagg`` v0.1.0: ``rhs_cp_P/Q``, ``rhs_tt_P/Q``, ``rhs_dense_P/Q``,
``rhs_total``, ``rk2_step`` and ``integrate``.

The arithmetic runs in hand-written sm_100a CUDA kernels (fp64) behind the
C-ABI in ``include/ttagg_b200.h``; this package is the Python mirror of the
reference's operator API on top of it.  ``install()`` swaps the GPU operators
into an imported reference package through its own module-level seams.
"""

__version__ = "0.1.0"

from .integrator import (
    InitialCondition,
    MomentSeries,
    StepFailureError,
    StepSizeWarning,
    TimeGrid,
    integrate,
    midpoint_step,
    moments,
    rk2_step,
)
from .kernels import CPKernel, DenseKernel, KernelError, TTKernel, constant_cp, constant_tt
from .parallel import SERIAL_PLAN, ExecutionPlan, lpt_rank_shards
from .rhs import (
    ConcentrationState,
    KernelSet,
    RhsResult,
    kernel_element,
    rhs_cp_P,
    rhs_cp_Q,
    rhs_dense_P,
    rhs_dense_Q,
    rhs_total,
    rhs_tt_P,
    rhs_tt_Q,
    sample_symmetry_violation,
)

__all__ = [
    "__version__",
    "CPKernel",
    "TTKernel",
    "DenseKernel",
    "KernelError",
    "constant_cp",
    "constant_tt",
    "ConcentrationState",
    "KernelSet",
    "RhsResult",
    "kernel_element",
    "sample_symmetry_violation",
    "rhs_cp_P",
    "rhs_cp_Q",
    "rhs_tt_P",
    "rhs_tt_Q",
    "rhs_dense_P",
    "rhs_dense_Q",
    "rhs_total",
    "TimeGrid",
    "InitialCondition",
    "MomentSeries",
    "StepFailureError",
    "StepSizeWarning",
    "midpoint_step",
    "rk2_step",
    "integrate",
    "moments",
    "ExecutionPlan",
    "SERIAL_PLAN",
    "lpt_rank_shards",
    "install",
]


def install(ttagg_module=None):
    """Route an imported reference package through the GPU operators.

    Patches the reference's own call-time lookups:
    ``ttagg.rhs.rhs_{cp,tt}_{P,Q}`` (used by its ``rhs_total``,
    rhs.py:446-451) and ``ttagg.integrator.rhs_total`` (used by its
    ``rk2_step``, integrator.py:16, 171), and the dense operators
    ``ttagg.rhs.rhs_dense_{P,Q}``.  Returns a function that undoes the patch.
    """
    import importlib

    from . import rhs as _rhs

    mod = ttagg_module or importlib.import_module("ttagg")
    rhs_mod = importlib.import_module(mod.__name__ + ".rhs")
    integ_mod = importlib.import_module(mod.__name__ + ".integrator")
    saved = {
        (rhs_mod, name): getattr(rhs_mod, name)
        for name in ("rhs_cp_P", "rhs_cp_Q", "rhs_tt_P", "rhs_tt_Q", "rhs_dense_P", "rhs_dense_Q")
    }
    saved[(integ_mod, "rhs_total")] = integ_mod.rhs_total
    for name in ("rhs_cp_P", "rhs_cp_Q", "rhs_tt_P", "rhs_tt_Q", "rhs_dense_P", "rhs_dense_Q"):
        setattr(rhs_mod, name, getattr(_rhs, name))

    ref_total = rhs_mod.rhs_total
    ref_result = rhs_mod.RhsResult

    def gpu_total(kernels, state, plan=None, *, breakdown=False):
        ks = [kernels[d] for d in kernels.orders]
        if all(hasattr(k, "factors") or hasattr(k, "cores") or hasattr(k, "values") for k in ks):
            r = _rhs.rhs_total(kernels, state, plan, breakdown=breakdown)
            return ref_result(p=r.p, q=r.q, s=r.s, by_order=r.by_order)
        return ref_total(kernels, state, plan, breakdown=breakdown)

    integ_mod.rhs_total = gpu_total

    def uninstall():
        for (m, name), fn in saved.items():
            setattr(m, name, fn)

    return uninstall
