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
    "dedup_identical_columns",
    "use_devices",
]


def use_devices(devices=None):
    """Evaluate rhs_total / rhs_*_P/Q / integrate on several GPUs of this
    process (a device group: rank-sharded kernels, one NCCL all-reduce per
    RHS, ttagg_group_*).  ``None`` or ``[]`` returns to one device.  The
    environment variable TTAGG_DEVICES="0,1,..." selects a group at first use,
    so the reference's own CLI scales after install() without code changes.
    Returns the group (or None)."""
    from . import _lib

    return _lib.set_group(list(devices) if devices else None)


def dedup_identical_columns(enabled: bool = True) -> bool:
    """Opt-in storage mode for CP kernels (no reference counterpart): identical
    factor columns are uploaded and transformed once (ttagg_cp_upload_dedup).
    Results are unchanged; kernels built from a few distinct vectors (the
    permutation-power / Brownian families) get much cheaper column
    transforms.  Off by default, so a rank-R kernel is evaluated as the R
    rank terms it is specified as.  Applies to kernels uploaded after the
    call; returns the previous setting."""
    from . import _lib

    prev = _lib.DEDUP
    _lib.DEDUP = bool(enabled)
    return prev


def install(ttagg_module=None):
    """Route an imported reference package through the GPU operators.

    Patches the reference's own call-time lookups:

    * ``ttagg.rhs.rhs_{cp,tt,dense}_{P,Q}`` (used by its ``rhs_total``,
      rhs.py:446-451);
    * ``ttagg.integrator.rhs_total`` (used by its ``rk2_step``,
      integrator.py:16, 171);
    * ``ttagg.integrator.integrate`` / ``ttagg.integrate`` and the name the
      CLI bound at import, ``ttagg.cli.integrate`` (cli.py:21, 102): the
      fused device RK2 (state resident, one CUDA graph per step).  Its
      ``run_scaling_benchmark`` imports ``integrate`` lazily from the
      integrator module (parallel.py:221-222) and picks the patch up too.
      Results come back as the reference's own types (ConcentrationState,
      MomentSeries, StepFailureError, StepSizeWarning), so the CLI's exit
      codes and CSV writers work unchanged.

    Returns a function that undoes the patch.
    """
    import importlib
    import warnings as _warnings

    from . import integrator as _integ
    from . import rhs as _rhs

    mod = ttagg_module or importlib.import_module("ttagg")
    rhs_mod = importlib.import_module(mod.__name__ + ".rhs")
    integ_mod = importlib.import_module(mod.__name__ + ".integrator")
    try:
        cli_mod = importlib.import_module(mod.__name__ + ".cli")
    except ImportError:
        cli_mod = None
    ops = ("rhs_cp_P", "rhs_cp_Q", "rhs_tt_P", "rhs_tt_Q", "rhs_dense_P", "rhs_dense_Q")
    saved = {(rhs_mod, name): getattr(rhs_mod, name) for name in ops}
    saved[(integ_mod, "rhs_total")] = integ_mod.rhs_total
    saved[(integ_mod, "integrate")] = integ_mod.integrate
    if hasattr(mod, "integrate"):
        saved[(mod, "integrate")] = mod.integrate
    if cli_mod is not None and hasattr(cli_mod, "integrate"):
        saved[(cli_mod, "integrate")] = cli_mod.integrate
    for name in ops:
        setattr(rhs_mod, name, getattr(_rhs, name))

    ref_total = rhs_mod.rhs_total
    ref_result = rhs_mod.RhsResult
    ref_state = rhs_mod.ConcentrationState

    def gpu_total(kernels, state, plan=None, *, breakdown=False):
        ks = [kernels[d] for d in kernels.orders]
        if all(hasattr(k, "factors") or hasattr(k, "cores") or hasattr(k, "values") for k in ks):
            r = _rhs.rhs_total(kernels, state, plan, breakdown=breakdown)
            return ref_result(p=r.p, q=r.q, s=r.s, by_order=r.by_order)
        return ref_total(kernels, state, plan, breakdown=breakdown)

    def to_ref_series(series):
        if series is None:
            return None
        out = integ_mod.MomentSeries()
        for name in ("times", "m0", "m1", "m2", "min_n", "m1_drift"):
            setattr(out, name, list(getattr(series, name)))
        out.negativity_flagged = series.negativity_flagged
        return out

    def gpu_integrate(config, kernels=None, plan=None, on_record=None):
        cb = None
        if on_record is not None:
            def cb(step, state):
                on_record(step, ref_state(state.n, state.t))
        with _warnings.catch_warnings(record=True) as caught:
            _warnings.simplefilter("always")
            try:
                final, series = _integ.integrate(config, kernels, plan, cb)
            except _integ.StepFailureError as exc:
                err = integ_mod.StepFailureError(str(exc), step_index=exc.step_index,
                                                 series=to_ref_series(exc.series))
                failure = err
            else:
                failure = None
        for w in caught:  # re-issued as the reference's own warning classes
            cat = integ_mod.StepSizeWarning if issubclass(w.category, _integ.StepSizeWarning) else w.category
            _warnings.warn(str(w.message), cat, stacklevel=2)
        if failure is not None:
            raise failure
        return ref_state(final.n, final.t), to_ref_series(series)

    integ_mod.rhs_total = gpu_total
    integ_mod.integrate = gpu_integrate
    if (mod, "integrate") in saved:
        mod.integrate = gpu_integrate
    if (cli_mod, "integrate") in saved:
        cli_mod.integrate = gpu_integrate

    def uninstall():
        for (m, name), fn in saved.items():
            setattr(m, name, fn)

    return uninstall
