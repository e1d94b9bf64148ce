"""Host-side mirror of the reference API: validation and error behaviour
(no GPU needed; these paths raise before any device call)."""

import warnings

import numpy as np
import pytest

import paper_1905_09071_b200 as g
import paper_1905_09071_b200.integrator as integrator_mod
from oracle import rhs_oracle as orc


def monodisperse(n_classes):
    n = np.zeros(n_classes)
    n[0] = 1.0
    return g.ConcentrationState(n)


def test_state_validation():  # rhs.py:54-79, test_rhs.py:400-408
    with pytest.raises(ValueError, match="non-finite"):
        g.ConcentrationState(np.array([1.0, np.inf]))
    with pytest.raises(ValueError, match="length"):
        g.ConcentrationState(np.array([1.0]))
    st = g.ConcentrationState(np.array([1.0, 2.0]), t=0.5)
    assert st.t == 0.5
    with pytest.raises(ValueError):
        st.n[0] = 3.0
    src = np.array([1.0, 2.0, 3.0])
    st = g.ConcentrationState(src)
    src[0] = 9.0
    assert st.n[0] == 1.0  # copied


def test_kernel_containers():  # kernels.py:137-215
    with pytest.raises(g.KernelError, match="two cores"):
        g.TTKernel((np.ones((1, 4, 1)),))
    with pytest.raises(g.KernelError, match="boundary"):
        g.TTKernel((np.ones((2, 4, 1)), np.ones((1, 4, 1))))
    with pytest.raises(g.KernelError, match="rank mismatch"):
        g.TTKernel((np.ones((1, 4, 2)), np.ones((3, 4, 1))))
    with pytest.raises(g.KernelError, match="same N x R"):
        g.CPKernel((np.ones((4, 2)), np.ones((4, 3))))
    k = g.TTKernel((np.ones((1, 5, 3)), np.ones((3, 5, 1))))
    assert k.ranks == (1, 3, 1) and k.dimension == 2 and k.n_classes == 5
    c = g.constant_cp(2.0, 3, 7)
    assert c.rank == 1 and c.dimension == 3 and c.factors[0][0, 0] == 2.0


def test_kernel_set_validation():  # test_rhs.py:373-389
    with pytest.raises(g.KernelError, match="order"):
        g.KernelSet({1: g.constant_tt(1.0, 2, 8)})
    with pytest.raises(g.KernelError, match="dimension"):
        g.KernelSet({3: g.constant_tt(1.0, 2, 8)})
    with pytest.raises(g.KernelError, match="same N"):
        g.KernelSet({2: g.constant_tt(1.0, 2, 8), 3: g.constant_tt(1.0, 3, 16)})
    with pytest.raises(g.KernelError, match="mode size"):
        g.KernelSet({}).n_classes
    assert g.KernelSet({3: g.constant_tt(1.0, 3, 8), 2: g.constant_tt(1.0, 2, 8)}).orders == (2, 3)
    rng = np.random.default_rng(79)
    lopsided = g.CPKernel(tuple(rng.random((12, 2)) for _ in range(3)))
    with pytest.raises(g.KernelError, match="not symmetric"):
        g.KernelSet({3: lopsided})
    assert g.sample_symmetry_violation(lopsided) > 1e-3


def test_rhs_total_errors_before_any_device_work():  # rhs.py:434-439
    with pytest.raises(g.KernelError, match="no collision orders"):
        g.rhs_total(g.KernelSet({}), monodisperse(8))
    with pytest.raises(g.KernelError, match="N"):
        g.rhs_total(g.KernelSet({2: g.constant_tt(1.0, 2, 8)}), monodisperse(9))
    with pytest.raises(g.KernelError, match="N"):
        g.rhs_cp_P(g.constant_cp(1.0, 2, 8), monodisperse(9))
    with pytest.raises(g.KernelError, match="TT"):
        g.rhs_tt_P(g.constant_cp(1.0, 2, 8), monodisperse(8))


def test_execution_plan():  # parallel.py:310-359
    with pytest.raises(g.KernelError):
        g.ExecutionPlan(workers=0)
    with pytest.raises(g.KernelError):
        g.ExecutionPlan(fft_length_policy="fast")
    assert g.ExecutionPlan().fft_length(3, 4096) == 16384
    assert g.ExecutionPlan(fft_length_policy="min").fft_length(3, 4096) == 12289


def test_midpoint_step_linear_decay():  # test_integrator.py:42-46
    n0 = np.array([2.0, 0.5, 1.25])
    dt = 0.1
    stepped = g.midpoint_step(n0, 0.0, dt, lambda n, t: -n)
    np.testing.assert_allclose(stepped, (1.0 - dt + dt**2 / 2.0) * n0, rtol=1e-15)


def test_rk2_step_seam_calls_rhs_exactly_twice(monkeypatch):
    """integrator.py:16, 171 plugin seam (test_integrator.py:57-69) — driven
    here by the CPU oracle so no device is needed."""
    calls = []

    def oracle_total(kernels, state, plan=None, *, breakdown=False):
        calls.append(1)
        ks = {d: {"kind": "tt", "arrays": kernels[d].cores} for d in kernels.orders}
        p, q, s = orc.rhs_total(ks, state.n)
        return g.RhsResult(p=p, q=q, s=s)

    monkeypatch.setattr(integrator_mod, "rhs_total", oracle_total)
    kernels = g.KernelSet({2: g.constant_tt(1.0, 2, 8)})
    st = g.rk2_step(g.ConcentrationState(np.full(8, 0.1), t=1.0), 1e-3, kernels)
    assert len(calls) == 2
    assert st.t == 1.0 + 1e-3
    with pytest.raises(ValueError, match="dt"):
        g.rk2_step(g.ConcentrationState(np.ones(8)), 0.0, kernels)


def test_rk2_step_failure_wraps_value_error(monkeypatch):
    def exploding(kernels, state, plan=None, *, breakdown=False):
        s = np.full(state.n.size, 1e308)
        return g.RhsResult(p=s, q=0 * s, s=s)

    monkeypatch.setattr(integrator_mod, "rhs_total", exploding)
    kernels = g.KernelSet({2: g.constant_tt(1.0, 2, 8)})
    with pytest.raises(g.StepFailureError):
        g.rk2_step(g.ConcentrationState(np.ones(8)), 10.0, kernels)


def test_moments_and_series():  # test_integrator.py:148-178
    st = g.ConcentrationState(np.array([1.0, 0.0, 0.0]))
    assert g.moments(st, (0, 1, 2)) == [1.0, 1.0, 1.0]
    st = g.ConcentrationState(np.array([0.0, 1.0, 0.0]))
    assert g.moments(st, (1, 2)) == [2.0, 4.0]
    with pytest.raises(ValueError):
        g.moments(st, (-1,))
    series = g.MomentSeries()
    series.record(g.ConcentrationState(np.ones(4), t=0.0))
    series.record(g.ConcentrationState(np.ones(4), t=1.0))
    with pytest.raises(ValueError, match="increasing"):
        series.record(g.ConcentrationState(np.ones(4), t=1.0))
    assert len(series) == 2 and series.m1_drift == [0.0, 0.0]


def test_time_grid_and_initial_condition():
    with pytest.raises(ValueError):
        g.TimeGrid(0.0, 1e-3, 0)
    with pytest.raises(ValueError):
        g.TimeGrid(0.0, 0.0, 10)
    with pytest.raises(ValueError, match="nonnegative"):
        g.InitialCondition.from_vector([1.0, -0.5])
    with pytest.raises(ValueError, match="kind"):
        g.InitialCondition(kind="bimodal")
    ic = g.InitialCondition.from_vector([0.5, 0.5, 0.0])
    with pytest.raises(ValueError, match="length"):
        ic.state(4)
    st = g.InitialCondition.monodisperse(2.0).state(4, t0=1.0)
    np.testing.assert_array_equal(st.n, [2.0, 0.0, 0.0, 0.0])
    assert st.t == 1.0


def test_integrate_stepwise_path_with_cpu_seam(monkeypatch):
    """integrate(on_record=...) steps through rk2_step; with the seam on the
    oracle it reproduces the oracle trajectory and the record/callback rule."""

    def oracle_total(kernels, state, plan=None, *, breakdown=False):
        ks = {d: {"kind": "tt", "arrays": kernels[d].cores} for d in kernels.orders}
        p, q, s = orc.rhs_total(ks, state.n)
        return g.RhsResult(p=p, q=q, s=s)

    monkeypatch.setattr(integrator_mod, "rhs_total", oracle_total)

    class Cfg:
        n_classes = 32
        initial = g.InitialCondition.monodisperse(1.0)
        time = g.TimeGrid(0.0, 1e-3, 10)
        record_every = 3

    seen = []
    ks = g.KernelSet({3: g.constant_tt(1.0, 3, 32)})
    final, series = g.integrate(Cfg, kernels=ks, on_record=lambda step, st: seen.append(step))
    assert seen == [0, 3, 6, 9] and len(series) == 4
    ref_n, _, ref_series = orc.integrate({3: {"kind": "tt", "arrays": ks[3].cores}}, Cfg.initial.state(32).n,
                                         dt=1e-3, steps=10, record_every=3)
    np.testing.assert_allclose(final.n, ref_n, rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(np.array(series.rows()), np.array(ref_series.rows()), rtol=1e-14)


def test_install_patches_reference_seams():
    import os
    import sys

    if os.path.isdir("/root/reference/pkg/src") and "/root/reference/pkg/src" not in sys.path:
        sys.dont_write_bytecode = True
        sys.path.append("/root/reference/pkg/src")
    ttagg = pytest.importorskip("ttagg")
    import ttagg.integrator as ti
    import ttagg.rhs as tr

    before = (tr.rhs_cp_P, tr.rhs_dense_P, tr.rhs_dense_Q, ti.rhs_total)
    undo = g.install(ttagg)
    try:
        assert tr.rhs_cp_P is g.rhs_cp_P and ti.rhs_total is not before[3]
        assert tr.rhs_dense_P is g.rhs_dense_P and tr.rhs_dense_Q is g.rhs_dense_Q
    finally:
        undo()
    assert (tr.rhs_cp_P, tr.rhs_dense_P, tr.rhs_dense_Q, ti.rhs_total) == before


def test_dense_kernel_container_and_budget():
    """DenseKernel validation (kernels.py:218-238) and the dense budget
    (rhs.py:188-199) are host-side: no GPU needed."""
    with pytest.raises(g.KernelError):
        g.DenseKernel(np.ones(5))
    with pytest.raises(g.KernelError):
        g.DenseKernel(np.ones((4, 5)))
    k = g.DenseKernel(np.arange(27.0).reshape(3, 3, 3))
    assert k.dimension == 3 and k.n_classes == 3
    assert g.kernel_element(k, (1, 2, 3)) == 5.0
    with pytest.raises(g.KernelError, match="budget"):
        g.rhs_dense_P(g.DenseKernel(np.zeros((8193, 8193))), g.ConcentrationState(np.ones(8193)))
    with pytest.raises(g.KernelError, match="budget"):
        g.rhs_total(g.KernelSet({2: g.DenseKernel(np.zeros((8193, 8193)))}), g.ConcentrationState(np.ones(8193)))


def _reference():
    import os
    import sys

    if os.path.isdir("/root/reference/pkg/src") and "/root/reference/pkg/src" not in sys.path:
        sys.dont_write_bytecode = True
        sys.path.append("/root/reference/pkg/src")
    return pytest.importorskip("ttagg")


def test_brownian_tt_matches_reference_builder():
    """construct.brownian_tt restates build_brownian_tt (kernels.py:332-363):
    the same cores, bit for bit, so integrate(config) needs no reference."""
    ttagg = _reference()
    from paper_1905_09071_b200.construct import brownian_tt

    for mus in ((0.3, -0.3), (0.2, -0.1, -0.1), (0.1, -0.1, 0.05, -0.05, 0.0)):
        ref = ttagg.build_brownian_tt(ttagg.BrownianSpec(mus), 257).cores
        got = brownian_tt(mus, 257)
        assert len(got) == len(ref)
        for a, b in zip(got, ref):
            assert a.shape == b.shape
            np.testing.assert_array_equal(a, b)


def test_kernel_set_from_config_matches_reference(tmp_path):
    """Brownian -> exact TT, constant -> rank-1 TT, table -> dense
    (config.py:231-242), from the reference's own SimulationConfig."""
    ttagg = _reference()
    from ttagg.config import build_kernel_set, config_from_dict

    from paper_1905_09071_b200.construct import kernel_set_from_config

    table = tmp_path / "k2.bin"
    rng = np.random.default_rng(5)
    vals = rng.random((16, 16))
    vals = vals + vals.T
    vals.astype("<f8").tofile(table)
    cfg = config_from_dict({"N": 16, "D": 4, "time": {"dt": 0.01, "steps": 1},
                            "kernels": {"2": {"type": "table", "table_path": str(table)},
                                        "3": {"type": "constant", "c": 2.5},
                                        "4": {"type": "brownian", "mu": [0.1, -0.1, 0.2, 0.0]}}})
    ref = build_kernel_set(cfg)
    got = kernel_set_from_config(cfg)
    np.testing.assert_array_equal(got[2].values, ref[2].values)
    for d in (3, 4):
        for a, b in zip(got[d].cores, ref[d].cores):
            np.testing.assert_array_equal(a, b)


def _oracle_total(kernels, state, plan=None, *, breakdown=False):
    """CPU stand-in for the GPU rhs_total (host-logic test double only)."""
    from types import SimpleNamespace

    from oracle import rhs_oracle as orc

    ks = {d: {"kind": "tt", "arrays": kernels[d].cores} for d in kernels.orders}
    p, q, s = orc.rhs_total(ks, state.n)
    return SimpleNamespace(p=p, q=q, s=s, by_order=None)


def test_install_routes_reference_cli_through_package_integrate(tmp_path, golden, monkeypatch):
    """After install(), the reference's own `ttagg simulate` (cli.py:80-110,
    which bound `integrate` at import, cli.py:21) runs the package's
    integrate: kernels built from the config's specs in-repo, records and
    snapshots through the reference's types and writers.  The device RHS is
    replaced by the oracle here (no GPU on this host); the GPU twin is
    tests/test_gpu_integrate.py::test_config_kernels_match_reference_cli."""
    import json

    ttagg = _reference()
    import ttagg.cli as tc
    import ttagg.integrator as ti

    import paper_1905_09071_b200.integrator as gi

    monkeypatch.setattr(gi, "rhs_total", _oracle_total)
    ref = golden("cli.npz")
    cfg = json.loads(str(ref["config"]))
    path = tmp_path / "run.json"
    path.write_text(json.dumps(cfg))
    undo = g.install(ttagg)
    try:
        assert tc.integrate is ti.integrate and ti.integrate is not gi.integrate
        assert tc.main(["simulate", "--config", str(path), "--output", str(tmp_path / "out")]) == 0
        rows = np.loadtxt(tmp_path / "out" / "moments.csv", delimiter=",", skiprows=1)
        snap = np.loadtxt(tmp_path / "out" / "n_40.csv", delimiter=",", skiprows=1)[:, 1]
        assert rows.shape == ref["rows"].shape
        from conftest import assert_rows

        assert_rows(rows, ref["rows"], 1e-9)  # FFT roundoff differs from the reference's plan
        np.testing.assert_allclose(snap, ref["n_final"], rtol=0, atol=1e-10 * np.abs(ref["n_final"]).max())
        # a diverging run maps to the CLI's numerical-failure exit code (cli.py:236-238)
        cfg_bad = dict(cfg, time={"t0": 0.0, "dt": 1e6, "steps": 3})
        path.write_text(json.dumps(cfg_bad))
        assert tc.main(["simulate", "--config", str(path), "--output", str(tmp_path / "bad")]) == 2
    finally:
        undo()
    assert tc.integrate is not ti.rhs_total and ti.integrate.__module__ == "ttagg.integrator"


def test_group_rank_split_covers_every_rank_once():
    """Device-group sharding (Group.shards): every CP rank term on exactly one
    device, balanced within one term, small orders spread over devices."""
    from paper_1905_09071_b200._lib import group_rank_split

    for n_dev in (1, 2, 3, 4, 8):
        owners = {}
        for d, R in ((2, 2), (3, 6), (4, 24), (5, 120)):
            split = group_rank_split(d, R, n_dev)
            assert len(split) == n_dev
            flat = sorted(r for sub in split for r in sub)
            assert flat == list(range(R))
            sizes = [len(sub) for sub in split]
            assert max(sizes) - min(sizes) <= 1
            for i, sub in enumerate(split):
                if sub:
                    owners.setdefault(i, []).append(d)
        if n_dev == 8:  # the rank-2 and rank-6 orders do not pile onto the same devices
            assert len(owners) == 8


def test_bench_launches_its_own_ranks():
    """`bench.py --gpus N` outside torchrun starts N ranks itself (torchrun on
    127.0.0.1) and reports n_gpus = the world actually used; a mismatched
    WORLD_SIZE is refused.  The launch plumbing runs here over gloo
    (--launcher-selftest: no GPU work)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["max_ms"] == 2.0
    assert sorted(r[0] for r in line["ranks"]) == [0, 1] and all(r[2] == 2 for r in line["ranks"])
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, env={**env, "WORLD_SIZE": "1"}, timeout=120)
    assert bad.returncode == 2 and "refusing" in bad.stderr
