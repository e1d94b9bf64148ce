"""Host-side kernel construction for the BASELINE configs (not on the hot path).

* ``tt_cross`` — TT-cross (alternating maxvol skeletons) of a function on the
  grid [1..N]^d, for config 4's kernel (i+j+l)^(1/2)(ijl)^(-1/6), which the
  reference cannot compress (TT-cross is a declared non-goal, SPEC.md:150;
  SURVEY.md §0.5, §8(f)).  The cores are built once and fed identically to
  every implementation, so RHS parity never depends on the approximation.
* ``c4_kernels`` — the C4 kernel set: exact rank-3 TT for (i^(1/3)+j^(1/3))^2
  (d = 2) and the cross-approximated d = 3 kernel (ranks <= 16, tol 1e-6).
* ``brownian_tt`` / ``kernel_set_from_config`` — the reference's default
  kernels for a ``SimulationConfig`` (config.py:231-242): the exact
  constructive TT of a generalized Brownian kernel (Theorem 1,
  kernels.py:332-363; ranks C(D, lam)), rank-1 constant TT, dense tables;
  restated here so ``integrate(config)`` needs no reference import.
* ``tt_rank_shard`` — slice a TT kernel over its first internal rank index:
  the gain and loss are linear in that index (rhs.py:277-290, 305-338), so
  the slices of all GPUs sum to the full RHS (TT rank sharding).
"""

from __future__ import annotations

import numpy as np

__all__ = ["maxvol", "tt_cross", "cores_from_skeleton", "c4_kernels", "c4_d2_cores", "c4_d3_from_skeleton",
           "tt_rank_shard", "brownian_tt", "kernel_set_from_config"]


def _orth(a: np.ndarray) -> np.ndarray:
    """Orthonormal basis of the columns of a tall matrix (CholeskyQR2, O(n r^2))."""
    q = a
    for _ in range(2):
        g = q.T @ q
        try:
            r = np.linalg.cholesky(g).T
        except np.linalg.LinAlgError:
            return np.linalg.qr(a)[0]
        q = np.linalg.solve(r.T, q.T).T
    return q


def maxvol(a: np.ndarray, tol: float = 1.05, max_iters: int = 64) -> np.ndarray:
    """Row indices of a (near) maximum-volume r x r submatrix of the n x r matrix a."""
    n, r = a.shape
    if n <= r:
        return np.arange(n)
    import scipy.linalg as sla

    # initial guess from LU with partial pivoting (O(n r^2))
    perm, _, _ = sla.lu(a, p_indices=True)
    idx = np.array(perm[:r])
    b = np.linalg.solve(a[idx].T, a.T).T  # n x r, b[idx] = I
    for _ in range(max_iters):
        flat = np.argmax(np.abs(b))
        i, j = divmod(int(flat), r)
        if abs(b[i, j]) <= tol:
            break
        bj = b[:, j].copy()
        bi = b[i, :].copy()
        bi[j] -= 1.0
        b -= np.outer(bj, bi / b[i, j])
        idx[j] = i
    return idx


def _fiber_fn(f, N: int, d: int):
    grid = np.arange(1, N + 1)

    def fiber(k, Ik, Jk1):
        # tensor of values f(I_k, i, J_{k+1}) with shape (r_k, N, r_{k+1})
        if hasattr(f, "fiber"):
            return f.fiber(Ik, grid, Jk1)
        a, b = Ik.shape[0], Jk1.shape[0]
        pts = np.empty((a, N, b, d), dtype=np.int64)
        pts[:, :, :, :k] = Ik[:, None, None, :]
        pts[:, :, :, k] = grid[None, :, None]
        pts[:, :, :, k + 1 :] = Jk1[None, None, :, :]
        return f(pts.reshape(-1, d)).reshape(a, N, b)

    return fiber


def cores_from_skeleton(f, n_classes: int, d: int, I, J):
    """TT cores of f through the cross skeleton (left index sets I[0..d-1],
    right index sets J[1..d]): C_k = f(I_k, :, J_{k+1}) times the inverse of
    f(I_{k+1}, J_{k+1}).  A few seconds at N = 2^20 — the skeleton (a few KB)
    is what fixtures store instead of the cores."""
    fiber = _fiber_fn(f, n_classes, d)
    cores = [None] * d
    for k in range(d):
        c = fiber(k, I[k], J[k + 1])
        if k < d - 1:
            r0, r1 = c.shape[0], c.shape[2]
            cmat = c.reshape(r0 * n_classes, r1)
            a = I[k + 1].shape[0]
            full = np.empty((a, J[k + 1].shape[0], d), dtype=np.int64)
            full[:, :, : k + 1] = I[k + 1][:, None, :]
            full[:, :, k + 1 :] = J[k + 1][None, :, :]
            m = f(full.reshape(-1, d)).reshape(a, -1)
            cmat = np.linalg.solve(m.T, cmat.T).T
            cores[k] = np.ascontiguousarray(cmat.reshape(r0, n_classes, r1))
        else:
            cores[k] = np.ascontiguousarray(c)
    return cores


def tt_cross(f, n_classes: int, d: int, rank: int, sweeps: int = 2, seed: int = 0, return_skeleton: bool = False):
    """TT-cross with fixed ranks (1, r, ..., r, 1) of f(idx) on [1..N]^d.

    ``f(points)`` evaluates the function on an (m, d) array of 1-based
    indices.  Returns d cores of shape (r_{k-1}, N, r_k) (and, with
    ``return_skeleton``, the index sets I, J that determine them).
    """
    rng = np.random.default_rng(seed)
    N = n_classes
    r = [1] + [min(rank, N ** min(k, d - k)) for k in range(1, d)] + [1]
    grid = np.arange(1, N + 1)
    # left index sets I[k]: (r[k], k) multi-indices; right sets J[k]: (r[k], d-k)
    J = [None] * (d + 1)
    J[d] = np.zeros((1, 0), dtype=np.int64)
    for k in range(d - 1, 0, -1):
        J[k] = rng.integers(1, N + 1, size=(r[k], d - k))
    I = [None] * (d + 1)
    I[0] = np.zeros((1, 0), dtype=np.int64)
    fiber = _fiber_fn(f, N, d)
    for _ in range(sweeps):
        # left-to-right: choose I[k+1]
        for k in range(d - 1):
            c = fiber(k, I[k], J[k + 1]).reshape(r[k] * N, r[k + 1])
            sel = maxvol(_orth(c))
            left = np.concatenate([np.repeat(I[k], N, axis=0), np.tile(grid, r[k])[:, None]], axis=1)
            I[k + 1] = left[sel]
        # right-to-left: choose J[k]
        for k in range(d - 1, 0, -1):
            c = fiber(k, I[k], J[k + 1]).reshape(r[k], N * r[k + 1])
            sel = maxvol(_orth(np.ascontiguousarray(c.T)))
            right = np.concatenate(
                [np.repeat(grid, r[k + 1])[:, None], np.tile(J[k + 1], (N, 1))], axis=1
            )
            J[k] = right[sel]
    cores = cores_from_skeleton(f, N, d, I, J)
    return (cores, I, J) if return_skeleton else cores


class _C4d3:
    """(i+j+l)^(1/2) (ijl)^(-1/6): pointwise and broadcast fiber evaluation."""

    def __call__(self, points: np.ndarray) -> np.ndarray:
        p = points.astype(np.float64)
        return np.sqrt(p.sum(axis=1)) * np.exp(-np.log(p).sum(axis=1) / 6.0)

    def fiber(self, Ik, grid, Jk1):
        left = Ik.astype(np.float64)
        right = Jk1.astype(np.float64)
        g = grid.astype(np.float64)
        sl = left.sum(axis=1)[:, None, None]
        sr = right.sum(axis=1)[None, None, :]
        pl = np.exp(-np.log(left).sum(axis=1) / 6.0)[:, None, None] if left.shape[1] else 1.0
        pr = np.exp(-np.log(right).sum(axis=1) / 6.0)[None, None, :] if right.shape[1] else 1.0
        out = np.sqrt(sl + g[None, :, None] + sr)
        out *= g[None, :, None] ** (-1.0 / 6.0)
        out *= pl
        out *= pr
        return out


_c4_d3 = _C4d3()


def c4_d2_cores(n_classes: int):
    """Exact rank-3 TT of (i^(1/3)+j^(1/3))^2 (config 4, d = 2)."""
    i = np.arange(1, n_classes + 1, dtype=np.float64)
    c1 = np.zeros((1, n_classes, 3))
    c1[0, :, 0], c1[0, :, 1], c1[0, :, 2] = i ** (2 / 3), 2 * i ** (1 / 3), 1.0
    c2 = np.zeros((3, n_classes, 1))
    c2[0, :, 0], c2[1, :, 0], c2[2, :, 0] = 1.0, i ** (1 / 3), i ** (2 / 3)
    return c1, c2


def c4_kernels(n_classes: int, rank: int = 16, seed: int = 0, return_skeleton: bool = False):
    """Config 4: {2: exact rank-3 TT of (i^(1/3)+j^(1/3))^2, 3: TT-cross of
    (i+j+l)^(1/2)(ijl)^(-1/6) with ranks <= rank}; returns (cores2, cores3)
    (and the d = 3 cross skeleton (I, J) with ``return_skeleton``)."""
    out = tt_cross(_c4_d3, n_classes, 3, rank, seed=seed, return_skeleton=return_skeleton)
    if return_skeleton:
        cores3, I, J = out
        return c4_d2_cores(n_classes), tuple(cores3), (I, J)
    return c4_d2_cores(n_classes), tuple(out)


def c4_d3_from_skeleton(n_classes: int, I, J):
    """The config-4 d = 3 cores from a stored cross skeleton."""
    return tuple(cores_from_skeleton(_c4_d3, n_classes, 3, I, J))


def tt_rank_shard(cores, world: int, rank: int):
    """Cores restricted to this GPU's share of the first internal rank index."""
    r1 = cores[0].shape[2]
    sel = np.array_split(np.arange(r1), world)[rank]
    if sel.size == 0:
        return None
    out = list(cores)
    out[0] = np.ascontiguousarray(cores[0][:, :, sel])
    out[1] = np.ascontiguousarray(cores[1][sel, :, :])
    return tuple(out)


# ---------------------------------------------------------------------------
# default kernels of a SimulationConfig (config.py:231-242)
# ---------------------------------------------------------------------------

def _colex_subsets(d: int, level: int):
    """level-subsets of the labels 1..d in colexicographic order (kernels.py:266-287)."""
    from itertools import combinations

    return sorted(combinations(range(1, d + 1), level), key=lambda t: t[::-1])


def brownian_tt(exponents, n_classes: int):
    """Exact TT cores of the generalized Brownian kernel with exponents mu
    (Theorem 1; the construction of build_brownian_tt, kernels.py:332-363).

    Rank index r at level lam is the r-th lam-subset S of the exponent labels
    (colex order); the fiber S -> T of core lam is the power vector
    i^mu_l = exp(mu_l log i) of the one label l = T \\ S when S is contained
    in T, and zero otherwise.  Ranks C(D, lam)."""
    mus = [float(m) for m in exponents]
    d = len(mus)
    if d < 2:
        raise ValueError("a Brownian kernel needs at least two exponents")
    sizes = np.arange(1, n_classes + 1, dtype=np.float64)
    logs = np.log(sizes)
    pows = [np.exp(mu * logs) for mu in mus]
    levels = [_colex_subsets(d, lam) for lam in range(d + 1)]
    index = [{sub: r for r, sub in enumerate(lv)} for lv in levels]
    cores = []
    for lam in range(1, d + 1):
        core = np.zeros((len(levels[lam - 1]), n_classes, len(levels[lam])))
        for rc, T in enumerate(levels[lam]):
            for label in T:
                S = tuple(x for x in T if x != label)
                core[index[lam - 1][S], :, rc] = pows[label - 1]
        cores.append(core)
    return tuple(cores)


def _load_table(path: str, d: int, n_classes: int) -> np.ndarray:
    """N^d coefficients, flat little-endian binary or text (kernels.py:404-422)."""
    import os

    from .kernels import KernelError

    expected = n_classes ** d
    if not os.path.exists(path):
        raise KernelError(f"kernel table file not found: {path}")
    if os.path.getsize(path) == expected * 8:
        flat = np.fromfile(path, dtype="<f8")
    else:
        try:
            flat = np.loadtxt(path, dtype=np.float64).ravel()
        except (ValueError, UnicodeDecodeError) as exc:
            raise KernelError(f"kernel table {path} could not be read ({exc})") from None
    if flat.size != expected:
        raise KernelError(f"kernel table {path} holds {flat.size} values, expected {expected}")
    return flat.reshape((n_classes,) * d)


def kernel_set_from_config(config):
    """KernelSet of a config's ``kernel_specs`` exactly as the reference's
    build_kernel_set (config.py:231-242): Brownian specs -> exact TT,
    constant specs -> rank-1 TT, tables -> dense.  Specs are recognised by
    their fields (``exponents`` / ``value`` / ``path``)."""
    from .kernels import DenseKernel, KernelError, TTKernel, constant_tt
    from .rhs import KernelSet

    N = int(config.n_classes)
    out = {}
    for d, spec in config.kernel_specs.items():
        if hasattr(spec, "exponents"):
            out[d] = TTKernel(brownian_tt(spec.exponents, N))
        elif hasattr(spec, "value"):
            out[d] = constant_tt(spec.value, d, N)
        elif hasattr(spec, "path"):
            if N ** d > 1 << 26:
                raise KernelError(f"dense kernel would hold {N ** d} elements, over the budget of {1 << 26}")
            out[d] = DenseKernel(_load_table(spec.path, spec.dimension, N))
        else:
            raise KernelError(f"unsupported kernel specification {type(spec).__name__}")
    return KernelSet(out)
