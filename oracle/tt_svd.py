"""Dense TT-SVD (Oseledets 2011) — test infrastructure for small C4-shaped cases.

The reference declares TT-cross/SVD compression a non-goal and
builds no compressed kernels; BASELINE config 4 asks for one.  This routine
produces the cores once on the host; the same cores are then fed to the
reference, the oracle and the GPU path, so parity never depends on it.
"""

from __future__ import annotations

import numpy as np


def tt_svd(tensor: np.ndarray, eps: float = 1e-6, rmax: int = 16) -> list[np.ndarray]:
    """Sequential truncated SVDs; relative Frobenius error <= eps (before the rank cap)."""
    shape = tensor.shape
    d = len(shape)
    delta = eps / np.sqrt(max(d - 1, 1)) * np.linalg.norm(tensor)
    cores = []
    c = tensor.reshape(shape[0], -1)
    r_prev = 1
    for k in range(d - 1):
        c = c.reshape(r_prev * shape[k], -1)
        u, s, vt = np.linalg.svd(c, full_matrices=False)
        tail = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]  # tail[i] = ||s[i:]||
        r = int(np.sum(tail > delta))
        r = max(1, min(r, rmax))
        cores.append(u[:, :r].reshape(r_prev, shape[k], r))
        c = s[:r, None] * vt[:r]
        r_prev = r
    cores.append(c.reshape(r_prev, shape[-1], 1))
    return [np.ascontiguousarray(x) for x in cores]
