"""numpy model of the GPU algorithm (same index maps) to validate the math."""
import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rhs_oracle as orc

def geom(N):
    Np = max(64, 1 << (N - 1).bit_length()); N1 = max(4, Np // 256); return Np, N1, Np // N1

def model_gain_cp(fs, n):
    d = len(fs); N = n.size; R = fs[0].shape[1]
    Np, N1, N2 = geom(N); L = d * Np; K = d * N1
    cols = []
    for r in range(R):
        for m in range(d):
            x = np.zeros(Np); x[:N] = fs[m][:, r] * n; cols.append(x)
    if len(cols) % 2: cols.append(np.zeros(Np))
    # residue rows
    rows = []  # (j, k1)
    for k1 in range(N1 // 2 + 1): rows.append((0, k1))
    for j in range(1, (d + 1) // 2):
        if 2 * j < d:
            for k1 in range(N1): rows.append((j, k1))
    if d % 2 == 0:
        for k1 in range(N1 // 2): rows.append((d // 2, k1))
    kap = np.array([j + d * k1 for j, k1 in rows])
    WK = lambda m: np.exp(-2j * np.pi * m / K)
    WL = lambda m: np.exp(-2j * np.pi * m / L)
    Tspec = []
    for p in range(len(cols) // 2):
        a = cols[2 * p].reshape(N1, N2); b = cols[2 * p + 1].reshape(N1, N2)   # [n1, n2]
        z = a + 1j * b
        Y = {}
        for j in range(d):
            tw = WK(j * np.arange(N1))[:, None]
            Y[j] = np.fft.fft(z * tw, axis=0)   # [k1, n2]
        Ta = np.zeros((len(rows), N2), complex); Tb = np.zeros_like(Ta)
        for ri, (j, k1) in enumerate(rows):
            kappa = j + d * k1
            mk = (K - kappa) % K; jm = mk % d; k1m = mk // d
            Z = Y[j][k1]; Zm = Y[jm][k1m]
            A = (Z + np.conj(Zm)) / 2; B = -1j * (Z - np.conj(Zm)) / 2
            w = WL(np.arange(N2) * kappa)
            Ta[ri] = A * w; Tb[ri] = B * w
        Tspec += [Ta, Tb]
    S = np.zeros((len(rows), N2), complex)
    for r in range(R):
        prod = np.ones((len(rows), N2), complex)
        for m in range(d):
            prod *= np.fft.fft(Tspec[r * d + m], axis=1)
        S += prod
    k = kap[:, None] + K * np.arange(N2)[None, :]
    S *= WL(((d - 1) * k) % L)
    u = np.fft.ifft(S, axis=1) * N2
    wgt = np.where((kap == 0) | (2 * kap == K), 1.0, 2.0)[:, None]
    U = wgt * np.conj(WL(np.arange(N2)[None, :] * kap[:, None])) * u    # [row, n2]
    s = np.zeros((N1, N2))
    for ri, (j, k1) in enumerate(rows):
        # contribution Re(U[row, n2] * W_K^{-n1 kappa})
        s += np.real(U[ri][None, :] * np.conj(WK(np.arange(N1)[:, None] * kap[ri])))
    s = s.reshape(-1)[:N] / L / np.math.factorial(d) if hasattr(np, 'math') else s.reshape(-1)[:N] / L
    import math
    s = s if hasattr(np, 'math') else s / math.factorial(d)
    p = s.copy(); p[:d - 1] = 0
    return p

rng = np.random.default_rng(0)
for N, d in ((64, 2), (64, 3), (50, 4), (100, 5), (300, 3)):
    fs = [rng.random((N, 2)) for _ in range(d)]; n = rng.random(N)
    p = model_gain_cp(fs, n); ref = orc.cp_gain(fs, n)
    print(N, d, np.abs(p - ref).max() / np.abs(ref).max())
