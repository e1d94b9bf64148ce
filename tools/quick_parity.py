"""Debug harness: GPU vs oracle on many shapes, prints errors (no asserts)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_09071_b200 as g
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.workloads import permutation_power_cp, CONFIGS, initial_state

def rel(a, b):
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s else 1.0)

rng = np.random.default_rng(1)
worst = 0
for N in (2, 3, 8, 16, 37, 64, 100, 257, 1000, 4096, 5000, 65536):
    for d in (2, 3, 4, 5):
        R = 3
        fs = tuple(rng.random((N, R)) for _ in range(d))
        n = rng.random(N)
        k = g.CPKernel(fs)
        st = g.ConcentrationState(n)
        try:
            P = g.rhs_cp_P(k, st); Q = g.rhs_cp_Q(k, st)
        except Exception as e:
            print("ERR", N, d, e); continue
        eP = rel(P, orc.cp_gain(fs, n)); eQ = rel(Q, orc.cp_loss(fs, n))
        worst = max(worst, eP, eQ)
        print(f"CP N={N} d={d}: P {eP:.2e} Q {eQ:.2e}", flush=True)
for N in (16, 64, 300, 4096):
    for d in (2, 3, 4):
        ranks = [1] + [int(x) for x in rng.integers(1, 5, d - 1)] + [1]
        cores = tuple(rng.random((ranks[l], N, ranks[l + 1])) for l in range(d))
        n = rng.random(N)
        k = g.TTKernel(cores); st = g.ConcentrationState(n)
        P = g.rhs_tt_P(k, st); Q = g.rhs_tt_Q(k, st)
        eP = rel(P, orc.tt_gain(cores, n)); eQ = rel(Q, orc.tt_loss(cores, n))
        worst = max(worst, eP, eQ)
        print(f"TT N={N} d={d} ranks={ranks}: P {eP:.2e} Q {eQ:.2e}", flush=True)
# C5 full N closed form for d=5 only (collapsed d-fold convolution)
N = 1 << 20
a = CONFIGS["C5"].exponents
n = initial_state("c5", N)
for d in (2, 3, 4, 5):
    fs = permutation_power_cp(a[:d], N)
    t0 = time.time()
    P = g.rhs_cp_P(g.CPKernel(fs), g.ConcentrationState(n))
    t1 = time.time()
    sz = np.arange(1, N + 1, dtype=np.float64)
    L = 1 << int(np.ceil(np.log2(d * N + 1)))
    spec = np.ones(L // 2 + 1, dtype=complex)
    for j in range(d):
        v = np.zeros(L); v[1:N + 1] = np.exp(a[j] * np.log(sz)) * n
        spec *= np.fft.rfft(v)
    conv = np.fft.irfft(spec, n=L)
    ref = np.zeros(N); ref[d - 1:] = conv[d:N + 1]
    e = rel(P, ref); worst = max(worst, e)
    print(f"C5 d={d} N=2^20 closed form: {e:.2e} ({t1-t0:.2f}s incl upload)", flush=True)
print("WORST", worst)
