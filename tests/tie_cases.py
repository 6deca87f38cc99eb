"""Inputs that put d*inv + u exactly on (and one fp32 step either side of) an integer.

Each group of G elements holds 0 and L = 2^b - 1, so mn = 0, range = L, inv = RZ(L / L) = 1
and T_i = d_i = x_i exactly (include/gact.h). Element i of the other slots is
x_i = N_i - (2 k_i + 1) 2^-9 + delta_i with k_i the element's 8-bit Philox byte (taken
from the oracle's generator, passed in as `lane`) and N_i in [1, L], so that
T_i + u_i = N_i + delta_i: the threshold test floor(T + u) sits exactly on its tie for
delta = 0 (q = N: the exact sum reaches N) and one fp32 step below / above it otherwise
(q = N - 1 / q = N). These are the cases where a GPU shortcut for the exact real
floor(T + u) (R5: fma.rm / fma.rn on the 2^-16 grid of [128, 256)) would go wrong first.
The expected codes are the closed form above, independent of both implementations.
"""
import numpy as np


def tie_groups(n_groups: int, G: int, bits: int, seed: int, lane, rng) -> tuple[np.ndarray, np.ndarray]:
    """(x float32[n_groups * G], expected codes uint8 or 255 where not constructed)."""
    L = (1 << bits) - 1
    n = n_groups * G
    x = np.zeros(n, dtype=np.float32)
    want = np.full(n, 255, dtype=np.int64)
    for g in range(n_groups):
        base = g * G
        x[base] = 0.0
        x[base + 1] = float(L)
        want[base], want[base + 1] = 0, L
        for j in range(2, G):
            i = base + j
            k = lane(seed, i)
            N = int(rng.integers(1, L + 1))
            which = j % 3  # 0: tie, 1: just below, 2: just above
            t = float(N) - (2 * k + 1) * 2.0 ** -9
            # one fp32 step of t (below / above), exactly representable by construction
            f = np.float32(t)
            if float(f) != t:  # not representable at this magnitude: plain integer instead
                x[i] = np.float32(N)
                want[i] = N
                continue
            if which == 1:
                f = np.nextafter(f, np.float32(-1.0))
                want[i] = N - 1
            elif which == 2:
                f = np.nextafter(f, np.float32(np.inf))
                want[i] = N
            else:
                want[i] = N
            x[i] = f
    return x, want
