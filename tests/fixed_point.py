"""NumPy restatement of the device's exact diagonal accumulation
(csrc/norm_observe.cu: fixed_split / observe_diag_fixed / fixed_to_double),
used by the tests as the checker: each |psi|^2 is split onto the grids
2^-30, 2^-70, 2^-110 and summed as int64 limbs, so sums are associative."""

import numpy as np

C2, C1, C0 = 1.5 * 2.0**22, 1.5 * 2.0**-18, 1.5 * 2.0**-58


def split(x):
    x = np.asarray(x, dtype=np.float64)
    a2 = (x + C2) - C2
    r1 = x - a2
    a1 = (r1 + C1) - C1
    r0 = r1 - a1
    a0 = (r0 + C0) - C0
    return np.stack([(a2 * 2.0**30).astype(np.int64), (a1 * 2.0**70).astype(np.int64),
                     (a0 * 2.0**110).astype(np.int64)])


def limbs(psi):
    """[3][D] int64 limbs of sum_r |psi_r|^2 for a (R, D) complex stack."""
    psi = np.asarray(psi)
    x = psi.real * psi.real + psi.imag * psi.imag
    return split(x).sum(axis=1) if x.ndim == 2 else split(x)


def to_double(acc):
    acc = np.asarray(acc, dtype=np.int64).copy()
    l2, l1, l0 = acc[0], acc[1], acc[2]
    c0 = l0 >> 40
    l0 = l0 - (c0 << 40)
    l1 = l1 + c0
    c1 = l1 >> 40
    l1 = l1 - (c1 << 40)
    l2 = l2 + c1
    lo = l1.astype(np.float64) * 2.0**-70 + l0.astype(np.float64) * 2.0**-110
    return l2.astype(np.float64) * 2.0**-30 + lo
