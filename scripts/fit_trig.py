"""Near-minimax polynomial coefficients for the device trig kernels (psso_trig.cuh).

cos(pi*s) = P(s^2), |s| <= 1/2   and   sin(r) = r*Q(r^2), |r| <= pi/2.
Least squares over Chebyshev nodes in 60-digit arithmetic (mpmath), then the
coefficients are rounded to the target type and the max abs error re-measured
with the rounded coefficients.  Prints the C initialisers.
"""
import mpmath as mp

mp.mp.dps = 60


def fit(f, zmax, deg, npts=400):
    nodes = [zmax * (1 - mp.cos(mp.pi * (k + 0.5) / npts)) / 2 for k in range(npts)]
    A = mp.matrix(npts, deg + 1)
    b = mp.matrix(npts, 1)
    for i, z in enumerate(nodes):
        for j in range(deg + 1):
            A[i, j] = z ** j
        b[i] = f(z)
    c = mp.lu_solve(A.T * A, A.T * b)
    return [c[j] for j in range(deg + 1)]


def rnd(c, single):
    import numpy as np
    t = np.float32 if single else np.float64
    return [float(t(float(x))) for x in c]


def err(f, c, zmax, scale, n=4000):
    m = 0
    for k in range(n + 1):
        z = zmax * mp.mpf(k) / n
        p = mp.mpf(0)
        for x in reversed(c):
            p = p * z + mp.mpf(x)
        m = max(m, abs((p - f(z)) * scale(z)))
    return float(m)


cosf_ = lambda z: mp.cos(mp.pi * mp.sqrt(z))                          # noqa: E731
sinq_ = lambda z: (mp.sin(mp.sqrt(z)) / mp.sqrt(z)) if z > 0 else mp.mpf(1)  # noqa: E731
for name, f, zmax, deg, single, scale in [
    ("COS_PI_D", cosf_, mp.mpf(1) / 4, 8, False, lambda z: 1),
    ("COS_PI_F", cosf_, mp.mpf(1) / 4, 5, True, lambda z: 1),
    ("SIN_Q_D", sinq_, (mp.pi / 2) ** 2, 9, False, lambda z: mp.sqrt(z)),
    ("SIN_Q_F", sinq_, (mp.pi / 2) ** 2, 5, True, lambda z: mp.sqrt(z)),
]:
    c = rnd(fit(f, zmax, deg), single)
    print(f"// {name}: degree {deg} in z, max abs error {err(f, c, zmax, scale):.3g}")
    print("{" + ", ".join(repr(x) for x in c) + "}")
