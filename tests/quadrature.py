"""Independent brute-force quadrature for the single-triangle potential
I(r;T) = int_T dS'/|r - r'|, used only to pin the oracle.

Method (not the oracle's edge formula): polar coordinates about the foot point
rho of r in the triangle's plane.  For a ray from rho at angle theta, the
triangle occupies radii [r1, r2]; the radial integral is exact,
  int_{r1}^{r2} s ds / sqrt(s^2 + h^2) = sqrt(r2^2 + h^2) - sqrt(r1^2 + h^2),
and the remaining 1-D integral over theta is done with adaptive Gauss-Kronrod
(scipy.integrate.quad) with break points at the vertex directions.
"""
import numpy as np
from scipy.integrate import quad


def _frame(v0, v1, v2):
    e1 = v1 - v0
    n = np.cross(e1, v2 - v0)
    n /= np.linalg.norm(n)
    ex = e1 / np.linalg.norm(e1)
    ey = np.cross(n, ex)
    return ex, ey, n


def _ray_interval(p, d, P):
    """Radii [r1,r2] (>=0) where ray p + s d, s>=0, lies in the 2-D triangle P."""
    lo, hi = 0.0, np.inf
    for i in range(3):
        a, b = P[i], P[(i + 1) % 3]
        c = P[(i + 2) % 3]
        # half-plane of edge (a,b) containing c: nrm.(x - a) >= 0
        t = b - a
        nrm = np.array([-t[1], t[0]])
        if nrm @ (c - a) < 0:
            nrm = -nrm
        num = nrm @ (p - a)
        den = nrm @ d
        if abs(den) < 1e-300:
            if num < 0:
                return 0.0, 0.0
            continue
        s = -num / den
        if den > 0:
            lo = max(lo, s)
        else:
            hi = min(hi, s)
    if hi <= lo:
        return 0.0, 0.0
    return lo, hi


def tri_potential_quad(r, v0, v1, v2, epsrel=1e-13):
    r, v0, v1, v2 = (np.asarray(x, dtype=np.float64) for x in (r, v0, v1, v2))
    ex, ey, n = _frame(v0, v1, v2)
    h = (r - v0) @ n
    rho = r - h * n
    P = np.array([[(v - rho) @ ex, (v - rho) @ ey] for v in (v0, v1, v2)])
    p0 = np.zeros(2)

    def f(th):
        d = np.array([np.cos(th), np.sin(th)])
        r1, r2 = _ray_interval(p0, d, P)
        if r2 <= r1:
            return 0.0
        return np.sqrt(r2 * r2 + h * h) - np.sqrt(r1 * r1 + h * h)

    angs = sorted({float(np.arctan2(q[1], q[0]) % (2 * np.pi)) for q in P if np.hypot(*q) > 0})
    pts = [a for a in angs if 0 < a < 2 * np.pi]
    val, err = quad(f, 0.0, 2 * np.pi, points=pts if pts else None, limit=400, epsabs=0.0, epsrel=epsrel)
    return val
