"""Element constants: closed-form hex8 stiffness, SIMP law, self-weight lumping.

Host-side constants (a 24x24 matrix per problem) with the reference's public
surface (element.py:30-133).  The device kernels never use the dense K0: they
use its factorized form (6 coefficients per level), derived
from the same lam / mu / h.  `unit_stiffness` is kept for API parity and for
the coarsest-level dense factorization check in tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["ElementStiffness", "MaterialModel", "unit_stiffness", "simp_scale",
           "simp_scale_derivative", "element_gravity_load", "lame"]


@dataclass(frozen=True)
class ElementStiffness:
    matrix: np.ndarray
    nu: float
    h: float


@dataclass(frozen=True)
class MaterialModel:
    """s(rho) = kmin_frac + rho**p (1 - kmin_frac); E scales K0 (element.py:40-58)."""

    p: float = 3.0
    kmin_frac: float = 1e-9
    E: float = 1.0

    def __post_init__(self):
        if self.p < 1:
            raise ValueError(f"penalization exponent must be >= 1, got {self.p}")
        if not 0 < self.kmin_frac < 1:
            raise ValueError(f"kmin_frac must lie in (0, 1), got {self.kmin_frac}")
        if self.E <= 0:
            raise ValueError("elastic modulus must be positive")


def lame(nu: float):
    return nu / ((1 + nu) * (1 - 2 * nu)), 1.0 / (2 * (1 + nu))


# 1-D integrals of the linear hat pair over [0,1]: value*value, grad*grad,
# grad*value (row = gradient).
_T_VV = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
_T_GG = np.array([[1.0, -1.0], [-1.0, 1.0]])
_T_GV = np.array([[-0.5, -0.5], [0.5, 0.5]])


def unit_stiffness(nu: float, h: float) -> ElementStiffness:
    """Closed-form 24x24 stiffness of an h-cube, E = 1 (element.py:82-99)."""
    if not 0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must lie in [0, 0.5), got {nu}")
    if not h > 0:
        raise ValueError(f"edge length must be positive, got {h}")
    lam, mu = lame(nu)

    def pick(axis, a, b):
        if axis == a and axis == b:
            return _T_GG
        if axis == a:
            return _T_GV
        if axis == b:
            return _T_GV.T
        return _T_VV

    grad = np.empty((3, 3, 8, 8))
    for a in range(3):
        for b in range(3):
            # x fastest in the corner index: kron(z, kron(y, x))
            grad[a, b] = np.kron(pick(2, a, b), np.kron(pick(1, a, b), pick(0, a, b))) * h
    trace = grad[0, 0] + grad[1, 1] + grad[2, 2]
    K = np.zeros((24, 24))
    for a in range(3):
        for b in range(3):
            blk = lam * grad[a, b] + mu * grad[b, a]
            if a == b:
                blk = blk + mu * trace
            K[a::3, b::3] = blk
    return ElementStiffness(K, float(nu), float(h))


def _check_rho(r):
    if np.any(r < 0) or np.any(r > 1):
        raise ValueError("density outside [0, 1]")


def simp_scale(rho, model: MaterialModel):
    """Scalar / host helper of s(rho) (element.py:102-108); the hot path
    evaluates it on the device (vt_scale_from_density)."""
    r = np.asarray(rho, dtype=np.float64)
    _check_rho(r)
    s = model.kmin_frac + r**model.p * (1.0 - model.kmin_frac)
    return s if s.ndim else float(s)


def simp_scale_derivative(rho, model: MaterialModel):
    r = np.asarray(rho, dtype=np.float64)
    _check_rho(r)
    d = model.p * r ** (model.p - 1.0) * (1.0 - model.kmin_frac)
    return d if d.ndim else float(d)


def element_gravity_load(rho: float, g: float, h: float, unit_weight: float, axis: int = 2):
    """Self-weight of one element, h^3/8 of it on each corner (element.py:121-133)."""
    if not 0 <= rho <= 1:
        raise ValueError("density outside [0, 1]")
    f = np.zeros(24)
    f[axis::3] = -rho * unit_weight * g * h**3 / 8.0
    return f


def gravity_coefficient(g: float, h: float, unit_weight: float) -> float:
    """Per-corner load of a unit-density element, same rounding as element_gravity_load(1.0, ...)."""
    return -1.0 * unit_weight * g * h**3 / 8.0
