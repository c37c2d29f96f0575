"""Ensemble observables from the diagonal of the averaged density matrix.

The reference builds the full ``<rho>`` as a dense D x D Gram product
(density.py:57-98) and reads everything off it (observables.py:34-101).
Every observable on the hot path except purity needs only its diagonal
``p(alpha) = mean_r |psi_r(alpha)|^2``; the device computes that sum
(``ctqw_observe_diag``), the cross-GPU all-reduce adds the shards, and
``ctqw_observe_reduce`` produces the populations and the participation-ratio
sums.  Purity is ``(1/R^2) sum_{r,s} |<psi_r|psi_s>|^2`` from the
realization overlaps (``ctqw_overlap_sumsq``), never the D x D matrix.

``DiagonalDensity`` stands in for the reference's ``DensityMatrix`` in the
``density_snapshot`` sink callback; the packed off-diagonal triangle (and the
``CTQWRHO1`` snapshot format built on it) is out of scope this round
(SURVEY.md section 8f-2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, ConsistencyError, NumericError

WRAP_EDGE_WINDOW = 2
WRAP_EDGE_MASS = 1e-3


@dataclass
class PositionStats:
    mean: float
    variance: float
    wrapped: bool


class DiagonalDensity:
    """diag(<rho>) with provenance; ``purity`` is set when it was requested.

    The diagonal may stay on the device (``device_diag``, the realization sum)
    until it is first read, so sinks that drop snapshots cost no transfer.
    """

    def __init__(self, diag, dim, sample_count, time_tag, purity=None, populations=None,
                 participation_ratio=None, device_diag=None):
        self._diag = None if diag is None else np.asarray(diag, dtype=np.float64)
        self._device_diag = device_diag
        self.dim = int(dim)
        self.sample_count = int(sample_count)
        self.time_tag = float(time_tag)
        self.purity = purity
        self.populations = populations
        self.participation_ratio = participation_ratio

    @property
    def diag(self) -> np.ndarray:
        if self._diag is None:
            self._diag = (self._device_diag / self.sample_count).cpu().numpy()
            self._device_diag = None
        return self._diag

    def diagonal(self) -> np.ndarray:
        return self.diag.astype(np.complex128)

    def trace(self) -> float:
        return float(self.diag.sum())


def joint_distribution(rho: DiagonalDensity) -> np.ndarray:
    return np.asarray(rho.diag, dtype=np.float64).copy()


def populations(rho: DiagonalDensity, space) -> np.ndarray:
    """Particle count per site, sums to m (observables.py:40-56)."""
    if rho.dim != space.dim:
        raise ConsistencyError(f"density dimension {rho.dim} does not match the space ({space.dim})")
    if rho.populations is not None:
        return rho.populations.copy()
    n = space.lattice.n_sites
    grid = np.asarray(rho.diag).reshape((n,) * space.m)
    out = np.zeros(n)
    for p in range(space.m):
        axes = tuple(a for a in range(space.m) if a != p)
        out += grid.sum(axis=axes) if axes else grid
    return out


def position_stats_from_populations(pops: np.ndarray, periodic: bool = True) -> PositionStats:
    """Mean/variance of a uniformly chosen particle's site (observables.py:59-83)."""
    total = pops.sum()
    if total <= 0:
        raise NumericError("population vector sums to zero")
    marginal = pops / total
    x = np.arange(marginal.shape[0], dtype=np.float64)
    mean = float(marginal @ x)
    variance = float(marginal @ (x - mean) ** 2)
    wrapped = False
    if periodic and marginal.shape[0] > 2 * WRAP_EDGE_WINDOW:
        low = marginal[:WRAP_EDGE_WINDOW].sum()
        high = marginal[-WRAP_EDGE_WINDOW:].sum()
        wrapped = bool(low > WRAP_EDGE_MASS and high > WRAP_EDGE_MASS)
    return PositionStats(mean=mean, variance=variance, wrapped=wrapped)


def position_variance(rho: DiagonalDensity, space) -> PositionStats:
    if space.lattice.q != 1:
        raise ConfigurationError("position variance needs a single direction")
    return position_stats_from_populations(populations(rho, space),
                                           space.lattice.boundary == "periodic")


def purity(rho: DiagonalDensity) -> float:
    if rho.purity is None:
        raise ConfigurationError("purity was not computed for this snapshot (select it in observables)")
    return float(rho.purity)


def participation_ratio(rho: DiagonalDensity) -> float:
    """1 / sum (p / sum p)^2 (observables.py:94-101)."""
    if rho.participation_ratio is not None:
        return float(rho.participation_ratio)
    probs = np.asarray(rho.diag, dtype=np.float64)
    denom = float(np.square(probs / probs.sum()).sum())
    if denom <= 0:
        raise NumericError("joint distribution has no weight")
    return 1.0 / denom
