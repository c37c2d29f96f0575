"""Lattice / joint-space description (host side).

Mirrors the reference's geometry API (``hilbert.py:45-173``): ``build_lattice``,
``LatticeTopology``, ``JointSpace``, ``joint_index``, ``joint_positions``.
``build_topology`` differs by design: the reference materialises an int64
neighbour table of ``dim x (2H+1)`` entries (``hilbert.py:278-359``, 40 MiB at
N = 1024); on the B200 path the kernels compute neighbours arithmetically, so
the "topology" is just the ring stencil descriptor ``RingStencil``.

Supported by the device path: one periodic direction, nearest-neighbour hops
(q = 1, k_half = 1), 1 <= m <= 3.  Other lattices validate here but are
rejected by ``build_topology`` (next round).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import CapacityError, ConfigurationError

BOUNDARY_PERIODIC = "periodic"
BOUNDARY_OPEN = "open"
MAX_JOINT_DIM = 2**62


@dataclass(frozen=True)
class LatticeTopology:
    dims: tuple
    k_half: tuple
    boundary: str = BOUNDARY_PERIODIC

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        hops = tuple(int(k) for k in self.k_half)
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "k_half", hops)
        if not dims:
            raise ConfigurationError("lattice needs at least one direction")
        if len(hops) != len(dims):
            raise ConfigurationError(f"k_half has {len(hops)} entries for {len(dims)} directions")
        for axis, (extent, k) in enumerate(zip(dims, hops)):
            if extent < 2:
                raise ConfigurationError(f"dims[{axis}] = {extent}; each extent must be >= 2")
            if k < 1:
                raise ConfigurationError(f"k_half[{axis}] = {k}; hop range must be >= 1")
            if 2 * k >= extent:
                raise ConfigurationError(
                    f"k_half[{axis}] = {k} too large for extent {extent}; need 2*k_half < extent"
                )
        if self.boundary not in (BOUNDARY_PERIODIC, BOUNDARY_OPEN):
            raise ConfigurationError(f"boundary {self.boundary!r} not recognized")

    @property
    def q(self) -> int:
        return len(self.dims)

    @property
    def n_sites(self) -> int:
        return math.prod(self.dims)

    @property
    def moves_half(self) -> int:
        return sum(self.k_half)

    @property
    def neighbors_per_site(self) -> int:
        return 2 * self.moves_half


def build_lattice(dims, k_half=None, boundary=BOUNDARY_PERIODIC) -> LatticeTopology:
    dims = tuple(dims)
    return LatticeTopology(dims=dims, k_half=tuple(k_half) if k_half is not None else (1,) * len(dims),
                           boundary=boundary)


@dataclass(frozen=True)
class JointSpace:
    lattice: LatticeTopology
    m: int

    def __post_init__(self):
        object.__setattr__(self, "m", int(self.m))
        if self.m < 1:
            raise ConfigurationError(f"m = {self.m}; need at least one particle")
        if self.dim > MAX_JOINT_DIM:
            raise CapacityError("joint dimension overflows the 64-bit index space")

    @property
    def dim(self) -> int:
        return self.lattice.n_sites ** self.m

    @property
    def moves_half(self) -> int:
        return self.m * self.lattice.moves_half


def joint_index(positions, space: JointSpace):
    """Row-major mixed-radix flattening, particle 0 most significant."""
    pos = np.asarray(positions, dtype=np.int64)
    n = space.lattice.n_sites
    if pos.shape[-1:] != (space.m,):
        raise ConfigurationError(f"expected {space.m} particle positions, got shape {pos.shape}")
    if np.any(pos < 0) or np.any(pos >= n):
        raise ConfigurationError(f"site index out of range [0, {n})")
    out = np.zeros(pos.shape[:-1], dtype=np.int64)
    for p in range(space.m):
        out = out * n + pos[..., p]
    return int(out) if out.ndim == 0 else out


def joint_positions(alpha, space: JointSpace):
    a = np.asarray(alpha, dtype=np.int64)
    n = space.lattice.n_sites
    if np.any(a < 0) or np.any(a >= space.dim):
        raise ConfigurationError(f"joint index out of range [0, {space.dim})")
    out = np.empty(a.shape + (space.m,), dtype=np.int64)
    rem = a.copy()
    for p in reversed(range(space.m)):
        out[..., p] = rem % n
        rem = rem // n
    return out


@dataclass(frozen=True)
class RingStencil:
    """The B200 'topology': m particles on a periodic N-ring, K = 1.

    Replaces the reference's materialised ``TopologyMatrix`` (hilbert.py:227-275);
    ``half`` and ``dim`` keep their meaning.
    """

    space: JointSpace

    @property
    def m(self) -> int:
        return self.space.m

    @property
    def n(self) -> int:
        return self.space.lattice.n_sites

    @property
    def dim(self) -> int:
        return self.space.dim

    @property
    def half(self) -> int:
        return self.space.moves_half

    @property
    def n_links(self) -> int:
        return self.n * self.space.lattice.moves_half


def check_supported(space: JointSpace):
    lat = space.lattice
    if lat.q != 1 or lat.k_half != (1,) or lat.boundary != BOUNDARY_PERIODIC:
        raise ConfigurationError(
            "the B200 path supports one periodic direction with nearest-neighbour hops "
            f"(got dims={lat.dims}, k_half={lat.k_half}, boundary={lat.boundary!r})"
        )
    if not 1 <= space.m <= 3:
        raise ConfigurationError(f"the B200 path supports 1 <= m <= 3 particles (got m={space.m})")
    if lat.n_sites < 3:
        raise ConfigurationError("ring needs at least 3 sites")


def build_topology(space: JointSpace) -> RingStencil:
    check_supported(space)
    return RingStencil(space=space)
