"""Lattice / joint-space description (host side).

Mirrors the reference's geometry API (``hilbert.py:45-173``): ``build_lattice``,
``LatticeTopology``, ``JointSpace``, ``joint_index``, ``joint_positions``.
``build_topology`` differs by design: the reference materialises an int64
neighbour table of ``dim x (2H+1)`` entries (``hilbert.py:278-359``, 40 MiB at
N = 1024); on the B200 path the kernels compute joint neighbours on the fly,
so the "topology" is the stencil descriptor ``LatticeStencil``: nothing for
the periodic nearest-neighbour ring (the fused kernels), and for any other
lattice -- q directions, k_half hops per direction, periodic or open -- the
single-particle move tables of ``_site_move_tables`` (``hilbert.py:189-224``,
N x K entries), which the generic kernels combine per particle.
1 <= m <= 3 particles.
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


def site_coordinates(lattice: LatticeTopology, sites=None) -> np.ndarray:
    """Row-major coordinates of each site (hilbert.py:176-186)."""
    if sites is None:
        sites = np.arange(lattice.n_sites, dtype=np.int64)
    rem = np.asarray(sites, dtype=np.int64).copy()
    coords = np.empty(rem.shape + (lattice.q,), dtype=np.int64)
    for i in range(lattice.q - 1, -1, -1):
        coords[..., i] = rem % lattice.dims[i]
        rem //= lattice.dims[i]
    return coords


def site_move_tables(lattice: LatticeTopology):
    """(pos, neg, directions, distances): targets of every signed
    single-particle move, -1 off an open lattice; slots run direction-major,
    distance 1..k_half within a direction (hilbert.py:189-224)."""
    n, q = lattice.n_sites, lattice.q
    coords = site_coordinates(lattice)
    strides = np.empty(q, dtype=np.int64)
    acc = 1
    for i in range(q - 1, -1, -1):
        strides[i] = acc
        acc *= lattice.dims[i]
    slots = [(i, dist) for i in range(q) for dist in range(1, lattice.k_half[i] + 1)]
    pos = np.empty((n, len(slots)), dtype=np.int64)
    neg = np.empty((n, len(slots)), dtype=np.int64)
    base = np.arange(n, dtype=np.int64)
    periodic = lattice.boundary == BOUNDARY_PERIODIC
    for s, (i, dist) in enumerate(slots):
        c = coords[:, i]
        extent = lattice.dims[i]
        if periodic:
            pos[:, s] = base + ((c + dist) % extent - c) * strides[i]
            neg[:, s] = base + ((c - dist) % extent - c) * strides[i]
        else:
            pos[:, s] = np.where(c + dist < extent, base + dist * strides[i], -1)
            neg[:, s] = np.where(c - dist >= 0, base - dist * strides[i], -1)
    directions = np.array([i for i, _ in slots], dtype=np.int64)
    distances = np.array([d for _, d in slots], dtype=np.int64)
    return pos, neg, directions, distances


@dataclass(frozen=True)
class LatticeStencil:
    """The B200 'topology' of m particles on a lattice.

    Replaces the reference's materialised ``TopologyMatrix``
    (hilbert.py:227-275); ``half`` and ``dim`` keep their meaning.  The
    periodic nearest-neighbour ring (``is_ring``) needs no tables; other
    lattices carry the single-particle move tables.
    """

    space: JointSpace

    @property
    def lattice(self) -> LatticeTopology:
        return self.space.lattice

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
    def K(self) -> int:
        return self.space.lattice.moves_half

    @property
    def n_links(self) -> int:
        return self.n * self.K

    @property
    def is_ring(self) -> bool:
        lat = self.space.lattice
        return lat.q == 1 and lat.k_half == (1,) and lat.boundary == BOUNDARY_PERIODIC

    def move_tables(self):
        """(pos, neg) int arrays (N, K) and the slot directions (K,)."""
        pos, neg, directions, _ = site_move_tables(self.space.lattice)
        return pos, neg, directions


RingStencil = LatticeStencil


def check_supported(space: JointSpace):
    lat = space.lattice
    if not 1 <= space.m <= 3:
        raise ConfigurationError(f"the B200 path supports 1 <= m <= 3 particles (got m={space.m})")
    if lat.q == 1 and lat.k_half == (1,) and lat.boundary == BOUNDARY_PERIODIC and lat.n_sites < 3:
        raise ConfigurationError("ring needs at least 3 sites")
    if lat.n_sites > 2**31 - 1:
        raise CapacityError("lattice too large for 32-bit site tables")


def build_topology(space: JointSpace) -> LatticeStencil:
    check_supported(space)
    return LatticeStencil(space=space)
