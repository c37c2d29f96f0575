"""Static noise: specification (host) and the per-realization draw (device).

``NoiseSpec`` keeps the reference's fields and validation (noise.py:29-68).
The draw replaces ``init_process`` (noise.py:128-159) for static disorder:
``ctqw_draw_noise`` runs NumPy's SeedSequence -> PCG64 -> ``choice`` per
realization on the GPU, so the values equal
``np.random.default_rng((master_seed, r)).choice(levels, n_links + n_sites)``
bit for bit, laid out ``[links (N) | sites (N)]`` per realization.

Dynamic telegraph noise (``rate > 0``, noise.py:165-206) is not on the B200
path yet; ``run`` rejects it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

NOISE_TUNNELING = "tunneling"
NOISE_ONSITE = "onsite"
NOISE_BOTH = "both"
TARGETS = (NOISE_TUNNELING, NOISE_ONSITE, NOISE_BOTH)


@dataclass(frozen=True)
class NoiseSpec:
    target: str = NOISE_TUNNELING
    levels: tuple = (-0.1, 0.1)
    rate: float = 0.1

    def __post_init__(self):
        object.__setattr__(self, "levels", tuple(float(v) for v in self.levels))
        object.__setattr__(self, "rate", float(self.rate))
        if self.target not in TARGETS:
            raise ConfigurationError(f"noise target {self.target!r} not recognized; use one of {TARGETS}")
        if not self.levels:
            raise ConfigurationError("noise level set is empty")
        if not all(np.isfinite(self.levels)):
            raise ConfigurationError("noise levels must be finite")
        if not np.isfinite(self.rate) or self.rate < 0:
            raise ConfigurationError(f"noise rate {self.rate} must be >= 0")

    @property
    def is_static(self) -> bool:
        return self.rate == 0.0

    @property
    def on_links(self) -> bool:
        return self.target in (NOISE_TUNNELING, NOISE_BOTH)

    @property
    def on_sites(self) -> bool:
        return self.target in (NOISE_ONSITE, NOISE_BOTH)

    def element_counts(self, n_sites: int, moves_half: int = 1):
        """(n_links, n_sites) of the ``[links | sites]`` layout (noise.py:121-125)."""
        return (n_sites * moves_half if self.on_links else 0, n_sites if self.on_sites else 0)


def draw_noise(handle, spec: NoiseSpec, master_seed: int, r0: int, count: int, counts=None):
    """Device tensor ``(count, n_links + n_sites)`` of realizations r0..r0+count-1."""
    import torch

    n_links, n_sites = counts if counts is not None else spec.element_counts(handle.n)
    total = n_links + n_sites
    out = torch.empty((count, max(total, 1)), dtype=torch.float64, device=f"cuda:{handle.device}")
    if total and count:
        if master_seed < 0 or r0 < 0:
            raise ConfigurationError("seeds must be non-negative")
        handle.draw_noise(master_seed, r0, count, spec.levels, total, out)
    return out[:, :total], n_links, n_sites


class StaticNoise:
    """Static disorder of one realization (the ``NoiseProcess`` of rate 0)."""

    __slots__ = ("spec", "n_links", "n_sites", "values", "switch_count", "time")

    def __init__(self, spec, n_links, n_sites, values):
        self.spec = spec
        self.n_links = n_links
        self.n_sites = n_sites
        self.values = values
        self.switch_count = 0
        self.time = 0.0

    @property
    def link_values(self):
        return self.values[: self.n_links]

    @property
    def site_values(self):
        return self.values[self.n_links:]


def init_process(spec: NoiseSpec, where, seed) -> StaticNoise:
    """Static-noise draw for one realization, seed ``(master_seed, r)``.

    Same values as the reference's ``init_process`` for ``rate == 0``.
    """
    from .hamiltonian import handle_for
    from .geometry import JointSpace, LatticeTopology, RingStencil

    if not spec.is_static:
        raise ConfigurationError("dynamic noise (rate > 0) is not on the B200 path")
    if isinstance(where, RingStencil):
        lattice = where.space.lattice
    elif isinstance(where, JointSpace):
        lattice = where.lattice
    elif isinstance(where, LatticeTopology):
        lattice = where
    else:
        raise ConfigurationError(f"cannot take a lattice from {type(where).__name__}")
    if not (isinstance(seed, (tuple, list)) and len(seed) == 2):
        raise ConfigurationError("the device draw takes seeds of the form (master_seed, r)")
    handle = handle_for(1, max(lattice.n_sites, 3), 0.0, 1.0, 0.0, 1.0)
    counts = spec.element_counts(lattice.n_sites, lattice.moves_half)
    vals, nl, ns = draw_noise(handle, spec, int(seed[0]), int(seed[1]), 1, counts)
    return StaticNoise(spec, nl, ns, vals[0].cpu().numpy())
