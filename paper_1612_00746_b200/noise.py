"""Static noise: specification (host) and the per-realization draw (device).

``NoiseSpec`` keeps the reference's fields and validation (noise.py:29-68).
The draw replaces ``init_process`` (noise.py:128-159) for static disorder:
``ctqw_draw_noise`` runs NumPy's SeedSequence -> PCG64 -> ``choice`` per
realization on the GPU, so the values equal
``np.random.default_rng((master_seed, r)).choice(levels, n_links + n_sites)``
bit for bit, laid out ``[links (N) | sites (N)]`` per realization.

Dynamic telegraph noise (``rate > 0``, noise.py:71-206) runs on the device as
well (``csrc/telegraph.cu``): ``ctqw_telegraph_init`` draws the values with
``choice`` and the switch times with ``exponential`` from the same
per-realization streams (NumPy's ziggurat, bit-compatible), and
``ctqw_evolve`` advances the process after every step.  ``init_process`` /
``advance`` below expose one realization's process with the reference's API.
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


@dataclass
class NoiseDelta:
    """Report of one advance window (noise.py:71-78)."""

    changed: bool
    links: np.ndarray
    sites: np.ndarray
    switches: int


class TelegraphProcess:
    """Telegraph state of one realization (the reference's ``NoiseProcess``
    for ``rate > 0``), held on the device by a one-realization handle."""

    def __init__(self, spec, n_links, n_sites, handle):
        self.spec = spec
        self.n_links = n_links
        self.n_sites = n_sites
        self._h = handle
        self._sync()

    def _sync(self):
        import torch

        total = self.n_links + self.n_sites
        dev = f"cuda:{self._h.device}"
        vals = torch.empty((1, max(total, 1)), dtype=torch.float64, device=dev)
        nxt = torch.empty_like(vals)
        times, sw = self._h.telegraph_read(1, vals if total else None, nxt if total else None)
        self.values = vals[0, :total].cpu().numpy()
        self.next_switch = nxt[0, :total].cpu().numpy()
        self.time = float(times[0])
        self.switch_count = int(sw[0])

    @property
    def link_values(self):
        return self.values[: self.n_links]

    @property
    def site_values(self):
        return self.values[self.n_links:]


def advance(process, dt: float) -> NoiseDelta:
    """Advance over ``(time, time + dt]`` (noise.py:165-206); a static process
    only moves its clock."""
    if dt < 0:
        raise ConfigurationError(f"advance window dt = {dt} must be >= 0")
    empty = np.empty(0, dtype=np.int64)
    if isinstance(process, StaticNoise):
        process.time += dt
        return NoiseDelta(False, empty, empty, 0)
    before = process.values.copy()
    switches0 = process.switch_count
    process._h.telegraph_advance(1, dt)
    process._sync()
    changed = process.values != before
    links = np.nonzero(changed[: process.n_links])[0]
    sites = np.nonzero(changed[process.n_links:])[0]
    return NoiseDelta(bool(links.size or sites.size), links, sites, process.switch_count - switches0)


def init_process(spec: NoiseSpec, where, seed):
    """Noise draw for one realization, seed ``(master_seed, r)``.

    Same values (and, for ``rate > 0``, switch times) as the reference's
    ``init_process``.
    """
    from .hamiltonian import handle_for
    from .geometry import JointSpace, LatticeTopology, RingStencil

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
    counts = spec.element_counts(lattice.n_sites, lattice.moves_half)
    if int(seed[0]) < 0 or int(seed[1]) < 0:
        raise ConfigurationError("seeds must be non-negative")
    if not spec.is_static:
        from .geometry import site_move_tables
        from .native import Handle

        n = lattice.n_sites
        ring = lattice.q == 1 and lattice.k_half == (1,) and lattice.boundary == "periodic" and n >= 3
        tables = None
        if not ring:
            pos, neg, _, _ = site_move_tables(lattice)
            tables = (pos, neg, np.ones(pos.shape[1]))
        handle = Handle(1, n, 0.0, 1.0, 0.0, 1.0, _device(), lattice=tables)
        handle.telegraph_init(int(seed[0]), int(seed[1]), 1, spec.levels, counts[0], counts[1], spec.rate)
        return TelegraphProcess(spec, counts[0], counts[1], handle)
    handle = handle_for(1, max(lattice.n_sites, 3), 0.0, 1.0, 0.0, 1.0)
    vals, nl, ns = draw_noise(handle, spec, int(seed[0]), int(seed[1]), 1, counts)
    return StaticNoise(spec, nl, ns, vals[0].cpu().numpy())


def _device() -> int:
    import torch

    if not torch.cuda.is_available():
        from .errors import NativeError

        raise NativeError("no CUDA device: the B200 path has no CPU fallback")
    return torch.cuda.current_device()
