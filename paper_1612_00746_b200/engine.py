"""Ensemble run: the drop-in replacement of ``ctqw.ensemble.run`` for static noise.

Keeps the reference's configuration and output API -- ``RunConfig``,
``InitialStateSpec``, ``build_initial_state``, ``OutputSinks`` /
``MemorySinks``, ``RunReport``, ``estimate_memory``, ``run(config, sinks)``
(ensemble.py:122-804) -- and replaces its engine:

* the realization stack lives in HBM for the whole run (one contiguous shard
  per GPU when torch.distributed is initialised, see ``sharding``);
* the noise draw and the stencil coefficients are generated on the device;
* each segment between collection points is one ``ctqw_evolve`` call (the
  reference's ``_evolve_segment``, ensemble.py:445-558) -- fused step kernels
  with the per-step norm policy on the device;
* at each collection point the diagonal of the ensemble-averaged density
  matrix is summed on the device, all-reduced across GPUs, and reduced to
  the observable rows in the reference's row order (ensemble.py:609-632).

Results match the reference's ``run(..., precision="double")`` to rounding
(1e-10 relative is the acceptance bar; bit-identical between renormalisation
events in ``exact`` mode).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import numpy as np

from . import sharding
from .errors import CapacityError, ConfigurationError, MemoryBudgetError, NormFailureError, NumericError
from .geometry import JointSpace, build_topology, joint_index
from .hamiltonian import CouplingModel, handle_for, model_handle
from .noise import NoiseSpec, draw_noise
from .observables import DiagonalDensity, position_stats_from_populations
from .profiling import (
    STAGE_DENSITY,
    STAGE_EVOLUTION,
    STAGE_HAMILTONIAN,
    STAGE_INITIALIZATION,
    StageProfile,
)
from .propagators import BACKEND_EIGEN, NormEvent, StepperConfig

PRECISION_SINGLE = "single"
PRECISION_DOUBLE = "double"
PRECISIONS = (PRECISION_SINGLE, PRECISION_DOUBLE)

KIND_AUTO = "auto"
KIND_SINGLE_SITE = "single_site"
KIND_PRODUCT = "product"
KIND_SYMMETRIZED = "symmetrized_pair"
KIND_ANTISYMMETRIZED = "antisymmetrized_pair"
KIND_CUSTOM = "custom_vector"
STATE_KINDS = (KIND_AUTO, KIND_SINGLE_SITE, KIND_PRODUCT, KIND_SYMMETRIZED,
               KIND_ANTISYMMETRIZED, KIND_CUSTOM)

OBS_POPULATIONS = "populations"
OBS_POSITION = "position_mean_variance"
OBS_PURITY = "purity"
OBS_PARTICIPATION = "participation_ratio"
OBS_JOINT = "joint_distribution"
KNOWN_OBSERVABLES = (OBS_POPULATIONS, OBS_POSITION, OBS_PURITY, OBS_PARTICIPATION, OBS_JOINT)

WORKERS_ENV = "CTQW_WORKERS"
MAX_EVENTS_PER_SEGMENT = 100
# sum_{r,s} |<psi_r|psi_s>|^2 costs R^2 * D complex multiply-adds per snapshot
PURITY_WORK_CAP = 2**40
PURITY_GATHER_CAP = 2 * 2**30


@dataclass(frozen=True)
class InitialStateSpec:
    kind: str = KIND_AUTO
    positions: tuple | None = None
    amplitudes: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in STATE_KINDS:
            raise ConfigurationError(f"initial state kind {self.kind!r} not recognized; use one of {STATE_KINDS}")
        if self.positions is not None:
            object.__setattr__(self, "positions", tuple(int(x) for x in self.positions))


# pinned host buffers for the initial-state upload, by dimension: [tensor,
# nonzero indices written last (None: unknown / dense), event of the last
# upload from it]
_PINNED: dict = {}


def _pinned_initial(dim: int) -> list:
    import torch

    pool = _PINNED.get(dim)
    if pool:
        buf = pool.pop()
        if buf[2] is not None:
            buf[2].synchronize()
        return buf
    return [torch.empty(dim, dtype=torch.complex128, pin_memory=torch.cuda.is_available()), None, None]


def _fill_pinned(buf: list, entries) -> None:
    arr = buf[0].numpy()
    if isinstance(entries, np.ndarray):
        arr[:] = entries
        buf[1] = None
        return
    if buf[1] is None:
        arr[:] = 0
    else:
        arr[list(buf[1])] = 0
    for k, v in entries.items():
        arr[k] = v
    buf[1] = tuple(entries.keys())


class _Entries(dict):
    """The nonzero entries of a closed-form initial state (psi[index] = value)."""


def build_initial_state(spec: InitialStateSpec, space: JointSpace) -> np.ndarray:
    """Unit-norm joint state (ensemble.py:147-216), complex128 on the host."""
    entries = initial_state_entries(spec, space)
    if isinstance(entries, np.ndarray):
        return entries
    psi = np.zeros(space.dim, dtype=np.complex128)
    for k, v in entries.items():
        psi[k] = v
    return psi


def initial_state_entries(spec: InitialStateSpec, space: JointSpace):
    """build_initial_state's state: the dense vector for custom amplitudes,
    else its few nonzero entries (an ``_Entries`` dict), so a pinned upload
    buffer can be updated in place instead of rewritten."""
    n, m = space.lattice.n_sites, space.m
    kind = spec.kind
    if kind == KIND_AUTO:
        kind = KIND_SINGLE_SITE if m == 1 else KIND_PRODUCT
    if kind == KIND_CUSTOM:
        if spec.amplitudes is None:
            raise ConfigurationError("custom_vector needs explicit amplitudes")
        amps = np.asarray(spec.amplitudes, dtype=np.complex128)
        if amps.shape != (space.dim,):
            raise ConfigurationError(f"custom vector has shape {amps.shape}, expected ({space.dim},)")
        norm = np.linalg.norm(amps)
        if norm == 0:
            raise ConfigurationError("custom vector has zero norm")
        return amps / norm
    psi = _Entries()
    if kind == KIND_SINGLE_SITE:
        if m != 1:
            raise ConfigurationError("single_site describes one particle only")
        pos = spec.positions if spec.positions is not None else ((n - 1) // 2,)
        if len(pos) != 1:
            raise ConfigurationError("single_site takes exactly one position")
        psi[joint_index(pos, space)] = 1.0
        return psi
    if kind == KIND_PRODUCT:
        pos = spec.positions
        if pos is None:
            if m > n:
                raise ConfigurationError(f"no default product placement for {m} particles on {n} sites")
            first = (n - m) // 2
            pos = tuple(range(first, first + m))
        if len(pos) != m:
            raise ConfigurationError(f"product state needs {m} positions, got {len(pos)}")
        psi[joint_index(pos, space)] = 1.0
        return psi
    if m != 2:
        raise ConfigurationError(f"{kind} requires exactly two particles")
    pos = spec.positions
    if pos is None:
        first = (n - 2) // 2
        pos = (first, first + 1)
    if len(pos) != 2:
        raise ConfigurationError(f"{kind} takes exactly two positions")
    x, y = pos
    if x == y:
        if kind == KIND_ANTISYMMETRIZED:
            raise ConfigurationError("antisymmetrized pair on one site vanishes identically")
        psi[joint_index((x, x), space)] = 1.0
        return psi
    amp = 1.0 / np.sqrt(2.0)
    psi[joint_index((x, y), space)] = amp
    psi[joint_index((y, x), space)] = (-1.0 if kind == KIND_ANTISYMMETRIZED else 1.0) * amp
    return psi


@dataclass(frozen=True)
class RunConfig:
    """The reference's run description (ensemble.py:219-294) plus two B200 knobs.

    ``exact``: reference operation order without FMA (bit-identical between
    renormalisations) vs FMA-contracted stencil.  ``device``: CUDA device
    index (default: the current device / LOCAL_RANK).
    """

    space: JointSpace
    model: CouplingModel = CouplingModel()
    noise: NoiseSpec = NoiseSpec()
    stepper: StepperConfig = StepperConfig()
    initial: InitialStateSpec = InitialStateSpec()
    realizations: int = 1000
    steps: int = 1500
    post_rate: int = 10
    master_seed: int = 1234
    workers: int = 0
    precision: str = PRECISION_SINGLE
    observables: tuple | None = None
    memory_budget: int = 4 * 2**30
    dense_cap: int = 4096
    exact: bool = True
    device: int | None = None

    def __post_init__(self):
        if self.realizations < 1:
            raise ConfigurationError(f"realizations = {self.realizations} must be >= 1")
        if self.steps < 0:
            raise ConfigurationError(f"steps = {self.steps} must be >= 0")
        if self.post_rate < 1:
            raise ConfigurationError(f"post_rate = {self.post_rate} must be >= 1")
        if self.steps > 0 and self.post_rate > self.steps:
            raise ConfigurationError(f"post_rate = {self.post_rate} exceeds steps = {self.steps}")
        if self.workers < 0:
            raise ConfigurationError(f"workers = {self.workers} must be >= 0")
        if self.precision not in PRECISIONS:
            raise ConfigurationError(f"precision {self.precision!r} not recognized; use one of {PRECISIONS}")
        if self.memory_budget <= 0:
            raise ConfigurationError("memory_budget must be positive")
        if self.observables is None:
            names = [OBS_POPULATIONS, OBS_PURITY, OBS_PARTICIPATION]
            if self.space.lattice.q == 1:
                names.insert(1, OBS_POSITION)
            object.__setattr__(self, "observables", tuple(names))
        else:
            object.__setattr__(self, "observables", tuple(self.observables))
            for name in self.observables:
                if name not in KNOWN_OBSERVABLES:
                    raise ConfigurationError(f"observable {name!r} not recognized; use one of {KNOWN_OBSERVABLES}")
            if not self.observables:
                raise ConfigurationError("observable selection is empty")
        if OBS_POSITION in self.observables and self.space.lattice.q != 1:
            raise ConfigurationError("position_mean_variance is only defined on one-direction lattices")

    @property
    def dtype(self):
        return np.complex128

    @property
    def schedule(self) -> tuple:
        if self.steps == 0:
            return (0,)
        pts = list(range(self.post_rate, self.steps + 1, self.post_rate))
        if pts[-1] != self.steps:
            pts.append(self.steps)
        return tuple(pts)


def kernel_path(config: RunConfig) -> str:
    """The step-kernel family ``ctqw_evolve`` will run for this configuration
    (the dispatch of csrc/api.cu): "resident", "plane3", "band4", "tile" or
    "generic"."""
    lat = config.space.lattice
    st = config.stepper
    m, n = config.space.m, lat.n_sites
    ring = lat.q == 1 and lat.k_half == (1,) and lat.boundary == "periodic" and n >= 3
    pinned = os.environ.get("CTQW_STREAM", "")
    order_ok = st.backend == "rk4" or 1 <= st.taylor_order <= 4
    if not ring or pinned == "generic":
        return "generic"
    if m == 2 and n <= 64 and pinned == "" and (st.backend == "rk4" or st.taylor_order <= 16):
        return "resident"
    if m == 3 and n == 128 and (st.backend == "rk4" or st.taylor_order == 4) and pinned in ("", "plane3"):
        return "plane3"
    if m == 2 and order_ok and n % 4 == 0 and n >= 16 and n // 4 <= 256 and pinned in ("", "band4"):
        return "band4"
    if m == 2 and n > 64 and (st.backend == "rk4" or st.taylor_order <= 4) and pinned in ("", "tile", "band4"):
        return "tile"
    return "generic"


# full state stacks each path keeps on the device (caller's + library's)
_PATH_BUFFERS = {"resident": 1, "plane3": 1, "band4": 2, "tile": 2, "generic": 4}


def estimate_memory(config: RunConfig, world: int = 1) -> dict:
    """Device working set per GPU in bytes (keys of ensemble.py:297-323).

    States are complex128 regardless of ``precision``.  The number of full
    state stacks follows the kernel path (``kernel_path``): one for the
    in-place resident and plane3 kernels, two for the ping-pong streaming
    kernels, four for the generic per-application path (stack, work and two
    library term buffers).  Plus O(N) coefficients per realization instead of
    the (D, H+1) value table, the per-realization norm statistics and event
    buffers, the telegraph process state for dynamic noise, no topology
    table, and the diagonal (limbs, sum, joint) instead of the packed rho.
    """
    space = config.space
    dim = space.dim
    n = space.lattice.n_sites
    r_local = -(-config.realizations // world)
    state = r_local * dim * 16
    path = kernel_path(config)
    buffers = _PATH_BUFFERS[path]
    k_links = n * sum(space.lattice.k_half)
    coeff = r_local * (k_links + n) * 8
    stats = r_local * (48 + 100 * 16 + 8 + 32 * 8)  # RealStat, EventRec[100], rescale, norm partials
    noise_state = 0
    if not config.noise.is_static:
        total = k_links + n
        noise_state = r_local * (total * (8 + 8 + 12) + 64)  # values, switch times, due lists, generator
    # the collection buffers of one group of points on the batched path
    # (_fused_groups): int64 limbs [P][3][D] + diagonal [P][D], P points per group
    points = max(1, min(len(config.schedule), FUSED_ACC_BYTES // (24 * dim),
                        max(1, FUSED_CALL_STEPS // max(config.post_rate, 1))))
    density = points * dim * (24 + 8) + dim * 8  # + the joint distribution
    if OBS_PURITY in config.observables:  # the states at every point of a group (enqueue_group)
        snap = points * r_local * dim * 16
        density += snap if snap <= SNAPSHOT_BYTES else 0
    return {
        "joint_dim": dim,
        "itemsize": 16,
        "kernel_path": path,
        "state_buffers": buffers,
        "state_bytes": buffers * state,
        "hamiltonian_bytes": coeff + noise_state,
        "statistics_bytes": stats,
        "topology_bytes": 0,
        "density_bytes": density,
        "total_bytes": buffers * state + coeff + noise_state + stats + density,
    }


def marches_in_place(config: RunConfig) -> bool:
    """The resident (m = 2, N <= 64) and m = 3, N = 128 cluster kernels update
    the states in place: one buffer (so twice the realizations per GPU --
    configs[4])."""
    return kernel_path(config) in ("resident", "plane3")


class OutputSinks:
    def observable_rows(self, time_tag: float, rows):
        pass

    def density_snapshot(self, rho, step: int):
        pass

    def norm_events(self, events):
        pass

    def message(self, text: str):
        pass

    def finish(self, report):
        pass


class MemorySinks(OutputSinks):
    """The reference's MemorySinks (ensemble.py:345-373).  ``dense=True`` asks
    ``run`` for the dense packed <rho> (``density.DensityMatrix``) at every
    collection point instead of its diagonal (``DiagonalDensity``)."""

    def __init__(self, keep_densities: bool = True, max_events: int = 1000, dense: bool = False):
        self.keep_densities = keep_densities
        self.dense_density = bool(dense) and keep_densities
        self.max_events = max_events
        self.rows = []
        self.densities = []
        self.events = []
        self.messages = []
        self.report = None

    def observable_rows(self, time_tag, rows):
        self.rows.extend((time_tag, name, idx, value) for name, idx, value in rows)

    def density_snapshot(self, rho, step):
        if self.keep_densities:
            self.densities.append(rho)

    def norm_events(self, events):
        room = self.max_events - len(self.events)
        if room > 0:
            self.events.extend(events[:room])

    def message(self, text):
        self.messages.append(text)

    def finish(self, report):
        self.report = report


@dataclass
class RunReport:
    config: RunConfig
    profile: StageProfile
    io_seconds: float
    wall_seconds: float
    workers: int
    snapshots: int
    max_norm_deviation: float
    norm_corrections: int
    norm_events: int
    switch_count: int
    memory_estimate: dict


def _default_device():
    import torch

    if not torch.cuda.is_available():
        from .errors import NativeError

        raise NativeError("no CUDA device: the B200 path has no CPU fallback")
    env = os.environ.get("LOCAL_RANK")
    if env is not None and torch.distributed.is_initialized():
        return int(env) % torch.cuda.device_count()
    return torch.cuda.current_device()


class EnsembleState:
    """Device-resident shard of one run: noise, coefficients, states.

    Exposed so benchmarks and tests can drive segments directly; ``run``
    is the public entry point.
    """

    def __init__(self, config: RunConfig, device: int, lo: int, hi: int):
        import torch

        self.config = config
        self.lo, self.hi = lo, hi
        self.count = hi - lo
        space = config.space
        self.topology = build_topology(space)
        model = config.model
        # a private handle: this ensemble's coefficient rows and telegraph
        # process stay bound for the whole run, whatever the caller does with
        # the cached handles of the single-step API in between
        self.handle = model_handle(self.topology, model, device=device, private=True)
        self.dev = torch.device(f"cuda:{device}")
        n = space.lattice.n_sites
        self.dynamic = not config.noise.is_static
        if self.dynamic:
            # telegraph process on the device (noise.py:128-206): values and
            # switch times drawn from the same NumPy-compatible streams, advanced
            # by ctqw_evolve after every step
            n_links, n_sites = config.noise.element_counts(n, space.lattice.moves_half)
            if config.master_seed < 0 or lo < 0:
                raise ConfigurationError("seeds must be non-negative")
            self.handle.telegraph_init(config.master_seed, lo, self.count, config.noise.levels, n_links,
                                       n_sites, config.noise.rate)
            noise = None
        else:
            noise, n_links, n_sites = draw_noise(self.handle, config.noise, config.master_seed, lo,
                                                 self.count,
                                                 config.noise.element_counts(n, space.lattice.moves_half))
        self.n_links, self.n_sites = n_links, n_sites
        self.hop = torch.empty((max(self.count, 1), self.topology.n_links), dtype=torch.float64, device=self.dev)
        self.site = (torch.empty((max(self.count, 1), n), dtype=torch.float64, device=self.dev)
                     if n_sites else None)
        if self.count:
            if self.dynamic:
                self.handle.build_coefficients_from_ptr(self.handle.telegraph_values_ptr(), self.count, n_links,
                                                        n_sites, self.hop, self.site)
            else:
                self.handle.build_coefficients(noise.contiguous(), self.count, n_links, n_sites,
                                               self.hop, self.site)
        self.handle.bind(self.hop, self.site, self.count, self.topology.n_links)
        self.handle.telegraph_enable(self.dynamic and self.count > 0)
        del noise
        # the initial state goes up from a pooled pinned buffer (asynchronous
        # copy on the stream); closed-form states only rewrite their few
        # nonzero entries in it
        self._pinned = _pinned_initial(space.dim)
        _fill_pinned(self._pinned, initial_state_entries(config.initial, space))
        self.psi0 = torch.empty(space.dim, dtype=torch.complex128, device=self.dev)
        self.psi0.copy_(self._pinned[0], non_blocking=True)
        self._pinned[2] = torch.cuda.Event()
        self._pinned[2].record(torch.cuda.current_stream(self.dev))  # the buffer is rewritten only after this copy
        self.psi = torch.empty((max(self.count, 1), space.dim), dtype=torch.complex128, device=self.dev)
        # one buffer when the step kernel marches in place (the library keeps a
        # second one itself if another path ends up running)
        self.work = self.psi if marches_in_place(config) else torch.empty_like(self.psi)
        # every realization starts from psi0: handed to the library lazily
        # (ctqw_set_initial), so the first step reads the one state instead of
        # a materialised R x D stack; anything that reads the states before
        # the first step materialises them (_materialise)
        self._initial_pending = False
        if self.count:
            self.handle.set_initial(self.psi0)
            self._initial_pending = True
        self.stepper = config.stepper.native(config.exact)

    def _materialise(self):
        if self._initial_pending:
            self.handle.fill_states(self.psi, self.count, self.psi0)
            self._initial_pending = False

    def evolve(self, first_step: int, n_steps: int):
        """Enqueue ``n_steps`` steps (asynchronous)."""
        if self.count == 0 or n_steps == 0:
            self._materialise()
            self.handle.evolve(self.psi, self.work, 0, first_step, 0, self.stepper)
            return
        swapped = self.handle.evolve(self.psi, self.work, self.count, first_step, n_steps,
                                     self.stepper)
        self._initial_pending = False
        if swapped and self.work is not self.psi:
            self.psi, self.work = self.work, self.psi

    def evolve_observe(self, first_step: int, n_steps: int, post_rate: int, acc, keep_stats: bool = False,
                       snap=None):
        """Enqueue ``n_steps`` steps and the collection points among them
        (every ``post_rate``-th step from ``first_step``, and the last one): acc[P][3][D]
        int64 receives each point's exact limbs of sum_r |psi_r|^2
        (ctqw_evolve_observe; fused into the step kernel on the resident
        N = 64 path)."""
        if self.count == 0:
            acc.zero_()
            self.handle.evolve(self.psi, self.work, 0, first_step, 0, self.stepper)  # empty statistics
            return
        swapped = self.handle.evolve_observe(self.psi, self.work, self.count, first_step, n_steps, post_rate, acc,
                                             self.stepper, keep_stats, snap)
        self._initial_pending = False
        if swapped and self.work is not self.psi:
            self.psi, self.work = self.work, self.psi

    def segment_events(self, step_lo: int, step_hi: int) -> list:
        st = self.handle.segment_events(self.lo, step_lo, step_hi)
        return [(e.deviation, bool(e.corrected), int(e.realization), int(e.step)) for e in st.events[: st.n_events]]

    def stats(self) -> dict:
        st = self.handle.segment_stats(self.lo)
        events = [(e.deviation, bool(e.corrected), int(e.realization), int(e.step))
                  for e in st.events[: st.n_events]]
        failure = None
        if st.failed:
            failure = (float(st.fail_deviation), int(st.fail_realization), int(st.fail_step))
        return {"event_count": int(st.event_count), "corrections": int(st.corrections),
                "max_deviation": float(st.max_deviation), "events": events, "failure": failure}

    def switch_count(self) -> int:
        """Telegraph switches processed so far in this shard (NoiseProcess.switch_count summed)."""
        if not self.dynamic or self.count == 0:
            return 0
        return int(sum(self.handle.telegraph_read(self.count)[1]))

    def diagonal_sum(self, out):
        self._materialise()
        self.handle.observe_diag(self.psi, self.count, out, accumulate=False)
        return out

    def diagonal_limbs(self, acc):
        """acc[3][D] int64 = exact fixed-point limbs of this shard's sum_r |psi_r|^2."""
        self._materialise()
        self.handle.observe_diag_fixed(self.psi, self.count, acc, accumulate=False)
        return acc

    def states(self):
        self._materialise()
        return self.psi[: self.count]

    def release(self):
        """Give the state buffers and the handle back now (not whenever the
        garbage collector gets to this object): a following run() then
        reuses the memory instead of mapping fresh tens of GiB."""
        from .hamiltonian import release_private_handle

        self.psi = self.work = self.psi0 = self.hop = self.site = None
        if self.handle is not None:
            release_private_handle(self.handle)
            self.handle = None
        if getattr(self, "_pinned", None) is not None:
            _PINNED.setdefault(self._pinned[0].numel(), []).append(self._pinned)
            self._pinned = None


def _observable_rows(config, pops, pr, purity, joint):
    rows = []
    for name in config.observables:
        if name == OBS_POPULATIONS:
            rows.extend(("population", i, float(v)) for i, v in enumerate(pops))
        elif name == OBS_POSITION:
            st = position_stats_from_populations(pops, config.space.lattice.boundary == "periodic")
            rows.append(("position_mean", 0, st.mean))
            rows.append(("position_variance", 0, st.variance))
            rows.append(("position_wrapped", 0, float(st.wrapped)))
        elif name == OBS_PURITY:
            rows.append(("purity", 0, purity))
        elif name == OBS_PARTICIPATION:
            rows.append(("participation_ratio", 0, pr))
        elif name == OBS_JOINT:
            rows.extend(("joint_probability", i, float(v)) for i, v in enumerate(joint))
    return rows


def _dense_snapshot(config, ens, group, time_tag):
    """Packed <rho> over all ranks (density.py:91-96): each rank's Gram sum of
    its shard, all-reduced, divided by R."""
    import torch

    from .density import DensityMatrix, packed_density_device, packed_length

    dim = config.space.dim
    if ens.count:
        part = packed_density_device(ens.states(), ens.count, scale=1.0)
    else:
        part = torch.zeros(packed_length(dim), dtype=torch.complex128, device=ens.dev)
    if group is not None and sharding._collective(group):
        import torch.distributed as dist

        real = torch.view_as_real(part).contiguous()
        dist.all_reduce(real, group=group)
        part = torch.view_as_complex(real)
    return DensityMatrix(None, dim=dim, sample_count=config.realizations, time_tag=float(time_tag),
                         device_packed=part * (1.0 / config.realizations))


class PendingObservables:
    """Observables of one collection point, enqueued on the device.

    Everything the rows need is packed into one small device buffer
    ``[populations (N) | sum p, sum p^2, PR | sum |<r|s>|^2]`` so reading the
    rows costs one device-to-host copy; the diagonal and the joint
    distribution stay on the device until asked for.
    """

    def __init__(self, config, packed, diag, joint, n):
        self.config = config
        self.packed = packed
        self.diag_dev = diag
        self.joint_dev = joint
        self.n = n
        self._host = None

    def host(self):
        if self._host is None:
            self._host = self.packed.cpu().numpy()
        return self._host

    @property
    def populations(self):
        return self.host()[: self.n].copy()

    @property
    def participation_ratio(self):
        h = self.host()
        s2 = float(h[self.n + 1])
        if s2 <= 0.0:  # NaN passes through (a blown-up state), as in observables.py:94-101
            raise NumericError("joint distribution has no weight")
        return float(h[self.n + 2])

    @property
    def purity(self):
        if OBS_PURITY not in self.config.observables:
            return None
        return float(self.host()[self.n + 3]) / float(self.config.realizations) ** 2

    def joint(self):
        return self.joint_dev.cpu().numpy() if self.joint_dev is not None else None


def collect_observables_async(config, ens: EnsembleState, group=None, want_joint=None):
    """Enqueue one collection point (diagonal sum, all-reduce, reductions, purity)."""
    import torch

    space = config.space
    dim = space.dim
    n = space.lattice.n_sites
    # exact int64 limbs: the all-reduce (and so every row) is bitwise the same
    # for any number of ranks and any split of the realizations
    acc = torch.empty((3, dim), dtype=torch.int64, device=ens.dev)
    ens.diagonal_limbs(acc)
    sharding.allreduce_sum_(acc, group)
    diag = torch.empty(dim, dtype=torch.float64, device=ens.dev)
    ens.handle.fixed_to_double(acc, diag)
    packed = torch.zeros(n + 4, dtype=torch.float64, device=ens.dev)
    need_joint = OBS_JOINT in config.observables if want_joint is None else want_joint
    joint = torch.empty(dim, dtype=torch.float64, device=ens.dev) if need_joint else None
    ens.handle.observe_reduce(diag, float(config.realizations), packed[:n], packed[n:n + 3], joint)
    if OBS_PURITY in config.observables:
        states = sharding.gather_states(ens.states(), group)
        ens.handle.overlap_sumsq(states, states.shape[0], states, states.shape[0], packed[n + 3:])
    return PendingObservables(config, packed, diag, joint, n)


def collect_observables(config, ens: EnsembleState, group=None, want_joint=None):
    """Device reduction of one collection point -> (pops, pr, purity, joint, diag)."""
    obs = collect_observables_async(config, ens, group, want_joint)
    return obs.populations, obs.participation_ratio, obs.purity, obs.joint(), obs.diag_dev


# steps per evolve_observe call in run(): each realization logs at most one
# event per step and keeps CTQW_MAX_EVENTS of them, so with calls of at most
# this many steps every segment's event list can be rebuilt exactly
FUSED_CALL_STEPS = MAX_EVENTS_PER_SEGMENT
FUSED_ACC_BYTES = 512 * 2**20
SNAPSHOT_BYTES = 1024 * 2**20  # states kept per group of points for purity


def fused_collection_ok(config: RunConfig, sinks, world: int) -> bool:
    """run() takes the batched path (ctqw_evolve_observe + ctqw_observe_points:
    one call per group of collection points instead of a segment call, a
    limb pass and four reductions per point, one host synchronisation and,
    sharded, one limb all-reduce plus two statistics all-gathers per group)
    unless the sink wants the dense rho.
    With purity, which needs the states at every point, the group issues one
    evolve_observe per segment plus the overlap kernel, still without a host
    synchronisation per point."""
    return not getattr(sinks, "dense_density", False) and config.steps > 0


def _fused_groups(config: RunConfig):
    """Consecutive schedule points grouped into evolve_observe calls."""
    dim = config.space.dim
    max_points = max(1, FUSED_ACC_BYTES // (24 * dim))
    groups, cur, start = [], [], 0
    for t in config.schedule:
        if cur and (t - start > FUSED_CALL_STEPS or len(cur) >= max_points):
            groups.append((start, cur))
            start, cur = cur[-1], []
        cur.append(t)
    if cur:
        groups.append((start, cur))
    return groups


def enqueue_group(config: RunConfig, ens, start: int, targets, group=None):
    """Enqueue one group of collection points on the batched path (no host
    synchronisation): the steps from ``start`` to ``targets[-1]`` with the
    exact diag limbs at every target (ctqw_evolve_observe; per segment, with
    the overlap kernel, when purity is requested), one all-reduce of the
    limbs, and ctqw_observe_points.  Returns device buffers (out[P][N+3],
    diag[P][D], purity sums[P] or None)."""
    import torch

    n, dim = config.space.lattice.n_sites, config.space.dim
    npts = len(targets)
    acc = torch.empty((npts, 3, dim), dtype=torch.int64, device=ens.dev)
    pur = None
    if OBS_PURITY in config.observables:
        pur = torch.empty(npts, dtype=torch.float64, device=ens.dev)
        if npts * max(ens.count, 1) * dim * 16 <= SNAPSHOT_BYTES and ens.count:
            # the states at every point written by the same call (the resident
            # kernel stores them from registers), then the overlap sums of all
            # points in one launch set (one pass per point across ranks, which
            # gathers every rank's states)
            snap = torch.empty((npts, ens.count, dim), dtype=torch.complex128, device=ens.dev)
            ens.evolve_observe(start, targets[-1] - start, config.post_rate, acc, snap=snap)
            if sharding.is_collective(group):
                for k in range(npts):
                    st = sharding.gather_states(snap[k], group)
                    ens.handle.overlap_sumsq(st, st.shape[0], st, st.shape[0], pur[k:k + 1])
            else:
                ens.handle.overlap_sumsq_points(snap, ens.count, npts, ens.count * dim, pur)
        else:
            prev = start
            for k, t in enumerate(targets):
                ens.evolve_observe(prev, t - prev, t - prev, acc[k:k + 1], keep_stats=k > 0)
                st = sharding.gather_states(ens.states(), group)
                ens.handle.overlap_sumsq(st, st.shape[0], st, st.shape[0], pur[k:k + 1])
                prev = t
    else:
        ens.evolve_observe(start, targets[-1] - start, config.post_rate, acc)
    sharding.allreduce_sum_(acc, group)
    out = torch.empty((npts, n + 3), dtype=torch.float64, device=ens.dev)
    diag = torch.empty((npts, dim), dtype=torch.float64, device=ens.dev)
    ens.handle.observe_points(acc, npts, float(config.realizations), out, diag)
    return out, diag, pur


def _run_fused(config, ens, sinks, emit, profile, clock, group=None):
    """The schedule loop of run() on the batched path; same rows, events,
    counters and failure semantics as the per-segment loop, for any number
    of ranks."""
    import torch

    n = config.space.lattice.n_sites
    dim = config.space.dim
    want_joint = OBS_JOINT in config.observables
    want_purity = OBS_PURITY in config.observables
    totals = {"corrections": 0, "events": 0, "max_dev": 0.0, "snapshots": 0}
    for start, targets in _fused_groups(config):
        t0 = clock()
        out, diag, pur = enqueue_group(config, ens, start, targets, group)
        local = sharding.merge_segment_stats(sharding.gather_stats(ens.stats(), group))  # synchronises
        host = out.cpu().numpy()
        seg_events = None
        if local["event_count"]:
            prevs = [start] + list(targets[:-1])
            seg_events = sharding.gather_segment_events(
                [ens.segment_events(lo, hi) if ens.count else [] for lo, hi in zip(prevs, targets)], group)
        pur_host = pur.cpu().numpy() if pur is not None else None
        profile.add(STAGE_EVOLUTION, clock() - t0, calls=config.realizations * (targets[-1] - start))
        profile.add(STAGE_HAMILTONIAN, 0.0, calls=config.realizations * (targets[-1] - start))
        fail = local["failure"]
        previous = start
        for k, target in enumerate(targets):
            if fail is not None and fail[2] <= target:
                dev, real, step = fail
                emit(sinks.message, f"aborted: norm deviation {dev:.3e} at realization {real}, step {step}; "
                                    f"reduce the time step")
                ens.release()
                raise NormFailureError(dev, realization=real, step=step)
            events = seg_events[k] if seg_events is not None else []
            if events:
                emit(sinks.norm_events, [NormEvent(deviation=d, corrected=c, realization=r, step=s)
                                         for d, c, r, s in events])
            with profile.stage(STAGE_DENSITY):
                pops = host[k, :n].copy()
                s2 = float(host[k, n + 1])
                if s2 <= 0.0:
                    raise NumericError("joint distribution has no weight")
                pr = float(host[k, n + 2])
                # p = diag / R divided as the reduction kernel does (IEEE division,
                # not torch's reciprocal multiply)
                joint = diag[k].cpu().numpy() / float(config.realizations) if want_joint else None
                time_tag = target * config.stepper.dt
                purity = float(pur_host[k]) / float(config.realizations) ** 2 if want_purity else None
                rows = _observable_rows(config, pops, pr, purity, joint)
                rho = DiagonalDensity(diag=None, dim=dim, sample_count=config.realizations,
                                      time_tag=float(time_tag), purity=purity, populations=pops,
                                      participation_ratio=pr, device_diag=diag[k])
            totals["snapshots"] += 1
            emit(sinks.observable_rows, rho.time_tag, rows)
            emit(sinks.density_snapshot, rho, target)
            previous = target
        totals["corrections"] += local["corrections"]
        totals["events"] += local["event_count"]
        totals["max_dev"] = max(totals["max_dev"], local["max_deviation"])
    return totals


def run(config: RunConfig, sinks: OutputSinks | None = None, group=None) -> RunReport:
    """Execute a full ensemble run on the GPU(s) (ensemble.py:635-804)."""
    import torch

    if sinks is None:
        sinks = MemorySinks()
    profile = StageProfile()
    io_seconds = 0.0
    clock = time.perf_counter
    wall_start = clock()

    def emit(method, *args):
        nonlocal io_seconds
        t0 = clock()
        method(*args)
        io_seconds += clock() - t0

    rank, world = sharding.world_info(group)
    with profile.stage(STAGE_INITIALIZATION):
        estimate = estimate_memory(config, world)
        if estimate["total_bytes"] > config.memory_budget:
            raise MemoryBudgetError(
                f"estimated device working set {estimate['total_bytes']:,} bytes exceeds the budget "
                f"of {config.memory_budget:,}; lower realizations, shrink the lattice, or raise memory_budget"
            )
        if config.stepper.backend == BACKEND_EIGEN:
            raise ConfigurationError(
                "the eigen backend (dense diagonalisation) is not on the B200 path; use 'taylor' or 'rk4'"
            )
        if OBS_PURITY in config.observables:
            work = float(config.realizations) ** 2 * config.space.dim
            if work > PURITY_WORK_CAP:
                raise CapacityError(
                    f"purity needs R^2*D = {work:.3g} overlap multiply-adds per snapshot "
                    f"(cap {PURITY_WORK_CAP:.3g}); drop it from observables"
                )
            if world > 1 and config.realizations * config.space.dim * 16 > PURITY_GATHER_CAP:
                raise CapacityError("multi-GPU purity gathers all states; too large for this run")
        build_topology(config.space)
        device = config.device if config.device is not None else _default_device()
        lo, hi = sharding.shard_bounds(config.realizations, world, rank)
        with torch.cuda.device(device):
            ens = EnsembleState(config, device, lo, hi)
    if config.precision == PRECISION_SINGLE:
        emit(sinks.message, "precision=single requested: the B200 path propagates in double")
    emit(sinks.message,
         f"run start: dim={config.space.dim} realizations={config.realizations} steps={config.steps} "
         f"backend={config.stepper.backend} precision={config.precision} workers={world} "
         f"snapshots={len(config.schedule)}")

    snapshots = 0
    max_deviation = 0.0
    corrections = 0
    event_total = 0
    previous = 0
    fused = fused_collection_ok(config, sinks, world)
    if fused:
        with torch.cuda.device(device):
            tot = _run_fused(config, ens, sinks, emit, profile, clock, group)
        snapshots, corrections = tot["snapshots"], tot["corrections"]
        event_total, max_deviation = tot["events"], tot["max_dev"]
    with torch.cuda.device(device):
        for target in (() if fused else config.schedule):
            span = target - previous
            if span > 0:
                t0 = clock()
                ens.evolve(previous, span)
                t_ev = clock()
            # the collection point is enqueued behind the segment; the single
            # synchronisation below (statistics) covers both
            t_obs0 = clock()
            pending = collect_observables_async(config, ens, group)
            t_obs1 = clock()
            if span > 0:
                local = ens.stats()
                merged = sharding.merge_segment_stats(sharding.gather_stats(local, group))
                profile.add(STAGE_EVOLUTION, (t_ev - t0) + (clock() - t_obs1),
                            calls=config.realizations * span)
                # the Hamiltonian is generated on the fly; dynamic noise rewrites the
                # switched couplings inside ctqw_evolve (timed with the evolution)
                profile.add(STAGE_HAMILTONIAN, 0.0, calls=config.realizations * span)
                if merged["failure"] is not None:
                    dev, real, step = merged["failure"]
                    emit(sinks.message,
                         f"aborted: norm deviation {dev:.3e} at realization {real}, step {step}; "
                         f"reduce the time step")
                    ens.release()
                    raise NormFailureError(dev, realization=real, step=step)
                corrections += merged["corrections"]
                event_total += merged["event_count"]
                max_deviation = max(max_deviation, merged["max_deviation"])
                if merged["events"]:
                    emit(sinks.norm_events,
                         [NormEvent(deviation=d, corrected=c, realization=r, step=s)
                          for d, c, r, s in merged["events"]])
            previous = target
            with profile.stage(STAGE_DENSITY):
                profile.add(STAGE_DENSITY, t_obs1 - t_obs0, calls=0)
                pops = pending.populations
                joint = pending.joint() if OBS_JOINT in config.observables else None
                time_tag = target * config.stepper.dt
                rows = _observable_rows(config, pops, pending.participation_ratio, pending.purity, joint)
                if getattr(sinks, "dense_density", False):
                    rho = _dense_snapshot(config, ens, group, time_tag)
                else:
                    rho = DiagonalDensity(diag=None, dim=config.space.dim, sample_count=config.realizations,
                                          time_tag=float(time_tag), purity=pending.purity, populations=pops,
                                          participation_ratio=pending.participation_ratio,
                                          device_diag=pending.diag_dev)
            snapshots += 1
            emit(sinks.observable_rows, rho.time_tag, rows)
            emit(sinks.density_snapshot, rho, target)

    with torch.cuda.device(device):
        switches = sharding.allreduce_int_([ens.switch_count()], group)[0]
        ens.release()
    report = RunReport(config=config, profile=profile, io_seconds=io_seconds,
                       wall_seconds=clock() - wall_start, workers=world, snapshots=snapshots,
                       max_norm_deviation=max_deviation, norm_corrections=corrections,
                       norm_events=event_total, switch_count=switches, memory_estimate=estimate)
    emit(sinks.message,
         f"run end: snapshots={snapshots} corrections={corrections} switches={switches} "
         f"max_norm_deviation={max_deviation:.3e}")
    sinks.finish(report)
    return report
