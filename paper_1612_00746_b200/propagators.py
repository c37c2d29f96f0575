"""Single-step propagators and the norm policy on the device.

API of the reference's ``propagators.py`` for the B200 path:
``StepperConfig`` (:61-86), ``step_taylor_values`` (:167-194),
``step_rk4_values`` (:197-241), ``check_norm_stack`` (:309-328),
``WaveFunction``, ``NormEvent``, ``step_taylor`` / ``step_rk4`` / ``check_norm``.
The eigen backend (dense O(D^3) diagonalisation, :99-140) is out of scope
 and rejected.

Arithmetic runs in libctqw's kernels; ``exact=True`` (default) reproduces the
reference's operation order without FMA contraction, so these calls return
the reference's bits.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, NormFailureError
from .hamiltonian import as_state_stack, bind_values, model_handle

BACKEND_EIGEN = "eigen"
BACKEND_RK4 = "rk4"
BACKEND_TAYLOR = "taylor"
BACKENDS = (BACKEND_EIGEN, BACKEND_RK4, BACKEND_TAYLOR)
DEVICE_BACKENDS = (BACKEND_TAYLOR, BACKEND_RK4)

DEFAULT_DT = 0.05
DEFAULT_TAYLOR_ORDER = 4
DEFAULT_TOL_NORM = 1e-6
DEFAULT_TOL_FAIL = 1e-3


@dataclass
class WaveFunction:
    amplitudes: object
    time_tag: float = 0.0

    def norm(self) -> float:
        return float(np.linalg.norm(np.asarray(self.amplitudes)))

    @property
    def dim(self) -> int:
        return self.amplitudes.shape[-1]


@dataclass(frozen=True)
class StepperConfig:
    backend: str = BACKEND_TAYLOR
    dt: float = DEFAULT_DT
    taylor_order: int = DEFAULT_TAYLOR_ORDER
    tol_norm: float = DEFAULT_TOL_NORM
    tol_fail: float = DEFAULT_TOL_FAIL
    renormalize: bool = True

    def __post_init__(self):
        if self.backend not in BACKENDS:
            raise ConfigurationError(f"backend {self.backend!r} not recognized; use one of {BACKENDS}")
        if not (np.isfinite(self.dt) and self.dt > 0):
            raise ConfigurationError(f"dt = {self.dt} must be positive and finite")
        if self.taylor_order < 1:
            raise ConfigurationError(f"taylor_order = {self.taylor_order} must be >= 1")
        if not (0 < self.tol_norm < self.tol_fail):
            raise ConfigurationError(
                f"need 0 < tol_norm < tol_fail, got {self.tol_norm} and {self.tol_fail}"
            )

    def native(self, exact: bool = True):
        from .native import make_stepper

        if self.backend not in DEVICE_BACKENDS:
            raise ConfigurationError(
                "the eigen backend (dense diagonalisation) is not on the B200 path; "
                "use 'taylor' or 'rk4'"
            )
        return make_stepper(self.backend, self.taylor_order, self.dt, self.tol_norm,
                            self.tol_fail, self.renormalize, exact)


@dataclass
class NormEvent:
    deviation: float
    corrected: bool
    realization: int | None = None
    step: int | None = None


def _step(backend, topology, values, psi, dt, hbar, order, out, exact):
    import torch

    h = model_handle(topology, values.model, hbar=hbar)
    dev = torch.device(f"cuda:{h.device}")
    stack, restore, _ = as_state_stack(psi, dev)
    if stack.shape[-1] != topology.dim:
        raise ConfigurationError(f"state has {stack.shape[-1]} amplitudes, expected {topology.dim}")
    result = torch.empty_like(stack)
    bind_values(h, values, stack.shape[0])
    cfg = StepperConfig(backend=backend, dt=dt, taylor_order=order)
    h.step(stack, result, stack.shape[0], cfg.native(exact))
    res = restore(result)
    if out is not None:
        out[...] = res
        return out
    return res


def step_taylor_values(topology, values, psi, dt: float, hbar: float = 1.0,
                       order: int = DEFAULT_TAYLOR_ORDER, out=None, scratch=None, exact=True):
    """Truncated-series step of a batch (propagators.py:167-194)."""
    return _step(BACKEND_TAYLOR, topology, values, psi, dt, hbar, order, out, exact)


def step_rk4_values(topology, values, psi, dt: float, hbar: float = 1.0, out=None,
                    scratch=None, exact=True):
    """Classical RK4 step of a batch (propagators.py:197-241)."""
    return _step(BACKEND_RK4, topology, values, psi, dt, hbar, 4, out, exact)


def step_taylor(h, psi, dt: float, order: int = DEFAULT_TAYLOR_ORDER):
    amps = psi.amplitudes if isinstance(psi, WaveFunction) else psi
    out = step_taylor_values(h.topology, h, amps, dt, hbar=h.model.hbar, order=order)
    return WaveFunction(out, psi.time_tag + dt) if isinstance(psi, WaveFunction) else out


def step_rk4(h, psi, dt: float):
    amps = psi.amplitudes if isinstance(psi, WaveFunction) else psi
    out = step_rk4_values(h.topology, h, amps, dt, hbar=h.model.hbar)
    return WaveFunction(out, psi.time_tag + dt) if isinstance(psi, WaveFunction) else out


def check_norm_stack(stack, stepper: StepperConfig, topology=None):
    """Norm policy over a stack, mutating it in place (propagators.py:309-328).

    Returns ``(deviations, corrected)`` as NumPy arrays; raises
    ``NormFailureError`` naming the worst row (before any rescale) when a
    row's squared-norm deviation exceeds ``tol_fail``.
    """
    import torch

    from .geometry import JointSpace, build_lattice, build_topology
    from .hamiltonian import CouplingModel

    is_torch = isinstance(stack, torch.Tensor)
    dim = stack.shape[-1]
    if topology is None:
        # any handle works (the norm does not depend on the operator)
        topology = build_topology(JointSpace(build_lattice([max(dim, 3)]), 1))
    h = model_handle(topology, CouplingModel())
    dev = torch.device(f"cuda:{h.device}")
    t, restore, shape = as_state_stack(stack, dev)
    rows = t.shape[0]
    deviations = torch.empty(rows, dtype=torch.float64, device=dev)
    corrected = torch.empty(rows, dtype=torch.int32, device=dev)
    try:
        h.check_norm(t, rows, stepper.native(), deviations, corrected)
    except NormFailureError:
        raise
    res = restore(t)
    if is_torch:
        if res.data_ptr() != stack.data_ptr():
            stack.copy_(res)
    else:
        np.copyto(stack, res)
    devs = deviations.cpu().numpy()
    corr = corrected.cpu().numpy().astype(bool)
    if len(shape) == 1:
        return devs[0], corr[0]
    return devs, corr


def check_norm(psi, stepper: StepperConfig):
    """Single-state norm policy (propagators.py:278-306)."""
    amps = np.array(psi.amplitudes if isinstance(psi, WaveFunction) else psi, dtype=np.complex128)
    stack = amps.reshape(1, -1)
    dev, corr = check_norm_stack(stack, stepper)
    dev = float(dev[0])
    if dev <= stepper.tol_norm:
        return psi, None
    new = stack[0]
    if isinstance(psi, WaveFunction):
        new_psi = WaveFunction(new, psi.time_tag) if stepper.renormalize else psi
    else:
        new_psi = new if stepper.renormalize else psi
    return new_psi, NormEvent(deviation=dev, corrected=bool(stepper.renormalize))
