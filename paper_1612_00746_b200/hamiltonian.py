"""Hamiltonian model and the matrix-free apply (device).

``CouplingModel`` keeps the reference's fields and validation
(hamiltonian.py:30-72).  ``assemble_values`` returns a ``StencilValues``
instead of the reference's ``(B, D, H+1)`` complex value table
(hamiltonian.py:105-144): for the ring stencil that table is fully determined
by the per-realization link couplings ``hop[x] = t + xi_link[x]`` and on-site
noise ``xi_site[x]`` -- O(N) instead of O(N^m) per realization -- and the
kernels regenerate every entry on the fly.  ``apply_values``
(hamiltonian.py:195-223) runs ``ctqw_apply`` in the reference's accumulation
order, bit-identical to it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

_HANDLES: dict = {}


@dataclass(frozen=True)
class CouplingModel:
    onsite_energy: float = 0.0
    tunneling: float | tuple = 1.0
    interaction: float = 0.0
    hbar: float = 1.0

    def __post_init__(self):
        if isinstance(self.tunneling, (list, tuple, np.ndarray)):
            object.__setattr__(self, "tunneling", tuple(float(v) for v in self.tunneling))
            amps = self.tunneling
        else:
            object.__setattr__(self, "tunneling", float(self.tunneling))
            amps = (self.tunneling,)
        for name in ("onsite_energy", "interaction", "hbar"):
            if not np.isfinite(getattr(self, name)):
                raise ConfigurationError(f"{name} = {getattr(self, name)} must be finite")
        if not all(np.isfinite(amps)):
            raise ConfigurationError("tunneling amplitudes must be finite")
        if self.hbar <= 0:
            raise ConfigurationError(f"hbar = {self.hbar} must be > 0")

    def tunneling_per_direction(self, q: int) -> np.ndarray:
        if isinstance(self.tunneling, tuple):
            if len(self.tunneling) != q:
                raise ConfigurationError(f"{len(self.tunneling)} tunneling amplitudes for {q} directions")
            return np.asarray(self.tunneling, dtype=np.float64)
        return np.full(q, self.tunneling, dtype=np.float64)

    def ring_tunneling(self) -> float:
        return float(self.tunneling_per_direction(1)[0])


def handle_for(m, n, onsite, tunneling, interaction, hbar, device=None, lattice=None, lattice_key=None):
    """Cached ``native.Handle`` for a model on a device (``lattice``: move
    tables of a non-ring lattice, identified by ``lattice_key``)."""
    import torch

    from .native import Handle

    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    key = (int(m), int(n), float(onsite), float(tunneling), float(interaction), float(hbar), int(device),
           lattice_key)
    h = _HANDLES.get(key)
    if h is None:
        h = Handle(m, n, onsite, tunneling, interaction, hbar, device, lattice=lattice)
        _HANDLES[key] = h
    return h


# Free private handles by model key: an ensemble takes one for its lifetime
# (exclusive: it binds its own coefficient rows and telegraph process) and
# gives it back when it is released, so repeated runs do not re-create the
# handle's device and pinned host buffers (cudaMallocHost / cudaFreeHost per
# run cost up to tens of milliseconds, and vary).
_PRIVATE_POOL: dict = {}


def release_private_handle(h):
    """Return a private handle to the pool (EnsembleState.release)."""
    key = getattr(h, "_pool_key", None)
    if key is None or not getattr(h, "_h", None):
        return
    h.telegraph_enable(False)
    h.set_initial(None)  # a pending initial state of the released ensemble must not leak into the next
    h._bound = None
    _PRIVATE_POOL.setdefault(key, []).append(h)


def model_handle(topology, model: CouplingModel, hbar=None, device=None, private: bool = False):
    """Handle for ``topology`` + ``model``: the ring as is, any other lattice
    with its move tables and the tunnelling of each slot's direction
    (slot_couplings, hamiltonian.py:92-97).

    ``private=True`` returns a new, uncached handle: an ensemble binds its own
    coefficient rows and telegraph process into its handle, so it must not
    share one with the single-step API or another ensemble."""
    import torch

    from .native import Handle

    hb = model.hbar if hbar is None else hbar

    def pooled(key, make):
        free = _PRIVATE_POOL.get(key)
        h = free.pop() if free else make()
        h._pool_key = key
        return h

    if topology.is_ring:
        args = (topology.m, topology.n, model.onsite_energy, model.ring_tunneling(), model.interaction, hb)
        if private:
            dev = torch.cuda.current_device() if device is None else device
            return pooled(("ring",) + tuple(float(a) for a in args) + (int(dev),), lambda: Handle(*args, dev))
        return handle_for(*args, device)
    lat = topology.lattice
    pos, neg, directions = topology.move_tables()
    t_slot = model.tunneling_per_direction(lat.q)[directions]
    if private:
        dev = torch.cuda.current_device() if device is None else device
        key = ("lattice", topology.m, lat.dims, lat.k_half, lat.boundary, tuple(float(v) for v in t_slot),
               float(model.onsite_energy), float(model.interaction), float(hb), int(dev))
        return pooled(key, lambda: Handle(topology.m, topology.n, model.onsite_energy, float(t_slot[0]),
                                          model.interaction, hb, dev, lattice=(pos, neg, t_slot)))
    key = (lat.dims, lat.k_half, lat.boundary, tuple(float(v) for v in t_slot))
    return handle_for(topology.m, topology.n, model.onsite_energy, float(t_slot[0]), model.interaction, hb,
                      device, lattice=(pos, neg, t_slot), lattice_key=key)


@dataclass
class StencilValues:
    """Per-realization couplings of the lattice operator (device tensors).

    ``hop``: ``batch + (N*K,)`` float64 (link x*K + s), ``site``: ``batch +
    (N,)`` or None.  ``batch`` is
    ``()`` for one Hamiltonian shared by every state, ``(B,)`` for a stack.
    """

    topology: object
    model: CouplingModel
    hop: object
    site: object | None

    @property
    def batch(self) -> tuple:
        return tuple(self.hop.shape[:-1])

    @property
    def dim(self) -> int:
        return self.topology.dim


def _device_array(x, device):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device=device)


def assemble_values(topology, model: CouplingModel, link_values=None, site_values=None,
                    out=None, dtype=np.complex128) -> StencilValues:
    """Stencil couplings from optional noise arrays (hamiltonian.py:105-144)."""
    import torch

    h = model_handle(topology, model)
    dev = torch.device(f"cuda:{h.device}")
    n = topology.n
    nl = topology.n_links
    has_link = link_values is not None and np.shape(link_values)[-1] != 0
    has_site = site_values is not None and np.shape(site_values)[-1] != 0
    batch = ()
    if has_link:
        batch = tuple(np.shape(link_values)[:-1])
    if has_site:
        batch = tuple(np.shape(site_values)[:-1])
    count = int(np.prod(batch)) if batch else 1
    noise_cols = []
    if has_link:
        if np.shape(link_values)[-1] != nl:
            raise ConfigurationError(f"link_values needs {nl} entries per realization")
        noise_cols.append(_device_array(link_values, dev).reshape(count, nl))
    if has_site:
        if np.shape(site_values)[-1] != n:
            raise ConfigurationError(f"site_values needs {n} entries per realization")
        noise_cols.append(_device_array(site_values, dev).reshape(count, n))
    hop = torch.empty((count, nl), dtype=torch.float64, device=dev)
    site = torch.empty((count, n), dtype=torch.float64, device=dev) if has_site else None
    noise = torch.cat(noise_cols, dim=1).contiguous() if noise_cols else None
    h.build_coefficients(noise, count, nl if has_link else 0, n if has_site else 0, hop, site)
    hop = hop.reshape(batch + (nl,))
    if site is not None:
        site = site.reshape(batch + (n,))
    return StencilValues(topology=topology, model=model, hop=hop, site=site)


def as_state_stack(psi, device):
    """(tensor (B, D) complex128 on device, restore-fn) for numpy or torch input."""
    import torch

    if isinstance(psi, torch.Tensor):
        shape = tuple(psi.shape)
        t = psi.to(device=device, dtype=torch.complex128).reshape(-1, shape[-1]).contiguous()
        return t, (lambda out: out.reshape(shape)), shape
    arr = np.asarray(psi)
    shape = arr.shape
    t = torch.as_tensor(np.ascontiguousarray(arr.reshape(-1, shape[-1]), dtype=np.complex128),
                        device=device)
    return t, (lambda out: out.reshape(shape).cpu().numpy()), shape


def bind_values(h, values: StencilValues, count: int):
    """Bind ``values`` for a batch of ``count`` states (broadcast or per row)."""
    vb = values.batch
    vcount = int(np.prod(vb)) if vb else 1
    if vb == () or vcount == 1 and count == 1:
        stride = 0
    elif vcount == count:
        stride = values.topology.n_links
    else:
        raise ConfigurationError(f"values batch {vb} does not match {count} states")
    hop = values.hop.reshape(-1, values.topology.n_links)
    site = values.site.reshape(-1, values.topology.n) if values.site is not None else None
    h.bind(hop, site, vcount, stride)


def apply_values(topology, values: StencilValues, psi, out=None, exact: bool = True):
    """``H psi`` through the on-the-fly stencil (hamiltonian.py:195-223)."""
    import torch

    h = model_handle(topology, values.model)
    dev = torch.device(f"cuda:{h.device}")
    stack, restore, _ = as_state_stack(psi, dev)
    if stack.shape[-1] != topology.dim:
        raise ConfigurationError(f"state has {stack.shape[-1]} amplitudes, expected {topology.dim}")
    result = torch.empty_like(stack)
    bind_values(h, values, stack.shape[0])
    h.apply(stack, result, stack.shape[0], exact)
    res = restore(result)
    if out is not None:
        out[...] = res
        return out
    return res
