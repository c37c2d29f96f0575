"""The binding a ``ctqw`` maintainer adds as ``ctqw/_b200.py``:
routes the reference's static-noise segment loop ``_evolve_segment``
(ensemble.py:445-558) through libctqw.so on sm_100a.

    import ctqw_b200_binding; ctqw_b200_binding.install()
    ctqw.run(config, sinks)          # workers = 1: segments run in-process

Inside the package the imports below become relative (``from .errors ...``).
Dynamic noise (rate > 0) and the eigen backend fall through to the
original loop: the binding replaces only the static-noise Taylor / RK4 path.
Executed by tests/test_gpu_integration.py against the reference's own run().
"""
import numpy as np
import torch

import ctqw.ensemble as _ens
from ctqw.errors import NormFailureError
from ctqw.propagators import NormEvent
from paper_1612_00746_b200 import native  # ctypes signatures of include/ctqw.h

_handles = {}
_original = _ens._evolve_segment


def _handle(ctx):
    topo, model = ctx.topology, ctx.model
    key = (topo.space.m, topo.space.lattice.n_sites, model.onsite_energy, float(model.tunneling),
           model.interaction, model.hbar)
    if key not in _handles:
        _handles[key] = native.Handle(*key, device=torch.cuda.current_device())
    return _handles[key]


def _supported(ctx, chunk):
    lat = ctx.topology.space.lattice
    ring = lat.q == 1 and tuple(lat.k_half) == (1,) and lat.boundary == "periodic"
    static = all(p.spec.rate == 0.0 for p in chunk.noise)
    return ring and static and ctx.stepper.backend in ("taylor", "rk4") and ctx.dtype_name == "complex128"


def evolve_segment_b200(ctx, chunk, start_step, n_steps):
    """Drop-in body for ctqw.ensemble._evolve_segment (static noise, taylor/rk4)."""
    if not _supported(ctx, chunk):
        return _original(ctx, chunk, start_step, n_steps)
    h = _handle(ctx)
    b, n = chunk.psi.shape[0], h.n
    dev = torch.device(f"cuda:{h.device}")
    nl, ns = chunk.noise[0].n_links, chunk.noise[0].n_sites
    noise = torch.as_tensor(np.stack([p.values for p in chunk.noise]), device=dev)
    hop = torch.empty((b, n), dtype=torch.float64, device=dev)
    site = torch.empty((b, n), dtype=torch.float64, device=dev) if ns else None
    h.build_coefficients(noise, b, nl, ns, hop, site)
    h.bind(hop, site, b, n)
    psi = torch.as_tensor(np.ascontiguousarray(chunk.psi, dtype=np.complex128), device=dev)
    work = torch.empty_like(psi)
    st = ctx.stepper
    stepper = native.make_stepper(st.backend, st.taylor_order, st.dt, st.tol_norm, st.tol_fail, st.renormalize,
                                  exact=True)
    swapped = h.evolve(psi, work, b, start_step, n_steps, stepper)
    s = h.segment_stats(chunk.r0)
    if s.failed:
        raise NormFailureError(s.fail_deviation, realization=s.fail_realization, step=s.fail_step)
    chunk.psi = (work if swapped else psi).cpu().numpy().astype(chunk.psi.dtype)
    events = [NormEvent(e.deviation, bool(e.corrected), e.realization, e.step) for e in s.events[: s.n_events]]
    stats = _ens._SegmentStats(0.0, 0.0, b * n_steps, b * n_steps, events, s.event_count, s.corrections,
                               s.max_deviation)
    return chunk, stats


def install():
    _ens._evolve_segment = evolve_segment_b200


def uninstall():
    _ens._evolve_segment = _original
