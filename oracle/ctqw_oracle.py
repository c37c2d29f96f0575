"""TEST INFRASTRUCTURE ONLY -- NumPy restatement of the reference hot path.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import it.  The product package ``paper_1612_00746_b200`` never imports
anything under ``oracle/``; its compute runs in ``libctqw.so`` on the GPU.

Scope: m particles (1..3) on a periodic 1-D ring of N sites, nearest-neighbour
hops (q = 1, k_half = 1), static noise, FP64 (complex128) states.  For that
geometry the reference's reduced operator (``hilbert.py:278-359`` +
``hamiltonian.py:105-144,195-223``) is the stencil

    (H psi)(x) = v0(x) psi(x)
               + sum_p [ hop[x_p] psi(x_p + 1) + hop[x_p - 1] psi(x_p - 1) ]

with ``hop[x] = t + xi_link[x]`` (``hamiltonian.py:137-141``; the mirrored
slot reads the value stored at the target row, ``:216``) and
``v0 = (m*eps0 + U*coincidence) + sum_p xi_site[x_p]`` (``:132-135``).

Every floating-point operation below is ordered exactly as the reference's
NumPy expression evaluates it (diagonal first, then per particle slot the
+move then the -move, ``hamiltonian.py:205-222``; Taylor ``product *= coeff/j;
out += term`` ``propagators.py:185-193``; RK4 stage arithmetic
``propagators.py:213-240``; the site sum left-associated as
``ndarray.sum(axis=-1)`` evaluates it).  So when the norm policy never
rescales, this restatement is bit-identical to the reference -- the golden
fixtures in ``tests/golden/`` (made by ``tests/golden/make_golden.py`` from the
reference itself) pin that.  The squared norm (``propagators.py:316-318``,
an ``einsum``) is only reproduced to rounding.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MAX_EVENTS_PER_SEGMENT = 100  # ensemble.py:119


# ----------------------------------------------------------------------------
# coefficients (hamiltonian.py:105-144)


@dataclass
class Stencil:
    """Per-realization stencil coefficients of the m-particle ring operator."""

    m: int
    n: int
    base: np.ndarray          # (4,) diagonal base per coincidence count c
    hop: np.ndarray           # (B, N) hop amplitude of link x -> x+1 (ring); (B, N*K) link x*K+s (lattice)
    site: np.ndarray | None   # (B, N) on-site noise, None when absent
    pos: np.ndarray | None = None    # (N, K) +move targets, -1 off-lattice (general lattices)
    neg: np.ndarray | None = None    # (N, K) -move targets
    t_slot: np.ndarray | None = None  # (K,) tunnelling per slot

    @property
    def dim(self) -> int:
        return self.n ** self.m


def diagonal_base(m: int, onsite: float, interaction: float) -> np.ndarray:
    """``m*eps0 + U*c`` for c = 0..3 pairs coinciding (hamiltonian.py:132)."""
    return np.array([m * onsite + interaction * c for c in range(4)], dtype=np.float64)


def make_stencil(m, n, onsite, tunneling, interaction, link=None, site=None, batch=1):
    """Assemble coefficients like ``assemble_values`` (hamiltonian.py:131-141)."""
    base = diagonal_base(m, onsite, interaction)
    if link is not None and np.shape(link)[-1]:
        link = np.atleast_2d(np.asarray(link, dtype=np.float64))
        hop = np.float64(tunneling) + link          # out[...,1:] = base; += link
    else:
        hop = np.full((batch, n), np.float64(tunneling))
    if site is not None and np.shape(site)[-1]:
        site = np.atleast_2d(np.asarray(site, dtype=np.float64))
    else:
        site = None
    return Stencil(m=m, n=n, base=base, hop=hop, site=site)


def make_lattice_stencil(m, dims, k_half, boundary, onsite, tunneling, interaction, link=None, site=None,
                         batch=1):
    """General lattice (hilbert.py:189-224, hamiltonian.py:92-141): the
    single-particle move tables in the reference's slot order and the link
    couplings ``t_dir(slot) + xi_link[x*K + s]``."""
    dims = [int(d) for d in dims]
    k_half = [int(k) for k in k_half]
    q = len(dims)
    n = int(np.prod(dims))
    coords = np.empty((n, q), dtype=np.int64)
    rem = np.arange(n, dtype=np.int64)
    for i in range(q - 1, -1, -1):
        coords[:, i] = rem % dims[i]
        rem //= dims[i]
    strides = [int(np.prod(dims[i + 1:])) for i in range(q)]
    slots = [(i, d) for i in range(q) for d in range(1, k_half[i] + 1)]
    pos = np.empty((n, len(slots)), dtype=np.int64)
    neg = np.empty((n, len(slots)), dtype=np.int64)
    base_sites = np.arange(n, dtype=np.int64)
    for sl, (i, d) in enumerate(slots):
        c = coords[:, i]
        if boundary == "periodic":
            pos[:, sl] = base_sites + ((c + d) % dims[i] - c) * strides[i]
            neg[:, sl] = base_sites + ((c - d) % dims[i] - c) * strides[i]
        else:
            pos[:, sl] = np.where(c + d < dims[i], base_sites + d * strides[i], -1)
            neg[:, sl] = np.where(c - d >= 0, base_sites - d * strides[i], -1)
    per_dir = (np.asarray(tunneling, dtype=np.float64) if np.ndim(tunneling)
               else np.full(q, float(tunneling)))
    t_slot = per_dir[[i for i, _ in slots]]
    K = len(slots)
    t_links = np.tile(t_slot, n)                    # link x*K + s
    if link is not None and np.shape(link)[-1]:
        hop = t_links + np.atleast_2d(np.asarray(link, dtype=np.float64))
    else:
        hop = np.broadcast_to(t_links, (batch, n * K)).copy()
    if site is not None and np.shape(site)[-1]:
        site = np.atleast_2d(np.asarray(site, dtype=np.float64))
    else:
        site = None
    return Stencil(m=m, n=n, base=diagonal_base(m, onsite, interaction), hop=hop, site=site, pos=pos, neg=neg,
                   t_slot=t_slot)


def _apply_lattice(st: Stencil, psi: np.ndarray, v0: np.ndarray) -> np.ndarray:
    """``apply_values`` on a general lattice, order: diagonal, then per
    particle p and slot s the +move, then the -move whose coupling is stored
    at its target row (hamiltonian.py:205-222); absent moves add an exact
    zero."""
    m, n, K = st.m, st.n, st.pos.shape[1]
    b = psi.shape[0]
    dim = psi.shape[1]
    out = v0.reshape(v0.shape[0], -1) * psi
    alpha = np.arange(dim, dtype=np.int64)
    digits = np.empty((dim, m), dtype=np.int64)
    rem = alpha.copy()
    for p in range(m - 1, -1, -1):
        digits[:, p] = rem % n
        rem //= n
    hop = st.hop if st.hop.shape[0] == b else np.broadcast_to(st.hop, (b, st.hop.shape[1]))
    for p in range(m):
        shift = n ** (m - 1 - p)
        xs = digits[:, p]
        for sl in range(K):
            tgt = st.pos[xs, sl]
            ok = tgt >= 0
            beta = np.where(ok, alpha + (tgt - xs) * shift, 0)
            out = out + np.where(ok, hop[:, xs * K + sl] * psi[:, beta], 0)
            src = st.neg[xs, sl]
            ok = src >= 0
            beta = np.where(ok, alpha + (src - xs) * shift, 0)
            out = out + np.where(ok, hop[:, np.where(ok, src, 0) * K + sl] * psi[:, beta], 0)
    return out


def diagonal_values(st: Stencil) -> np.ndarray:
    """v0 per joint state, shape (B, N, ..., N) (hamiltonian.py:132-135)."""
    m, n = st.m, st.n
    grids = np.meshgrid(*([np.arange(n)] * m), indexing="ij")
    coinc = np.zeros(grids[0].shape, dtype=np.int64)
    for p in range(m):
        for r in range(p + 1, m):
            coinc += grids[p] == grids[r]
    v0 = st.base[coinc][None]                      # (1, N, .., N)
    if st.site is not None:
        b = st.site.shape[0]
        total = None
        for p in range(m):
            shape = [b] + [1] * m
            shape[1 + p] = n
            term = st.site.reshape(shape)
            total = term if total is None else total + term   # left-assoc sum
        v0 = v0 + total
    return v0


# ----------------------------------------------------------------------------
# apply (hamiltonian.py:195-223)


def apply_stencil(st: Stencil, psi: np.ndarray, v0: np.ndarray | None = None) -> np.ndarray:
    """``H psi`` for a (B, D) complex128 stack, reference accumulation order."""
    if st.pos is not None:
        return _apply_lattice(st, psi, diagonal_values(st) if v0 is None else v0)
    m, n = st.m, st.n
    b = psi.shape[0]
    shp = (b,) + (n,) * m
    x = psi.reshape(shp)
    if v0 is None:
        v0 = diagonal_values(st)
    out = v0 * x                                   # np.multiply(values[...,0], psi)
    hop = st.hop
    hop_m1 = np.roll(hop, 1, axis=-1)              # hop[x-1]: stored at the -move target
    for p in range(m):
        bshape = [hop.shape[0]] + [1] * m
        bshape[1 + p] = n
        axis = 1 + p
        out = out + hop.reshape(bshape) * np.roll(x, -1, axis=axis)      # +move
        out = out + hop_m1.reshape(bshape) * np.roll(x, 1, axis=axis)    # -move
    return out.reshape(b, -1)


# ----------------------------------------------------------------------------
# propagators (propagators.py:167-241)


def taylor_coefficients(dt: float, hbar: float, order: int):
    """``coeff/j`` with ``coeff = -1j*dt/hbar`` (propagators.py:185,191)."""
    coeff = -1j * dt / hbar
    return [coeff / j for j in range(1, order + 1)]


def _times_coeff(z: np.ndarray, c: complex) -> np.ndarray:
    out = z.copy()
    out *= c
    return out


def taylor_step(st, psi, dt, hbar=1.0, order=4, v0=None):
    """``step_taylor_values`` restated (propagators.py:167-194)."""
    if v0 is None:
        v0 = diagonal_values(st)
    out = psi.copy()
    term = psi
    for c in taylor_coefficients(dt, hbar, order):
        product = apply_stencil(st, term, v0)
        product *= c
        term = product
        out += term
    return out


def rk4_step(st, psi, dt, hbar=1.0, v0=None):
    """``step_rk4_values`` restated (propagators.py:197-241)."""
    if v0 is None:
        v0 = diagonal_values(st)
    coeff = -1j * dt / hbar
    stage = apply_stencil(st, psi, v0)
    stage *= coeff
    arg = stage * 0.5
    arg += psi
    out = psi.copy()
    stage *= 1.0 / 6.0
    out += stage
    stage = apply_stencil(st, arg, v0)
    stage *= coeff
    arg = stage * 0.5
    arg += psi
    stage *= 1.0 / 3.0
    out += stage
    stage = apply_stencil(st, arg, v0)
    stage *= coeff
    arg = stage.copy()
    arg += psi
    stage *= 1.0 / 3.0
    out += stage
    stage = apply_stencil(st, arg, v0)
    stage *= coeff
    stage *= 1.0 / 6.0
    out += stage
    return out


# ----------------------------------------------------------------------------
# norm policy (propagators.py:309-328)


class NormFailure(Exception):
    def __init__(self, deviation, realization=None, step=None):
        super().__init__(f"norm deviation {deviation:.3e} (realization {realization}, step {step})")
        self.deviation = float(deviation)
        self.realization = realization
        self.step = step


def check_norm_stack(stack, tol_norm, tol_fail, renormalize=True):
    """Mutates ``stack``; returns (deviations, corrected) like the reference."""
    norm_sq = np.einsum("...i,...i->...", stack.real, stack.real, dtype=np.float64) + np.einsum(
        "...i,...i->...", stack.imag, stack.imag, dtype=np.float64
    )
    dev = np.abs(norm_sq - 1.0)
    failed = dev > tol_fail
    if np.any(failed):
        row = int(np.argmax(dev))
        raise NormFailure(float(dev[row]), realization=row)
    over = dev > tol_norm
    if renormalize and np.any(over):
        stack[over] /= np.sqrt(norm_sq[over])[..., None]
        return dev, over
    return dev, np.zeros_like(over)


# ----------------------------------------------------------------------------
# segment loop (ensemble.py:445-558) and diagonal observables


@dataclass
class SegmentStats:
    events: list = field(default_factory=list)   # (deviation, corrected, realization, step)
    event_count: int = 0
    corrections: int = 0
    max_deviation: float = 0.0


def refresh_stencil(st, noise, tunneling):
    """Couplings after a telegraph advance: a fresh ``assemble_values``
    (hamiltonian.py:131-141), which the reference's incremental ``update``
    reproduces bit for bit (test_hamiltonian.py:124-139)."""
    if noise.n_links:
        t = np.tile(st.t_slot, st.n) if st.t_slot is not None else np.float64(tunneling)
        st.hop = t + noise.link_values()
    if noise.n_sites:
        st.site = noise.site_values().copy()


def evolve_segment(st, psi, start_step, n_steps, dt, hbar=1.0, backend="taylor", order=4,
                   tol_norm=1e-6, tol_fail=1e-3, renormalize=True, r0=0, noise=None, tunneling=1.0):
    """Advance a (B, D) stack ``n_steps`` with the per-step norm policy.

    ``noise`` (a ``TelegraphOracle``) is advanced by ``dt`` after every
    step's norm check and the couplings rebuilt (ensemble.py:536-544)."""
    v0 = diagonal_values(st)
    stats = SegmentStats()
    for s in range(n_steps):
        step_number = start_step + s + 1
        if backend == "taylor":
            psi = taylor_step(st, psi, dt, hbar, order, v0)
        else:
            psi = rk4_step(st, psi, dt, hbar, v0)
        try:
            dev, corrected = check_norm_stack(psi, tol_norm, tol_fail, renormalize)
        except NormFailure as exc:
            raise NormFailure(exc.deviation, r0 + (exc.realization or 0), step_number) from None
        stats.max_deviation = max(stats.max_deviation, float(dev.max()))
        over = dev > tol_norm
        if over.any():
            stats.corrections += int(corrected.sum())
            for row in np.nonzero(over)[0]:
                stats.event_count += 1
                if len(stats.events) < MAX_EVENTS_PER_SEGMENT:
                    stats.events.append((float(dev[row]), bool(corrected[row]), r0 + int(row), step_number))
        if noise is not None:
            noise.advance(dt)
            refresh_stencil(st, noise, tunneling)
            v0 = diagonal_values(st)
    return psi, stats


def joint_distribution(stack: np.ndarray) -> np.ndarray:
    """diag of ``accumulate_density`` (density.py:91-96): mean_r |psi_r|^2."""
    return (stack.real ** 2 + stack.imag ** 2).sum(axis=0) / stack.shape[0]


def populations(jd: np.ndarray, m: int, n: int) -> np.ndarray:
    """``observables.populations`` (observables.py:40-56)."""
    grid = jd.reshape((n,) * m)
    out = np.zeros(n)
    for p in range(m):
        axes = tuple(a for a in range(m) if a != p)
        out += grid.sum(axis=axes) if axes else grid
    return out


def position_stats(pops: np.ndarray, window=2, mass=1e-3, periodic=True):
    """``observables.position_variance`` (observables.py:59-83); the wrap flag
    only on a periodic lattice."""
    marginal = pops / pops.sum()
    x = np.arange(marginal.shape[0], dtype=np.float64)
    mean = float(marginal @ x)
    var = float(marginal @ (x - mean) ** 2)
    wrapped = False
    if periodic and marginal.shape[0] > 2 * window:
        wrapped = bool(marginal[:window].sum() > mass and marginal[-window:].sum() > mass)
    return mean, var, wrapped


def participation_ratio(jd: np.ndarray) -> float:
    """observables.py:94-101."""
    return 1.0 / float(np.square(jd / jd.sum()).sum())


def purity(stack: np.ndarray) -> float:
    """Tr rho^2 of the ensemble average = (1/R^2) sum_{r,s} |<psi_r|psi_s>|^2 (observables.py:86-91)."""
    g = stack.conj() @ stack.T
    return float((np.abs(g) ** 2).sum() / stack.shape[0] ** 2)


def observable_rows(stack, m, n, observables, periodic=True):
    """Row list in ``_observable_rows`` order (ensemble.py:609-632)."""
    jd = joint_distribution(stack)
    rows = []
    for name in observables:
        if name == "populations":
            rows.extend(("population", i, float(v)) for i, v in enumerate(populations(jd, m, n)))
        elif name == "position_mean_variance":
            mean, var, wrapped = position_stats(populations(jd, m, n), periodic=periodic)
            rows += [("position_mean", 0, mean), ("position_variance", 0, var),
                     ("position_wrapped", 0, float(wrapped))]
        elif name == "purity":
            rows.append(("purity", 0, purity(stack)))
        elif name == "participation_ratio":
            rows.append(("participation_ratio", 0, participation_ratio(jd)))
        elif name == "joint_distribution":
            rows.extend(("joint_probability", i, float(v)) for i, v in enumerate(jd))
    return rows


def product_state(m: int, n: int, positions=None) -> np.ndarray:
    """``build_initial_state`` auto/product kind (ensemble.py:178-193)."""
    if positions is None:
        start = (n - m) // 2
        positions = tuple(range(start, start + m))
    psi = np.zeros(n ** m, dtype=np.complex128)
    idx = 0
    for x in positions:
        idx = idx * n + int(x)
    psi[idx] = 1.0
    return psi


def schedule(steps: int, post_rate: int):
    """``RunConfig.schedule`` (ensemble.py:286-294)."""
    if steps == 0:
        return (0,)
    pts = list(range(post_rate, steps + 1, post_rate))
    if pts[-1] != steps:
        pts.append(steps)
    return tuple(pts)


def run_rows(st, psi0, realizations, steps, post_rate, dt, hbar=1.0, backend="taylor", order=4,
             observables=("populations", "position_mean_variance", "purity", "participation_ratio"),
             tol_norm=1e-6, tol_fail=1e-3, renormalize=True, noise=None, tunneling=1.0, periodic=True):
    """Diagonal-observable restatement of ``run`` (ensemble.py:635-804)."""
    psi = np.tile(psi0, (realizations, 1))
    out = []
    totals = SegmentStats()
    prev = 0
    for target in schedule(steps, post_rate):
        span = target - prev
        if span > 0:
            psi, stats = evolve_segment(st, psi, prev, span, dt, hbar, backend, order,
                                        tol_norm, tol_fail, renormalize, noise=noise, tunneling=tunneling)
            totals.event_count += stats.event_count
            totals.corrections += stats.corrections
            totals.max_deviation = max(totals.max_deviation, stats.max_deviation)
            totals.events.extend(stats.events)
        prev = target
        out.append((target * dt, observable_rows(psi, st.m, st.n, observables, periodic)))
    return out, psi, totals
