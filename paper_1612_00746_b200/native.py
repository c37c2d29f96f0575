"""ctypes binding to ``libctqw.so`` (the C ABI declared in ``include/ctqw.h``).

There is no fallback: if the library or a CUDA device is missing, every
compute entry point raises.  Device buffers are torch tensors (plumbing for
device memory and streams only); the arithmetic runs in the library's sm_100a
kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (
    CapacityError,
    ConfigurationError,
    CtqwError,
    NativeError,
    NormFailureError,
    NumericError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTQW_LIB", os.path.join(_HERE, "lib", "libctqw.so"))

MAX_EVENTS = 100
BACKEND_CODES = {"taylor": 0, "rk4": 1}


class Model(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32),
        ("n_sites", ctypes.c_int32),
        ("k_half", ctypes.c_int32),
        ("periodic", ctypes.c_int32),
        ("onsite_energy", ctypes.c_double),
        ("tunneling", ctypes.c_double),
        ("interaction", ctypes.c_double),
        ("hbar", ctypes.c_double),
    ]


class Stepper(ctypes.Structure):
    _fields_ = [
        ("backend", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("dt", ctypes.c_double),
        ("tol_norm", ctypes.c_double),
        ("tol_fail", ctypes.c_double),
        ("renormalize", ctypes.c_int32),
        ("exact", ctypes.c_int32),
    ]


class NormEventC(ctypes.Structure):
    _fields_ = [
        ("deviation", ctypes.c_double),
        ("realization", ctypes.c_int64),
        ("step", ctypes.c_int64),
        ("corrected", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class SegmentStats(ctypes.Structure):
    _fields_ = [
        ("event_count", ctypes.c_int64),
        ("corrections", ctypes.c_int64),
        ("max_deviation", ctypes.c_double),
        ("failed", ctypes.c_int32),
        ("n_events", ctypes.c_int32),
        ("fail_realization", ctypes.c_int64),
        ("fail_step", ctypes.c_int64),
        ("fail_deviation", ctypes.c_double),
        ("events", NormEventC * MAX_EVENTS),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

# name -> (restype, argtypes); the exact symbol set of include/ctqw.h
SIGNATURES = {
    "ctqw_abi_version": (ctypes.c_int, []),
    "ctqw_last_error": (ctypes.c_char_p, [_P]),
    "ctqw_create": (ctypes.c_int, [ctypes.POINTER(Model), _I32, ctypes.POINTER(_P)]),
    "ctqw_destroy": (ctypes.c_int, [_P]),
    "ctqw_draw_noise": (ctypes.c_int, [_P, ctypes.c_uint64, _I64, _I64, ctypes.POINTER(_D), _I32,
                                       _I64, _P, _P]),
    "ctqw_build_coefficients": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _P, _P]),
    "ctqw_bind_coefficients": (ctypes.c_int, [_P, _I64, _P, _P, _I64]),
    "ctqw_fill_states": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "ctqw_apply": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _P]),
    "ctqw_step": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(Stepper), _P]),
    "ctqw_check_norm": (ctypes.c_int, [_P, _P, _I64, ctypes.POINTER(Stepper), _P, _P,
                                       ctypes.POINTER(_I64), ctypes.POINTER(_D), _P]),
    "ctqw_evolve": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, ctypes.POINTER(Stepper),
                                   ctypes.POINTER(_I32), _P]),
    "ctqw_segment_stats": (ctypes.c_int, [_P, _I64, ctypes.POINTER(SegmentStats), _P]),
    "ctqw_observe_diag": (ctypes.c_int, [_P, _P, _I64, _P, _I32, _P]),
    "ctqw_observe_diag_fixed": (ctypes.c_int, [_P, _P, _I64, _P, _I32, _P]),
    "ctqw_fixed_to_double": (ctypes.c_int, [_P, _P, _P, _P]),
    "ctqw_observe_reduce": (ctypes.c_int, [_P, _P, _D, _P, _P, _P, _P]),
    "ctqw_overlap_sumsq": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _P, _P]),
    "ctqw_overlap_sumsq_points": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _P]),
    "ctqw_packed_gram": (ctypes.c_int, [_P, _I64, _I64, _D, _P, _I32, _P]),
    "ctqw_set_initial": (ctypes.c_int, [_P, _P]),
    "ctqw_evolve_observe": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, ctypes.POINTER(Stepper),
                                           _I32, ctypes.POINTER(_I32), _P]),
    "ctqw_segment_events": (ctypes.c_int, [_P, _I64, _I64, _I64, ctypes.POINTER(SegmentStats), _P]),
    "ctqw_observe_points": (ctypes.c_int, [_P, _P, _I64, _D, _P, _P, _P]),
    "ctqw_launch_count": (ctypes.c_int64, [_P]),
    "ctqw_kernel_timing": (ctypes.c_int, [_P, _I32]),
    "ctqw_kernel_time": (ctypes.c_int, [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64), _P]),
    "ctqw_step_kernel": (ctypes.c_char_p, [_P]),
    "ctqw_step_variant": (ctypes.c_char_p, [_P]),
    "ctqw_set_lattice": (ctypes.c_int, [_P, _I32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(_D)]),
    "ctqw_telegraph_init": (ctypes.c_int, [_P, ctypes.c_uint64, _I64, _I64, ctypes.POINTER(_D), _I32, _I64,
                                           _I64, _D, _P]),
    "ctqw_telegraph_values": (ctypes.c_void_p, [_P]),
    "ctqw_telegraph_enable": (ctypes.c_int, [_P, _I32]),
    "ctqw_telegraph_advance": (ctypes.c_int, [_P, _I64, _D, _P]),
    "ctqw_telegraph_read": (ctypes.c_int, [_P, _P, _P, ctypes.POINTER(_D), ctypes.POINTER(_I64), _P]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load and type the shared library (no CUDA context is touched)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        target = path or LIB_PATH
        if not os.path.exists(target):
            raise NativeError(
                f"libctqw.so not found at {target}; build it with "
                f"`make -C paper_1612_00746_b200/csrc` (the B200 path has no CPU fallback)"
            )
        lib = ctypes.CDLL(target)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _raise_for(code: int, handle=None):
    if code == 0:
        return
    lib = load_library()
    msg = (lib.ctqw_last_error(handle) or b"").decode(errors="replace")
    if code == 2:
        raise ConfigurationError(msg)
    if code == 3:
        raise NumericError(msg)
    if code == 4:
        raise CapacityError(msg)
    raise NativeError(msg or f"libctqw error {code}")


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(device_index: int) -> int:
    import torch

    return int(torch.cuda.current_stream(device_index).cuda_stream)


def make_stepper(backend: str, order: int, dt: float, tol_norm: float, tol_fail: float,
                 renormalize: bool, exact: bool) -> Stepper:
    if backend not in BACKEND_CODES:
        raise ConfigurationError(
            f"backend {backend!r} is not on the B200 path; use 'taylor' or 'rk4'"
        )
    return Stepper(BACKEND_CODES[backend], int(order), float(dt), float(tol_norm),
                   float(tol_fail), 1 if renormalize else 0, 1 if exact else 0)


class Handle:
    """One ``ctqw_handle_t``: a model bound to a CUDA device."""

    def __init__(self, m: int, n_sites: int, onsite: float, tunneling: float,
                 interaction: float, hbar: float, device: int = 0, lattice=None):
        """``lattice`` = (pos, neg, t_slot) move tables of a general lattice
        ((N, K) int arrays, -1 off-lattice; (K,) tunnelling per slot), None
        for the periodic nearest-neighbour ring."""
        import torch

        if not torch.cuda.is_available():
            raise NativeError("no CUDA device: the B200 path has no CPU fallback")
        self.lib = load_library()
        self.device = int(device)
        self.m = int(m)
        self.n = int(n_sites)
        self.dim = self.n ** self.m
        self.K = 1 if lattice is None else int(np.shape(lattice[0])[1])
        model = Model(self.m, self.n, self.K, 1 if lattice is None else 0, float(onsite), float(tunneling),
                      float(interaction), float(hbar))
        h = _P()
        code = self.lib.ctqw_create(ctypes.byref(model), self.device, ctypes.byref(h))
        _raise_for(code, None)
        self._h = h
        self._bound = None  # keep coefficient tensors alive
        if lattice is not None:
            pos = np.ascontiguousarray(lattice[0], dtype=np.int32)
            neg = np.ascontiguousarray(lattice[1], dtype=np.int32)
            ts = np.ascontiguousarray(lattice[2], dtype=np.float64)
            self._check(self.lib.ctqw_set_lattice(
                self._h, self.K, pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                neg.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ts.ctypes.data_as(ctypes.POINTER(_D))))

    # -- lifecycle -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self.lib.ctqw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code):
        _raise_for(code, self._h)

    @property
    def stream(self) -> int:
        return _stream(self.device)

    @property
    def launches(self) -> int:
        return int(self.lib.ctqw_launch_count(self._h))

    # -- noise and coefficients -----------------------------------------
    def draw_noise(self, master_seed: int, r0: int, count: int, levels, total: int, out):
        arr = (ctypes.c_double * len(levels))(*[float(v) for v in levels])
        self._check(self.lib.ctqw_draw_noise(self._h, int(master_seed), int(r0), int(count), arr,
                                             len(levels), int(total), _ptr(out), self.stream))

    def telegraph_init(self, master_seed: int, r0: int, count: int, levels, n_links: int, n_sites: int,
                       rate: float):
        arr = (ctypes.c_double * len(levels))(*[float(v) for v in levels])
        self._check(self.lib.ctqw_telegraph_init(self._h, int(master_seed), int(r0), int(count), arr, len(levels),
                                                 int(n_links), int(n_sites), float(rate), self.stream))

    def telegraph_values_ptr(self) -> int:
        """Device pointer of the process values ``[count][n_links + n_sites]``."""
        return int(self.lib.ctqw_telegraph_values(self._h) or 0)

    def telegraph_advance(self, count: int, dt: float):
        self._check(self.lib.ctqw_telegraph_advance(self._h, int(count), float(dt), self.stream))

    def telegraph_enable(self, enable: bool):
        self._check(self.lib.ctqw_telegraph_enable(self._h, 1 if enable else 0))

    def telegraph_read(self, count: int, values=None, next_switch=None):
        """(times, switch counts) per realization; optionally copies values /
        next switch times into the given ``(count, total)`` device tensors."""
        times = (ctypes.c_double * max(count, 1))()
        sw = (ctypes.c_int64 * max(count, 1))()
        self._check(self.lib.ctqw_telegraph_read(self._h, _ptr(values), _ptr(next_switch), times, sw,
                                                 self.stream))
        return [times[i] for i in range(count)], [sw[i] for i in range(count)]

    def build_coefficients_from_ptr(self, noise_ptr: int, count: int, n_links: int, n_sites: int, hop, site):
        self._check(self.lib.ctqw_build_coefficients(self._h, ctypes.c_void_p(noise_ptr), int(count),
                                                     int(n_links), int(n_sites), _ptr(hop), _ptr(site),
                                                     self.stream))

    def build_coefficients(self, noise, count: int, n_links: int, n_sites: int, hop, site):
        self._check(self.lib.ctqw_build_coefficients(self._h, _ptr(noise), int(count), int(n_links),
                                                     int(n_sites), _ptr(hop), _ptr(site),
                                                     self.stream))

    def bind(self, hop, site, count: int, stride: int):
        self._bound = (hop, site)
        self._check(self.lib.ctqw_bind_coefficients(self._h, int(count), _ptr(hop), _ptr(site),
                                                    int(stride)))

    # -- compute ----------------------------------------------------------
    def fill_states(self, psi, count: int, psi0):
        self._check(self.lib.ctqw_fill_states(self._h, _ptr(psi), int(count), _ptr(psi0),
                                              self.stream))

    def apply(self, psi, out, count: int, exact: bool = True):
        self._check(self.lib.ctqw_apply(self._h, _ptr(psi), _ptr(out), int(count),
                                        1 if exact else 0, self.stream))

    def step(self, psi, out, count: int, stepper: Stepper):
        self._check(self.lib.ctqw_step(self._h, _ptr(psi), _ptr(out), int(count),
                                       ctypes.byref(stepper), self.stream))

    def check_norm(self, psi, count: int, stepper: Stepper, deviations, corrected):
        row = _I64(-1)
        dev = _D(0.0)
        code = self.lib.ctqw_check_norm(self._h, _ptr(psi), int(count), ctypes.byref(stepper),
                                        _ptr(deviations), _ptr(corrected), ctypes.byref(row),
                                        ctypes.byref(dev), self.stream)
        if code == 3:
            raise NormFailureError(dev.value, realization=int(row.value))
        self._check(code)

    def evolve(self, psi, work, count: int, first_step: int, n_steps: int,
               stepper: Stepper) -> bool:
        flag = _I32(0)
        self._check(self.lib.ctqw_evolve(self._h, _ptr(psi), _ptr(work), int(count),
                                         int(first_step), int(n_steps), ctypes.byref(stepper),
                                         ctypes.byref(flag), self.stream))
        return bool(flag.value)

    def set_initial(self, psi0):
        self._initial = psi0  # kept alive until the next evolve reads it
        self._check(self.lib.ctqw_set_initial(self._h, _ptr(psi0)))

    def evolve_observe(self, psi, work, count: int, first_step: int, n_steps: int, post_rate: int, acc,
                       stepper: Stepper, keep_stats: bool = False, snap=None) -> bool:
        flag = _I32(0)
        self._check(self.lib.ctqw_evolve_observe(self._h, _ptr(psi), _ptr(work), int(count), int(first_step),
                                                 int(n_steps), int(post_rate), _ptr(acc), _ptr(snap),
                                                 ctypes.byref(stepper), int(bool(keep_stats)), ctypes.byref(flag),
                                                 self.stream))
        return bool(flag.value)

    def segment_events(self, r0: int, step_lo: int, step_hi: int) -> SegmentStats:
        st = SegmentStats()
        self._check(self.lib.ctqw_segment_events(self._h, int(r0), int(step_lo), int(step_hi), ctypes.byref(st),
                                                 self.stream))
        return st

    def observe_points(self, acc, npoints: int, total: float, out, diag=None):
        self._check(self.lib.ctqw_observe_points(self._h, _ptr(acc), int(npoints), float(total), _ptr(out),
                                                 _ptr(diag), self.stream))

    def segment_stats(self, r0: int = 0) -> SegmentStats:
        st = SegmentStats()
        code = self.lib.ctqw_segment_stats(self._h, int(r0), ctypes.byref(st), self.stream)
        if code not in (0, 3):
            self._check(code)
        return st

    def observe_diag(self, psi, count: int, diag_sum, accumulate: bool = False):
        self._check(self.lib.ctqw_observe_diag(self._h, _ptr(psi), int(count), _ptr(diag_sum),
                                               1 if accumulate else 0, self.stream))

    def observe_diag_fixed(self, psi, count: int, acc, accumulate: bool = False):
        """acc[3][D] (int64) (+)= exact limbs of sum_r |psi_r|^2 (order independent)."""
        self._check(self.lib.ctqw_observe_diag_fixed(self._h, _ptr(psi) if count else None, int(count), _ptr(acc),
                                                     int(bool(accumulate)), self.stream))

    def fixed_to_double(self, acc, diag):
        self._check(self.lib.ctqw_fixed_to_double(self._h, _ptr(acc), _ptr(diag), self.stream))

    def observe_reduce(self, diag_sum, total: float, pops, scalars, joint=None):
        self._check(self.lib.ctqw_observe_reduce(self._h, _ptr(diag_sum), float(total), _ptr(pops),
                                                 _ptr(scalars), _ptr(joint), self.stream))

    def kernel_timing(self, enable: bool):
        self._check(self.lib.ctqw_kernel_timing(self._h, 1 if enable else 0))

    def kernel_time(self):
        """(summed ms, bracketed launches) since timing was enabled/last read."""
        ms = _D(0.0)
        n = _I64(0)
        self._check(self.lib.ctqw_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n), self.stream))
        return float(ms.value), int(n.value)

    def step_kernel(self) -> str:
        """Name of the dominant kernel the last evolve ran ('' = generic path)."""
        return (self.lib.ctqw_step_kernel(self._h) or b"").decode()

    def step_variant(self) -> str:
        """Its compile-time specialization (template arguments)."""
        return (self.lib.ctqw_step_variant(self._h) or b"").decode()

    def overlap_sumsq(self, a, count_a: int, b, count_b: int, out):
        self._check(self.lib.ctqw_overlap_sumsq(self._h, _ptr(a), int(count_a), _ptr(b),
                                                int(count_b), _ptr(out), self.stream))

    def overlap_sumsq_points(self, stacks, count: int, npoints: int, point_stride: int, out):
        """out[p] = sum_{i,j} |<a_i|a_j>|^2 for the stack at stacks + p * point_stride."""
        self._check(self.lib.ctqw_overlap_sumsq_points(self._h, _ptr(stacks), int(count), int(npoints),
                                                       int(point_stride), _ptr(out), self.stream))


def packed_gram(stack, count: int, packed, scale: float):
    """packed[i(i+1)/2 + j] = scale * sum_r stack[r, i] conj(stack[r, j]), j <= i
    (hand-written triangle-only kernel; density.py:91-95)."""
    lib = load_library()
    dev = stack.device.index
    code = lib.ctqw_packed_gram(_ptr(stack), int(count), int(stack.shape[1]), float(scale), _ptr(packed),
                                int(dev), _stream(dev))
    _raise_for(code, None)


def exported_symbols(path: str | None = None) -> list[str]:
    """Names of the C-ABI entry points the library exports (CPU-safe check)."""
    lib = load_library(path)
    return [name for name in SIGNATURES if hasattr(lib, name)]


__all__ = ["Handle", "Model", "Stepper", "SegmentStats", "load_library", "exported_symbols",
           "make_stepper", "packed_gram", "CtqwError", "LIB_PATH", "SIGNATURES"]
