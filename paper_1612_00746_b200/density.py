"""Dense ensemble-averaged density matrix.

The reference's ``accumulate_density`` (``density.py:57-98``) forms
``gram = stack.T @ stack.conj()`` over the whole (R, D) stack, keeps the
lower triangle row-major (``packed[i*(i+1)/2 + j]`` = entry (i, j), j <= i)
and divides by R.  The hot path only needs diag(rho) (``observables.py``:
``DiagonalDensity``); this module provides the dense rho for callers and
sinks that want it:

* ``accumulate_density(states, time_tag)`` -- the reference's function, on
  the GPU: the Gram product runs in a hand-written triangle-only kernel
  (``csrc/density_gram.cu``, HERK-style: half the multiply-adds of the
  reference's full GEMM, no D x D transient) that writes the packed lower
  triangle directly; it reaches the host only when ``DensityMatrix.packed``
  is read;
* ``run`` computes it at every collection point for sinks whose
  ``dense_density`` attribute is true (``MemorySinks(dense=True)``), within
  the reference's own size limit (the D x D transient).

Results equal the reference's to rounding (BLAS summation order), checked to
1e-15 against its own output in ``tests/test_gpu_parity.py``.
"""

from __future__ import annotations

import numpy as np

from .errors import CapacityError, ConsistencyError

TIME_TAG_SLACK = 1e-9
# D x D complex128 transient of the Gram product; the reference's own
# feasibility limit under its default 4 GiB budget is D ~ 22.8k
DENSE_DIM_CAP = 32768


def packed_length(dim: int) -> int:
    return dim * (dim + 1) // 2


class DensityMatrix:
    """Lower-triangle ensemble average rho(t) with its provenance counts
    (the reference's ``DensityMatrix``, density.py:26-54).  ``packed`` may
    stay on the device until first read."""

    def __init__(self, packed, dim, sample_count, time_tag, device_packed=None):
        self._packed = None if packed is None else np.asarray(packed, dtype=np.complex128)
        self._device_packed = device_packed
        self.dim = int(dim)
        self.sample_count = int(sample_count)
        self.time_tag = float(time_tag)
        n = self._packed.shape[0] if self._packed is not None else int(device_packed.shape[0])
        if n != packed_length(self.dim):
            raise ConsistencyError(f"packed length ({n},) does not fit dimension {self.dim}")

    @property
    def packed(self) -> np.ndarray:
        if self._packed is None:
            self._packed = self._device_packed.cpu().numpy()
            self._device_packed = None
        return self._packed

    def diagonal(self) -> np.ndarray:
        idx = np.arange(self.dim, dtype=np.int64)
        return self.packed[idx * (idx + 1) // 2 + idx]

    def trace(self) -> float:
        return float(self.diagonal().real.sum())

    def dense(self) -> np.ndarray:
        """Expand to the full Hermitian matrix (quadratic memory)."""
        out = np.zeros((self.dim, self.dim), dtype=np.complex128)
        rows, cols = np.tril_indices(self.dim)
        out[rows, cols] = self.packed
        out[cols, rows] = np.conj(self.packed)
        return out

    @property
    def purity(self) -> float:
        """tr(rho^2) = 2 sum |packed|^2 - sum |diag|^2 (observables.py:86-91)."""
        p = self.packed
        d = self.diagonal()
        return float(2.0 * np.sum(np.abs(p) ** 2) - np.sum(np.abs(d) ** 2))


def packed_density_device(stack_dev, count: int, scale: float | None = None):
    """Packed scale * lower(stack^T conj(stack)) of a device (R, D) complex128
    stack (density.py:91-96; default scale 1/R, NumPy's ``packed /= r``
    multiplies by the reciprocal), by ``ctqw_packed_gram``."""
    import torch

    from . import native

    dim = stack_dev.shape[1]
    if dim > DENSE_DIM_CAP:
        raise CapacityError(f"dense density of dimension {dim} exceeds the cap {DENSE_DIM_CAP}")
    s = stack_dev[:count].contiguous()
    packed = torch.empty(packed_length(dim), dtype=torch.complex128, device=s.device)
    native.packed_gram(s, count, packed, 1.0 / count if scale is None else scale)
    return packed


def accumulate_density(states, time_tag: float | None = None) -> DensityMatrix:
    """Average projectors over a stack of realizations (density.py:57-98).

    ``states`` is a sequence of ``WaveFunction`` (agreeing time tags) or a
    bare (R, dim) array / CUDA tensor with an explicit ``time_tag``."""
    import torch

    from .engine import _default_device

    if isinstance(states, (np.ndarray, torch.Tensor)):
        stack = states
        if stack.ndim != 2:
            raise ConsistencyError(f"expected an (R, dim) stack, got {tuple(stack.shape)}")
        if time_tag is None:
            raise ConsistencyError("a bare stack needs an explicit time_tag")
    else:
        states = list(states)
        if not states:
            raise ConsistencyError("no states to average")
        tags = np.array([w.time_tag for w in states], dtype=np.float64)
        spread = tags.max() - tags.min()
        if spread > TIME_TAG_SLACK * max(1.0, abs(float(tags[0]))):
            raise ConsistencyError(
                f"states carry mixed time tags (spread {spread:.3e}); "
                f"an average across different times is not a state")
        if time_tag is None:
            time_tag = float(tags[0])
        stack = np.stack([w.amplitudes for w in states])
    if isinstance(stack, torch.Tensor) and stack.is_cuda:
        dev = stack.to(torch.complex128)
    else:
        dev = torch.as_tensor(np.asarray(stack).astype(np.complex128, copy=False),
                              device=f"cuda:{_default_device()}")
    r = int(dev.shape[0])
    packed = packed_density_device(dev, r)
    return DensityMatrix(None, dim=int(dev.shape[1]), sample_count=r, time_tag=float(time_tag),
                         device_packed=packed)
