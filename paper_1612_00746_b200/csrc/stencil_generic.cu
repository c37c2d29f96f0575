// General-m stencil kernels (m = 1, 2, 3 on a periodic ring, any Taylor
// order): one launch per operator application, neighbours gathered through
// L1/L2.  This is the coverage path -- every (m, order, backend) the
// reference's propagators support on this geometry -- and the engine behind
// the single-step API (apply_values / step_taylor_values / step_rk4_values,
// hamiltonian.py:195-223, propagators.py:167-241).  The m = 2 hot path runs
// through the fused tile kernels in step_tile.cu instead.
#include "ctqw_device.cuh"
#include "kernels.h"

namespace ctqw {

namespace {

constexpr int kBlock = 256;

template <int M>
struct Digits {
  int x[M];
};

template <int M>
__device__ __forceinline__ Digits<M> digits_of(int64_t a, int n) {
  Digits<M> d;
  int64_t rem = a;
#pragma unroll
  for (int p = M - 1; p >= 0; --p) {
    d.x[p] = (int)(rem % n);
    rem /= n;
  }
  return d;
}

// (H t)(a) in the reference accumulation order: diagonal, then for each
// particle slot p the +move then the -move (hamiltonian.py:205-222).  The
// -move reads the coupling stored at its target row, hop[x_p - 1]
// (hamiltonian.py:216).  SCALE multiplies every loaded amplitude by s first
// (the pending norm rescale of the previous step, see evolve).
template <int M, bool EXACT, bool SITE, bool SCALE>
__device__ __forceinline__ double2 stencil_point(const double2* __restrict__ t, int64_t a, int n,
                                                 const double* __restrict__ hop,
                                                 const double* __restrict__ site,
                                                 const StencilConst& k, double s) {
  const Digits<M> d = digits_of<M>(a, n);
  int c = 0;
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = p + 1; q < M; ++q) c += (d.x[p] == d.x[q]);
  double v0 = k.base[c];
  if (SITE) {
    double ss = site[d.x[0]];
#pragma unroll
    for (int p = 1; p < M; ++p) ss = __dadd_rn(ss, site[d.x[p]]);  // ndarray.sum, left-assoc
    v0 = __dadd_rn(v0, ss);
  }
  double2 self = t[a];
  if (SCALE) self = rmul(s, self);
  double2 acc = rmul(v0, self);
  int64_t stride = 1;
  int64_t strides[M];
#pragma unroll
  for (int p = M - 1; p >= 0; --p) {
    strides[p] = stride;
    stride *= n;
  }
#pragma unroll
  for (int p = 0; p < M; ++p) {
    const int xp = d.x[p];
    const int64_t st = strides[p];
    const int64_t ap = (xp == n - 1) ? a - (int64_t)(n - 1) * st : a + st;
    const int64_t am = (xp == 0) ? a + (int64_t)(n - 1) * st : a - st;
    double2 up = t[ap], dn = t[am];
    if (SCALE) {
      up = rmul(s, up);
      dn = rmul(s, dn);
    }
    acc = madd<EXACT>(acc, hop[xp], up);
    acc = madd<EXACT>(acc, hop[xp == 0 ? n - 1 : xp - 1], dn);
  }
  return acc;
}

// General lattices (q >= 1, K = sum(k_half) slots per site, periodic or
// open): the same accumulation order -- diagonal, then for each particle p
// and site slot s the +move and the -move (stored slot j = 1 + p*K + s,
// hamiltonian.py:205-222).  The -move reads the coupling stored at its
// target row: the link of the target site, hop[neg*K + s].  Moves off an
// open lattice contribute nothing (the reference adds an exact zero).
template <int M, bool EXACT, bool SITE, bool SCALE>
__device__ __forceinline__ double2 stencil_point_lat(const double2* __restrict__ t, int64_t a, int n,
                                                     const double* __restrict__ hop,
                                                     const double* __restrict__ site, const Coef& coef,
                                                     const StencilConst& k, double s) {
  const Digits<M> d = digits_of<M>(a, n);
  int c = 0;
#pragma unroll
  for (int p = 0; p < M; ++p)
#pragma unroll
    for (int q = p + 1; q < M; ++q) c += (d.x[p] == d.x[q]);
  double v0 = k.base[c];
  if (SITE) {
    double ss = site[d.x[0]];
#pragma unroll
    for (int p = 1; p < M; ++p) ss = __dadd_rn(ss, site[d.x[p]]);
    v0 = __dadd_rn(v0, ss);
  }
  double2 self = t[a];
  if (SCALE) self = rmul(s, self);
  double2 acc = rmul(v0, self);
  int64_t stride = 1;
  int64_t strides[M];
#pragma unroll
  for (int p = M - 1; p >= 0; --p) {
    strides[p] = stride;
    stride *= n;
  }
  const int K = coef.K;
#pragma unroll
  for (int p = 0; p < M; ++p) {
    const int xp = d.x[p];
    for (int sl = 0; sl < K; ++sl) {
      const int tgt = coef.pos[xp * K + sl];
      if (tgt >= 0) {
        double2 z = t[a + (int64_t)(tgt - xp) * strides[p]];
        if (SCALE) z = rmul(s, z);
        acc = madd<EXACT>(acc, hop[xp * K + sl], z);
      }
      const int src = coef.neg[xp * K + sl];
      if (src >= 0) {
        double2 z = t[a + (int64_t)(src - xp) * strides[p]];
        if (SCALE) z = rmul(s, z);
        acc = madd<EXACT>(acc, hop[src * K + sl], z);
      }
    }
  }
  return acc;
}

template <int M, bool EXACT, bool SITE, bool SCALE>
__device__ __forceinline__ double2 stencil_any(const double2* __restrict__ t, int64_t a, int n,
                                               const double* __restrict__ hop, const double* __restrict__ site,
                                               const Coef& coef, const StencilConst& k, double s) {
  if (coef.pos) return stencil_point_lat<M, EXACT, SITE, SCALE>(t, a, n, hop, site, coef, k, s);
  return stencil_point<M, EXACT, SITE, SCALE>(t, a, n, hop, site, k, s);
}

template <int M, bool EXACT, bool SITE>
__global__ void __launch_bounds__(kBlock) apply_kernel(const double2* __restrict__ psi,
                                                       double2* __restrict__ out, int64_t dim,
                                                       int n, Coef coef, StencilConst k,
                                                       int64_t r_base) {
  const int64_t r = r_base + blockIdx.y;
  const double2* t = psi + r * dim;
  const double* hop = coef.hop + r * coef.stride;
  const double* site = SITE ? coef.site + r * coef.site_stride : nullptr;
  for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * kBlock)
    out[r * dim + a] = stencil_any<M, EXACT, SITE, false>(t, a, n, hop, site, coef, k, 1.0);
}

// One Taylor order: term_out = (coeff/j) * H term_in; acc_out = acc_in + term_out
// (propagators.py:189-193).  SCALE: term_in and acc_in are the step's input
// state with its pending rescale.  term_out may be null (last order).
// partial (optional) receives per-block sums of |acc_out|^2.
template <int M, bool EXACT, bool SITE, bool SCALE>
__global__ void __launch_bounds__(kBlock) taylor_order_kernel(
    const double2* __restrict__ term_in, double2* __restrict__ term_out,
    const double2* acc_in, double2* acc_out, int64_t dim, int n, Coef coef, StencilConst k,
    double ci, const double* __restrict__ scl, double* __restrict__ partial, int nparts,
    int64_t r_base, const long long* __restrict__ fail_step) {
  __shared__ double red[kBlock / 32];
  if (fail_step && *fail_step != kNoFail) return;
  const int64_t r = r_base + blockIdx.y;
  const double s = SCALE ? scl[r] : 1.0;
  const double2* t = term_in + r * dim;
  const double* hop = coef.hop + r * coef.stride;
  const double* site = SITE ? coef.site + r * coef.site_stride : nullptr;
  double nrm = 0.0;
  for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * kBlock) {
    const double2 h = stencil_any<M, EXACT, SITE, SCALE>(t, a, n, hop, site, coef, k, s);
    const double2 tk = times_i(ci, h);
    double2 acc = acc_in[r * dim + a];
    if (SCALE) acc = rmul(s, acc);
    acc = cadd(acc, tk);
    if (term_out) term_out[r * dim + a] = tk;
    acc_out[r * dim + a] = acc;
    nrm += norm2(acc);
  }
  if (partial) {
    const double b = block_sum(nrm, red);
    if (threadIdx.x == 0) partial[r * nparts + blockIdx.x] = b;
  }
}

// One RK4 stage (propagators.py:213-240).  stage = coeff * H arg_in, then
//   1: arg = 0.5*stage + psi ; out = psi + stage/6
//   2: arg = 0.5*stage + psi ; out += stage/3
//   3: arg = stage + psi     ; out += stage/3
//   4:                         out += stage/6
template <int M, bool EXACT, bool SITE, bool SCALE>
__global__ void __launch_bounds__(kBlock) rk4_stage_kernel(
    int stage, const double2* __restrict__ arg_in, const double2* psi,
    const double2* out_in, double2* __restrict__ arg_out, double2* out_out, int64_t dim, int n,
    Coef coef, StencilConst k, double ci, const double* __restrict__ scl,
    double* __restrict__ partial, int nparts, int64_t r_base,
    const long long* __restrict__ fail_step) {
  __shared__ double red[kBlock / 32];
  if (fail_step && *fail_step != kNoFail) return;
  const int64_t r = r_base + blockIdx.y;
  const double s = SCALE ? scl[r] : 1.0;
  const double* hop = coef.hop + r * coef.stride;
  const double* site = SITE ? coef.site + r * coef.site_stride : nullptr;
  const double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  double nrm = 0.0;
  for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * kBlock) {
    const int64_t g = r * dim + a;
    // arg_in of stage 1 is psi itself (scaled); later stages read unscaled scratch
    double2 h;
    if (stage == 1)
      h = stencil_any<M, EXACT, SITE, SCALE>(arg_in + r * dim, a, n, hop, site, coef, k, s);
    else
      h = stencil_any<M, EXACT, SITE, false>(arg_in + r * dim, a, n, hop, site, coef, k, 1.0);
    const double2 st = times_i(ci, h);
    double2 p0 = make_double2(0.0, 0.0);
    if (stage < 4) {
      p0 = psi[g];
      if (SCALE) p0 = rmul(s, p0);
    }
    double2 o;
    if (stage == 1) {
      arg_out[g] = cadd(rmul(0.5, st), p0);
      o = cadd(p0, rmul(c16, st));
    } else if (stage == 2) {
      arg_out[g] = cadd(rmul(0.5, st), p0);
      o = cadd(out_in[g], rmul(c13, st));
    } else if (stage == 3) {
      arg_out[g] = cadd(st, p0);
      o = cadd(out_in[g], rmul(c13, st));
    } else {
      o = cadd(out_in[g], rmul(c16, st));
    }
    out_out[g] = o;
    if (stage == 4) nrm += norm2(o);
  }
  if (partial && stage == 4) {
    const double b = block_sum(nrm, red);
    if (threadIdx.x == 0) partial[r * nparts + blockIdx.x] = b;
  }
}

__global__ void __launch_bounds__(kBlock) norm_partial_kernel(const double2* __restrict__ psi,
                                                              int64_t dim, double* partial,
                                                              int nparts, int64_t r_base) {
  __shared__ double red[kBlock / 32];
  const int64_t r = r_base + blockIdx.y;
  double nrm = 0.0;
  for (int64_t a = (int64_t)blockIdx.x * kBlock + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * kBlock)
    nrm += norm2(psi[r * dim + a]);
  const double b = block_sum(nrm, red);
  if (threadIdx.x == 0) partial[r * nparts + blockIdx.x] = b;
}

inline dim3 grid_for(int64_t dim, int64_t rows, int nparts) {
  (void)dim;
  return dim3((unsigned)nparts, (unsigned)rows);
}

template <int M>
cudaError_t apply_m(const double2* psi, double2* out, int64_t count, int64_t dim, int n,
                    const Coef& coef, const StencilConst& k, bool exact, cudaStream_t s) {
  const int nparts = generic_parts(dim);
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    const dim3 grid = grid_for(dim, rows, nparts);
    const bool site = coef.site != nullptr;
    if (exact && site) apply_kernel<M, true, true><<<grid, kBlock, 0, s>>>(psi, out, dim, n, coef, k, r0);
    else if (exact) apply_kernel<M, true, false><<<grid, kBlock, 0, s>>>(psi, out, dim, n, coef, k, r0);
    else if (site) apply_kernel<M, false, true><<<grid, kBlock, 0, s>>>(psi, out, dim, n, coef, k, r0);
    else apply_kernel<M, false, false><<<grid, kBlock, 0, s>>>(psi, out, dim, n, coef, k, r0);
  }
  return cudaGetLastError();
}

template <int M, bool EXACT, bool SITE>
void taylor_dispatch(bool scale, dim3 grid, cudaStream_t s, const double2* ti, double2* to,
                     const double2* ai, double2* ao, int64_t dim, int n, const Coef& coef,
                     const StencilConst& k, double ci, const double* scl, double* partial,
                     int nparts, int64_t r0, const long long* fail) {
  if (scale)
    taylor_order_kernel<M, EXACT, SITE, true><<<grid, kBlock, 0, s>>>(
        ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else
    taylor_order_kernel<M, EXACT, SITE, false><<<grid, kBlock, 0, s>>>(
        ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
}

template <int M, bool EXACT, bool SITE>
void rk4_dispatch(bool scale, dim3 grid, cudaStream_t s, int stage, const double2* ai,
                  const double2* psi, const double2* oi, double2* ao, double2* oo, int64_t dim,
                  int n, const Coef& coef, const StencilConst& k, double ci, const double* scl,
                  double* partial, int nparts, int64_t r0, const long long* fail) {
  if (scale)
    rk4_stage_kernel<M, EXACT, SITE, true><<<grid, kBlock, 0, s>>>(
        stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else
    rk4_stage_kernel<M, EXACT, SITE, false><<<grid, kBlock, 0, s>>>(
        stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
}

template <int M>
void taylor_m(bool exact, bool site, bool scale, dim3 grid, cudaStream_t s, const double2* ti,
              double2* to, const double2* ai, double2* ao, int64_t dim, int n, const Coef& coef,
              const StencilConst& k, double ci, const double* scl, double* partial, int nparts,
              int64_t r0, const long long* fail) {
  if (exact && site) taylor_dispatch<M, true, true>(scale, grid, s, ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else if (exact) taylor_dispatch<M, true, false>(scale, grid, s, ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else if (site) taylor_dispatch<M, false, true>(scale, grid, s, ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else taylor_dispatch<M, false, false>(scale, grid, s, ti, to, ai, ao, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
}

template <int M>
void rk4_m(bool exact, bool site, bool scale, dim3 grid, cudaStream_t s, int stage,
           const double2* ai, const double2* psi, const double2* oi, double2* ao, double2* oo,
           int64_t dim, int n, const Coef& coef, const StencilConst& k, double ci,
           const double* scl, double* partial, int nparts, int64_t r0, const long long* fail) {
  if (exact && site) rk4_dispatch<M, true, true>(scale, grid, s, stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else if (exact) rk4_dispatch<M, true, false>(scale, grid, s, stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else if (site) rk4_dispatch<M, false, true>(scale, grid, s, stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
  else rk4_dispatch<M, false, false>(scale, grid, s, stage, ai, psi, oi, ao, oo, dim, n, coef, k, ci, scl, partial, nparts, r0, fail);
}

}  // namespace

int generic_parts(int64_t dim) {
  const int64_t blocks = (dim + kBlock - 1) / kBlock;
  return (int)(blocks < kMaxParts ? blocks : kMaxParts);
}

cudaError_t launch_apply(int m, const double2* psi, double2* out, int64_t count, int64_t dim,
                         int n, const Coef& coef, const StencilConst& k, bool exact,
                         cudaStream_t s) {
  switch (m) {
    case 1: return apply_m<1>(psi, out, count, dim, n, coef, k, exact, s);
    case 2: return apply_m<2>(psi, out, count, dim, n, coef, k, exact, s);
    case 3: return apply_m<3>(psi, out, count, dim, n, coef, k, exact, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_taylor_order(int m, bool exact, bool scale, const double2* term_in,
                                double2* term_out, const double2* acc_in, double2* acc_out,
                                int64_t count, int64_t dim, int n, const Coef& coef,
                                const StencilConst& k, double ci, const double* scl,
                                double* partial, const long long* fail, cudaStream_t s) {
  const int nparts = generic_parts(dim);
  const bool site = coef.site != nullptr;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    const dim3 grid = grid_for(dim, rows, nparts);
    switch (m) {
      case 1: taylor_m<1>(exact, site, scale, grid, s, term_in, term_out, acc_in, acc_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      case 2: taylor_m<2>(exact, site, scale, grid, s, term_in, term_out, acc_in, acc_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      case 3: taylor_m<3>(exact, site, scale, grid, s, term_in, term_out, acc_in, acc_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_rk4_stage(int m, bool exact, bool scale, int stage, const double2* arg_in,
                             const double2* psi, const double2* out_in, double2* arg_out,
                             double2* out_out, int64_t count, int64_t dim, int n,
                             const Coef& coef, const StencilConst& k, double ci,
                             const double* scl, double* partial, const long long* fail,
                             cudaStream_t s) {
  const int nparts = generic_parts(dim);
  const bool site = coef.site != nullptr;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    const dim3 grid = grid_for(dim, rows, nparts);
    switch (m) {
      case 1: rk4_m<1>(exact, site, scale, grid, s, stage, arg_in, psi, out_in, arg_out, out_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      case 2: rk4_m<2>(exact, site, scale, grid, s, stage, arg_in, psi, out_in, arg_out, out_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      case 3: rk4_m<3>(exact, site, scale, grid, s, stage, arg_in, psi, out_in, arg_out, out_out, dim, n, coef, k, ci, scl, partial, nparts, r0, fail); break;
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_norm_partial(const double2* psi, int64_t count, int64_t dim, double* partial,
                                cudaStream_t s) {
  const int nparts = generic_parts(dim);
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    norm_partial_kernel<<<grid_for(dim, rows, nparts), kBlock, 0, s>>>(psi, dim, partial, nparts, r0);
  }
  return cudaGetLastError();
}

}  // namespace ctqw
