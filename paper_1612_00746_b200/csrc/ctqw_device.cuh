// Shared device-side definitions for libctqw (sm_100a).
//
// Complex128 amplitudes are double2 {re, im}.  Two arithmetic modes:
//   EXACT = true : every product and sum rounded separately, in the order the
//                  reference's NumPy expressions evaluate them
//                  (hamiltonian.py:205-222, propagators.py:185-193,213-240), so
//                  results are bit-identical to the reference between rescales.
//   EXACT = false: the neighbour accumulations contract into DFMA (fewer FP64
//                  instructions, one rounding per term instead of two).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ctqw {

constexpr int kMaxEvents = 100;     // ensemble.py:119
constexpr long long kNoFail = 0x7fffffffffffffffLL;

// Coefficient rows of a batch: realization i reads hop + i*stride and
// site + i*site_stride.  Ring (q = 1, K = 1, periodic): hop[x] couples
// x -> x+1.  General lattices (pos != nullptr, generic kernels only):
// hop[x*K + s] couples x -> pos[x*K + s] (the reference's link
// x*K + s, hilbert.py:303-314), pos / neg = targets of the signed moves,
// -1 off-lattice (hilbert.py:189-224).
struct Coef {
  const double* hop;    // [.][N*K]  t_dir + xi_link
  const double* site;   // [.][N]    xi_site[x], nullptr when absent
  int64_t stride;       // 0 = broadcast
  int64_t site_stride;
  const int* pos = nullptr;  // [N][K] general lattice move tables (device)
  const int* neg = nullptr;
  int K = 1;
};

// Norm policy, StepperConfig (propagators.py:61-86).
struct NormPolicy {
  double tol_norm;
  double tol_fail;
  int renormalize;
};

// Per-realization statistics of one evolve call (ensemble.py:459-533).
struct RealStat {
  long long events;
  long long corrections;
  long long fail_step;    // kNoFail if none
  double max_dev;
  double fail_dev;
  int n_ev;               // events stored (<= kMaxEvents)
  int pad;
};

struct EventRec {
  double dev;
  int step_lo;            // step number (fits 31 bits for any practical run)
  int corrected;
};

__device__ __forceinline__ double2 cmake(double re, double im) { return make_double2(re, im); }

// acc + v*z for a real coupling v (values are complex with zero imaginary
// part in the reference; (v + 0i)*z rounds exactly like v*z component-wise).
template <bool EXACT>
__device__ __forceinline__ double2 madd(double2 acc, double v, double2 z) {
  if (EXACT) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, z.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, z.y));
  } else {
    acc.x = fma(v, z.x, acc.x);
    acc.y = fma(v, z.y, acc.y);
  }
  return acc;
}

__device__ __forceinline__ double2 rmul(double v, double2 z) {
  return cmake(__dmul_rn(v, z.x), __dmul_rn(v, z.y));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return cmake(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// z * (0 + ci i): the Taylor/RK4 coefficient -1j*dt/hbar/j has a zero real
// part, so NumPy's complex product reduces to (-b*ci, a*ci) exactly.
__device__ __forceinline__ double2 times_i(double ci, double2 z) {
  return cmake(__dmul_rn(-z.y, ci), __dmul_rn(z.x, ci));
}

// x + (0 + w i) * h with one DFMA per component (FMA-mode stage arithmetic:
// the Taylor/RK4 coefficient times i folded into the accumulation)
__device__ __forceinline__ double2 ifma(double2 x, double w, double2 h) {
  return cmake(fma(-w, h.y, x.x), fma(w, h.x, x.y));
}

__device__ __forceinline__ double norm2(double2 z) { return z.x * z.x + z.y * z.y; }

__device__ __forceinline__ int wrap(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// Block-wide sum; result valid in thread 0.  Deterministic for a fixed
// block size (fixed shuffle tree, fixed warp order).
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nwarps; ++w) s += red[w];
  return s;
}

// The norm policy for one realization after one step (propagators.py:316-327
// + ensemble.py:509-533).  Returns the factor the state must be multiplied
// by (1/sqrt(n2) when corrected -- NumPy's complex division by a real
// multiplies by the reciprocal -- else exactly 1.0).  Sets *failed.
__device__ __forceinline__ double norm_decide(double n2, long long step, const NormPolicy& pol,
                                              RealStat* st, EventRec* ev, int* failed) {
  const double dev = fabs(n2 - 1.0);
  *failed = 0;
  if (dev > pol.tol_fail) {
    if (st->fail_step == kNoFail) {
      st->fail_step = step;
      st->fail_dev = dev;
    }
    *failed = 1;
    return 1.0;
  }
  if (dev > st->max_dev) st->max_dev = dev;
  if (dev > pol.tol_norm) {
    const int corrected = pol.renormalize ? 1 : 0;
    st->events += 1;
    st->corrections += corrected;
    if (st->n_ev < kMaxEvents) {
      EventRec e;
      e.dev = dev;
      e.step_lo = (int)step;
      e.corrected = corrected;
      ev[st->n_ev] = e;
      st->n_ev += 1;
    }
    if (corrected) return __ddiv_rn(1.0, __dsqrt_rn(n2));
  }
  return 1.0;
}

// Exact (order-independent) ensemble sums of |psi_r(alpha)|^2.
//
// Each term x = |psi|^2 (x <= 2^22) is split, exactly and deterministically,
// into three pieces on the fixed grids 2^-30, 2^-70 and 2^-110
// (x = a2 + a1 + a0 + (rounding below 2^-111)), and each piece is added as an
// int64 multiple of its grid: limb k of [3][dim].  Integer addition is
// associative, so the sum is the same bits for any realization order, any
// split of the realizations over blocks, atomics or GPUs (the all-reduce of
// the limbs is an int64 SUM).  This is what makes the observables identical
// across 1/2/4/8 GPUs, as the reference's are across worker counts
// (pkg/README.md:174-180).  Limbs hold up to 2^23 realizations without
// overflow.  Terms below 2^-111 (far beneath the 1e-10 relative bar on any
// entry above 1e-30) are dropped.
__device__ __forceinline__ void fixed_split(double x, long long& l2, long long& l1, long long& l0) {
  const double c2 = 0x1.8p22, c1 = 0x1.8p-18, c0 = 0x1.8p-58;
  const double a2 = __dsub_rn(__dadd_rn(x, c2), c2);  // nearest multiple of 2^-30
  const double r1 = __dsub_rn(x, a2);                 // exact
  const double a1 = __dsub_rn(__dadd_rn(r1, c1), c1); // nearest multiple of 2^-70
  const double r0 = __dsub_rn(r1, a1);                // exact
  const double a0 = __dsub_rn(__dadd_rn(r0, c0), c0); // nearest multiple of 2^-110
  l2 = __double2ll_rn(__dmul_rn(a2, 0x1p30));
  l1 = __double2ll_rn(__dmul_rn(a1, 0x1p70));
  l0 = __double2ll_rn(__dmul_rn(a0, 0x1p110));
}

// |z|^2 = re*re + im*im, each product rounded (no FMA contraction), as NumPy
// forms it: the term -- and so its limbs -- is a pure function of z.
__device__ __forceinline__ double norm2_rn(double2 z) { return __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y)); }

}  // namespace ctqw
