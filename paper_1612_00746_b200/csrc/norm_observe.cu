// Norm policy bookkeeping and ensemble observables.
//
// Norm policy (propagators.py:309-328, ensemble.py:509-533): the step kernels
// leave per-realization |psi|^2 partials; norm_decide_kernel sums them in a
// fixed order, records deviation statistics/events and the rescale factor,
// which the NEXT step's kernel applies while loading (the step is linear, so a
// lazy rescale is exact).  rescale_kernel applies the last step's factor at
// the end of a segment.
//
// Observables: only diag(rho) = mean_r |psi_r|^2 is needed for populations,
// position moments, participation ratio and the joint distribution
// (observables.py:34-101); purity needs the realization overlaps
// sum_{r,s} |<psi_r|psi_s>|^2 instead of the dense D x D Gram
// (density.py:91-92).
#include "ctqw_device.cuh"
#include "kernels.h"

namespace ctqw {

namespace {

__global__ void norm_decide_kernel(const double* __restrict__ partial, int nparts, int64_t count,
                                   long long step, NormPolicy pol, double* scl, RealStat* stats,
                                   EventRec* events, long long* fail) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= count) return;
  if (*fail < step) return;  // an earlier step already failed: run is over
  double n2 = 0.0;
  const double* p = partial + r * nparts;
  for (int i = 0; i < nparts; ++i) n2 += p[i];
  int failed = 0;
  scl[r] = norm_decide(n2, step, pol, stats + r, events + r * kMaxEvents, &failed);
  if (failed) atomicMin(reinterpret_cast<unsigned long long*>(fail), (unsigned long long)step);
}

__global__ void rescale_kernel(double2* psi, int64_t dim, double* scl) {
  const int64_t r = blockIdx.y;
  const double s = scl[r];
  if (s == 1.0) return;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * blockDim.x)
    psi[r * dim + a] = rmul(s, psi[r * dim + a]);
}

__global__ void reset_scale_kernel(double* scl, int64_t count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < count) scl[r] = 1.0;
}

__global__ void reset_stats_kernel(RealStat* stats, double* scl, int64_t count, long long* fail) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) *fail = kNoFail;
  if (r >= count) return;
  RealStat z;
  z.events = 0;
  z.corrections = 0;
  z.fail_step = kNoFail;
  z.max_dev = 0.0;
  z.fail_dev = 0.0;
  z.n_ev = 0;
  z.pad = 0;
  stats[r] = z;
  scl[r] = 1.0;
}

// Totals over realizations; the failure is the earliest failing step, and at
// that step the largest deviation (np.argmax picks the lowest row on ties).
__global__ void stats_reduce_kernel(const RealStat* __restrict__ stats, int64_t count,
                                    Summary* out) {
  __shared__ long long s_ev[1024], s_cor[1024], s_fs[1024], s_fr[1024];
  __shared__ double s_md[1024], s_fd[1024];
  const int tid = threadIdx.x;
  long long ev = 0, cor = 0, fs = kNoFail, fr = -1;
  double md = 0.0, fd = 0.0;
  for (int64_t r = tid; r < count; r += blockDim.x) {
    const RealStat st = stats[r];
    ev += st.events;
    cor += st.corrections;
    if (st.max_dev > md) md = st.max_dev;
    if (st.fail_step != kNoFail) {
      if (st.fail_step < fs || (st.fail_step == fs && (st.fail_dev > fd || (st.fail_dev == fd && r < fr)))) {
        fs = st.fail_step;
        fd = st.fail_dev;
        fr = r;
      }
    }
  }
  s_ev[tid] = ev;
  s_cor[tid] = cor;
  s_md[tid] = md;
  s_fs[tid] = fs;
  s_fd[tid] = fd;
  s_fr[tid] = fr;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) {
      s_ev[tid] += s_ev[tid + o];
      s_cor[tid] += s_cor[tid + o];
      if (s_md[tid + o] > s_md[tid]) s_md[tid] = s_md[tid + o];
      const long long fs2 = s_fs[tid + o];
      const double fd2 = s_fd[tid + o];
      const long long fr2 = s_fr[tid + o];
      if (fs2 != kNoFail &&
          (fs2 < s_fs[tid] || (fs2 == s_fs[tid] && (fd2 > s_fd[tid] || (fd2 == s_fd[tid] && fr2 < s_fr[tid]))))) {
        s_fs[tid] = fs2;
        s_fd[tid] = fd2;
        s_fr[tid] = fr2;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    Summary sm;
    sm.events = s_ev[0];
    sm.corrections = s_cor[0];
    sm.max_dev = s_md[0];
    sm.fail_step = s_fs[0];
    sm.fail_row = s_fr[0];
    sm.fail_dev = s_fd[0];
    *out = sm;
  }
}

__global__ void norm_sum_kernel(const double* __restrict__ partial, int nparts, int64_t count,
                                double* n2) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= count) return;
  double s = 0.0;
  for (int i = 0; i < nparts; ++i) s += partial[r * nparts + i];
  n2[r] = s;
}

// fixed_split / norm2_rn: ctqw_device.cuh (shared with the fused
// collection of resident64.cu)

// acc[k][alpha] += sum_{r in this block's realization range} limb_k(|psi_r(alpha)|^2)
__global__ void observe_diag_fixed_kernel(const double2* __restrict__ psi, int64_t count, int64_t dim,
                                          int64_t rspan, unsigned long long* __restrict__ acc) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= dim) return;
  const int64_t r0 = (int64_t)blockIdx.y * rspan;
  const int64_t r1 = r0 + rspan < count ? r0 + rspan : count;
  long long s2 = 0, s1 = 0, s0 = 0;
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = norm2_rn(__ldg(psi + (r + u) * dim + a));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      long long l2, l1, l0;
      fixed_split(v[u], l2, l1, l0);
      s2 += l2;
      s1 += l1;
      s0 += l0;
    }
  }
  for (; r < r1; ++r) {
    long long l2, l1, l0;
    fixed_split(norm2_rn(__ldg(psi + r * dim + a)), l2, l1, l0);
    s2 += l2;
    s1 += l1;
    s0 += l0;
  }
  if (gridDim.y == 1) {
    acc[a] += (unsigned long long)s2;
    acc[dim + a] += (unsigned long long)s1;
    acc[2 * dim + a] += (unsigned long long)s0;
  } else {
    atomicAdd(acc + a, (unsigned long long)s2);
    atomicAdd(acc + dim + a, (unsigned long long)s1);
    atomicAdd(acc + 2 * dim + a, (unsigned long long)s0);
  }
}

// acc <- limbs of the doubles in diag (to accumulate onto an existing sum)
__global__ void fixed_from_double_kernel(const double* __restrict__ diag, int64_t dim,
                                         unsigned long long* __restrict__ acc) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= dim) return;
  long long l2, l1, l0;
  fixed_split(diag[a], l2, l1, l0);
  acc[a] = (unsigned long long)l2;
  acc[dim + a] = (unsigned long long)l1;
  acc[2 * dim + a] = (unsigned long long)l0;
}

// diag[alpha] = value of the limbs: carries normalised in integers, then
// L2 * 2^-30 (exact) + (L1 * 2^-70 + L0 * 2^-110) (one rounding each).
__global__ void fixed_to_double_kernel(const unsigned long long* __restrict__ acc, int64_t dim,
                                       double* __restrict__ diag) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= dim) return;
  long long l2 = (long long)acc[a], l1 = (long long)acc[dim + a], l0 = (long long)acc[2 * dim + a];
  const long long c0 = l0 >> 40;  // floor
  l0 -= c0 << 40;
  l1 += c0;
  const long long c1 = l1 >> 40;
  l1 -= c1 << 40;
  l2 += c1;
  const double lo = __dadd_rn(__dmul_rn((double)l1, 0x1p-70), __dmul_rn((double)l0, 0x1p-110));
  diag[a] = __dadd_rn(__dmul_rn((double)l2, 0x1p-30), lo);
}

// populations[x] = sum_p sum_{alpha: x_p = x} p(alpha), p = diag/total.
__global__ void populations_kernel(int m, int n, const double* __restrict__ diag, double total,
                                   double* pops) {
  __shared__ double red[32];
  const int x = blockIdx.x;
  const int64_t plane = m == 1 ? 1 : (m == 2 ? (int64_t)n : (int64_t)n * n);
  double acc = 0.0;
  for (int p = 0; p < m; ++p) {
    // joint states with digit p equal to x: enumerate the other m-1 digits
    int64_t stride_p = 1;
    for (int q = p + 1; q < m; ++q) stride_p *= n;
    for (int64_t j = threadIdx.x; j < plane; j += blockDim.x) {
      // j enumerates the remaining digits; split into high (above p) and low parts
      const int64_t low = j % stride_p;
      const int64_t high = j / stride_p;
      const int64_t alpha = (high * n + x) * stride_p + low;
      acc += diag[alpha] / total;
    }
  }
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) pops[x] = b;
}

__global__ void joint_sums_kernel(const double* __restrict__ diag, int64_t dim, double total,
                                  double* partial, double* joint) {
  __shared__ double red[32];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < dim;
       a += (int64_t)gridDim.x * blockDim.x) {
    const double p = diag[a] / total;
    if (joint) joint[a] = p;
    s1 += p;
    s2 += p * p;
  }
  const double b1 = block_sum(s1, red);
  const double b2 = block_sum(s2, red);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = b1;
    partial[2 * blockIdx.x + 1] = b2;
  }
}

// The block partials of the two joint sums, reduced by one warp in a fixed
// order (lane l takes partials l, l+32, ..., then a shuffle tree): the same
// bits on the per-point and the batched path.
__device__ __forceinline__ void joint_final_warp(const double* __restrict__ pp, int nparts, double& s1,
                                                 double& s2) {
  const int lane = threadIdx.x & 31;
  s1 = 0.0;
  s2 = 0.0;
  for (int i = lane; i < nparts; i += 32) {
    s1 += pp[2 * i];
    s2 += pp[2 * i + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
}

__global__ void joint_final_kernel(const double* __restrict__ partial, int nparts,
                                   double* scalars) {
  if (blockIdx.x != 0) return;
  double s1, s2;
  joint_final_warp(partial, nparts, s1, s2);
  if (threadIdx.x != 0) return;
  scalars[0] = s1;
  scalars[1] = s2;
  // participation ratio 1 / sum (p/S1)^2 = S1^2 / S2  (observables.py:94-101)
  // NaN states give NaN; a zero-weight distribution gives NaN too and the
  // host raises NumericError on s2 <= 0, as observables.py:98-99 does
  scalars[2] = s2 > 0.0 ? (s1 * s1) / s2 : (s2 == s2 ? __longlong_as_double(0x7ff8000000000000LL) : s2);
}

// sum_{i,j} |<a_i|b_j>|^2 : 32 x 32 tiles of the overlap matrix G = A^H B,
// 64 threads per tile, each a 4 x 4 register block (rows ty + 8u, columns
// tx + 8v: a warp's row reads are broadcasts and its column reads one
// 128-byte wavefront, 64 DFMA per 8 shared loads), D split over `ksplit`
// blocks per tile (partial G tiles summed in a fixed order afterwards ->
// deterministic).  blockIdx.z is the collection point.
constexpr int kOT = 32;   // overlap tile
constexpr int kOK = 16;   // D chunk staged through shared memory
constexpr int kOThreads = 64;
constexpr int kOReg = 16;  // accumulators per thread

__global__ void __launch_bounds__(kOThreads) overlap_partial_kernel(const double2* __restrict__ a, int64_t ra,
                                                                    const double2* __restrict__ b, int64_t rb,
                                                                    int64_t dim, int same, int64_t ntj,
                                                                    int64_t kspan, int64_t pstride,
                                                                    double2* __restrict__ gpart) {
  __shared__ double2 sa[kOK][kOT + 1];
  __shared__ double2 sb[kOK][kOT + 1];
  a += (int64_t)blockIdx.z * pstride;
  b += (int64_t)blockIdx.z * pstride;
  gpart += (int64_t)blockIdx.z * gridDim.x * gridDim.y * kOThreads * kOReg;
  const int64_t tile = blockIdx.x;
  const int64_t ti = tile / ntj, tj = tile % ntj;
  const int ks = blockIdx.y;
  const int tid = threadIdx.x;
  if (same && tj < ti) return;
  const int ty = tid >> 3, tx = tid & 7;
  double2 g[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) g[u][v] = make_double2(0.0, 0.0);
  const int64_t klo = ks * kspan;
  const int64_t khi = klo + kspan < dim ? klo + kspan : dim;
  for (int64_t k0 = klo; k0 < khi; k0 += kOK) {
#pragma unroll
    for (int e = tid; e < kOK * kOT; e += kOThreads) {
      const int kk = e % kOK, rr = e / kOK;
      const int64_t gi = ti * kOT + rr, gj = tj * kOT + rr, gk = k0 + kk;
      sa[kk][rr] = (gi < ra && gk < khi) ? a[gi * dim + gk] : make_double2(0.0, 0.0);
      sb[kk][rr] = (gj < rb && gk < khi) ? b[gj * dim + gk] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kOK; ++kk) {
      double2 av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = sa[kk][ty + 8 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = sb[kk][tx + 8 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          // conj(a) * b
          g[u][v].x = fma(av[u].x, bv[v].x, fma(av[u].y, bv[v].y, g[u][v].x));
          g[u][v].y = fma(av[u].x, bv[v].y, fma(-av[u].y, bv[v].x, g[u][v].y));
        }
    }
    __syncthreads();
  }
  double2* out = gpart + ((tile * gridDim.y + ks) * kOThreads + tid) * kOReg;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) out[u * 4 + v] = g[u][v];
}

// one thread per G entry of the tile (kOThreads x kOReg = 1024), summing the
// D split in order with coalesced loads
__global__ void __launch_bounds__(kOThreads * kOReg) overlap_finish_kernel(const double2* __restrict__ gpart,
                                                                           int ksplit, int same, int64_t ntj,
                                                                           double* partial) {
  __shared__ double red[32];
  constexpr int kE = kOThreads * kOReg;
  gpart += (int64_t)blockIdx.y * gridDim.x * ksplit * kE;
  partial += (int64_t)blockIdx.y * gridDim.x;
  const int64_t tile = blockIdx.x;
  const int64_t ti = tile / ntj, tj = tile % ntj;
  const int e = threadIdx.x;
  if (same && tj < ti) {
    if (e == 0) partial[tile] = 0.0;
    return;
  }
  double2 g = make_double2(0.0, 0.0);
  for (int ks = 0; ks < ksplit; ++ks) g = cadd(g, gpart[(tile * ksplit + ks) * kE + e]);
  const double tot = block_sum(norm2(g), red);
  if (e == 0) partial[tile] = (same && tj > ti) ? 2.0 * tot : tot;
}

// Small stacks (one stack against itself, R <= kTriMaxR, the purity case):
// the upper triangle of G = A A^H in 4 x 4 register blocks, every block
// (bi <= bj) one thread, so neither the padding of R to a tile nor the lower
// half of the diagonal tiles is computed (R = 100: 325 blocks, half the work
// of the 32 x 32 tiles).  Grid (ksplit, point); D split over ksplit CTAs in a
// fixed way (independent of the point count), partial blocks summed in order.
// Shared memory holds a 16-wide k chunk as [row mod 4][k][row / 4], so the
// column reads of a warp (consecutive bj) are contiguous.
constexpr int kTriMaxR = 124;     // 31 x 32 / 2 = 496 blocks
constexpr int kTriK = 16;
constexpr int kTriThreads = 512;  // 128 registers per thread

__device__ __forceinline__ void cpa16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

__global__ void __launch_bounds__(kTriThreads, 1) overlap_tri_kernel(const double2* __restrict__ a, int64_t R,
                                                                     int64_t dim, int nb, int nbp, int nblk,
                                                                     int64_t kspan, int64_t pstride,
                                                                     double2* __restrict__ gpart) {
  extern __shared__ double2 tri_st[];  // two buffers of [4][kTriK][nbp]
  const int bufsz = 4 * kTriK * nbp;
  a += (int64_t)blockIdx.y * pstride;
  gpart += ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * nblk * 16;
  const int tid = threadIdx.x;
  // rows R .. 4 nb - 1 are never staged: zero them once (both buffers)
  for (int e = tid; e < 2 * bufsz; e += blockDim.x) tri_st[e] = make_double2(0.0, 0.0);
  // my block: row-major over the upper triangle
  int bi = 0, rem = tid;
  while (bi < nb && rem >= nb - bi) {
    rem -= nb - bi;
    ++bi;
  }
  const bool active = tid < nblk;
  const int bj = active ? bi + rem : 0;
  if (!active) bi = 0;
  double2 g[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) g[u][v] = make_double2(0.0, 0.0);
  const int64_t klo = (int64_t)blockIdx.x * kspan;
  const int64_t khi = klo + kspan < dim ? klo + kspan : dim;
  const int nchunk = (int)((khi - klo + kTriK - 1) / kTriK);
  __syncthreads();
  // k chunks staged with cp.async, double-buffered: chunk c + 1 is in flight
  // while chunk c is multiplied
  auto stage = [&](int c) {
    double2* st = tri_st + (c & 1) * bufsz;
    const int64_t k0 = klo + (int64_t)c * kTriK;
    for (int e = tid; e < kTriK * R; e += blockDim.x) {
      const int kk = e % kTriK, r = e / kTriK;
      const int64_t gk = k0 + kk;
      const bool ok = gk < khi;
      cpa16_zfill(st + ((r & 3) * kTriK + kk) * nbp + (r >> 2), a + r * dim + (ok ? gk : klo), ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  stage(0);
  for (int c = 0; c < nchunk; ++c) {
    if (c + 1 < nchunk) {
      stage(c + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double2* st = tri_st + (c & 1) * bufsz;
    if (active) {
#pragma unroll 4
      for (int kk = 0; kk < kTriK; ++kk) {
        double2 av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = st[(u * kTriK + kk) * nbp + bi];
#pragma unroll
        for (int v = 0; v < 4; ++v) bv[v] = st[(v * kTriK + kk) * nbp + bj];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            // conj(a) * b
            g[u][v].x = fma(av[u].x, bv[v].x, fma(av[u].y, bv[v].y, g[u][v].x));
            g[u][v].y = fma(av[u].x, bv[v].y, fma(-av[u].y, bv[v].x, g[u][v].y));
          }
      }
    }
    __syncthreads();  // buffer c & 1 is restaged for chunk c + 2
  }
  if (active) {
    double2* out = gpart + (int64_t)tid * 16;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) out[u * 4 + v] = g[u][v];
  }
}

// sum over the D split, |.|^2, weight 2 off the diagonal blocks: one thread
// per G entry (coalesced over the [ks][block][16] partials), one partial per
// 256 entries and point
__global__ void __launch_bounds__(256) overlap_tri_finish_kernel(const double2* __restrict__ gpart, int ksplit,
                                                                 int nb, int nblk, double* partial) {
  __shared__ double red[32];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = nblk * 16;
  const double2* gp = gpart + (int64_t)blockIdx.y * ksplit * n;
  double sq = 0.0;
  if (e < n) {
    double2 g = make_double2(0.0, 0.0);
    for (int ks = 0; ks < ksplit; ++ks) g = cadd(g, gp[(int64_t)ks * n + e]);
    int bi = 0, rem = e >> 4;
    while (bi < nb && rem >= nb - bi) {
      rem -= nb - bi;
      ++bi;
    }
    sq = (rem == 0 ? 1.0 : 2.0) * norm2(g);  // bj == bi: the diagonal block holds both halves
  }
  const double tot = block_sum(sq, red);
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
}

__global__ void sum_kernel(const double* __restrict__ partial, int64_t nparts, double* out) {
  __shared__ double red[32];
  partial += (int64_t)blockIdx.x * nparts;  // one block per collection point
  out += blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  const double b = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = b;
}

}  // namespace

cudaError_t launch_norm_decide(const double* partial, int nparts, int64_t count, long long step,
                               const NormPolicy& pol, double* scl, RealStat* stats,
                               EventRec* events, long long* fail, cudaStream_t s) {
  const int bs = 128;
  norm_decide_kernel<<<(unsigned)((count + bs - 1) / bs), bs, 0, s>>>(partial, nparts, count, step,
                                                                       pol, scl, stats, events, fail);
  return cudaGetLastError();
}

cudaError_t launch_rescale(double2* psi, int64_t count, int64_t dim, double* scl, cudaStream_t s) {
  const int bs = 256;
  int64_t blocks = (dim + bs - 1) / bs;
  if (blocks > 64) blocks = 64;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    rescale_kernel<<<dim3((unsigned)blocks, (unsigned)rows), bs, 0, s>>>(psi + r0 * dim, dim, scl + r0);
  }
  reset_scale_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(scl, count);
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(double2* psi, int64_t count, int64_t dim, const double* scl,
                              cudaStream_t s) {
  const int bs = 256;
  int64_t blocks = (dim + bs - 1) / bs;
  if (blocks > 64) blocks = 64;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    rescale_kernel<<<dim3((unsigned)blocks, (unsigned)rows), bs, 0, s>>>(psi + r0 * dim, dim,
                                                                         const_cast<double*>(scl) + r0);
  }
  return cudaGetLastError();
}

cudaError_t launch_reset_stats(RealStat* stats, double* scl, int64_t count, long long* fail,
                               cudaStream_t s) {
  const int64_t work = count > 0 ? count : 1;
  reset_stats_kernel<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(stats, scl, count, fail);
  return cudaGetLastError();
}

cudaError_t launch_stats_reduce(const RealStat* stats, int64_t count, Summary* out, cudaStream_t s) {
  stats_reduce_kernel<<<1, 1024, 0, s>>>(stats, count, out);
  return cudaGetLastError();
}

cudaError_t launch_norm_sum(const double* partial, int nparts, int64_t count, double* n2,
                            cudaStream_t s) {
  norm_sum_kernel<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(partial, nparts, count, n2);
  return cudaGetLastError();
}

cudaError_t launch_observe_diag_fixed(const double2* psi, int64_t count, int64_t dim, unsigned long long* acc,
                                      bool accumulate, cudaStream_t s) {
  if (!accumulate) {
    cudaError_t e = cudaMemsetAsync(acc, 0, (size_t)3 * dim * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  if (count <= 0 || dim <= 0) return cudaSuccess;
  const int bs = 256;
  const int64_t bx = (dim + bs - 1) / bs;
  // enough blocks to fill the GPU: split the realizations over blockIdx.y
  // (exact integer atomics make the split invisible in the result)
  int64_t ny = (4 * 148 + bx - 1) / bx;
  if (ny > count) ny = count;
  if (ny > 65535) ny = 65535;
  if (ny < 1) ny = 1;
  const int64_t rspan = (count + ny - 1) / ny;
  ny = (count + rspan - 1) / rspan;
  observe_diag_fixed_kernel<<<dim3((unsigned)bx, (unsigned)ny), bs, 0, s>>>(psi, count, dim, rspan, acc);
  return cudaGetLastError();
}

cudaError_t launch_fixed_from_double(const double* diag, int64_t dim, unsigned long long* acc, cudaStream_t s) {
  if (dim <= 0) return cudaSuccess;
  fixed_from_double_kernel<<<(unsigned)((dim + 255) / 256), 256, 0, s>>>(diag, dim, acc);
  return cudaGetLastError();
}

cudaError_t launch_fixed_to_double(const unsigned long long* acc, int64_t dim, double* diag, cudaStream_t s) {
  if (dim <= 0) return cudaSuccess;
  fixed_to_double_kernel<<<(unsigned)((dim + 255) / 256), 256, 0, s>>>(acc, dim, diag);
  return cudaGetLastError();
}

cudaError_t launch_observe_reduce(int m, int n, int64_t dim, const double* diag_sum, double total,
                                  double* pops, double* scalars, double* joint, double* scratch,
                                  cudaStream_t s) {
  if (pops) populations_kernel<<<n, 256, 0, s>>>(m, n, diag_sum, total, pops);
  const int nparts = 148;
  joint_sums_kernel<<<nparts, 256, 0, s>>>(diag_sum, dim, total, scratch, joint);
  joint_final_kernel<<<1, 32, 0, s>>>(scratch, nparts, scalars);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Batched post-processing of P collection points (ctqw_observe_points): the
// per-point kernels above with the point on blockIdx.y, four launches for
// any number of points.

__global__ void fixed_to_double_points_kernel(const unsigned long long* __restrict__ acc, int64_t dim,
                                              double* __restrict__ diag) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= dim) return;
  const unsigned long long* ap = acc + (int64_t)blockIdx.y * 3 * dim;
  long long l2 = (long long)ap[a], l1 = (long long)ap[dim + a], l0 = (long long)ap[2 * dim + a];
  const long long c0 = l0 >> 40;
  l0 -= c0 << 40;
  l1 += c0;
  const long long c1 = l1 >> 40;
  l1 -= c1 << 40;
  l2 += c1;
  const double lo = __dadd_rn(__dmul_rn((double)l1, 0x1p-70), __dmul_rn((double)l0, 0x1p-110));
  diag[(int64_t)blockIdx.y * dim + a] = __dadd_rn(__dmul_rn((double)l2, 0x1p-30), lo);
}

__global__ void populations_points_kernel(int m, int n, int64_t dim, const double* __restrict__ diag, double total,
                                          double* out, int64_t out_stride) {
  __shared__ double red[32];
  const int x = blockIdx.x;
  const double* dp = diag + (int64_t)blockIdx.y * dim;
  const int64_t plane = m == 1 ? 1 : (m == 2 ? (int64_t)n : (int64_t)n * n);
  double acc = 0.0;
  for (int p = 0; p < m; ++p) {
    int64_t stride_p = 1;
    for (int q = p + 1; q < m; ++q) stride_p *= n;
    for (int64_t j = threadIdx.x; j < plane; j += blockDim.x) {
      const int64_t low = j % stride_p, high = j / stride_p;
      acc += dp[(high * n + x) * stride_p + low] / total;
    }
  }
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) out[(int64_t)blockIdx.y * out_stride + x] = b;
}

__global__ void joint_sums_points_kernel(const double* __restrict__ diag, int64_t dim, double total,
                                         double* partial) {
  __shared__ double red[32];
  const double* dp = diag + (int64_t)blockIdx.y * dim;
  double s1 = 0.0, s2 = 0.0;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < dim; a += (int64_t)gridDim.x * blockDim.x) {
    const double p = dp[a] / total;
    s1 += p;
    s2 += p * p;
  }
  const double b1 = block_sum(s1, red);
  const double b2 = block_sum(s2, red);
  if (threadIdx.x == 0) {
    double* pp = partial + (int64_t)blockIdx.y * 2 * gridDim.x;
    pp[2 * blockIdx.x] = b1;
    pp[2 * blockIdx.x + 1] = b2;
  }
}

__global__ void joint_final_points_kernel(const double* __restrict__ partial, int nparts, double* out,
                                          int64_t out_stride, int n) {
  double s1, s2;
  joint_final_warp(partial + (int64_t)blockIdx.x * 2 * nparts, nparts, s1, s2);
  if (threadIdx.x != 0) return;
  double* o = out + (int64_t)blockIdx.x * out_stride + n;
  o[0] = s1;
  o[1] = s2;
  o[2] = s2 > 0.0 ? (s1 * s1) / s2 : (s2 == s2 ? __longlong_as_double(0x7ff8000000000000LL) : s2);
}

cudaError_t launch_observe_points(int m, int n, int64_t dim, const unsigned long long* acc, int64_t npoints,
                                  double total, double* diag, double* out, double* scratch, cudaStream_t s) {
  if (npoints <= 0) return cudaSuccess;
  if (npoints > 65535) return cudaErrorInvalidValue;
  const unsigned P = (unsigned)npoints;
  const int nparts = 148;
  const int64_t stride = n + 3;
  fixed_to_double_points_kernel<<<dim3((unsigned)((dim + 255) / 256), P), 256, 0, s>>>(acc, dim, diag);
  populations_points_kernel<<<dim3((unsigned)n, P), 256, 0, s>>>(m, n, dim, diag, total, out, stride);
  joint_sums_points_kernel<<<dim3(nparts, P), 256, 0, s>>>(diag, dim, total, scratch);
  joint_final_points_kernel<<<P, 32, 0, s>>>(scratch, nparts, out, stride, n);
  return cudaGetLastError();
}

// (independent of the number of points, so a point's sum does not depend on
// how the points are batched)
static int overlap_ksplit(int64_t ra, int64_t rb, bool same, int64_t dim) {
  const int64_t ti = (ra + kOT - 1) / kOT, tj = (rb + kOT - 1) / kOT;
  const int64_t active = same ? ti * (ti + 1) / 2 : ti * tj;
  int64_t ks = (296 + active - 1) / active;
  const int64_t kmax = dim / 256 > 0 ? dim / 256 : 1;
  if (ks > kmax) ks = kmax;
  if (ks > 64) ks = 64;
  return (int)(ks < 1 ? 1 : ks);
}

int64_t overlap_parts(int64_t ra, int64_t rb, bool same) {
  (void)same;
  const int64_t ti = (ra + kOT - 1) / kOT, tj = (rb + kOT - 1) / kOT;
  return ti * tj;
}

static bool overlap_tri(int64_t ra, int64_t rb, bool same) { return same && ra == rb && ra <= kTriMaxR; }
static int tri_nb(int64_t r) { return (int)((r + 3) / 4); }
static int tri_ksplit(int64_t dim) {
  int64_t ks = dim / 64;
  return (int)(ks < 1 ? 1 : (ks > 64 ? 64 : ks));
}

int64_t overlap_scratch_doubles(int64_t ra, int64_t rb, bool same, int64_t dim, int64_t npoints) {
  if (overlap_tri(ra, rb, same)) {
    const int64_t nb = tri_nb(ra), nblk = nb * (nb + 1) / 2, chunks = (nblk * 16 + 255) / 256;
    return npoints * (((chunks + 1) & ~int64_t(1)) + (int64_t)tri_ksplit(dim) * nblk * 16 * 2);
  }
  const int64_t tiles = overlap_parts(ra, rb, same);
  const int64_t per = ((tiles + 1) & ~int64_t(1)) + tiles * overlap_ksplit(ra, rb, same, dim) * kOThreads * kOReg * 2;
  return per * npoints;
}

// npoints stacks (a and b each advance pstride elements per point): the
// P overlap sums in one launch set, grid dimension z = point.
cudaError_t launch_overlap_sumsq(const double2* a, int64_t ra, const double2* b, int64_t rb,
                                 int64_t dim, double* scratch, int64_t scratch_cap, double* out,
                                 cudaStream_t s, int64_t npoints, int64_t pstride) {
  if (npoints < 1 || npoints > 65535) return cudaErrorInvalidValue;
  const bool same = (a == b) && (ra == rb);
  if (overlap_tri(ra, rb, same)) {
    if (overlap_scratch_doubles(ra, rb, same, dim, npoints) > scratch_cap) return cudaErrorInvalidValue;
    const int nb = tri_nb(ra), nbp = nb | 1, nblk = nb * (nb + 1) / 2, chunks = (nblk * 16 + 255) / 256;
    const int ks = tri_ksplit(dim);
    int64_t kspan = (dim + ks - 1) / ks;
    kspan = ((kspan + kTriK - 1) / kTriK) * kTriK;
    const int ksn = (int)((dim + kspan - 1) / kspan);  // CTAs with work
    double* partial = scratch;  // [P][chunks]
    double2* gpart = reinterpret_cast<double2*>(scratch + ((chunks * npoints + 1) & ~int64_t(1)));
    const int threads = ((nblk + 31) / 32) * 32;
    const size_t smem = (size_t)2 * 4 * kTriK * nbp * sizeof(double2);
    static DeviceOnce once;
    if (once.first()) {
      const cudaError_t e = cudaFuncSetAttribute(overlap_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(2 * 4 * kTriK * ((kTriMaxR + 3) / 4 | 1) * sizeof(double2)));
      if (e != cudaSuccess) return e;
    }
    overlap_tri_kernel<<<dim3((unsigned)ksn, (unsigned)npoints), threads, smem, s>>>(a, ra, dim, nb, nbp, nblk, kspan,
                                                                                     pstride, gpart);
    overlap_tri_finish_kernel<<<dim3((unsigned)chunks, (unsigned)npoints), 256, 0, s>>>(gpart, ksn, nb, nblk, partial);
    sum_kernel<<<(unsigned)npoints, 1024, 0, s>>>(partial, chunks, out);
    return cudaGetLastError();
  }
  const int64_t ntj = (rb + kOT - 1) / kOT;
  const int64_t tiles = overlap_parts(ra, rb, same);
  const int ks = overlap_ksplit(ra, rb, same, dim);
  if (overlap_scratch_doubles(ra, rb, same, dim, npoints) > scratch_cap) return cudaErrorInvalidValue;
  double* partial = scratch;  // [P][tiles]
  double2* gpart = reinterpret_cast<double2*>(scratch + ((tiles * npoints + 1) & ~int64_t(1)));
  int64_t kspan = (dim + ks - 1) / ks;
  kspan = ((kspan + kOK - 1) / kOK) * kOK;
  overlap_partial_kernel<<<dim3((unsigned)tiles, (unsigned)ks, (unsigned)npoints), kOThreads, 0, s>>>(
      a, ra, b, rb, dim, same ? 1 : 0, ntj, kspan, pstride, gpart);
  overlap_finish_kernel<<<dim3((unsigned)tiles, (unsigned)npoints), kOThreads * kOReg, 0, s>>>(gpart, ks, same ? 1 : 0,
                                                                                               ntj, partial);
  sum_kernel<<<(unsigned)npoints, 1024, 0, s>>>(partial, tiles, out);
  return cudaGetLastError();
}

}  // namespace ctqw
