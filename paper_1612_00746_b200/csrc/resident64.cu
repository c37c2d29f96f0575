// Resident whole-realization step kernel for N = 64 (BASELINE configs[0]):
// one CTA per realization keeps the 64 x 64 state on chip for a whole
// segment, all steps and the per-step norm policy included (HBM is touched
// at segment ends only).
//
// Why a second resident kernel.  The generic one (step_tile.cu) gives each
// thread one column of an 8-row strip, so every application reads both
// in-row neighbours of every amplitude from shared memory and writes every
// amplitude back: 3 shared-memory accesses per amplitude and application,
// which bounds it (ncu: shared memory ahead of a 17 % busy FP64 pipe).
// Here each of 256 threads owns a 4 x 4 block: the neighbours inside the
// block come from registers, only the block's rim is read (16 loads per 16
// amplitudes) and only the rim is written (12 of 16, ping-pong buffers,
// one barrier per application).  Columns are stored XOR-swizzled by 16-byte
// chunk (zo below), so every access pattern is bank-conflict free.
//
// Arithmetic is the reference's (hamiltonian.py:205-222, propagators.py:
// 167-241): diagonal, particle 0 +move / -move, particle 1 +move / -move,
// Taylor terms summed in order, RK4 stage arithmetic.  EXACT rounds every
// product and sum separately (bit-identical between renormalisations);
// otherwise the neighbour terms contract into DFMA and the Taylor series
// runs in Horner form (as band4_kernel.cuh).
#include "ctqw_device.cuh"
#include "kernels.h"

namespace ctqw {

namespace {

constexpr int kN64 = 64;
constexpr int kB64 = 4;                        // block edge
constexpr int kG64 = kN64 / kB64;              // blocks per row / column
constexpr int kThreads64 = kG64 * kG64;        // 256
constexpr int kPlane64 = kN64 * kN64;          // amplitudes

struct Res64Args {
  double2* psi;
  int64_t r_base;
  Coef coef;
  StencilConst k;
  double ci[4];
  NormPolicy pol;
  long long first_step;
  long long n_steps;
  RealStat* stats;
  EventRec* events;
  long long* fail;
  // fused collection (ctqw_evolve_observe): at every global step g with
  // (g - origin) % post_rate == 0 or g == final_step, the exact limbs of
  // |psi_r(g)|^2 are added into obs[idx][3][N^2], idx = ceil((g - origin) / post_rate) - 1
  const double2* psi0;  // non-null: every realization starts from this one state
  unsigned long long* obs;
  long long post_rate;
  long long origin;
  long long final_step;
  double2* snap;        // optional: the states at each point, [point][count][N^2] (purity)
  int64_t count;
};

// 16-byte chunk x of row y at x ^ ((x >> 3) & 3): the block-row loads
// (x = 4p + q) and the rim-column loads (x = 4p - 1, 4p + 4, wrapping) of a
// quarter warp then hit eight distinct bank groups.
__device__ __forceinline__ int zo(int y, int x) { return y * kN64 + (x ^ ((x >> 3) & 3)); }
// the block's rim (row 0 / 3, column 0 / 3): the only amplitudes other
// threads read; interior ones are never stored
__device__ __forceinline__ constexpr bool rim(int i, int q) { return i == 0 || i == kB64 - 1 || q == 0 || q == kB64 - 1; }
__device__ __forceinline__ int w64(int v) { return v & (kN64 - 1); }

__device__ __forceinline__ void st_v4(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

template <bool RK4, bool SITE, bool EXACT, bool ZD, int NAPP>
__global__ void __launch_bounds__(kThreads64, 1) resident64_kernel(const __grid_constant__ Res64Args a) {
  extern __shared__ __align__(16) double2 sm64[];
  double2* zb[2] = {sm64, sm64 + kPlane64};
  double2* psis = sm64 + 2 * kPlane64;  // RK4: psi at the start of the step
  double* hv = reinterpret_cast<double*>(sm64 + (RK4 ? 3 : 2) * kPlane64);
  double* sv = hv + kN64;
  double* red = sv + kN64;
  // Taylor with a collection (ctqw_evolve_observe): the point's limbs [3][N^2]
  unsigned long long* lbuf = reinterpret_cast<unsigned long long*>(red + 16);
  constexpr bool HORN = !RK4 && !EXACT;

  const int64_t r = a.r_base + blockIdx.x;
  const int tid = threadIdx.x, p = tid % kG64, g = tid / kG64;
  const int x0 = kB64 * p, y0 = kB64 * g;
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.site_stride : nullptr;
  if (tid < kN64) {
    hv[tid] = hop[tid];
    if (SITE) sv[tid] = site[tid];
  }
  double2* gpsi = a.psi + r * (int64_t)kPlane64;
  double2 cur[kB64][kB64], acc[kB64][kB64];
#pragma unroll
  for (int i = 0; i < kB64; ++i)
#pragma unroll
    for (int q = 0; q < kB64; ++q) {
      cur[i][q] = (a.psi0 ? a.psi0 : gpsi)[(y0 + i) * kN64 + x0 + q];
      acc[i][q] = cur[i][q];
      if (rim(i, q)) zb[0][zo(y0 + i, x0 + q)] = cur[i][q];
      if (RK4) psis[zo(y0 + i, x0 + q)] = cur[i][q];
    }
  __syncthreads();
  // couplings of the block's rows and columns: hr[i] = hop[y0 + i - 1]
  // (particle 0 -move of row i, +move of row i - 1), hc likewise for columns
  double hr[kB64 + 1], hc[kB64 + 1], sr[kB64], sc[kB64];
#pragma unroll
  for (int i = 0; i <= kB64; ++i) {
    hr[i] = hv[w64(y0 + i - 1)];
    hc[i] = hv[w64(x0 + i - 1)];
  }
#pragma unroll
  for (int i = 0; i < kB64; ++i) {
    sr[i] = SITE ? sv[y0 + i] : 0.0;
    sc[i] = SITE ? sv[x0 + i] : 0.0;
  }
  const double base0 = a.k.base[0], base1 = a.k.base[1];
  const bool diag_block = g == p;  // amplitudes with x0 == x1 lie in the diagonal blocks
  constexpr double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  RealStat* st_r = a.stats + r;
  // the realization's statistics live in thread 0's registers for the whole
  // segment (written back at the end): the per-step norm decision then needs
  // no global load, which would hold warp 0 -- and at the next barrier every
  // warp -- for a memory round trip per step
  RealStat st_l;
  if (tid == 0) st_l = *st_r;
  EventRec* ev_r = a.events + r * kMaxEvents;
  int b = 0;  // buffer holding the current stage input

#pragma unroll 1
  for (long long step = 0; step < a.n_steps; ++step) {
#pragma unroll
    for (int k = 0; k < NAPP; ++k) {
      const double2* zs = zb[b];
      double2* zd = zb[b ^ 1];
      const double ci = RK4 ? a.ci[0] : (HORN ? a.ci[NAPP - 1 - k] : a.ci[k]);
      const bool last = k == NAPP - 1;
      double2 prev[kB64];
#pragma unroll
      for (int q = 0; q < kB64; ++q) prev[q] = zs[zo(w64(y0 - 1), x0 + q)];
#pragma unroll
      for (int i = 0; i < kB64; ++i) {
        const int y = y0 + i;
        double2 dn[kB64];
#pragma unroll
        for (int q = 0; q < kB64; ++q) dn[q] = i + 1 < kB64 ? cur[i + 1][q] : zs[zo(w64(y0 + kB64), x0 + q)];
        const double2 lf = zs[zo(y, w64(x0 - 1))];
        const double2 rt = zs[zo(y, w64(x0 + kB64))];
        double2 out[kB64];
#pragma unroll
        for (int q = 0; q < kB64; ++q) {
          const double2 mid = cur[i][q];
          const double2 l = q > 0 ? cur[i][q - 1] : lf;
          const double2 rr = q + 1 < kB64 ? cur[i][q + 1] : rt;
          double2 h;
          if constexpr (ZD) {
            h = rmul(hr[i + 1], dn[q]);  // 0 * mid + x == x: the reference's bits
          } else {
            double v0 = (diag_block && i == q) ? base1 : base0;
            if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sr[i], sc[q]));  // base + (site[x0] + site[x1])
            h = madd<EXACT>(rmul(v0, mid), hr[i + 1], dn[q]);      // particle 0 +move, hop[x0]
          }
          h = madd<EXACT>(h, hr[i], prev[q]);    // particle 0 -move, hop[x0 - 1]
          h = madd<EXACT>(h, hc[q + 1], rr);     // particle 1 +move, hop[x1]
          h = madd<EXACT>(h, hc[q], l);          // particle 1 -move, hop[x1 - 1]
          if constexpr (HORN) {
            out[q] = ifma(acc[i][q], ci, h);     // psi + i c H z
          } else if constexpr (!RK4) {
            out[q] = times_i(ci, h);
            acc[i][q] = cadd(acc[i][q], out[q]);
          } else {
            const double2 stg = times_i(ci, h);
            const double2 p0 = psis[zo(y, x0 + q)];
            if (k == 0) {
              out[q] = cadd(rmul(0.5, stg), p0);
              acc[i][q] = cadd(p0, rmul(c16, stg));
            } else if (k == 1) {
              out[q] = cadd(rmul(0.5, stg), p0);
              acc[i][q] = cadd(acc[i][q], rmul(c13, stg));
            } else if (k == 2) {
              out[q] = cadd(stg, p0);
              acc[i][q] = cadd(acc[i][q], rmul(c13, stg));
            } else {
              acc[i][q] = cadd(acc[i][q], rmul(c16, stg));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kB64; ++q) {
          prev[q] = cur[i][q];
          // the last application leaves psi' in the other buffer: Horner's
          // output is psi', the exact series and RK4 have it in acc
          cur[i][q] = (last && !HORN) ? acc[i][q] : out[q];
          if (rim(i, q)) zd[zo(y, x0 + q)] = cur[i][q];
        }
      }
      if (last) {
        // |psi'|^2 of this warp's blocks, published before the application's
        // barrier: every thread then sums the eight warp partials in warp
        // order itself (block_sum's order), so the norm decision costs no
        // extra barrier
        double nrm = 0.0;
#pragma unroll
        for (int i = 0; i < kB64; ++i)
#pragma unroll
          for (int q = 0; q < kB64; ++q) nrm += norm2(cur[i][q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nrm += __shfl_down_sync(0xffffffffu, nrm, o);
        if ((tid & 31) == 0) red[(step & 1) * 8 + (tid >> 5)] = nrm;  // by step parity: order-1 steps have no barrier in between
      }
      __syncthreads();
      b ^= 1;
    }
    // norm policy for this step (propagators.py:309-328): cur holds psi'
    double n2 = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads64 / 32; ++w) n2 += red[(step & 1) * 8 + w];
    const long long step_no = a.first_step + step + 1;
    if (tid == 0) {  // statistics, events and the failure flag
      int failed = 0;
      norm_decide(n2, step_no, a.pol, &st_l, ev_r, &failed);
      if (failed) atomicMin(reinterpret_cast<unsigned long long*>(a.fail), (unsigned long long)step_no);
    }
    const double dev = fabs(n2 - 1.0);
    if (dev > a.pol.tol_fail) break;  // the same decision in every thread
    const double scl = (dev > a.pol.tol_norm && a.pol.renormalize) ? __ddiv_rn(1.0, __dsqrt_rn(n2)) : 1.0;
    if (scl != 1.0) {
#pragma unroll
      for (int i = 0; i < kB64; ++i)
#pragma unroll
        for (int q = 0; q < kB64; ++q) {
          cur[i][q] = rmul(scl, cur[i][q]);
          if (rim(i, q)) zb[b][zo(y0 + i, x0 + q)] = cur[i][q];
        }
    }
#pragma unroll
    for (int i = 0; i < kB64; ++i)
#pragma unroll
      for (int q = 0; q < kB64; ++q) {
        acc[i][q] = cur[i][q];
        if (RK4) psis[zo(y0 + i, x0 + q)] = cur[i][q];
      }
    if (scl != 1.0 || RK4) __syncthreads();
    if (a.obs) {
      // diag(rho) fused into the step (ensemble.py:761-769, density.py:91-95):
      // this realization's |psi|^2 as exact int64 limbs, added with L2
      // reductions -- integer addition, so the sum's bits do not depend on
      // the order the realizations arrive in
      const long long gs = a.first_step + step + 1, rel = gs - a.origin;
      if (rel % a.post_rate == 0 || gs == a.final_step) {
        const long long idx = (rel + a.post_rate - 1) / a.post_rate - 1;
        unsigned long long* o = a.obs + idx * 3 * (int64_t)kPlane64;
        if constexpr (!RK4) {
          // staged through shared memory, so a warp's reductions cover 256
          // contiguous bytes (8 sectors) instead of 32 sectors: the L2 sector
          // operations, not the adds, bound the scattered form (measured
          // 6.5 -> 2 us per point at R = 100).  The previous point's reads of
          // lbuf finished before the step's application barriers.
#pragma unroll
          for (int i = 0; i < kB64; ++i) {
            long long l[3][kB64];
#pragma unroll
            for (int q = 0; q < kB64; ++q) fixed_split(norm2_rn(cur[i][q]), l[0][q], l[1][q], l[2][q]);
            const int al = (y0 + i) * kN64 + x0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              ulonglong2* d = reinterpret_cast<ulonglong2*>(lbuf + c * kPlane64 + al);
              d[0] = make_ulonglong2((unsigned long long)l[c][0], (unsigned long long)l[c][1]);
              d[1] = make_ulonglong2((unsigned long long)l[c][2], (unsigned long long)l[c][3]);
            }
          }
          __syncthreads();
#pragma unroll 4
          for (int f = tid; f < 3 * kPlane64; f += kThreads64) atomicAdd(o + f, lbuf[f]);
        } else {
#pragma unroll
          for (int i = 0; i < kB64; ++i)
#pragma unroll
            for (int q = 0; q < kB64; ++q) {
              long long l2, l1, l0;
              fixed_split(norm2_rn(cur[i][q]), l2, l1, l0);
              const int al = (y0 + i) * kN64 + x0 + q;
              atomicAdd(o + al, (unsigned long long)l2);
              atomicAdd(o + kPlane64 + al, (unsigned long long)l1);
              atomicAdd(o + 2 * kPlane64 + al, (unsigned long long)l0);
            }
        }
        if (a.snap) {
          double2* sp = a.snap + (idx * a.count + r) * (int64_t)kPlane64;
          // 32-byte stores: whole L2 sectors
#pragma unroll
          for (int i = 0; i < kB64; ++i)
#pragma unroll
            for (int q = 0; q < kB64; q += 2) st_v4(sp + (y0 + i) * kN64 + x0 + q, cur[i][q], cur[i][q + 1]);
        }
      }
    }
  }
  if (tid == 0) *st_r = st_l;
#pragma unroll
  for (int i = 0; i < kB64; ++i)
#pragma unroll
    for (int q = 0; q < kB64; q += 2) st_v4(gpsi + (y0 + i) * kN64 + x0 + q, acc[i][q], acc[i][q + 1]);
}

template <bool RK4, bool SITE, bool EXACT, bool ZD, int NAPP>
cudaError_t launch64(const Res64Args& a, int64_t count, cudaStream_t s) {
  constexpr size_t smem0 = (size_t)(RK4 ? 3 : 2) * kPlane64 * sizeof(double2) + (2 * kN64 + 16) * sizeof(double);
  constexpr size_t smem_obs = smem0 + (RK4 ? 0 : (size_t)3 * kPlane64 * sizeof(unsigned long long));
  static_assert(smem_obs <= 227 * 1024, "resident64 shared memory");
  const size_t smem = a.obs ? smem_obs : smem0;
  auto kern = resident64_kernel<RK4, SITE, EXACT, ZD, NAPP>;
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_obs);
    if (e != cudaSuccess) return e;
  }
  Res64Args b = a;
  for (int64_t r0 = 0; r0 < count; r0 += 2147483647LL) {
    b.r_base = r0;
    const int64_t rows = count - r0 < 2147483647LL ? count - r0 : 2147483647LL;
    kern<<<(unsigned)rows, kThreads64, smem, s>>>(b);
  }
  return cudaGetLastError();
}

template <bool RK4, bool SITE, bool EXACT, bool ZD>
cudaError_t launch64_o(const Res64Args& a, int64_t count, int napp, cudaStream_t s) {
  if constexpr (RK4) {
    return launch64<true, SITE, EXACT, ZD, 4>(a, count, s);
  } else {
    switch (napp) {
      case 1: return launch64<false, SITE, EXACT, ZD, 1>(a, count, s);
      case 2: return launch64<false, SITE, EXACT, ZD, 2>(a, count, s);
      case 3: return launch64<false, SITE, EXACT, ZD, 3>(a, count, s);
      case 4: return launch64<false, SITE, EXACT, ZD, 4>(a, count, s);
      default: return cudaErrorInvalidValue;
    }
  }
}

template <bool RK4, bool SITE, bool EXACT>
cudaError_t launch64_z(const Res64Args& a, int64_t count, int napp, bool zd, cudaStream_t s) {
  if constexpr (!SITE) {
    if (zd) return launch64_o<RK4, false, EXACT, true>(a, count, napp, s);
  }
  return launch64_o<RK4, SITE, EXACT, false>(a, count, napp, s);
}

}  // namespace

bool resident64_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n == kN64 && (sc.backend == 1 || (sc.order >= 1 && sc.order <= 4));
}

cudaError_t launch_resident64(double2* psi, int64_t count, const Coef& coef, const StencilConst& k,
                              const StepScalars& sc, bool exact, const NormPolicy& pol, long long first_step,
                              long long n_steps, RealStat* stats, EventRec* events, long long* fail,
                              cudaStream_t s, unsigned long long* obs, long long post_rate, long long origin,
                              long long final_step, const double2* psi0, double2* snap) {
  Res64Args a;
  a.psi0 = psi0;
  a.snap = snap;
  a.count = count;
  a.obs = obs;
  a.post_rate = post_rate > 0 ? post_rate : 1;
  a.origin = origin;
  a.final_step = final_step;
  a.psi = psi;
  a.r_base = 0;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.pol = pol;
  a.first_step = first_step;
  a.n_steps = n_steps;
  a.stats = stats;
  a.events = events;
  a.fail = fail;
  const bool site = coef.site != nullptr;
  const bool rk4 = sc.backend == 1;
  const int napp = rk4 ? 4 : sc.order;
  // eps0 = U = 0 and no site noise: the diagonal is zero
  const bool zd = !site && k.base[0] == 0.0 && k.base[1] == 0.0;
  if (count <= 0 || n_steps <= 0) return cudaSuccess;
  if (rk4) {
    if (site && exact) return launch64_z<true, true, true>(a, count, napp, zd, s);
    if (site) return launch64_z<true, true, false>(a, count, napp, zd, s);
    if (exact) return launch64_z<true, false, true>(a, count, napp, zd, s);
    return launch64_z<true, false, false>(a, count, napp, zd, s);
  }
  if (site && exact) return launch64_z<false, true, true>(a, count, napp, zd, s);
  if (site) return launch64_z<false, true, false>(a, count, napp, zd, s);
  if (exact) return launch64_z<false, false, true>(a, count, napp, zd, s);
  return launch64_z<false, false, false>(a, count, napp, zd, s);
}

}  // namespace ctqw
