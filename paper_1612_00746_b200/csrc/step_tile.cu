// Fused m = 2 step kernels: every stencil application of one time step runs
// on chip, HBM is touched once per step (streaming tile path) or once per
// segment (resident path).
//
// The two-particle ring operator is a 5-point stencil on the N x N torus of
// joint positions (x0 = row, particle 0; x1 = column, particle 1):
//   (H t)(y,x) = v0(y,x) t(y,x) + hop[y] t(y+1,x) + hop[y-1] t(y-1,x)
//                               + hop[x] t(y,x+1) + hop[x-1] t(y,x-1)
// accumulated in exactly that order (hamiltonian.py:205-222, slot 1 = particle
// 0, slot 2 = particle 1, +move before -move).
//
// Thread mapping (both kernels): thread (strip, x) owns column x of a strip
// of S consecutive rows; its rows live in registers across the orders, so per
// application it reads only the two strip-end rows and the left/right columns
// from shared memory and writes its S new values back once.
//
// Streaming tile kernel: a (64 + 2H)^2 tile with an H-deep halo is loaded once
// from HBM (periodic wrap in the index math), the H applications of the step
// (Taylor order H, or the 4 RK4 stages) shrink the valid region by one per
// application, and the 64 x 64 interior is written back with its |psi|^2 norm
// partial.  Halo rows are shared with neighbouring tiles through L2.
//
// Resident kernel (N <= 64): one CTA holds a whole realization in shared
// memory + registers for the entire segment, including the per-step norm
// policy (propagators.py:309-328) -- HBM traffic only at segment ends.
#include "ctqw_device.cuh"
#include "kernels.h"

namespace ctqw {

namespace {

constexpr int kTI = 64;   // tile interior
constexpr int kS = 9;     // rows per strip (tile kernel)
constexpr int kSR = 8;    // rows per strip (resident kernel)
constexpr int kResidentMax = 64;

// One tile geometry for every Taylor order <= 4 and RK4: a 64 x 64 interior
// with a 4-deep halo; fewer applications simply leave a wider valid region.
constexpr int kHalo = 4;
constexpr int kT = kTI + 2 * kHalo;          // 72
constexpr int kNStrip = kT / kS;             // 8
constexpr int kTileThreads = kNStrip * kT;   // 576
static_assert(kNStrip * kS == kT, "strips must tile the rows exactly");

struct TileArgs {
  const double2* psi_in;
  double2* psi_out;
  int n;
  int nt;
  int64_t r_base;
  Coef coef;
  StencilConst k;
  double ci[4];
  int napp;
  const double* scl;
  double* partial;
  int nparts;
  const long long* fail;
};

template <bool RK4>
constexpr size_t tile_smem_bytes() {
  constexpr int T = kT;
  return (size_t)T * T * sizeof(double2) * (RK4 ? 2 : 1) + (size_t)(4 * T + 2 + 32) * sizeof(double);
}

template <bool RK4, bool SITE, bool EXACT>
__global__ void __launch_bounds__(kTileThreads, 1) tile_step_kernel(TileArgs a) {
  constexpr int T = kT;
  constexpr int NT = kTileThreads;
  constexpr int H = kHalo;
  extern __shared__ double4 smem_raw[];
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  double2* psis = tile + T * T;                                   // RK4 only
  double* hr = reinterpret_cast<double*>(tile + (RK4 ? 2 : 1) * T * T);
  double* hc = hr + (T + 1);
  double* sr = hc + (T + 1);
  double* sc = sr + T;
  double* red = sc + T;

  if (*a.fail != kNoFail) return;
  const int n = a.n;
  const int64_t dim = (int64_t)n * n;
  const int64_t r = a.r_base + blockIdx.y;
  const int tid = threadIdx.x;
  const int ty = blockIdx.x / a.nt, tx = blockIdx.x % a.nt;
  const int gy0 = ty * kTI - H, gx0 = tx * kTI - H;
  const int strip = tid / T, x = tid % T;
  const int y0 = strip * kS;
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.stride : nullptr;

  for (int i = tid; i <= T; i += NT) {
    hr[i] = hop[wrap(gy0 - 1 + i, n)];
    hc[i] = hop[wrap(gx0 - 1 + i, n)];
  }
  if (SITE)
    for (int i = tid; i < T; i += NT) {
      sr[i] = site[wrap(gy0 + i, n)];
      sc[i] = site[wrap(gx0 + i, n)];
    }

  const double s = a.scl ? a.scl[r] : 1.0;  // pending rescale of the previous step
  const int gx = wrap(gx0 + x, n);
  const double2* src = a.psi_in + r * dim;
  double2 cur[kS], acc[kS];
  unsigned cmask = 0;  // rows whose joint state has both particles on one site
#pragma unroll
  for (int i = 0; i < kS; ++i) {
    const int y = y0 + i;
    const int gy = wrap(gy0 + y, n);
    if (gy == gx) cmask |= 1u << i;
    cur[i] = rmul(s, __ldg(src + (int64_t)gy * n + gx));
    tile[y * T + x] = cur[i];
    if (RK4) psis[y * T + x] = cur[i];
    acc[i] = cur[i];
  }
  __syncthreads();

  const double base0 = a.k.base[0], base1 = a.k.base[1];
  const double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  const int xl = x > 0 ? x - 1 : x, xr = x < T - 1 ? x + 1 : x;
  const int napp = RK4 ? 4 : a.napp;
#pragma unroll 1
  for (int k = 0; k < napp; ++k) {
    const double ci = RK4 ? a.ci[0] : a.ci[k];
    double2 prev = y0 > 0 ? tile[(y0 - 1) * T + x] : cur[0];
#pragma unroll
    for (int i = 0; i < kS; ++i) {
      const int y = y0 + i;
      {
        double2 nxt;
        if (i + 1 < kS) nxt = cur[i + 1];
        else nxt = y + 1 < T ? tile[(y + 1) * T + x] : cur[i];
        const double2 lf = tile[y * T + xl];
        const double2 rt = tile[y * T + xr];
        double v0 = ((cmask >> i) & 1u) ? base1 : base0;
        if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sr[y], sc[x]));
        double2 h = rmul(v0, cur[i]);
        h = madd<EXACT>(h, hr[y + 1], nxt);
        h = madd<EXACT>(h, hr[y], prev);
        h = madd<EXACT>(h, hc[x + 1], rt);
        h = madd<EXACT>(h, hc[x], lf);
        prev = cur[i];
        const double2 st = times_i(ci, h);
        if (!RK4) {
          cur[i] = st;
          acc[i] = cadd(acc[i], st);
        } else {
          const double2 p0 = psis[y * T + x];
          if (k == 0) {
            cur[i] = cadd(rmul(0.5, st), p0);
            acc[i] = cadd(p0, rmul(c16, st));
          } else if (k == 1) {
            cur[i] = cadd(rmul(0.5, st), p0);
            acc[i] = cadd(acc[i], rmul(c13, st));
          } else if (k == 2) {
            cur[i] = cadd(st, p0);
            acc[i] = cadd(acc[i], rmul(c13, st));
          } else {
            acc[i] = cadd(acc[i], rmul(c16, st));
          }
        }
      }
    }
    if (k + 1 < napp) {
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kS; ++i) tile[(y0 + i) * T + x] = cur[i];
      __syncthreads();
    }
  }

  // interior write-back + norm partial
  double nrm = 0.0;
  const bool col_ok = x >= H && x < T - H && (tx * kTI + x - H) < n;
  double2* dst = a.psi_out + r * dim;
#pragma unroll
  for (int i = 0; i < kS; ++i) {
    const int y = y0 + i;
    if (col_ok && y >= H && y < T - H && (ty * kTI + y - H) < n) {
      const int gy = gy0 + y;  // in [0, n) for interior rows
      dst[(int64_t)gy * n + gx] = acc[i];
      nrm += norm2(acc[i]);
    }
  }
  const double b = block_sum(nrm, red);
  if (tid == 0 && a.partial) a.partial[r * a.nparts + blockIdx.x] = b;
}

// ---------------------------------------------------------------------------
// resident whole-realization kernel (N <= 64), all steps of a segment

struct ResArgs {
  double2* psi;
  int n;
  int64_t r_base;
  Coef coef;
  StencilConst k;
  int order;
  double ci[kMaxTaylorOrder];
  NormPolicy pol;
  long long first_step;
  long long n_steps;
  RealStat* stats;
  EventRec* events;
  long long* fail;
};

template <bool RK4, bool SITE, bool EXACT>
__global__ void __launch_bounds__(512, 1) resident_kernel(ResArgs a) {
  extern __shared__ double4 smem_raw[];
  const int n = a.n;
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  double2* psis = tile + n * n;
  double* hv = reinterpret_cast<double*>(tile + (RK4 ? 2 : 1) * n * n);
  double* sv = hv + n;
  double* red = sv + n;
  __shared__ double s_scale;
  __shared__ int s_failed;

  const int64_t r = a.r_base + blockIdx.x;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const int strip = tid / n, x = tid % n;
  const int y0 = strip * kSR;
  const bool active = strip * kSR < n;
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.stride : nullptr;
  for (int i = tid; i < n; i += nthreads) {
    hv[i] = hop[i];
    if (SITE) sv[i] = site[i];
  }
  double2* psi = a.psi + r * (int64_t)n * n;
  double2 cur[kSR], acc[kSR];
  unsigned cmask = 0;
#pragma unroll
  for (int i = 0; i < kSR; ++i) {
    const int y = y0 + i;
    cur[i] = make_double2(0.0, 0.0);
    if (active && y < n) {
      if (y == x) cmask |= 1u << i;
      cur[i] = psi[y * n + x];
      tile[y * n + x] = cur[i];
      if (RK4) psis[y * n + x] = cur[i];
    }
    acc[i] = cur[i];
  }
  __syncthreads();

  const double base0 = a.k.base[0], base1 = a.k.base[1];
  const double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  const int xl = x == 0 ? n - 1 : x - 1, xr = x == n - 1 ? 0 : x + 1;
  const double hx = active ? hv[x] : 0.0, hxl = active ? hv[xl] : 0.0;
  const double sxv = (SITE && active) ? sv[x] : 0.0;
  const int applications = RK4 ? 4 : a.order;
  // FMA-mode Taylor in Horner form (see step_band4.cu): application k applies
  // c_{order-k} and adds psi (held in acc through the step)
  constexpr bool HORN = !RK4 && !EXACT;
  RealStat* st_r = a.stats + r;
  EventRec* ev_r = a.events + r * kMaxEvents;

#pragma unroll 1
  for (long long step = 0; step < a.n_steps; ++step) {
#pragma unroll 1
    for (int k = 0; k < applications; ++k) {
      const double ci = RK4 ? a.ci[0] : (HORN ? a.ci[applications - 1 - k] : a.ci[k]);
      if (active) {
        double2 prev = tile[(y0 == 0 ? n - 1 : y0 - 1) * n + x];
#pragma unroll
        for (int i = 0; i < kSR; ++i) {
          const int y = y0 + i;
          if (y < n) {
            double2 nxt;
            if (i + 1 < kSR && y + 1 < n) nxt = cur[i + 1];
            else nxt = tile[(y + 1 == n ? 0 : y + 1) * n + x];
            const double2 lf = tile[y * n + xl];
            const double2 rt = tile[y * n + xr];
            double v0 = ((cmask >> i) & 1u) ? base1 : base0;
            if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sv[y], sxv));
            double2 h = rmul(v0, cur[i]);
            h = madd<EXACT>(h, hv[y], nxt);
            h = madd<EXACT>(h, hv[y == 0 ? n - 1 : y - 1], prev);
            h = madd<EXACT>(h, hx, rt);
            h = madd<EXACT>(h, hxl, lf);
            prev = cur[i];
            if (HORN) {
              cur[i] = cmake(fma(-ci, h.y, acc[i].x), fma(ci, h.x, acc[i].y));
              continue;
            }
            const double2 stg = times_i(ci, h);
            if (!RK4) {
              cur[i] = stg;
              acc[i] = cadd(acc[i], stg);
            } else {
              const double2 p0 = psis[y * n + x];
              if (k == 0) {
                cur[i] = cadd(rmul(0.5, stg), p0);
                acc[i] = cadd(p0, rmul(c16, stg));
              } else if (k == 1) {
                cur[i] = cadd(rmul(0.5, stg), p0);
                acc[i] = cadd(acc[i], rmul(c13, stg));
              } else if (k == 2) {
                cur[i] = cadd(stg, p0);
                acc[i] = cadd(acc[i], rmul(c13, stg));
              } else {
                acc[i] = cadd(acc[i], rmul(c16, stg));
              }
            }
          }
        }
      }
      __syncthreads();
      if (active && k + 1 < applications) {
#pragma unroll
        for (int i = 0; i < kSR; ++i)
          if (y0 + i < n) tile[(y0 + i) * n + x] = cur[i];
      }
      __syncthreads();
    }
    if (HORN && active) {
#pragma unroll
      for (int i = 0; i < kSR; ++i) acc[i] = cur[i];
    }
    // norm policy for this step
    double nrm = 0.0;
    if (active) {
#pragma unroll
      for (int i = 0; i < kSR; ++i)
        if (y0 + i < n) nrm += norm2(acc[i]);
    }
    const double n2 = block_sum(nrm, red);
    if (tid == 0) {
      int failed = 0;
      s_scale = norm_decide(n2, a.first_step + step + 1, a.pol, st_r, ev_r, &failed);
      s_failed = failed;
      if (failed) atomicMin(reinterpret_cast<unsigned long long*>(a.fail),
                            (unsigned long long)(a.first_step + step + 1));
    }
    __syncthreads();
    if (s_failed) break;
    const double sc = s_scale;
    if (active) {
#pragma unroll
      for (int i = 0; i < kSR; ++i) {
        const int y = y0 + i;
        if (y < n) {
          acc[i] = rmul(sc, acc[i]);
          cur[i] = acc[i];
          tile[y * n + x] = acc[i];
          if (RK4) psis[y * n + x] = acc[i];
        }
      }
    }
    __syncthreads();
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < kSR; ++i)
      if (y0 + i < n) psi[(y0 + i) * n + x] = acc[i];
  }
}

template <bool RK4, bool SITE, bool EXACT>
cudaError_t launch_tile_t(const TileArgs& args, int64_t count, cudaStream_t s) {
  constexpr size_t smem = tile_smem_bytes<RK4>();
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(tile_step_kernel<RK4, SITE, EXACT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  TileArgs a = args;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    a.r_base = r0;
    tile_step_kernel<RK4, SITE, EXACT>
        <<<dim3((unsigned)(args.nt * args.nt), (unsigned)rows), kTileThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <bool RK4>
cudaError_t launch_tile_b(const TileArgs& a, int64_t count, bool site, bool exact, cudaStream_t s) {
  if (site && exact) return launch_tile_t<RK4, true, true>(a, count, s);
  if (site) return launch_tile_t<RK4, true, false>(a, count, s);
  if (exact) return launch_tile_t<RK4, false, true>(a, count, s);
  return launch_tile_t<RK4, false, false>(a, count, s);
}

template <bool RK4, bool SITE, bool EXACT>
cudaError_t launch_res_t(const ResArgs& args, int64_t count, cudaStream_t s) {
  const int n = args.n;
  const size_t smem = (size_t)n * n * sizeof(double2) * (RK4 ? 2 : 1) + (size_t)(2 * n + 32) * sizeof(double);
  static DeviceOnce once;
  if (once.first()) {
    const int maxs = kResidentMax * kResidentMax * (int)sizeof(double2) * 2 + (2 * kResidentMax + 32) * 8;
    cudaError_t e = cudaFuncSetAttribute(resident_kernel<RK4, SITE, EXACT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
    if (e != cudaSuccess) return e;
  }
  const int threads = ((n + kSR - 1) / kSR) * n;
  ResArgs a = args;
  for (int64_t r0 = 0; r0 < count; r0 += 2147483647LL) {
    const int64_t rows = count - r0;
    a.r_base = r0;
    resident_kernel<RK4, SITE, EXACT><<<(unsigned)rows, threads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace

bool tile_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n > kResidentMax && (sc.backend == 1 || (sc.order >= 1 && sc.order <= kHalo));
}

bool resident_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n >= 3 && n <= kResidentMax && (sc.backend == 1 || (sc.order >= 1 && sc.order <= 16));
}

int tile_parts(int n, const StepScalars& sc) {
  (void)sc;
  const int nt = (n + kTI - 1) / kTI;
  return nt * nt;
}

cudaError_t launch_tile_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                             const Coef& coef, const StencilConst& k, const StepScalars& sc,
                             bool exact, const double* scl, double* partial,
                             const long long* fail, cudaStream_t s) {
  TileArgs a;
  a.psi_in = psi_in;
  a.psi_out = psi_out;
  a.n = n;
  a.nt = (n + kTI - 1) / kTI;
  a.r_base = 0;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.scl = scl;
  a.partial = partial;
  a.nparts = a.nt * a.nt;
  a.fail = fail;
  a.napp = sc.backend == 1 ? 4 : sc.order;
  const bool site = coef.site != nullptr;
  if (sc.backend == 1) return launch_tile_b<true>(a, count, site, exact, s);
  if (sc.order < 1 || sc.order > kHalo) return cudaErrorInvalidValue;
  return launch_tile_b<false>(a, count, site, exact, s);
}

cudaError_t launch_resident(double2* psi, int64_t count, int n, const Coef& coef,
                            const StencilConst& k, const StepScalars& sc, bool exact,
                            const NormPolicy& pol, long long first_step, long long n_steps,
                            RealStat* stats, EventRec* events, long long* fail,
                            cudaStream_t s) {
  ResArgs a;
  a.psi = psi;
  a.n = n;
  a.r_base = 0;
  a.coef = coef;
  a.k = k;
  a.order = sc.order;
  for (int i = 0; i < kMaxTaylorOrder; ++i) a.ci[i] = sc.ci[i];
  a.pol = pol;
  a.first_step = first_step;
  a.n_steps = n_steps;
  a.stats = stats;
  a.events = events;
  a.fail = fail;
  const bool site = coef.site != nullptr;
  const bool rk4 = sc.backend == 1;
  if (rk4) {
    if (site && exact) return launch_res_t<true, true, true>(a, count, s);
    if (site) return launch_res_t<true, true, false>(a, count, s);
    if (exact) return launch_res_t<true, false, true>(a, count, s);
    return launch_res_t<true, false, false>(a, count, s);
  }
  if (site && exact) return launch_res_t<false, true, true>(a, count, s);
  if (site) return launch_res_t<false, true, false>(a, count, s);
  if (exact) return launch_res_t<false, false, true>(a, count, s);
  return launch_res_t<false, false, false>(a, count, s);
}

}  // namespace ctqw
