// Row-marching streaming step kernel for m = 2, two columns per thread.
//
// Same pipeline as step_band.cu (every stencil application of a step as a
// software pipeline over rows, stage k computing row j-2k+1 at iteration j,
// three-row register windows per stage, one __syncthreads per row, cp.async
// ring of psi rows), but each thread owns the column pair (2p, 2p+1).  The
// pair's inner neighbours are in registers, so per application a thread
// publishes its two values and reads one value on each side -- a third less
// shared-memory traffic than one column per thread, which is what bounds the
// one-column kernels (ncu: L1/TEX 87 % busy).
//
// Shared-memory rows are stored split by parity -- E[p] = column 2p,
// O[p] = column 2p+1 -- so a warp's 16-byte accesses to E[...] or O[...] are
// contiguous and bank-conflict free.
//
// Arithmetic: identical to the reference (hamiltonian.py:205-222,
// propagators.py:185-193 / 213-240); EXACT keeps every product and sum
// separately rounded in the reference order.
#include "ctqw_device.cuh"
#include "kernels.h"

#include <cmath>
#include <cstdlib>

namespace ctqw {

namespace {

constexpr int kRing2 = 16;       // psi rows resident (8 prefetched ahead)
constexpr int kPref2 = kRing2 / 2;
constexpr int kHalo2 = 4;
constexpr int kPad2 = 8;         // coefficient rows padded by wrap on both sides
constexpr int kMaxPairs = 128;   // threads per CTA (two CTAs per SM)

struct Band2Args {
  const double2* psi_in;
  double2* psi_out;
  int n;
  int W;          // interior columns per band
  int nbands;
  int seg_len;
  int nseg;
  int64_t r_base;
  Coef coef;
  StencilConst k;
  double ci[4];
  const double* scl;
  double* partial;
  int nparts;
  const long long* fail;
};

__device__ __forceinline__ void cp_async16b(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_b() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_b() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int wrap_r(int r, int n) { return r < 0 ? r + n : (r >= n ? r - n : r); }

template <bool EXACT>
__device__ __forceinline__ double2 st5(double v0, double2 up, double2 mid, double2 dn, double2 lf, double2 rt,
                                       double hr, double hrm, double hc, double hcm) {
  double2 h = rmul(v0, mid);
  h = madd<EXACT>(h, hr, dn);   // particle 0 +move (row r+1), coupling hop[r]
  h = madd<EXACT>(h, hrm, up);  // particle 0 -move (row r-1), coupling hop[r-1]
  h = madd<EXACT>(h, hc, rt);   // particle 1 +move
  h = madd<EXACT>(h, hcm, lf);  // particle 1 -move
  return h;
}

struct Pair {
  double2 c[2];
};

struct Band2Thread {
  const double2* ringp;  // ring + p  (E part; O part at + NP)
  double2* rowp;         // stage rows + p
  int NP;                // pairs per row (row stride = 2 * NP)
  int dl, dr;            // O[p-1] and E[p+1] offsets relative to p
  const double2* hop2;   // (hop[r-1], hop[r]) at hop2[r]
  const double* sitex;
  int gx0, gx1;
  double hxm0, hx0, hx1, sx0, sx1;
  bool w0, w1;           // writes column 2p / 2p+1
};

template <int NAPP>
struct Band2Regs {
  static constexpr int NACC = 2 * NAPP - 2 > 0 ? 2 * NAPP - 2 : 1;
  Pair win[NAPP][3];
  Pair acc[NACC];
  double nrm;
};

constexpr int gcd2(int a, int b) { return b == 0 ? a : gcd2(b, a % b); }
template <int NAPP>
struct Band2Period {
  static constexpr int NACC = Band2Regs<NAPP>::NACC;
  static constexpr int value = 3 * NACC / gcd2(3, NACC);
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH>
__device__ __forceinline__ void band2_iter(const Band2Args& a, const Band2Thread& T, Band2Regs<NAPP>& R,
                                           int j, int slot, double2* outp, bool store, double s) {
  constexpr int NACC = Band2Regs<NAPP>::NACC;
  constexpr int P0 = PH % 3, P1 = (PH + 1) % 3, P2 = (PH + 2) % 3;
  const double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  const int n = a.n;
  const int RS = 2 * T.NP;  // row stride
  const double2* h2 = T.hop2 + j;
  const double* sj = T.sitex + j;
  const double b0 = a.k.base[0], b1 = a.k.base[1];

#pragma unroll
  for (int k = NAPP; k >= 2; --k) {
    const int rr = j - 2 * k + 1;
    const Pair up = R.win[k - 1][P0], mid = R.win[k - 1][P1], dn = R.win[k - 1][P2];
    const double2* prow = T.rowp + ((k - 2) * 3 + P1) * RS;
    const double2 lf0 = prow[T.NP + T.dl];  // O[p-1]
    const double2 rt1 = prow[T.dr];         // E[p+1]
    const int gy = wrap_r(rr, n);
    double v0 = gy == T.gx0 ? b1 : b0;
    double v1 = gy == T.gx1 ? b1 : b0;
    if (SITE) {
      v0 = __dadd_rn(v0, __dadd_rn(sj[1 - 2 * k], T.sx0));
      v1 = __dadd_rn(v1, __dadd_rn(sj[1 - 2 * k], T.sx1));
    }
    const double2 hp = h2[1 - 2 * k];
    const double ci = RK4 ? a.ci[0] : a.ci[k - 1];
    const double2 st0 = times_i(ci, st5<EXACT>(v0, up.c[0], mid.c[0], dn.c[0], lf0, mid.c[1], hp.y, hp.x, T.hx0, T.hxm0));
    const double2 st1 = times_i(ci, st5<EXACT>(v1, up.c[1], mid.c[1], dn.c[1], mid.c[0], rt1, hp.y, hp.x, T.hx1, T.hx0));
    const int AS = ((PH - 2 * k + 2) % NACC + NACC) % NACC;
    Pair newt;
    if (!RK4) {
      if (k == NAPP) {
        const double2 o0 = cadd(R.acc[AS].c[0], st0), o1 = cadd(R.acc[AS].c[1], st1);
        if (store) {
          if (T.w0) {
            outp[0] = o0;
            R.nrm += norm2(o0);
          }
          if (T.w1) {
            outp[1] = o1;
            R.nrm += norm2(o1);
          }
        }
      } else {
        R.acc[AS].c[0] = cadd(R.acc[AS].c[0], st0);
        R.acc[AS].c[1] = cadd(R.acc[AS].c[1], st1);
        newt.c[0] = st0;
        newt.c[1] = st1;
      }
    } else {
      if (k == 4) {
        const double2 o0 = cadd(R.acc[AS].c[0], rmul(c16, st0)), o1 = cadd(R.acc[AS].c[1], rmul(c16, st1));
        if (store) {
          if (T.w0) {
            outp[0] = o0;
            R.nrm += norm2(o0);
          }
          if (T.w1) {
            outp[1] = o1;
            R.nrm += norm2(o1);
          }
        }
      } else {
        const double2* rowr = T.ringp + ((slot - 2 * k + 1) & (kRing2 - 1)) * RS;
        const double2 p0 = rmul(s, rowr[0]), p1 = rmul(s, rowr[T.NP]);
        if (k == 2) {
          newt.c[0] = cadd(rmul(0.5, st0), p0);
          newt.c[1] = cadd(rmul(0.5, st1), p1);
        } else {
          newt.c[0] = cadd(st0, p0);
          newt.c[1] = cadd(st1, p1);
        }
        R.acc[AS].c[0] = cadd(R.acc[AS].c[0], rmul(c13, st0));
        R.acc[AS].c[1] = cadd(R.acc[AS].c[1], rmul(c13, st1));
      }
    }
    if (k < NAPP) {
      R.win[k][P0] = newt;
      double2* wrow = T.rowp + ((k - 1) * 3 + P0) * RS;
      wrow[0] = newt.c[0];
      wrow[T.NP] = newt.c[1];
    }
  }
  // ---- stage 1 ----
  {
    const int rr = j - 1;
    const double2* rowj = T.ringp + slot * RS;
    Pair pj;
    pj.c[0] = rmul(s, rowj[0]);
    pj.c[1] = rmul(s, rowj[T.NP]);
    R.win[0][P0] = pj;
    const Pair mid = R.win[0][P2], up = R.win[0][P1];
    const double2* rowm = T.ringp + ((slot - 1) & (kRing2 - 1)) * RS;
    const double2 lf0 = rmul(s, rowm[T.NP + T.dl]), rt1 = rmul(s, rowm[T.dr]);
    const int gy = wrap_r(rr, n);
    double v0 = gy == T.gx0 ? b1 : b0;
    double v1 = gy == T.gx1 ? b1 : b0;
    if (SITE) {
      v0 = __dadd_rn(v0, __dadd_rn(sj[-1], T.sx0));
      v1 = __dadd_rn(v1, __dadd_rn(sj[-1], T.sx1));
    }
    const double2 hp = h2[-1];
    const double2 st0 = times_i(a.ci[0], st5<EXACT>(v0, up.c[0], mid.c[0], pj.c[0], lf0, mid.c[1], hp.y, hp.x, T.hx0, T.hxm0));
    const double2 st1 = times_i(a.ci[0], st5<EXACT>(v1, up.c[1], mid.c[1], pj.c[1], mid.c[0], rt1, hp.y, hp.x, T.hx1, T.hx0));
    Pair newt, newacc;
    if (!RK4) {
      if (NAPP == 1) {
        const double2 o0 = cadd(mid.c[0], st0), o1 = cadd(mid.c[1], st1);
        if (store) {
          if (T.w0) {
            outp[0] = o0;
            R.nrm += norm2(o0);
          }
          if (T.w1) {
            outp[1] = o1;
            R.nrm += norm2(o1);
          }
        }
      } else {
        newacc.c[0] = cadd(mid.c[0], st0);
        newacc.c[1] = cadd(mid.c[1], st1);
        newt.c[0] = st0;
        newt.c[1] = st1;
      }
    } else {
      newt.c[0] = cadd(rmul(0.5, st0), mid.c[0]);
      newt.c[1] = cadd(rmul(0.5, st1), mid.c[1]);
      newacc.c[0] = cadd(mid.c[0], rmul(c16, st0));
      newacc.c[1] = cadd(mid.c[1], rmul(c16, st1));
    }
    if (NAPP > 1) {
      R.acc[PH % NACC] = newacc;
      R.win[1][P0] = newt;
      double2* wrow = T.rowp + (0 * 3 + P0) * RS;
      wrow[0] = newt.c[0];
      wrow[T.NP] = newt.c[1];
    }
  }
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int PERIOD>
struct Band2Phases {
  __device__ __forceinline__ static void run(const Band2Args& a, const Band2Thread& T, Band2Regs<NAPP>& R,
                                             int& j, int& slot, double2*& outp, int& ldrow, const double2* src0,
                                             const double2* src1, double2* ringw, int jload, int ya, int yb,
                                             bool wany, double s) {
    cp_async_wait_b<kPref2 - 1>();
    __syncthreads();
    if (j + kPref2 <= jload) {
      double2* dst = ringw + ((slot + kPref2) & (kRing2 - 1)) * (2 * T.NP);
      const int64_t off = (int64_t)ldrow * a.n;
      cp_async16b(dst, src0 + off);
      cp_async16b(dst + T.NP, src1 + off);
    }
    cp_async_commit_b();
    ldrow = ldrow + 1 == a.n ? 0 : ldrow + 1;
    const int rout = j - 2 * NAPP + 1;
    const bool store = wany && rout >= ya && rout < yb;
    band2_iter<NAPP, RK4, SITE, EXACT, PH>(a, T, R, j, slot, outp, store, s);
    ++j;
    slot = (slot + 1) & (kRing2 - 1);
    outp += a.n;
    if constexpr (PH + 1 < PERIOD)
      Band2Phases<NAPP, RK4, SITE, EXACT, PH + 1, PERIOD>::run(a, T, R, j, slot, outp, ldrow, src0, src1, ringw,
                                                               jload, ya, yb, wany, s);
  }
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL>
__global__ void __launch_bounds__(kMaxPairs, 2) band2_kernel(const __grid_constant__ Band2Args a) {
  extern __shared__ double4 smem_raw[];
  constexpr int PERIOD = Band2Period<NAPP>::value;
  constexpr int NROWS = NAPP > 1 ? (NAPP - 1) * 3 : 1;
  constexpr int X = kPad2;
  const int NP = blockDim.x;
  const int RS = 2 * NP;
  const int n = a.n;
  double2* ring = reinterpret_cast<double2*>(smem_raw);  // [kRing2][2][NP]
  double2* rows = ring + kRing2 * RS;                    // [NROWS][2][NP]
  double2* hop2 = rows + NROWS * RS;                     // [n + 2X]
  double* sitex = reinterpret_cast<double*>(hop2 + n + 2 * X);
  double* red = sitex + (SITE ? n + 2 * X : 0);

  if (*a.fail != kNoFail) return;
  const int64_t dim = (int64_t)n * n;
  const int p = threadIdx.x;
  const int band = blockIdx.x % a.nbands;
  const int seg = blockIdx.x / a.nbands;
  const int64_t r = a.r_base + blockIdx.y;
  const int halo = FULL ? 0 : kHalo2;
  const int col0 = band * a.W - halo;
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.stride : nullptr;
  for (int i = p; i < n + 2 * X; i += NP) {
    const int g = wrap(i - X, n);
    hop2[i] = make_double2(hop[g == 0 ? n - 1 : g - 1], hop[g]);
    if (SITE) sitex[i] = site[g];
  }
  Band2Thread T;
  T.NP = NP;
  T.gx0 = wrap(col0 + 2 * p, n);
  T.gx1 = wrap(col0 + 2 * p + 1, n);
  T.hxm0 = hop[T.gx0 == 0 ? n - 1 : T.gx0 - 1];
  T.hx0 = hop[T.gx0];
  T.hx1 = hop[T.gx1];
  T.sx0 = SITE ? site[T.gx0] : 0.0;
  T.sx1 = SITE ? site[T.gx1] : 0.0;
  int pl, pr;
  if (FULL) {
    pl = p == 0 ? NP - 1 : p - 1;
    pr = p == NP - 1 ? 0 : p + 1;
  } else {
    pl = p > 0 ? p - 1 : p;
    pr = p < NP - 1 ? p + 1 : p;
  }
  T.dl = pl - p;
  T.dr = pr - p;
  T.ringp = ring + p;
  T.rowp = rows + p;
  T.hop2 = hop2 + X;
  T.sitex = sitex + X;
  const int c0 = 2 * p, c1 = 2 * p + 1;
  T.w0 = FULL || (c0 >= halo && c0 < halo + a.W && band * a.W + c0 - halo < n);
  T.w1 = FULL || (c1 >= halo && c1 < halo + a.W && band * a.W + c1 - halo < n);
  const bool wany = T.w0 || T.w1;
  const double s = a.scl ? a.scl[r] : 1.0;  // pending rescale of the previous step (1.0 is exact)
  const int ya = seg * a.seg_len;
  const int yb = min(n, ya + a.seg_len);
  const int j0 = ya - NAPP;
  const int jload = yb - 1 + NAPP;
  const int j1 = yb + 2 * NAPP - 2;
  const double2* src0 = a.psi_in + r * dim + T.gx0;
  const double2* src1 = a.psi_in + r * dim + T.gx1;
  // in full-row mode the pair is contiguous in HBM (gx1 = gx0 + 1)
  double2* outp = a.psi_out + r * dim + T.gx0 + (int64_t)(j0 - 2 * NAPP + 1) * n;

  for (int i = p; i < (kRing2 + NROWS) * RS; i += NP) ring[i] = make_double2(0.0, 0.0);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kPref2; ++q) {
    const int jr = j0 + q;
    if (jr <= jload) {
      const int64_t off = (int64_t)wrap_r(jr, n) * n;
      cp_async16b(ring + q * RS + p, src0 + off);
      cp_async16b(ring + q * RS + NP + p, src1 + off);
    }
    cp_async_commit_b();
  }
  int ldrow = wrap_r(j0 + kPref2, n);

  Band2Regs<NAPP> R;
#pragma unroll
  for (int k = 0; k < NAPP; ++k)
#pragma unroll
    for (int q = 0; q < 3; ++q) R.win[k][q].c[0] = R.win[k][q].c[1] = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < Band2Regs<NAPP>::NACC; ++q) R.acc[q].c[0] = R.acc[q].c[1] = make_double2(0.0, 0.0);
  R.nrm = 0.0;
  int slot = 0;
  int j = j0;
  const int iters = j1 - j0 + 1;
  // outp indexes column gx0; column gx1 is outp[1] only when adjacent in HBM
  // (always in full-row mode; haloed bands wrap inside the band otherwise)
#pragma unroll 1
  for (int t = 0; t < iters; t += PERIOD)
    Band2Phases<NAPP, RK4, SITE, EXACT, 0, PERIOD>::run(a, T, R, j, slot, outp, ldrow, src0, src1, ring + p,
                                                       jload, ya, yb, wany, s);
  cp_async_wait_b<0>();
  const double b = block_sum(R.nrm, red);
  if (p == 0 && a.partial) a.partial[r * a.nparts + blockIdx.x] = b;
}

struct Band2Plan {
  bool full;
  int W, nbands, threads, nseg, seg_len;
  size_t smem;
};

Band2Plan plan_band2(int n, int napp, bool site, int64_t count, int num_sms) {
  Band2Plan p{};
  p.full = (n % 64 == 0) && n / 2 <= kMaxPairs;
  if (p.full) {
    p.W = n;
    p.nbands = 1;
    p.threads = n / 2;
  } else {
    // haloed bands of <= 2*kMaxPairs - 2*halo columns, an even number so the
    // pairs of the interior stay aligned to even global columns
    const int wmax = 2 * kMaxPairs - 2 * kHalo2;
    p.nbands = (n + wmax - 1) / wmax;
    p.W = (n + p.nbands - 1) / p.nbands;
    p.W += p.W & 1;
    p.threads = (((p.W + 2 * kHalo2 + 1) / 2 + 31) / 32) * 32;
  }
  const int rows = napp > 1 ? (napp - 1) * 3 : 1;
  p.smem = (size_t)(kRing2 + rows) * 2 * p.threads * sizeof(double2) + (size_t)(n + 2 * kPad2) * sizeof(double2) +
           (size_t)((site ? n + 2 * kPad2 : 0) + 32) * sizeof(double);
  const int per_sm = (int)std::min<size_t>(2, (227 * 1024) / (p.smem + 1024));
  const int slots = num_sms * (per_sm > 0 ? per_sm : 1);
  double best = 1e30;
  p.nseg = 1;
  for (int ns = 1; ns <= 8; ++ns) {
    const int len = (n + ns - 1) / ns;
    if (len < 4 * napp) break;
    const double items = (double)count * p.nbands * ns;
    const double waves = items / slots;
    const double cost = (waves <= 1.0 ? 1.0 : std::ceil(waves)) * (len + 3.0 * napp - 1.0);
    if (cost < best - 1e-9) {
      best = cost;
      p.nseg = ns;
    }
  }
  p.seg_len = (n + p.nseg - 1) / p.nseg;
  return p;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL>
cudaError_t launch_b2(const Band2Args& args, const Band2Plan& p, int64_t count, cudaStream_t s) {
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(band2_kernel<NAPP, RK4, SITE, EXACT, FULL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  Band2Args a = args;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    a.r_base = r0;
    band2_kernel<NAPP, RK4, SITE, EXACT, FULL>
        <<<dim3((unsigned)(p.nbands * p.nseg), (unsigned)rows), p.threads, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <int NAPP, bool RK4>
cudaError_t launch_b2_n(const Band2Args& a, const Band2Plan& p, int64_t count, bool site, bool exact,
                        cudaStream_t s) {
  if (p.full) {
    if (site && exact) return launch_b2<NAPP, RK4, true, true, true>(a, p, count, s);
    if (site) return launch_b2<NAPP, RK4, true, false, true>(a, p, count, s);
    if (exact) return launch_b2<NAPP, RK4, false, true, true>(a, p, count, s);
    return launch_b2<NAPP, RK4, false, false, true>(a, p, count, s);
  }
  if (site && exact) return launch_b2<NAPP, RK4, true, true, false>(a, p, count, s);
  if (site) return launch_b2<NAPP, RK4, true, false, false>(a, p, count, s);
  if (exact) return launch_b2<NAPP, RK4, false, true, false>(a, p, count, s);
  return launch_b2<NAPP, RK4, false, false, false>(a, p, count, s);
}

int sm_count2() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

}  // namespace

bool band2_supported(int m, int n, const StepScalars& sc, bool exact, bool force) {
  // Measured on B200: before the four-column kernel,
  // the two-column kernel won for Taylor steps in FMA mode and for N = 512;
  // the warp-specialised one-column kernel for exact-order Taylor at
  // N <= 256, for RK4 (the pair kernel spills) and for haloed bands.
  const bool ok = m == 2 && n >= 16 && (sc.backend == 1 || (sc.order >= 1 && sc.order <= 4));
  if (!ok) return false;
  if (force) return true;
  return sc.backend == 0 && n <= 512 && (!exact || n > 256);
}

int band2_parts(int n, const StepScalars& sc, bool site, int64_t count) {
  const Band2Plan p = plan_band2(n, sc.backend == 1 ? 4 : sc.order, site, count, sm_count2());
  return p.nbands * p.nseg;
}

cudaError_t launch_band2_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                              const Coef& coef, const StencilConst& k, const StepScalars& sc,
                              bool exact, const double* scl, double* partial,
                              const long long* fail, cudaStream_t s) {
  const bool site = coef.site != nullptr;
  const int napp = sc.backend == 1 ? 4 : sc.order;
  const Band2Plan p = plan_band2(n, napp, site, count, sm_count2());
  Band2Args a;
  a.psi_in = psi_in;
  a.psi_out = psi_out;
  a.n = n;
  a.W = p.W;
  a.nbands = p.nbands;
  a.seg_len = p.seg_len;
  a.nseg = p.nseg;
  a.r_base = 0;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.scl = scl;
  a.partial = partial;
  a.nparts = p.nbands * p.nseg;
  a.fail = fail;
  if (sc.backend == 1) return launch_b2_n<4, true>(a, p, count, site, exact, s);
  switch (napp) {
    case 1: return launch_b2_n<1, false>(a, p, count, site, exact, s);
    case 2: return launch_b2_n<2, false>(a, p, count, site, exact, s);
    case 3: return launch_b2_n<3, false>(a, p, count, site, exact, s);
    case 4: return launch_b2_n<4, false>(a, p, count, site, exact, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ctqw
