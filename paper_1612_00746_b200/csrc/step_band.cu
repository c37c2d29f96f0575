// Row-marching streaming step kernel for m = 2 (the HBM-bound hot path).
//
// One CTA owns one realization's column band (the full ring when N is a
// multiple of 32 and <= 512, otherwise a band with a 4-column halo on each
// side) and marches down the N rows of the joint grid once per time step.
// Every thread owns one column.  All stencil applications of the step run
// as a software pipeline over rows: at iteration j
//
//   stage 1 computes t1 for row j-1   (needs psi rows j-2, j-1, j)
//   stage k computes t_k for row j-2k+1 (needs t_{k-1} rows j-2k .. j-2k+2)
//
// so each stage lags the previous one by two rows.  A thread keeps, per
// stage, the three-row window of its column in registers (vertical
// neighbours) and gets the horizontal neighbours of the centre row from its
// lanes by warp shuffles; the two warp-edge lanes read them from a small
// shared-memory slot published two iterations earlier, so one __syncthreads
// per row is the only block-wide synchronisation.  Rows of psi stream in
// through a 16-row cp.async ring (8 rows of prefetch) and each finished row
// is written straight from registers, so HBM sees the state once in and once
// out per step (plus 3*napp-1 wrap rows per row segment) -- no y-halo and no
// reliance on L2 for halo re-reads.
//
// Arithmetic is the same as the reference's (hamiltonian.py:205-222,
// propagators.py:185-193 / 213-240): EXACT keeps every product and sum
// separately rounded in the reference order; the running Taylor sum is
// accumulated term by term ((((psi + t1) + t2) + t3) + t4).
#include "ctqw_device.cuh"
#include "kernels.h"

#include <cmath>
#include <cstdlib>

namespace ctqw {

namespace {

// psi rows resident in shared memory (half of them prefetched ahead): one
// 256-thread CTA per SM keeps 16 rows in flight, 512-thread CTAs 8.
constexpr int ring_rows(int maxt) { return maxt <= 256 ? 32 : 16; }
constexpr int kBandHalo = 4;    // x halo (non-full-row bands)
constexpr int kBandMaxThreads = 512;
constexpr int kCoefPad = 8;      // coefficient rows padded by wrap on both sides

struct BandArgs {
  const double2* psi_in;
  double2* psi_out;
  int n;
  int W;          // interior columns per band
  int nbands;
  int seg_len;    // output rows per row segment
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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_down2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

__device__ __forceinline__ int wrap_row(int r, int n) { return r < 0 ? r + n : (r >= n ? r - n : r); }

// (H t)(row r, column x) in the reference order: diagonal, particle 0 +/-
// (rows), particle 1 +/- (columns).
template <bool EXACT>
__device__ __forceinline__ double2 stencil5(double v0, double2 up, double2 mid, double2 dn, double2 lf,
                                            double2 rt, double hr, double hrm, double hc, double hcm) {
  double2 h = rmul(v0, mid);
  h = madd<EXACT>(h, hr, dn);
  h = madd<EXACT>(h, hrm, up);
  h = madd<EXACT>(h, hc, rt);
  h = madd<EXACT>(h, hcm, lf);
  return h;
}

// Per-thread values of one band CTA (kept few: everything uniform comes from
// the kernel parameters, i.e. the constant bank).
struct BandThread {
  const double2* ringc;   // own column of the psi ring
  double2* rowc;          // own column of the stage row buffers (warp-specialised kernel)
  int dl, dr;             // offsets of the left / right neighbour columns
  const double* hopx;     // hop[wrap(row)] at hopx[row]
  const double2* hop2;    // (hop[row-1], hop[row]) at hop2[row]
  const double* sitex;
  const double2* edl;     // edge slots: left / right neighbour warps, own lane
  const double2* edr;
  double2* edw;
  int NT;
  int gx;
  double hx, hxm, sx;
  bool writer, takeL, takeR, publish;
};

template <int NAPP>
struct BandRegs {
  static constexpr int NACC = 2 * NAPP - 2 > 0 ? 2 * NAPP - 2 : 1;
  double2 win[NAPP][3];   // per-stage 3-row windows, physical slot = producing iteration mod 3
  double2 acc[NACC];      // running sums of rows in flight, slot = creating iteration mod NACC
  double nrm;
};

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
template <int NAPP>
struct BandPeriod {
  static constexpr int NACC = BandRegs<NAPP>::NACC;
  static constexpr int value = 3 * NACC / gcd_c(3, NACC);  // lcm(3, NACC)
};

// One row iteration at phase PH = (j - j0) mod period.  All register-array
// indices are compile-time, so the rotating windows need no moves.  Stages
// run unconditionally: during the pipeline ramp they compute rows outside
// the segment whose values are never consumed by an in-range row (each
// stage's in-range rows only read in-range rows of the previous stage), and
// only in-range rows of the last stage are stored.
//
// Horizontal neighbours come from warp shuffles of the centre row; only the
// two warp-edge lanes exchange through shared memory (slots published two
// iterations earlier), so the shared-memory datapath carries just the psi
// ring and a few edge values per warp.
template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int RING>
__device__ __forceinline__ void band_iter(const BandArgs& a, const BandThread& T, BandRegs<NAPP>& R,
                                          int j, int slot, double2* outp, bool store, double s) {
  constexpr int NACC = BandRegs<NAPP>::NACC;
  constexpr int ES = NAPP > 1 ? (NAPP - 1) * 3 : 1;
  constexpr int P0 = PH % 3, P1 = (PH + 1) % 3, P2 = (PH + 2) % 3;
  const double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  const int n = a.n;
  const int NT = T.NT;
  const double2* h2 = T.hop2 + j;
  const double* sj = T.sitex + j;
  // ---- stages NAPP .. 2 ----
#pragma unroll
  for (int k = NAPP; k >= 2; --k) {
    const int rr = j - 2 * k + 1;
    const double2 up = R.win[k - 1][P0], mid = R.win[k - 1][P1], dn = R.win[k - 1][P2];
    double2 lf = shfl_up2(mid), rt = shfl_down2(mid);
    if (T.takeL) lf = T.edl[(k - 2) * 3 + P1];
    if (T.takeR) rt = T.edr[(k - 2) * 3 + P1];
    const int gy = wrap_row(rr, n);
    double v0 = gy == T.gx ? a.k.base[1] : a.k.base[0];
    if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sj[1 - 2 * k], T.sx));
    const double2 hp = h2[1 - 2 * k];  // (hop[rr-1], hop[rr])
    const double2 h = stencil5<EXACT>(v0, up, mid, dn, lf, rt, hp.y, hp.x, T.hx, T.hxm);
    const double2 st = times_i(RK4 ? a.ci[0] : a.ci[k - 1], h);
    const int AS = ((PH - 2 * k + 2) % NACC + NACC) % NACC;
    double2 newt;
    if (!RK4) {
      if (k == NAPP) {
        const double2 out = cadd(R.acc[AS], st);
        if (store) {
          *outp = out;
          R.nrm += norm2(out);
        }
      } else {
        R.acc[AS] = cadd(R.acc[AS], st);
        newt = st;
      }
    } else {
      if (k == 4) {
        const double2 out = cadd(R.acc[AS], rmul(c16, st));
        if (store) {
          *outp = out;
          R.nrm += norm2(out);
        }
      } else {
        const double2 p0 = rmul(s, T.ringc[((slot - 2 * k + 1) & (RING - 1)) * NT]);
        if (k == 2) {
          newt = cadd(rmul(0.5, st), p0);
          R.acc[AS] = cadd(R.acc[AS], rmul(c13, st));
        } else {
          newt = cadd(st, p0);
          R.acc[AS] = cadd(R.acc[AS], rmul(c13, st));
        }
      }
    }
    if (k < NAPP) {
      R.win[k][P0] = newt;
      if (T.publish) T.edw[(k - 1) * 3 + P0] = newt;
    }
  }
  // ---- stage 1: psi rows j-2, j-1, j (row j from the ring) ----
  {
    const int rr = j - 1;
    const double2 pj = rmul(s, T.ringc[slot * NT]);
    R.win[0][P0] = pj;
    const double2 mid = R.win[0][P2];
    double2 lf = shfl_up2(mid), rt = shfl_down2(mid);
    const double2* rowm = T.ringc + ((slot - 1) & (RING - 1)) * NT;
    if (T.takeL) lf = rmul(s, rowm[T.dl]);
    if (T.takeR) rt = rmul(s, rowm[T.dr]);
    const int gy = wrap_row(rr, n);
    double v0 = gy == T.gx ? a.k.base[1] : a.k.base[0];
    if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sj[-1], T.sx));
    const double2 hp = h2[-1];
    const double2 h = stencil5<EXACT>(v0, R.win[0][P1], mid, pj, lf, rt, hp.y, hp.x, T.hx, T.hxm);
    const double2 st = times_i(a.ci[0], h);
    double2 newt, newacc;
    if (!RK4) {
      if (NAPP == 1) {
        const double2 out = cadd(mid, st);
        if (store) {
          *outp = out;
          R.nrm += norm2(out);
        }
      } else {
        newacc = cadd(mid, st);
        newt = st;
      }
    } else {
      newt = cadd(rmul(0.5, st), mid);
      newacc = cadd(mid, rmul(c16, st));
    }
    if (NAPP > 1) {
      R.acc[PH % NACC] = newacc;
      R.win[1][P0] = newt;
      if (T.publish) T.edw[0 * 3 + P0] = newt;
    }
  }
  (void)ES;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int PERIOD, int RING>
struct BandPhases {
  static constexpr int PREF = RING / 2;
  __device__ __forceinline__ static void run(const BandArgs& a, const BandThread& T, BandRegs<NAPP>& R,
                                             int& j, int& slot, double2*& outp, int& ldrow,
                                             const double2* srcc, double2* ringw, int jload, int ya,
                                             int yb, double s) {
    cp_async_wait<PREF - 1>();
    __syncthreads();
    if (j + PREF <= jload) cp_async16(ringw + ((slot + PREF) & (RING - 1)) * T.NT, srcc + (int64_t)ldrow * a.n);
    cp_async_commit();
    ldrow = ldrow + 1 == a.n ? 0 : ldrow + 1;
    const int rout = j - 2 * NAPP + 1;  // row finished by the last stage
    const bool store = T.writer && rout >= ya && rout < yb;
    band_iter<NAPP, RK4, SITE, EXACT, PH, RING>(a, T, R, j, slot, outp, store, s);
    ++j;
    slot = (slot + 1) & (RING - 1);
    outp += a.n;
    BandPhases<NAPP, RK4, SITE, EXACT, PH + 1, PERIOD, RING>::run(a, T, R, j, slot, outp, ldrow, srcc, ringw, jload,
                                                            ya, yb, s);
  }
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PERIOD, int RING>
struct BandPhases<NAPP, RK4, SITE, EXACT, PERIOD, PERIOD, RING> {
  __device__ __forceinline__ static void run(const BandArgs&, const BandThread&, BandRegs<NAPP>&, int&, int&,
                                             double2*&, int&, const double2*, double2*, int, int, int,
                                             double) {}
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) band_step_kernel(const __grid_constant__ BandArgs a) {
  extern __shared__ double4 smem_raw[];
  constexpr int RING = ring_rows(MAXT);
  constexpr int PREF = RING / 2;
  constexpr int PERIOD = BandPeriod<NAPP>::value;
  constexpr int ES = NAPP > 1 ? (NAPP - 1) * 3 : 1;
  const int NT = blockDim.x;
  const int nwarps = NT >> 5;
  const int n = a.n;
  constexpr int X = kCoefPad;
  double2* ring = reinterpret_cast<double2*>(smem_raw);                 // [RING][NT]
  double2* edges = ring + RING * NT;                                    // [nwarps][2][ES]
  double2* hop2 = edges + nwarps * 2 * ES;                              // [n + 2X]
  double* hopx = reinterpret_cast<double*>(hop2 + n + 2 * X);           // [n + 2X]
  double* sitex = hopx + n + 2 * X;
  double* red = sitex + (SITE ? n + 2 * X : 0);

  if (*a.fail != kNoFail) return;
  const int64_t dim = (int64_t)n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int band = blockIdx.x % a.nbands;
  const int seg = blockIdx.x / a.nbands;
  const int64_t r = a.r_base + blockIdx.y;
  const int halo = FULL ? 0 : kBandHalo;
  const int c = tid;
  const int gx = wrap(band * a.W - halo + c, n);
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.stride : nullptr;
  for (int i = tid; i < n + 2 * X; i += NT) {
    const int g = wrap(i - X, n);
    hopx[i] = hop[g];
    hop2[i] = make_double2(hop[g == 0 ? n - 1 : g - 1], hop[g]);
    if (SITE) sitex[i] = site[g];
  }
  BandThread T;
  T.NT = NT;
  T.gx = gx;
  T.hx = hop[gx];
  T.hxm = hop[gx == 0 ? n - 1 : gx - 1];
  T.sx = SITE ? site[gx] : 0.0;
  int cl, cr;
  if (FULL) {
    cl = c == 0 ? NT - 1 : c - 1;
    cr = c == NT - 1 ? 0 : c + 1;
  } else {
    cl = c > 0 ? c - 1 : c;
    cr = c < NT - 1 ? c + 1 : c;
  }
  T.ringc = ring + c;
  T.rowc = nullptr;
  T.dl = cl - c;
  T.dr = cr - c;
  T.hopx = hopx + X;
  T.hop2 = hop2 + X;
  T.sitex = sitex + X;
  T.edl = edges + (((warp + nwarps - 1) % nwarps) * 2 + 1) * ES;
  T.edr = edges + (((warp + 1) % nwarps) * 2 + 0) * ES;
  T.edw = edges + (warp * 2 + (lane == 31 ? 1 : 0)) * ES;
  T.takeL = lane == 0 && (FULL || warp > 0);
  T.takeR = lane == 31 && (FULL || warp < nwarps - 1);
  T.publish = lane == 0 || lane == 31;
  T.writer = FULL || (c >= halo && c < halo + a.W && band * a.W + c - halo < n);
  const double s = a.scl ? a.scl[r] : 1.0;  // pending rescale of the previous step (1.0 is exact)
  const int ya = seg * a.seg_len;
  const int yb = min(n, ya + a.seg_len);
  const int j0 = ya - NAPP;           // first loaded row == first iteration
  const int jload = yb - 1 + NAPP;    // last loaded row
  const int j1 = yb + 2 * NAPP - 2;   // last iteration
  const double2* srcc = a.psi_in + r * dim + gx;
  double2* outp = a.psi_out + r * dim + gx + (int64_t)(j0 - 2 * NAPP + 1) * n;

  // ring slots read before they are first loaded must hold finite values
  for (int i = tid; i < RING * NT + nwarps * 2 * ES; i += NT) ring[i] = make_double2(0.0, 0.0);
  __syncthreads();
#pragma unroll
  for (int p = 0; p < PREF; ++p) {
    const int jr = j0 + p;
    if (jr <= jload) cp_async16(ring + p * NT + c, srcc + (int64_t)wrap_row(jr, n) * n);
    cp_async_commit();
  }
  int ldrow = wrap_row(j0 + PREF, n);

  BandRegs<NAPP> R;
#pragma unroll
  for (int k = 0; k < NAPP; ++k)
#pragma unroll
    for (int q = 0; q < 3; ++q) R.win[k][q] = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < BandRegs<NAPP>::NACC; ++q) R.acc[q] = make_double2(0.0, 0.0);
  R.nrm = 0.0;
  int slot = 0;
  int j = j0;
  const int iters = j1 - j0 + 1;
#pragma unroll 1
  for (int t = 0; t < iters; t += PERIOD)
    BandPhases<NAPP, RK4, SITE, EXACT, 0, PERIOD, RING>::run(a, T, R, j, slot, outp, ldrow, srcc, ring + c,
                                                             jload, ya, yb, s);
  cp_async_wait<0>();
  const double b = block_sum(R.nrm, red);
  if (tid == 0 && a.partial) a.partial[r * a.nparts + blockIdx.x] = b;
}

// ---------------------------------------------------------------------------
// Warp-specialised variant: the 256 columns of a band are processed by two
// thread groups of one thread per column.  Group A runs stages 1..KA, group B
// stages KA+1..NAPP; A hands B each finished t_KA row and the matching running
// sum through shared memory (the same two-iteration lag as the x-neighbour
// rows, so one __syncthreads per row still suffices).  Each thread holds half
// the pipeline's registers, which doubles the warps per SM (16 instead of 8)
// for latency hiding at the same shared-memory footprint.

template <int NAPP>
struct WsSplit {
  static constexpr int KA = (NAPP + 1) / 2;                         // stages in group A
  static constexpr int NA = 2 * KA - 2 > 0 ? 2 * KA - 2 : 1;        // A running-sum ring
  static constexpr int NB = 2 * (NAPP - KA - 1) > 0 ? 2 * (NAPP - KA - 1) : 1;  // B ring
  static constexpr int PERIOD = 6;  // lcm(3, NA, NB) for NAPP <= 4
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int RING>
__device__ __forceinline__ void ws_iter_a(const BandArgs& a, const BandThread& T, double2 (&win)[WsSplit<NAPP>::KA][3],
                                          double2 (&acc)[WsSplit<NAPP>::NA], double2* acch, int j, int slot,
                                          double s) {
  constexpr int KA = WsSplit<NAPP>::KA, NA = WsSplit<NAPP>::NA;
  constexpr int P0 = PH % 3, P1 = (PH + 1) % 3, P2 = (PH + 2) % 3;
  const double c13 = 1.0 / 3.0, c16 = 1.0 / 6.0;
  const int n = a.n, NT = T.NT;
  const double2* hj = T.hop2 + j;
  const double* sj = T.sitex + j;
#pragma unroll
  for (int k = KA; k >= 2; --k) {
    const int rr = j - 2 * k + 1;
    const double2 up = win[k - 1][P0], mid = win[k - 1][P1], dn = win[k - 1][P2];
    const double2* prow = T.rowc + ((k - 2) * 3 + P1) * NT;
    const double2 lf = prow[T.dl], rt = prow[T.dr];
    const int gy = wrap_row(rr, n);
    double v0 = gy == T.gx ? a.k.base[1] : a.k.base[0];
    if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sj[1 - 2 * k], T.sx));
    const double2 h = stencil5<EXACT>(v0, up, mid, dn, lf, rt, hj[1 - 2 * k].y, hj[1 - 2 * k].x, T.hx, T.hxm);
    const double2 st = times_i(RK4 ? a.ci[0] : a.ci[k - 1], h);
    const int AS = ((PH - 2 * k + 2) % NA + NA) % NA;
    double2 newt;
    if (!RK4) {
      acc[AS] = cadd(acc[AS], st);
      newt = st;
    } else {  // k == 2
      const double2 p0 = rmul(s, T.ringc[((slot - 2 * k + 1) & (RING - 1)) * NT]);
      newt = cadd(rmul(0.5, st), p0);
      acc[AS] = cadd(acc[AS], rmul(c13, st));
    }
    if (k < KA) win[k][P0] = newt;
    T.rowc[((k - 1) * 3 + P0) * NT] = newt;
    if (k == KA) acch[P0 * NT] = acc[AS];
  }
  // stage 1
  const int rr = j - 1;
  const double2* rowm = T.ringc + ((slot - 1) & (RING - 1)) * NT;
  const double2 pj = rmul(s, T.ringc[slot * NT]);
  const double2 lf = rmul(s, rowm[T.dl]), rt = rmul(s, rowm[T.dr]);
  win[0][P0] = pj;
  const int gy = wrap_row(rr, n);
  double v0 = gy == T.gx ? a.k.base[1] : a.k.base[0];
  if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sj[-1], T.sx));
  const double2 mid = win[0][P2];
  const double2 h = stencil5<EXACT>(v0, win[0][P1], mid, pj, lf, rt, hj[-1].y, hj[-1].x, T.hx, T.hxm);
  const double2 st = times_i(a.ci[0], h);
  double2 newt, newacc;
  if (!RK4) {
    newacc = cadd(mid, st);
    newt = st;
  } else {
    newt = cadd(rmul(0.5, st), mid);
    newacc = cadd(mid, rmul(c16, st));
  }
  if (KA > 1) {
    acc[PH % NA] = newacc;
    win[KA > 1 ? 1 : 0][P0] = newt;
  } else {
    acch[P0 * NT] = newacc;
  }
  T.rowc[(0 * 3 + P0) * NT] = newt;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int RING>
__device__ __forceinline__ void ws_iter_b(const BandArgs& a, const BandThread& T,
                                          double2 (&win)[NAPP - WsSplit<NAPP>::KA][3],
                                          double2 (&acc)[WsSplit<NAPP>::NB], const double2* acch, int j,
                                          int slot, double2* outp, bool store, double s, double& nrm) {
  constexpr int KA = WsSplit<NAPP>::KA, NB = WsSplit<NAPP>::NB;
  constexpr int P0 = PH % 3, P1 = (PH + 1) % 3, P2 = (PH + 2) % 3;
  const double c13 = 1.0 / 3.0, c16 = 1.0 / 6.0;
  const int n = a.n, NT = T.NT;
  const double2* hj = T.hop2 + j;
  const double* sj = T.sitex + j;
  // newest t_KA row (produced by A last iteration)
  win[0][P2] = T.rowc[((KA - 1) * 3 + P2) * NT];
#pragma unroll
  for (int k = NAPP; k >= KA + 1; --k) {
    const int w = k - 1 - KA;  // B-local window index of t_{k-1}
    // the running sum A finished two iterations ago enters the B ring only
    // after the last stage has consumed the slot it reuses
    if (k == KA + 1) acc[PH % NB] = acch[P1 * NT];
    const int rr = j - 2 * k + 1;
    const double2 up = win[w][P0], mid = win[w][P1], dn = win[w][P2];
    const double2* prow = T.rowc + ((k - 2) * 3 + P1) * NT;
    const double2 lf = prow[T.dl], rt = prow[T.dr];
    const int gy = wrap_row(rr, n);
    double v0 = gy == T.gx ? a.k.base[1] : a.k.base[0];
    if (SITE) v0 = __dadd_rn(v0, __dadd_rn(sj[1 - 2 * k], T.sx));
    const double2 h = stencil5<EXACT>(v0, up, mid, dn, lf, rt, hj[1 - 2 * k].y, hj[1 - 2 * k].x, T.hx, T.hxm);
    const double2 st = times_i(RK4 ? a.ci[0] : a.ci[k - 1], h);
    const int AS = ((PH - 2 * (k - KA - 1)) % NB + NB) % NB;
    if (k == NAPP) {
      const double2 out = RK4 ? cadd(acc[AS], rmul(c16, st)) : cadd(acc[AS], st);
      if (store) {
        *outp = out;
        nrm += norm2(out);
      }
    } else {
      double2 newt;
      if (!RK4) {
        acc[AS] = cadd(acc[AS], st);
        newt = st;
      } else {  // k == 3
        const double2 p0 = rmul(s, T.ringc[((slot - 2 * k + 1) & (RING - 1)) * NT]);
        newt = cadd(st, p0);
        acc[AS] = cadd(acc[AS], rmul(c13, st));
      }
      win[w + 1][P0] = newt;
      T.rowc[((k - 1) * 3 + P0) * NT] = newt;
    }
  }
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int RING>
struct WsPhases {
  static constexpr int PREF = RING / 2;
  static constexpr int KA = WsSplit<NAPP>::KA;
  __device__ __forceinline__ static void run_a(const BandArgs& a, const BandThread& T, double2 (&win)[KA][3],
                                               double2 (&acc)[WsSplit<NAPP>::NA], double2* acch, int& j,
                                               int& slot, int& ldrow, const double2* srcc, double2* ringw,
                                               int jload, double s) {
    cp_async_wait<PREF - 1>();
    __syncthreads();
    if (j + PREF <= jload) cp_async16(ringw + ((slot + PREF) & (RING - 1)) * T.NT, srcc + (int64_t)ldrow * a.n);
    cp_async_commit();
    ldrow = ldrow + 1 == a.n ? 0 : ldrow + 1;
    ws_iter_a<NAPP, RK4, SITE, EXACT, PH, RING>(a, T, win, acc, acch, j, slot, s);
    ++j;
    slot = (slot + 1) & (RING - 1);
    if constexpr (PH + 1 < WsSplit<NAPP>::PERIOD)
      WsPhases<NAPP, RK4, SITE, EXACT, PH + 1, RING>::run_a(a, T, win, acc, acch, j, slot, ldrow,
                                                                                  srcc, ringw, jload, s);
  }
  __device__ __forceinline__ static void run_b(const BandArgs& a, const BandThread& T,
                                               double2 (&win)[NAPP - KA][3], double2 (&acc)[WsSplit<NAPP>::NB],
                                               const double2* acch, int& j, int& slot, double2*& outp, int ya,
                                               int yb, double s, double& nrm) {
    __syncthreads();
    const int rout = j - 2 * NAPP + 1;
    const bool store = T.writer && rout >= ya && rout < yb;
    ws_iter_b<NAPP, RK4, SITE, EXACT, PH, RING>(a, T, win, acc, acch, j, slot, outp, store, s, nrm);
    ++j;
    slot = (slot + 1) & (RING - 1);
    outp += a.n;
    if constexpr (PH + 1 < WsSplit<NAPP>::PERIOD)
      WsPhases<NAPP, RK4, SITE, EXACT, PH + 1, RING>::run_b(a, T, win, acc, acch, j, slot, outp,
                                                                                  ya, yb, s, nrm);
  }
};

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL>
__global__ void __launch_bounds__(512, 1) band_ws_kernel(const __grid_constant__ BandArgs a) {
  extern __shared__ double4 smem_raw[];
  constexpr int RING = 32;
  constexpr int PREF = RING / 2;
  constexpr int KA = WsSplit<NAPP>::KA;
  constexpr int PERIOD = WsSplit<NAPP>::PERIOD;
  constexpr int NROWBUF = (NAPP - 1) * 3;
  const int NT = blockDim.x >> 1;  // columns
  const int n = a.n;
  constexpr int X = kCoefPad;
  double2* ring = reinterpret_cast<double2*>(smem_raw);   // [RING][NT]
  double2* rows = ring + RING * NT;                      // [NAPP-1][3][NT]
  double2* acch = rows + NROWBUF * NT;                   // [3][NT]
  double2* hop2 = acch + 3 * NT;                         // (hop[r-1], hop[r])
  double* hopx = reinterpret_cast<double*>(hop2 + n + 2 * X);
  double* sitex = hopx + n + 2 * X;
  double* red = sitex + (SITE ? n + 2 * X : 0);

  if (*a.fail != kNoFail) return;
  const int64_t dim = (int64_t)n * n;
  const int tid = threadIdx.x;
  const bool groupA = tid < NT;
  const int c = groupA ? tid : tid - NT;
  const int band = blockIdx.x % a.nbands;
  const int seg = blockIdx.x / a.nbands;
  const int64_t r = a.r_base + blockIdx.y;
  const int halo = FULL ? 0 : kBandHalo;
  const int gx = wrap(band * a.W - halo + c, n);
  const double* hop = a.coef.hop + r * a.coef.stride;
  const double* site = SITE ? a.coef.site + r * a.coef.stride : nullptr;
  for (int i = tid; i < n + 2 * X; i += blockDim.x) {
    const int g = wrap(i - X, n);
    hopx[i] = hop[g];
    hop2[i] = make_double2(hop[g == 0 ? n - 1 : g - 1], hop[g]);
    if (SITE) sitex[i] = site[g];
  }
  BandThread T;
  T.NT = NT;
  T.gx = gx;
  T.hx = hop[gx];
  T.hxm = hop[gx == 0 ? n - 1 : gx - 1];
  T.sx = SITE ? site[gx] : 0.0;
  int cl, cr;
  if (FULL) {
    cl = c == 0 ? NT - 1 : c - 1;
    cr = c == NT - 1 ? 0 : c + 1;
  } else {
    cl = c > 0 ? c - 1 : c;
    cr = c < NT - 1 ? c + 1 : c;
  }
  T.ringc = ring + c;
  T.rowc = rows + c;
  T.dl = cl - c;
  T.dr = cr - c;
  T.hopx = hopx + X;
  T.hop2 = hop2 + X;
  T.sitex = sitex + X;
  T.edl = T.edr = nullptr;
  T.edw = nullptr;
  T.takeL = T.takeR = T.publish = false;
  T.writer = FULL || (c >= halo && c < halo + a.W && band * a.W + c - halo < n);
  const double s = a.scl ? a.scl[r] : 1.0;
  const int ya = seg * a.seg_len;
  const int yb = min(n, ya + a.seg_len);
  const int j0 = ya - NAPP;
  const int jload = yb - 1 + NAPP;
  const int j1 = yb + 2 * NAPP - 2;
  const double2* srcc = a.psi_in + r * dim + gx;

  for (int i = tid; i < (RING + NROWBUF + 3) * NT; i += blockDim.x) ring[i] = make_double2(0.0, 0.0);
  __syncthreads();
  int ldrow = wrap_row(j0 + PREF, n);
  if (groupA) {
#pragma unroll
    for (int p = 0; p < PREF; ++p) {
      const int jr = j0 + p;
      if (jr <= jload) cp_async16(ring + p * NT + c, srcc + (int64_t)wrap_row(jr, n) * n);
      cp_async_commit();
    }
  }
  const int iters = j1 - j0 + 1;
  int slot = 0;
  int j = j0;
  double nrm = 0.0;
  if (groupA) {
    double2 win[KA][3];
    double2 acc[WsSplit<NAPP>::NA];
#pragma unroll
    for (int k = 0; k < KA; ++k)
#pragma unroll
      for (int q = 0; q < 3; ++q) win[k][q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < WsSplit<NAPP>::NA; ++q) acc[q] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int t = 0; t < iters; t += PERIOD)
      WsPhases<NAPP, RK4, SITE, EXACT, 0, RING>::run_a(a, T, win, acc, acch + c, j, slot, ldrow, srcc, ring + c,
                                                       jload, s);
    cp_async_wait<0>();
  } else {
    double2 win[NAPP - KA][3];
    double2 acc[WsSplit<NAPP>::NB];
#pragma unroll
    for (int k = 0; k < NAPP - KA; ++k)
#pragma unroll
      for (int q = 0; q < 3; ++q) win[k][q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < WsSplit<NAPP>::NB; ++q) acc[q] = make_double2(0.0, 0.0);
    double2* outp = a.psi_out + r * dim + gx + (int64_t)(j0 - 2 * NAPP + 1) * n;
#pragma unroll 1
    for (int t = 0; t < iters; t += PERIOD)
      WsPhases<NAPP, RK4, SITE, EXACT, 0, RING>::run_b(a, T, win, acc, acch + c, j, slot, outp, ya, yb, s, nrm);
  }
  const double b = block_sum(nrm, red);
  if (tid == 0 && a.partial) a.partial[r * a.nparts + blockIdx.x] = b;
}

struct BandPlan {
  bool full;
  bool ws;  // warp-specialised two-group kernel
  int W, nbands, threads, nseg, seg_len, maxt;
  size_t smem;
};

int ctas_per_sm(const BandPlan& p) {
  // 256-thread variants use up to 255 registers (one CTA per SM); the
  // 512-thread variants are capped at 128 registers.
  const int by_regs = p.maxt <= 256 ? 1 : 65536 / (p.threads * 128);
  const int by_smem = (int)((227 * 1024) / (p.smem + 1024));
  const int c = by_regs < by_smem ? by_regs : by_smem;
  return c > 0 ? c : 1;
}

int env_band_ws() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("CTQW_BAND_WS");
    v = e ? std::atoi(e) : 1;
  }
  return v;
}

int env_band_maxt() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("CTQW_BAND_MAXT");
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

BandPlan plan_band(int n, int napp, bool site, int64_t count, int num_sms) {
  BandPlan p{};
  // full rows need one thread per column; beyond 256 columns the pipeline's
  // ~210 registers per thread no longer fit, so wider rings use haloed bands
  const int full_max = env_band_maxt() == 512 ? kBandMaxThreads : 256;
  p.full = (n % 32 == 0) && n <= full_max;
  if (p.full) {
    p.W = n;
    p.nbands = 1;
    p.threads = n;
    p.maxt = n <= 256 && env_band_maxt() != 512 ? 256 : 512;
  } else {
    const int wmax = 256 - 2 * kBandHalo;
    p.nbands = (n + wmax - 1) / wmax;
    p.W = (n + p.nbands - 1) / p.nbands;
    p.threads = ((p.W + 2 * kBandHalo + 31) / 32) * 32;
    p.maxt = 256;
  }
  const int rows = napp > 1 ? napp - 1 : 1;
  p.ws = env_band_ws() != 0 && napp >= 2 && p.threads <= 256;
  if (p.ws) {
    // two thread groups of `threads` columns each; 32-row ring
    p.smem = (size_t)32 * p.threads * sizeof(double2) + (size_t)(rows * 3 + 3) * p.threads * sizeof(double2) +
             (size_t)(n + 2 * kCoefPad) * sizeof(double2) +
             (size_t)((n + 2 * kCoefPad) * (site ? 2 : 1) + 32) * sizeof(double);
  } else {
    const int ES = napp > 1 ? (napp - 1) * 3 : 1;
    p.smem = (size_t)ring_rows(p.maxt) * p.threads * sizeof(double2) + (size_t)(p.threads / 32) * 2 * ES * sizeof(double2) +
             (size_t)(n + 2 * kCoefPad) * sizeof(double2) +
             (size_t)((n + 2 * kCoefPad) * (site ? 2 : 1) + 32) * sizeof(double);
  }
  // row segments: balance the wave quantisation against the pipeline ramp
  const int slots = num_sms * ctas_per_sm(p);
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

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL, int MAXT>
cudaError_t launch_band_t(const BandArgs& args, const BandPlan& p, int64_t count, cudaStream_t s) {
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(band_step_kernel<NAPP, RK4, SITE, EXACT, FULL, MAXT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  BandArgs a = args;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    a.r_base = r0;
    band_step_kernel<NAPP, RK4, SITE, EXACT, FULL, MAXT>
        <<<dim3((unsigned)(p.nbands * p.nseg), (unsigned)rows), p.threads, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool FULL>
cudaError_t launch_ws_t(const BandArgs& args, const BandPlan& p, int64_t count, cudaStream_t s) {
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(band_ws_kernel<NAPP, RK4, SITE, EXACT, FULL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  BandArgs a = args;
  for (int64_t r0 = 0; r0 < count; r0 += kMaxGridY) {
    const int64_t rows = count - r0 < kMaxGridY ? count - r0 : kMaxGridY;
    a.r_base = r0;
    band_ws_kernel<NAPP, RK4, SITE, EXACT, FULL>
        <<<dim3((unsigned)(p.nbands * p.nseg), (unsigned)rows), 2 * p.threads, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <int NAPP, bool RK4, bool SITE, bool EXACT>
cudaError_t launch_band_f(const BandArgs& a, const BandPlan& p, int64_t count, cudaStream_t s) {
  if constexpr (NAPP >= 2) {
    if (p.ws)
      return p.full ? launch_ws_t<NAPP, RK4, SITE, EXACT, true>(a, p, count, s)
                    : launch_ws_t<NAPP, RK4, SITE, EXACT, false>(a, p, count, s);
  }
  if (!p.full) return launch_band_t<NAPP, RK4, SITE, EXACT, false, 256>(a, p, count, s);
  return p.maxt <= 256 ? launch_band_t<NAPP, RK4, SITE, EXACT, true, 256>(a, p, count, s)
                       : launch_band_t<NAPP, RK4, SITE, EXACT, true, 512>(a, p, count, s);
}

template <int NAPP, bool RK4>
cudaError_t launch_band_n(const BandArgs& a, const BandPlan& p, int64_t count, bool site, bool exact,
                          cudaStream_t s) {
  if (site && exact) return launch_band_f<NAPP, RK4, true, true>(a, p, count, s);
  if (site) return launch_band_f<NAPP, RK4, true, false>(a, p, count, s);
  if (exact) return launch_band_f<NAPP, RK4, false, true>(a, p, count, s);
  return launch_band_f<NAPP, RK4, false, false>(a, p, count, s);
}

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

}  // namespace

bool band_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n >= 8 && (sc.backend == 1 || (sc.order >= 1 && sc.order <= 4));
}

int band_parts(int n, const StepScalars& sc, bool site, int64_t count) {
  const BandPlan p = plan_band(n, sc.backend == 1 ? 4 : sc.order, site, count, num_sms());
  return p.nbands * p.nseg;
}

cudaError_t launch_band_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                             const Coef& coef, const StencilConst& k, const StepScalars& sc,
                             bool exact, const double* scl, double* partial,
                             const long long* fail, cudaStream_t s) {
  const bool site = coef.site != nullptr;
  const int napp = sc.backend == 1 ? 4 : sc.order;
  const BandPlan p = plan_band(n, napp, site, count, num_sms());
  BandArgs a;
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
  if (sc.backend == 1) return launch_band_n<4, true>(a, p, count, site, exact, s);
  switch (napp) {
    case 1: return launch_band_n<1, false>(a, p, count, site, exact, s);
    case 2: return launch_band_n<2, false>(a, p, count, site, exact, s);
    case 3: return launch_band_n<3, false>(a, p, count, site, exact, s);
    case 4: return launch_band_n<4, false>(a, p, count, site, exact, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ctqw
