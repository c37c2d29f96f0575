// Dispatch of the four-column row-marching m = 2 step (band4_kernel.cuh):
// picks the compiled variant for (order, integrator, site noise, arithmetic,
// lattice size, diagonal form) and launches it.  The variants are compiled in
// band4_inst_*.cu.
#include "band4.h"

namespace ctqw {
namespace b4 {

Band4Plan plan_band4(int n, int napp, bool site, int64_t count) {
  (void)count;
  Band4Plan p{};
  p.threads = n / kCols;
  p.npad = (n + 7) & ~7;
  p.rb = (n % kRB == 0) ? kRB : n;
  p.nblk = n / p.rb;
  const int nx = napp > 1 ? napp - 1 : 1;
  p.smem = (size_t)kRing4 * p.npad * sizeof(double2) + (size_t)nx * 4 * p.threads * sizeof(double2) +
           (size_t)n * sizeof(double2) + (size_t)((site ? n : 0) + 64 + (site ? 9 : 5) * p.threads) * sizeof(double) +
           (kRing4 + 2) * sizeof(uint64_t);
  if (napp == 4 && (n == 256 || n == 512 || n == 1024) && stash_fits(n, site))
    p.smem += 16 + (size_t)4 * p.threads * sizeof(double2);  // RK4 stash (also sized for Taylor-4: harmless)
  return p;
}


namespace {

// compile-time lattice sizes and the zero-diagonal form only for the
// four-application steps (the BASELINE configurations: Taylor-4 and RK4 at
// N = 256, 512, 1024)
template <int NAPP, bool RK4, bool SITE, bool EXACT>
cudaError_t launch_b4_nn(const Band4Args& a, Band4Plan p, bool zero_diag, cudaStream_t s) {
  if constexpr (NAPP != 4) {
    return launch_b4<NAPP, RK4, SITE, EXACT, 0, 2>(a, p, s);
  } else {
    if (zero_diag) {
      switch (a.n) {
        case 256: return launch_b4<NAPP, RK4, SITE, EXACT, 256, 0>(a, p, s);
        case 512: return launch_b4<NAPP, RK4, SITE, EXACT, 512, 0>(a, p, s);
        case 1024: return launch_b4<NAPP, RK4, SITE, EXACT, 1024, 0>(a, p, s);
        default: break;
      }
    }
    switch (a.n) {
      case 256: return launch_b4<NAPP, RK4, SITE, EXACT, 256, 2>(a, p, s);
      case 512: return launch_b4<NAPP, RK4, SITE, EXACT, 512, 2>(a, p, s);
      case 1024: return launch_b4<NAPP, RK4, SITE, EXACT, 1024, 2>(a, p, s);
      default: return launch_b4<NAPP, RK4, SITE, EXACT, 0, 2>(a, p, s);
    }
  }
}

template <int NAPP, bool RK4>
cudaError_t launch_b4_n(const Band4Args& a, Band4Plan p, bool site, bool exact, bool zero_diag, cudaStream_t s) {
  if (site && exact) return launch_b4_nn<NAPP, RK4, true, true>(a, p, zero_diag, s);
  if (site) return launch_b4_nn<NAPP, RK4, true, false>(a, p, zero_diag, s);
  if (exact) return launch_b4_nn<NAPP, RK4, false, true>(a, p, zero_diag, s);
  return launch_b4_nn<NAPP, RK4, false, false>(a, p, zero_diag, s);
}

}  // namespace
}  // namespace b4

using namespace b4;

bool band4_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n % kCols == 0 && n >= 16 && n / kCols <= kMaxThreads4 &&
         (sc.backend == 1 || (sc.order >= 1 && sc.order <= 4));
}

int band4_parts(int n) { return (n % kRB == 0) ? n / kRB : 1; }

cudaError_t launch_band4_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                              const Coef& coef, const StencilConst& k, const StepScalars& sc,
                              bool exact, const double* scl, double* partial,
                              const long long* fail, cudaStream_t s, bool bcast_in) {
  const bool site = coef.site != nullptr;
  const int napp = sc.backend == 1 ? 4 : sc.order;
  const Band4Plan p = plan_band4(n, napp, site, count);
  Band4Args a;
  a.psi_in = psi_in;
  a.psi_out = psi_out;
  a.n = n;
  a.npad = p.npad;
  a.rb = p.rb;
  a.nblk = p.nblk;
  a.total = count * p.nblk;
  a.count = count;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.rkw[0] = 0.5 * sc.ci[0];
  a.rkw[1] = sc.ci[0] * (1.0 / 3.0);
  a.rkw[2] = sc.ci[0] * (1.0 / 6.0);
  a.rkw[3] = 0.0;
  a.scl = scl;
  a.partial = partial;
  a.fail = fail;
  a.bcast = bcast_in ? 1 : 0;
  if (count == 0) return cudaSuccess;
  // eps0 = U = 0: the diagonal base is zero (no multiply, no coincidence select)
  const bool zd = k.base[0] == 0.0 && k.base[1] == 0.0 && k.base[2] == 0.0 && k.base[3] == 0.0;
  if (sc.backend == 1) return launch_b4_n<4, true>(a, p, site, exact, zd, s);
  switch (napp) {
    case 1: return launch_b4_n<1, false>(a, p, site, exact, zd, s);
    case 2: return launch_b4_n<2, false>(a, p, site, exact, zd, s);
    case 3: return launch_b4_n<3, false>(a, p, site, exact, zd, s);
    case 4: return launch_b4_n<4, false>(a, p, site, exact, zd, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ctqw
