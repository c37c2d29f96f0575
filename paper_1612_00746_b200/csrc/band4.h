// band4.h -- host-side interface of the four-column row-marching m = 2
// kernel family (band4_kernel.cuh): constants, launch arguments, plan, and
// the launch template.  The kernel instantiations are spread over several
// translation units (band4_inst_*.cu) so they compile in parallel;
// step_band4.cu dispatches to them.
#pragma once

#include "ctqw_device.cuh"
#include "kernels.h"

#include <cuda.h>

namespace ctqw {
namespace b4 {

constexpr int kCols = 4;        // columns per thread
constexpr int kRing4 = 8;       // psi rows resident
constexpr int kPref4 = 5;       // rows requested ahead of the one consumed
constexpr int kRB = 32;         // rows per norm block
constexpr int kMaxThreads4 = 256;

struct Band4Args {
  CUtensorMap tmap;   // psi_in as [count*n rows][n/8 lines][16 doubles], 128B-swizzled boxes of one row
  const double2* psi_in;
  double2* psi_out;
  int n;
  int npad;         // ring row stride in 16-byte chunks (n rounded up to 8)
  int rb;           // rows per norm block
  int nblk;         // norm blocks per realization (= nparts)
  int64_t total;    // count * nblk
  int64_t count;
  Coef coef;
  StencilConst k;
  double ci[4];
  double rkw[4];    // FMA-mode RK4 weights times c: c/2, c/3, c/6 (constant bank operands)
  const double* scl;
  double* partial;
  const long long* fail;
  int bcast;          // psi_in is one state shared by every realization
};

struct Band4Plan {
  int threads, npad, rb, nblk, grid;
  size_t smem;
};

// Does the RK4 stash fit next to the rest (compile-time sizes only)?
constexpr bool stash_fits(int nn, bool site) {
  return nn > 0 && (size_t)kRing4 * nn * 16 + (size_t)3 * 4 * (nn / 4) * 16 + (size_t)nn * 16 +
                           (size_t)((site ? nn : 0) + 64 + (site ? 9 : 5) * (nn / 4)) * 8 + (kRing4 + 2) * 8 + 16 +
                           (size_t)4 * (nn / 4) * 16 <=
                       227 * 1024;
}

Band4Plan plan_band4(int n, int napp, bool site, int64_t count);

// DG: diagonal form -- 0 zero base (eps0 = U = 0), 2 general (coincidence
// select; also used for a uniform nonzero base)
template <int NAPP, bool RK4, bool SITE, bool EXACT, int NN, int DG>
cudaError_t launch_b4(const Band4Args& args, Band4Plan p, cudaStream_t s);

}  // namespace b4
}  // namespace ctqw
