// Packed ensemble density matrix: the lower triangle of
//   rho[i][j] = scale * sum_r psi_r[i] * conj(psi_r[j]),   j <= i,
// written straight into the reference's packed layout packed[i(i+1)/2 + j]
// (density.py:91-95: gram = stack.T @ stack.conj(); packed = gram[tril];
// packed /= r).  A Hermitian rank-R update restricted to the triangle
// (HERK-style): half the multiply-adds of the full complex GEMM the
// reference's BLAS call does, and no D x D transient.
//
// FP64 bound: 8 flops per (i, j, r) complex multiply-add; the packed output
// (16 B per entry) is written once.  One CTA per 64 x 64 tile of the
// triangle (bj <= bi), 256 threads, each thread a 4 x 4 register block of
// complex accumulators (rows ty + 16a, columns tx + 16c: the tile's row
// reads are broadcasts and its column reads consecutive, so shared memory
// is conflict-free, and a warp's stores are 256-byte runs of a packed row).
// Realizations are staged 16 at a time in shared memory; every accumulator
// sums r = 0 .. R-1 in order, so the result is deterministic.
#include "ctqw_device.cuh"
#include "kernels.h"

namespace ctqw {

namespace {

constexpr int kGT = 64;   // tile edge
constexpr int kGK = 16;   // realizations per shared-memory stage
constexpr int kGThreads = 256;

__global__ void __launch_bounds__(kGThreads) packed_gram_kernel(const double2* __restrict__ psi, int64_t count,
                                                                 int64_t dim, int64_t tiles_per_edge,
                                                                 double scale, double2* __restrict__ packed) {
  __shared__ double2 sa[kGK][kGT];
  __shared__ double2 sb[kGK][kGT];
  // tile t -> (bi, bj), bj <= bi, row-major over the triangle of tiles
  const int64_t t = blockIdx.x;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  const int64_t bj = t - bi * (bi + 1) / 2;
  (void)tiles_per_edge;
  const int64_t i0 = bi * kGT, j0 = bj * kGT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;

  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = make_double2(0.0, 0.0);

  for (int64_t r0 = 0; r0 < count; r0 += kGK) {
    // stage psi[r0 .. r0+16)[i0 .. i0+64) and [j0 .. j0+64): 4 + 4 per thread
#pragma unroll
    for (int e = 0; e < (kGK * kGT) / kGThreads; ++e) {
      const int idx = e * kGThreads + threadIdx.x;
      const int k = idx / kGT, col = idx % kGT;
      const int64_t r = r0 + k;
      const bool rk = r < count;
      const int64_t gi = i0 + col, gj = j0 + col;
      sa[k][col] = (rk && gi < dim) ? __ldg(psi + r * dim + gi) : make_double2(0.0, 0.0);
      sb[k][col] = (rk && gj < dim) ? __ldg(psi + r * dim + gj) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int kn = count - r0 < kGK ? (int)(count - r0) : kGK;
    for (int k = 0; k < kn; ++k) {
      double2 av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[k][ty + 16 * a];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = sb[k][tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // a * conj(b) = (ar br + ai bi) + i (ai br - ar bi)
          acc[a][c].x = fma(av[a].x, bv[c].x, acc[a][c].x);
          acc[a][c].x = fma(av[a].y, bv[c].y, acc[a][c].x);
          acc[a][c].y = fma(av[a].y, bv[c].x, acc[a][c].y);
          acc[a][c].y = fma(-av[a].x, bv[c].y, acc[a][c].y);
        }
    }
    __syncthreads();
  }

#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = i0 + ty + 16 * a;
    if (i >= dim) continue;
    double2* row = packed + i * (i + 1) / 2;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t j = j0 + tx + 16 * c;
      if (j <= i) row[j] = make_double2(acc[a][c].x * scale, acc[a][c].y * scale);
    }
  }
}

}  // namespace

cudaError_t launch_packed_gram(const double2* psi, int64_t count, int64_t dim, double scale, double2* packed,
                               cudaStream_t s) {
  if (count <= 0 || dim <= 0) return cudaSuccess;
  const int64_t te = (dim + kGT - 1) / kGT;
  const int64_t tiles = te * (te + 1) / 2;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  packed_gram_kernel<<<(unsigned)tiles, kGThreads, 0, s>>>(psi, count, dim, te, scale, packed);
  return cudaGetLastError();
}

}  // namespace ctqw
