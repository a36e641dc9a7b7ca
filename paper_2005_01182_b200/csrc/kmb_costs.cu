// GPU cost construction: the reference's
// build_instance (datasets.cpp:184-214) — C_ij = llround(scale * ||a_i - b_j||)
// with the distance accumulated in double over the dimensions in order — plus
// the squared-distance mode BASELINE configs 2 and 4 use.  Every operation is an
// explicitly rounded IEEE double op (__dsub_rn / __dmul_rn / __dadd_rn, no FMA
// contraction; sqrt is correctly rounded), so the int32 costs are bit-identical
// to the reference's and to the host generators (csrc/kmb_gen.c, built with
// -ffp-contract=off) on the same points.
//
// Layout: a is n x dim, b is m x dim (row-major); a CTA computes a 32 x 32 tile
// of C from point tiles staged in shared memory (dim chunked by 32).  Points are
// double (configs 2 and 4) or float promoted to double (config 3's 300-D fp32
// vectors, batched instances).
#include <cuda_runtime.h>

#include <cstdint>

#include "kmb_internal.h"

namespace kmb {

template <typename P>
__global__ void __launch_bounds__(256) k_costs(const P* __restrict__ A, const P* __restrict__ B,
                                               int32_t n, int32_t m, int32_t dim, double scale,
                                               int32_t squared, int32_t* __restrict__ out,
                                               int64_t a_stride, int64_t b_stride,
                                               int64_t out_stride, int32_t* __restrict__ bad) {
  constexpr int TI = 32, TJ = 32, TK = 32;
  __shared__ double sa[TI][TK + 1];
  __shared__ double sb[TJ][TK + 1];
  const int inst = blockIdx.z;
  const P* a = A + inst * a_stride;
  const P* b = B + inst * b_stride;
  const int i0 = blockIdx.y * TI, j0 = blockIdx.x * TJ;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  double acc[TI / 8];
#pragma unroll
  for (int r = 0; r < TI / 8; ++r) acc[r] = 0.0;
  for (int k0 = 0; k0 < dim; k0 += TK) {
    for (int t = threadIdx.x; t < TI * TK; t += blockDim.x) {
      const int r = t / TK, k = t % TK;
      const int gi = i0 + r, gj = j0 + r, gk = k0 + k;
      sa[r][k] = (gi < n && gk < dim) ? static_cast<double>(a[static_cast<int64_t>(gi) * dim + gk]) : 0.0;
      sb[r][k] = (gj < m && gk < dim) ? static_cast<double>(b[static_cast<int64_t>(gj) * dim + gk]) : 0.0;
    }
    __syncthreads();
    const int kk = min(TK, dim - k0);
    for (int k = 0; k < kk; ++k) {  // dimension order preserved (datasets.cpp:16-22)
      const double bj = sb[tx][k];
#pragma unroll
      for (int r = 0; r < TI / 8; ++r) {
        const double d = __dsub_rn(sa[ty + 8 * r][k], bj);
        acc[r] = __dadd_rn(acc[r], __dmul_rn(d, d));
      }
    }
    __syncthreads();
  }
  const int j = j0 + tx;
  if (j >= m) return;
#pragma unroll
  for (int r = 0; r < TI / 8; ++r) {
    const int i = i0 + ty + 8 * r;
    if (i >= n) continue;
    const double dist = squared ? acc[r] : sqrt(acc[r]);
    const double x = __dmul_rn(scale, dist);
    if (!(x < 2147483647.0)) {  // llround would overflow int32
      atomicMax(bad, 1);
      continue;
    }
    out[inst * out_stride + static_cast<int64_t>(i) * m + j] = static_cast<int32_t>(llround(x));
  }
}

template <typename P>
cudaError_t launch_costs(const P* a, const P* b, int32_t batch, int32_t n, int32_t m, int32_t dim,
                         double scale, int32_t squared, int32_t* out, int32_t* bad,
                         cudaStream_t st) {
  dim3 grid((m + 31) / 32, (n + 31) / 32, batch);
  k_costs<P><<<grid, 256, 0, st>>>(a, b, n, m, dim, scale, squared, out,
                                    static_cast<int64_t>(n) * dim, static_cast<int64_t>(m) * dim,
                                    static_cast<int64_t>(n) * m, bad);
  return cudaGetLastError();
}

template cudaError_t launch_costs<double>(const double*, const double*, int32_t, int32_t, int32_t,
                                          int32_t, double, int32_t, int32_t*, int32_t*, cudaStream_t);
template cudaError_t launch_costs<float>(const float*, const float*, int32_t, int32_t, int32_t,
                                         int32_t, double, int32_t, int32_t*, int32_t*, cudaStream_t);

}  // namespace kmb
