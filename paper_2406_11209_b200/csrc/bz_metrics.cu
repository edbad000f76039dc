// bz_metrics.cu -- per-block error predictors and round-trip errors on the
// device (metrics.py:108-148).  One warp per block:
//
//   bin_bound[b]   = N / (2r + 1)                       (IEEE division, exact)
//   loose_linf[b]  = max|C| * prod(i)                    (exact: power of two)
//   l2_coeff[b]    = sqrt(sum (Chat - C)^2), Chat = (F N)/r at kept
//                    positions, 0 at pruned ones (codec.py:337-361)
//
// and, for two blocked f64 arrays X, Y: per-block sqrt(sum (X - Y)^2) plus
// the global max |X - Y| and sum (X - Y)^2 (deterministic: per-block values
// reduced in block order by the host-visible second stage).
#include "bz_common.cuh"
#include "bz_kernels.cuh"

namespace bz {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax_abs(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_error_bounds(Geo g, const void* __restrict__ maxima,
                               const void* __restrict__ indices,
                               const double* __restrict__ coeffs, double* __restrict__ bin_bound,
                               double* __restrict__ loose_linf, double* __restrict__ l2_coeff) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double r = radius_f64(g.index_kind);
  for (int64_t b = warp; b < g.nblocks; b += nwarps) {
    const double n = load_kind_rt(maxima, b, g.float_kind);
    double err = 0.0, mx = 0.0;
    for (int p = lane; p < g.bsize; p += 32) {
      const double c = coeffs[b * g.bsize + p];
      const int j = g.rank[p];
      const double f = j >= 0 ? (double)load_index_rt(indices, b * g.kept + j, g.index_kind) : 0.0;
      const double chat = j >= 0 ? __ddiv_rn(__dmul_rn(f, n), r) : 0.0;
      const double dlt = chat - c;
      err = __fma_rn(dlt, dlt, err);
      mx = nanmax_abs(mx, c);
    }
    err = warp_sum(err);
    mx = warp_nanmax(mx);
    if (lane == 0) {
      bin_bound[b] = __ddiv_rn(n, 2.0 * r + 1.0);
      loose_linf[b] = mx * (double)g.bsize;
      l2_coeff[b] = sqrt(err);
    }
  }
}

__global__ void k_block_diff(int64_t nblocks, int bsize, const double* __restrict__ x,
                             const double* __restrict__ y, double* __restrict__ l2,
                             double* __restrict__ maxabs) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nblocks; b += nwarps) {
    double s = 0.0, m = 0.0;
    for (int p = lane; p < bsize; p += 32) {
      const double d = x[b * bsize + p] - y[b * bsize + p];
      s = __fma_rn(d, d, s);
      m = nanmax_abs(m, d);
    }
    s = warp_sum(s);
    m = warp_nanmax(m);
    if (lane == 0) {
      l2[b] = s;  // squared; the host takes roots after the global sum
      maxabs[b] = m;
    }
  }
}

int launch_error_bounds(const Geo& g, const void* maxima, const void* indices,
                        const double* coeffs, double* bin_bound, double* loose_linf,
                        double* l2_coeff, cudaStream_t s) {
  if (g.nblocks == 0) return BZ_OK;
  k_error_bounds<<<grid_for(g.nblocks * 32, 256, 8), 256, 0, s>>>(g, maxima, indices, coeffs,
                                                                  bin_bound, loose_linf, l2_coeff);
  return check_launch("error_bounds");
}

int launch_block_diff(int64_t nblocks, int bsize, const double* x, const double* y, double* l2sq,
                      double* maxabs, cudaStream_t s) {
  if (nblocks == 0) return BZ_OK;
  k_block_diff<<<grid_for(nblocks * 32, 256, 8), 256, 0, s>>>(nblocks, bsize, x, y, l2sq, maxabs);
  return check_launch("block_diff");
}

}  // namespace bz
