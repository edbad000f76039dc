// bz_generic.cu -- general-purpose kernels: every d, every power-of-two block,
// every kind, both transform families, any mask.  They restate the reference
// pipeline operation by operation (dense per-axis matrix contractions in axis
// order, exact IEEE binning) and serve
//   * the API building blocks (block/unblock/transform/bin/prune/unflatten/...),
//   * compress/decompress for layouts the fused kernels (bz_fast.cu) do not cover,
//   * the exact fix-up of "special" blocks found by the fused compress kernel.
#include <cstdarg>
#include <cstdio>

#include "bz_common.cuh"
#include "bz_kernels.cuh"

namespace bz {

// --------------------------------------------------------------- rounding --
__global__ void k_round_to_kind(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                                int32_t* mismatch) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = load_kind_rt(in, i, in_kind);
    double r = round_to_kind_rt(v, out_kind);
    if (out) store_kind_rt(out, i, r, out_kind);
    if (mismatch && !(r == v || (isnan(r) && isnan(v)))) atomicExch(mismatch, 1);
  }
}

// gradient_array (arrays.py:193-208): sum of zero-based indices / sum(s-1)
struct ShapeArg { int ndim; int64_t shape[BZ_MAX_DIMS]; };
__global__ void k_gradient(ShapeArg s, int kind, void* out, int64_t n, double denom) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i;
    int64_t coord[BZ_MAX_DIMS];
    for (int a = s.ndim - 1; a >= 0; --a) { coord[a] = rem % s.shape[a]; rem /= s.shape[a]; }
    double total = 0.0;  // same accumulation order as the reference: axis 0 first
    for (int a = 0; a < s.ndim; ++a) total = total + (double)coord[a];
    store_kind_rt(out, i, round_to_kind_rt(__ddiv_rn(total, denom), kind), kind);
  }
}

// counter-based synthetic data: splitmix64 of (seed, global index)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit_open(uint64_t h) {  // (0, 1)
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__global__ void k_fill_random(void* out, int kind, int64_t n, int64_t offset, uint64_t seed,
                              int dist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t g = (uint64_t)(offset + i);
    uint64_t h1 = mix64(seed * 0x632be59bd9b4e019ull ^ (2 * g));
    double v;
    if (dist == 1) {
      v = (double)(h1 >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
    } else {
      uint64_t h2 = mix64(seed * 0x632be59bd9b4e019ull ^ (2 * g + 1));
      double u1 = unit_open(h1), u2 = unit_open(h2);
      v = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    store_kind_rt(out, i, round_to_kind_rt(v, kind), kind);
  }
}

// widen / narrow stored indices (mixed index kinds in reductions, ops.py:100-116)
__global__ void k_convert_indices(const void* in, int in_kind, void* out, int out_kind, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_index_rt(out, i, load_index_rt(in, i, in_kind), out_kind);
}

int launch_convert_indices(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                           cudaStream_t s) {
  if (n <= 0) return BZ_OK;
  k_convert_indices<<<grid_for(n, 256), 256, 0, s>>>(in, in_kind, out, out_kind, n);
  return check_launch("convert_indices");
}

// ------------------------------------------------------- block / unblock --
__global__ void k_block(Geo g, const void* x, int x_kind, double* blocks, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / g.bsize;
    int pos = (int)(i - b * g.bsize);
    int64_t off = element_offset(g, b, pos);
    blocks[i] = off >= 0 ? load_kind_rt(x, off, x_kind) : 0.0;
  }
}

__device__ __forceinline__ void dense_to_block(const Geo& g, int64_t i, int64_t& b, int& pos) {
  int64_t rem = i;
  b = 0;
  int64_t bmul = 1;
  pos = 0;
  int pmul = 1;
  for (int a = g.ndim - 1; a >= 0; --a) {
    int64_t c = rem % g.shape[a];
    rem /= g.shape[a];
    b += (c / g.block[a]) * bmul;
    bmul *= g.grid[a];
    pos += (int)(c % g.block[a]) * pmul;
    pmul *= g.block[a];
  }
}

__global__ void k_unblock(Geo g, const double* blocks, void* out, int out_kind, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b;
    int pos;
    dense_to_block(g, i, b, pos);
    store_kind_rt(out, i, round_to_kind_rt(blocks[b * g.bsize + pos], out_kind), out_kind);
  }
}

// ---------------------------------------------------- per-axis transform --
// out[b][.. k_a ..] = sum_j in[b][.. j ..] * H_a[j][k_a]      (forward)
// out[b][.. n_a ..] = sum_j in[b][.. j ..] * H_a[n_a][j]      (inverse)
__global__ void k_transform_axis(Geo g, const double* in, double* out, int axis, int inverse,
                                 int64_t total) {
  int inner = 1;
  for (int a = axis + 1; a < g.ndim; ++a) inner *= g.block[a];
  const int E = g.block[axis];
  const double* H = g.matrices + g.mat_off[axis];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / g.bsize;
    int pos = (int)(i - b * g.bsize);
    int k = (pos / inner) % E;
    int base = pos - k * inner;
    const double* src = in + b * g.bsize + base;
    double acc = 0.0;
    for (int j = 0; j < E; ++j) {
      double h = inverse ? H[k * E + j] : H[j * E + k];
      acc = __fma_rn(src[j * inner], h, acc);
    }
    out[i] = acc;
  }
}

// ------------------------------------------------------------ binning ----
__device__ __forceinline__ double warp_nanmax(double m) {
  for (int o = 16; o > 0; o >>= 1) {
    double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (isnan(t) || isnan(m)) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, t);
  }
  return m;
}

// bin_coefficients on blocked f64 coefficients: warp per block (codec.py:253-278)
__global__ void k_bin(Geo g, const double* coeffs, void* maxima, void* full) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double r = radius_f64(g.index_kind), bound = clamp_bound_f64(g.index_kind);
  for (int64_t b = warp; b < g.nblocks; b += nwarps) {
    const double* c = coeffs + b * g.bsize;
    double m = 0.0;
    for (int p = lane; p < g.bsize; p += 32) m = nanmax_abs(m, c[p]);
    m = warp_nanmax(m);
    double n = round_to_kind_rt(m, g.float_kind);
    if (lane == 0) store_kind_rt(maxima, b, n, g.float_kind);
    for (int p = lane; p < g.bsize; p += 32)
      store_index_rt(full, b * g.bsize + p, bin_exact(c[p], n, r, bound), g.index_kind);
  }
}

__global__ void k_prune(Geo g, const void* full, void* flat, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / g.kept;
    int j = (int)(i - b * g.kept);
    store_index_rt(flat, i, load_index_rt(full, b * g.bsize + g.kept_pos[j], g.index_kind),
                   g.index_kind);
  }
}

__global__ void k_unflatten(Geo g, const void* flat, void* full, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / g.bsize;
    int p = (int)(i - b * g.bsize);
    int j = g.rank[p];
    int64_t v = j >= 0 ? load_index_rt(flat, b * g.kept + j, g.index_kind) : 0;
    store_index_rt(full, i, v, g.index_kind);
  }
}

// (F * N) / r, multiply before divide (codec.py:337-350)
__global__ void k_specified(Geo g, const void* maxima, const void* flat, double* out,
                            int64_t total) {
  const double r = radius_f64(g.index_kind);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / g.bsize;
    int p = (int)(i - b * g.bsize);
    int j = g.rank[p];
    double f = j >= 0 ? (double)load_index_rt(flat, b * g.kept + j, g.index_kind) : 0.0;
    double n = load_kind_rt(maxima, b, g.float_kind);
    out[i] = __ddiv_rn(__dmul_rn(f, n), r);
  }
}

// ---------------------------------------- exact per-block compress (warp) --
// Restates codec.py:321-334 for one block per warp, scratch in smem or global.
// `list` (optional) restricts the work to listed block ids (fix-up of blocks
// the fused kernel flagged); list[-1] style count lives in *count.
__device__ void exact_compress_block(const Geo& g, const void* x, int x_kind, int64_t b,
                                     double* A, double* B, void* maxima, void* indices) {
  const int lane = threadIdx.x & 31;
  for (int p = lane; p < g.bsize; p += 32) {
    int64_t off = element_offset(g, b, p);
    A[p] = off >= 0 ? round_to_kind_rt(load_kind_rt(x, off, x_kind), g.float_kind) : 0.0;
  }
  __syncwarp();
  int inner = g.bsize;
  for (int a = 0; a < g.ndim; ++a) {
    const int E = g.block[a];
    inner /= E;
    const double* H = g.matrices + g.mat_off[a];
    for (int p = lane; p < g.bsize; p += 32) {
      int k = (p / inner) % E;
      const double* src = A + (p - k * inner);
      double acc = 0.0;
      for (int j = 0; j < E; ++j) acc = __fma_rn(src[j * inner], H[j * E + k], acc);
      B[p] = acc;
    }
    __syncwarp();
    double* t = A; A = B; B = t;
  }
  double m = 0.0;
  for (int p = lane; p < g.bsize; p += 32) m = nanmax_abs(m, A[p]);
  m = warp_nanmax(m);
  const double n = round_to_kind_rt(m, g.float_kind);
  if (lane == 0) store_kind_rt(maxima, b, n, g.float_kind);
  const double r = radius_f64(g.index_kind), bound = clamp_bound_f64(g.index_kind);
  for (int j = lane; j < g.kept; j += 32)
    store_index_rt(indices, b * g.kept + j, bin_exact(A[g.kept_pos[j]], n, r, bound),
                   g.index_kind);
  __syncwarp();
}

__global__ void k_exact_compress(Geo g, const void* x, int x_kind, void* maxima, void* indices,
                                 double* gscratch, const int32_t* list, const int32_t* count,
                                 void* dc) {
  extern __shared__ double smem[];
  const int wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double* A = gscratch ? gscratch + warp * 2 * (int64_t)g.bsize : smem + wib * 2 * g.bsize;
  double* B = A + g.bsize;
  const int64_t total = list ? (int64_t)*count : g.nblocks;
  for (int64_t w = warp; w < total; w += nwarps) {
    int64_t b = list ? (int64_t)list[w] : w;
    exact_compress_block(g, x, x_kind, b, A, B, maxima, indices);
    // DC plane: lane 0 stored flat position 0 (the first coefficient)
    if (dc && (threadIdx.x & 31) == 0)
      store_index_rt(dc, b, load_index_rt(indices, b * g.kept, g.index_kind), g.index_kind);
  }
}

// DC plane from the indices: dc[b] = F[b][0] (strided gather; the producers
// that know F0 in registers write the plane themselves)
template <typename IT>
__global__ void k_extract_dc(int64_t nblocks, int kept, const IT* __restrict__ indices,
                             IT* __restrict__ dc) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x)
    dc[b] = __ldcs(indices + b * (int64_t)kept);
}

int launch_extract_dc(const Geo& g, const void* indices, void* dc, cudaStream_t s) {
  if (!dc || g.nblocks == 0) return BZ_OK;
  if (!g.keeps_first) { set_error("extract_dc: mask drops the first coefficient"); return BZ_E_INVALID; }
  const int grid = grid_for(g.nblocks, 256, 8);
  switch (g.index_kind) {
    case BZ_I8: k_extract_dc<<<grid, 256, 0, s>>>(g.nblocks, g.kept, (const int8_t*)indices, (int8_t*)dc); break;
    case BZ_I16: k_extract_dc<<<grid, 256, 0, s>>>(g.nblocks, g.kept, (const int16_t*)indices, (int16_t*)dc); break;
    case BZ_I32: k_extract_dc<<<grid, 256, 0, s>>>(g.nblocks, g.kept, (const int32_t*)indices, (int32_t*)dc); break;
    default: k_extract_dc<<<grid, 256, 0, s>>>(g.nblocks, g.kept, (const int64_t*)indices, (int64_t*)dc); break;
  }
  return check_launch("extract_dc");
}

// ------------------------------------- exact per-block decompress (warp) --
// codec.py:364-384: inverse transform of the raw indices, then *N, then /r.
__global__ void k_exact_decompress(Geo g, const void* maxima, const void* indices, void* out,
                                   int out_kind, double* gscratch) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double* A0 = gscratch ? gscratch + warp * 2 * (int64_t)g.bsize : smem + wib * 2 * g.bsize;
  const double r = radius_f64(g.index_kind);
  for (int64_t b = warp; b < g.nblocks; b += nwarps) {
    double* A = A0;
    double* B = A0 + g.bsize;
    for (int p = lane; p < g.bsize; p += 32) {
      int j = g.rank[p];
      A[p] = j >= 0 ? (double)load_index_rt(indices, b * g.kept + j, g.index_kind) : 0.0;
    }
    __syncwarp();
    int inner = g.bsize;
    for (int a = 0; a < g.ndim; ++a) {
      const int E = g.block[a];
      inner /= E;
      const double* H = g.matrices + g.mat_off[a];
      for (int p = lane; p < g.bsize; p += 32) {
        int k = (p / inner) % E;
        const double* src = A + (p - k * inner);
        double acc = 0.0;
        for (int j = 0; j < E; ++j) acc = __fma_rn(src[j * inner], H[k * E + j], acc);
        B[p] = acc;
      }
      __syncwarp();
      double* t = A; A = B; B = t;
    }
    const double n = load_kind_rt(maxima, b, g.float_kind);
    for (int p = lane; p < g.bsize; p += 32) {
      int64_t off = element_offset(g, b, p);
      if (off >= 0) {
        double v = __ddiv_rn(__dmul_rn(A[p], n), r);
        store_kind_rt(out, off, round_to_kind_rt(v, out_kind), out_kind);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------- launchers --
static constexpr int kGenericWarps = 4;

size_t exact_scratch_bytes(const Geo& g, int blocks_in_grid, bool& use_smem) {
  size_t per_warp = 2 * (size_t)g.bsize * sizeof(double);
  use_smem = per_warp * kGenericWarps <= 160 * 1024;
  return use_smem ? 0 : per_warp * kGenericWarps * blocks_in_grid;
}

int launch_exact_compress(const Geo& g, const void* x, int x_kind, void* maxima, void* indices,
                          const int32_t* list, const int32_t* count, int64_t max_blocks,
                          void* ws, size_t ws_bytes, cudaStream_t s, void* dc) {
  if (dc && !g.keeps_first) dc = nullptr;
  bool use_smem;
  int grid = grid_for(max_blocks, kGenericWarps, 16);
  size_t need = exact_scratch_bytes(g, grid, use_smem);
  if (!use_smem) {
    // shrink the grid to the workspace we have
    size_t per_cta = 2 * (size_t)g.bsize * sizeof(double) * kGenericWarps;
    if (ws_bytes < per_cta) { set_error("compress: workspace too small (%zu < %zu)", ws_bytes, per_cta); return BZ_E_WORKSPACE; }
    grid = (int)std::min<size_t>((size_t)grid, ws_bytes / per_cta);
    need = per_cta * grid;
  }
  size_t smem = use_smem ? 2 * (size_t)g.bsize * sizeof(double) * kGenericWarps : 0;
  if (smem > 48 * 1024) occupancy((const void*)k_exact_compress, 32 * kGenericWarps, smem);
  k_exact_compress<<<grid, 32 * kGenericWarps, smem, s>>>(g, x, x_kind, maxima, indices,
                                                           use_smem ? nullptr : (double*)ws, list,
                                                           count, dc);
  (void)need;
  return check_launch("exact_compress");
}

size_t exact_compress_workspace(const Geo& g, int64_t max_blocks) {
  bool use_smem;
  int grid = grid_for(max_blocks, kGenericWarps, 16);
  return exact_scratch_bytes(g, grid, use_smem);
}

int launch_exact_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                            int out_kind, void* ws, size_t ws_bytes, cudaStream_t s) {
  bool use_smem;
  int grid = grid_for(g.nblocks, kGenericWarps, 16);
  exact_scratch_bytes(g, grid, use_smem);
  if (!use_smem) {
    size_t per_cta = 2 * (size_t)g.bsize * sizeof(double) * kGenericWarps;
    if (ws_bytes < per_cta) { set_error("decompress: workspace too small"); return BZ_E_WORKSPACE; }
    grid = (int)std::min<size_t>((size_t)grid, ws_bytes / per_cta);
  }
  size_t smem = use_smem ? 2 * (size_t)g.bsize * sizeof(double) * kGenericWarps : 0;
  if (smem > 48 * 1024) occupancy((const void*)k_exact_decompress, 32 * kGenericWarps, smem);
  k_exact_decompress<<<grid, 32 * kGenericWarps, smem, s>>>(
      g, maxima, indices, out, out_kind, use_smem ? nullptr : (double*)ws);
  return check_launch("exact_decompress");
}

int launch_round_to_kind(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                         int32_t* mismatch, cudaStream_t s) {
  if (n <= 0) return BZ_OK;
  k_round_to_kind<<<grid_for(n, 256), 256, 0, s>>>(in, in_kind, out, out_kind, n, mismatch);
  return check_launch("round_to_kind");
}

int launch_gradient(int ndim, const int64_t* shape, int kind, void* out, cudaStream_t s) {
  ShapeArg a{};
  a.ndim = ndim;
  int64_t n = 1, denom = 0;
  for (int i = 0; i < ndim; ++i) { a.shape[i] = shape[i]; n *= shape[i]; denom += shape[i] - 1; }
  if (denom == 0) { set_error("gradient: degenerate shape"); return BZ_E_INVALID; }
  k_gradient<<<grid_for(n, 256), 256, 0, s>>>(a, kind, out, n, (double)denom);
  return check_launch("gradient");
}

int launch_fill_random(void* out, int kind, int64_t n, int64_t offset, uint64_t seed, int dist,
                       cudaStream_t s) {
  if (n <= 0) return BZ_OK;
  k_fill_random<<<grid_for(n, 256, 16), 256, 0, s>>>(out, kind, n, offset, seed, dist);
  return check_launch("fill_random");
}

int launch_block(const Geo& g, const void* x, int x_kind, double* blocks, cudaStream_t s) {
  int64_t total = g.nblocks * g.bsize;
  if (total == 0) return BZ_OK;
  k_block<<<grid_for(total, 256), 256, 0, s>>>(g, x, x_kind, blocks, total);
  return check_launch("block");
}

int launch_unblock(const Geo& g, const double* blocks, void* out, int out_kind, cudaStream_t s) {
  int64_t n = 1;
  for (int a = 0; a < g.ndim; ++a) n *= g.shape[a];
  k_unblock<<<grid_for(n, 256), 256, 0, s>>>(g, blocks, out, out_kind, n);
  return check_launch("unblock");
}

int launch_transform(const Geo& g, const double* in, double* out, int inverse, void* ws,
                     size_t ws_bytes, cudaStream_t s) {
  int64_t total = g.nblocks * g.bsize;
  if (total == 0) return BZ_OK;
  if (g.ndim > 1 && ws_bytes < (size_t)total * sizeof(double)) {
    set_error("transform: workspace too small");
    return BZ_E_WORKSPACE;
  }
  const double* src = in;
  double* tmp = (double*)ws;
  for (int a = 0; a < g.ndim; ++a) {
    double* dst = ((g.ndim - 1 - a) % 2 == 0) ? out : tmp;
    k_transform_axis<<<grid_for(total, 256), 256, 0, s>>>(g, src, dst, a, inverse, total);
    src = dst;
  }
  return check_launch("transform");
}

int launch_bin(const Geo& g, const double* coeffs, void* maxima, void* full, cudaStream_t s) {
  if (g.nblocks == 0) return BZ_OK;
  k_bin<<<grid_for(g.nblocks * 32, 256), 256, 0, s>>>(g, coeffs, maxima, full);
  return check_launch("bin");
}

int launch_prune(const Geo& g, const void* full, void* flat, cudaStream_t s) {
  int64_t total = g.nblocks * g.kept;
  if (total == 0) return BZ_OK;
  k_prune<<<grid_for(total, 256), 256, 0, s>>>(g, full, flat, total);
  return check_launch("prune");
}

int launch_unflatten(const Geo& g, const void* flat, void* full, cudaStream_t s) {
  int64_t total = g.nblocks * g.bsize;
  if (total == 0) return BZ_OK;
  k_unflatten<<<grid_for(total, 256), 256, 0, s>>>(g, flat, full, total);
  return check_launch("unflatten");
}

int launch_specified(const Geo& g, const void* maxima, const void* flat, double* out,
                     cudaStream_t s) {
  int64_t total = g.nblocks * g.bsize;
  if (total == 0) return BZ_OK;
  k_specified<<<grid_for(total, 256), 256, 0, s>>>(g, maxima, flat, out, total);
  return check_launch("specified");
}

}  // namespace bz
