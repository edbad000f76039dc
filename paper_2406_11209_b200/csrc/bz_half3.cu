// bz_half3.cu -- fused compress / decompress for 8x8x8 blocks with half slices.
//
// 16 threads own a block; each holds 32 values (an 8 x 4 half slice), so the
// kernel stays far below the register ceiling (the full-slice kernel needs
// 64 doubles per thread and runs at 2 warps per scheduler).  Reference axis
// order (axis 0 first), reference FMA chains (bz_fast.cuh):
//   A  thread (y, xh): rows z = 0..7 of x in half xh, straight from HBM (a
//      warp covers 16 blocks x 32 bytes = 512 contiguous bytes per row)
//      -> axis 0 over z -> canonical smem tile
//   B  thread (kz, xh): 8 y x 4 x  -> axis 1 over y -> in place
//   C  thread (kz, kyh): 4 ky x 8 x -> axis 2 over x -> 32 coefficients at
//      positions kz*64 + kyh*32 .. +32 (contiguous in the compressed layout)
// Two shared-memory exchanges (16-byte accesses, XOR-swizzled by block slot:
// conflict-free).  Decompress runs the mirror image.
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

namespace h3 {
constexpr int E = 8, BS = 512, TB = 16, NT = 256, BPC = NT / TB;  // 16 blocks per tile
constexpr int BSP = BS;                                           // block stride (doubles)

// canonical position -> swizzled smem index within the block region
__device__ __forceinline__ int sw(int pos, int key) { return (((pos >> 1) ^ key) << 1) | (pos & 1); }

__device__ __forceinline__ void st2(double* blk, int pos, int key, double a, double b) {
  *reinterpret_cast<double2*>(blk + sw(pos, key)) = make_double2(a, b);
}
__device__ __forceinline__ double2 ld2(const double* blk, int pos, int key) {
  return *reinterpret_cast<const double2*>(blk + sw(pos, key));
}
}  // namespace h3

// 8-point reference FMA chain on a strided register line
template <int S, bool INV>
__device__ __forceinline__ void line8(double* v, const double (&H)[64]) {
  double in[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) in[i] = v[i * S];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < 8; ++n) acc = __fma_rn(in[n], INV ? H[k * 8 + n] : H[n * 8 + k], acc);
    v[k * S] = acc;
  }
}

template <typename TIn, int FK, typename IT>
__global__ void __launch_bounds__(256, 2)
k_half3_compress(const FastParams p, const TIn* __restrict__ x, void* __restrict__ maxima,
                 IT* __restrict__ indices) {
  using namespace h3;
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);                                   // BPC*BSP
  unsigned long long* red = reinterpret_cast<unsigned long long*>(xs + BPC * BSP);    // NT
  unsigned char* stage = reinterpret_cast<unsigned char*>(red + NT);                  // pruned out
  const size_t stage_sz = f.full_mask ? 0 : ((size_t)BPC * f.kept * sizeof(IT) + 16 + 15) / 16 * 16;
  int16_t* rks = reinterpret_cast<int16_t*>(stage + stage_sz);
  if (!f.full_mask) {
    for (int i = threadIdx.x; i < BS; i += NT) rks[i] = (int16_t)f.rank[i];
    __syncthreads();
  }

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;       // 0..15
  const int hi = o >> 1, half = o & 1;
  const int key = lb & 7;
  double* blk = xs + lb * BSP;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const int64_t s0 = f.stride[0], s1 = f.stride[1];
  constexpr bool VEC = (4 * sizeof(TIn)) % 16 == 0;

  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)BPC, f.nblocks - b0);

    // ---- A: rows z of (y = hi, x in half), axis 0
    double v[32];  // [8][4] (rows z, cols x)
    {
      int64_t gc[4] = {0, 0, 0, 0};
      if (valid) block_coords<3>(f, b, gc);
      const int64_t z0 = gc[0] * E, y = gc[1] * E + hi, x0 = gc[2] * E + half * 4;
      const TIn* src = x + z0 * s0 + y * s1 + x0;
      const bool full = valid && z0 + E <= f.shape[0] && y < f.shape[1] && x0 + 4 <= f.shape[2];
      if (VEC && full && f.vec_dense) {
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          if constexpr (VEC) {
            const uint4 w = __ldcs(reinterpret_cast<const uint4*>(src + z * s0));
            if constexpr (sizeof(TIn) == 4) {
              v[z * 4 + 0] = (double)__uint_as_float(w.x);
              v[z * 4 + 1] = (double)__uint_as_float(w.y);
              v[z * 4 + 2] = (double)__uint_as_float(w.z);
              v[z * 4 + 3] = (double)__uint_as_float(w.w);
            }
          }
        }
      } else if (sizeof(TIn) == 8 && full && f.vec_dense) {
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          const double2 w0 = __ldcs(reinterpret_cast<const double2*>(src + z * s0));
          const double2 w1 = __ldcs(reinterpret_cast<const double2*>(src + z * s0) + 1);
          v[z * 4 + 0] = w0.x; v[z * 4 + 1] = w0.y; v[z * 4 + 2] = w1.x; v[z * 4 + 3] = w1.y;
        }
      } else {
        const bool okyx = valid && y < f.shape[1];
#pragma unroll
        for (int z = 0; z < 8; ++z)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[z * 4 + j] = (okyx && z0 + z < f.shape[0] && x0 + j < f.shape[2])
                               ? widen(src[z * s0 + j]) : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) line8<4, false>(v + j, p.H);  // axis 0 over z
#pragma unroll
    for (int z = 0; z < 8; ++z)
#pragma unroll
      for (int j = 0; j < 4; j += 2)
        st2(blk, z * 64 + hi * 8 + half * 4 + j, key, v[z * 4 + j], v[z * 4 + j + 1]);
    __syncthreads();

    // ---- B: (kz = hi, x in half), 8 y x 4 x, axis 1 in place
#pragma unroll
    for (int yy = 0; yy < 8; ++yy)
#pragma unroll
      for (int j = 0; j < 4; j += 2) {
        const double2 w = ld2(blk, hi * 64 + yy * 8 + half * 4 + j, key);
        v[yy * 4 + j] = w.x;
        v[yy * 4 + j + 1] = w.y;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) line8<4, false>(v + j, p.H);  // axis 1 over y
#pragma unroll
    for (int yy = 0; yy < 8; ++yy)
#pragma unroll
      for (int j = 0; j < 4; j += 2)
        st2(blk, hi * 64 + yy * 8 + half * 4 + j, key, v[yy * 4 + j], v[yy * 4 + j + 1]);
    __syncthreads();

    // ---- C: (kz = hi, ky in half), 4 ky x 8 x, axis 2
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int xx = 0; xx < 8; xx += 2) {
        const double2 w = ld2(blk, hi * 64 + (half * 4 + i) * 8 + xx, key);
        v[i * 8 + xx] = w.x;
        v[i * 8 + xx + 1] = w.y;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) line8<1, false>(v + i * 8, p.H);  // axis 2 over x
    // v[i*8 + kx] = C[kz][half*4+i][kx] at canonical position hi*64 + half*32 + i*8 + kx

    // ---- block maximum over the 16 threads of the block
    unsigned long long mkey = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const unsigned long long k2 = abs_key(v[q]);
      mkey = k2 > mkey ? k2 : mkey;
    }
    red[lb * TB + o] = mkey;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const unsigned long long k2 = red[lb * TB + j];
      mkey = k2 > mkey ? k2 : mkey;
    }
    const double mx = __longlong_as_double((long long)mkey);
    const double n = round_to_kind<FK>(mx);
    constexpr bool CLAMP = !(FK == BZ_F32 || FK == BZ_F64);
    const BinCtx bc = bin_ctx<CLAMP>(n, rr, mx);
    if (valid && o == 0) store_kind<FK>(maxima, b, n);
        const int ir = (int)rr;
    auto bin_q = [&](double c) -> int {
      if constexpr (sizeof(IT) <= 2) {
        unsigned nr = 0;
        const int qv = fast_index32<IT, CLAMP>(c, bc.R, ir, nr);
        return (nr | !bc.fast) ? (int)bin_exact_ctx(c, bc, rr, rr) : qv;
      } else {
        bool nr = false;
        const int qv = bc.fast ? fast_index<IT>(c, bc.R, rr, nr) : 0;
        return (nr || !bc.fast) ? (int)bin_exact_ctx(c, bc, rr, rr) : qv;
      }
    };

    // ---- bin + store (32 contiguous positions)
    const int pos0 = hi * 64 + half * 32;
    if (f.full_mask) {
      if (valid) {
        IT* dst = indices + b * (int64_t)BS + pos0;
        constexpr int PER = 16 / sizeof(IT);
#pragma unroll
        for (int cch = 0; cch < 32 / PER; ++cch) {
          int q[PER];
          if constexpr (sizeof(IT) <= 2) {
            unsigned nacc = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) q[e] = fast_index32<IT, CLAMP>(v[cch * PER + e], bc.R, ir, nacc);
            if (nacc | !bc.fast) {
#pragma unroll
              for (int e = 0; e < PER; ++e) q[e] = bin_q(v[cch * PER + e]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < PER; ++e) q[e] = bin_q(v[cch * PER + e]);
          }
          __stcs(reinterpret_cast<uint4*>(dst) + cch, pack16<IT>(q));
        }
      }
      __syncthreads();  // red / xs reused by the next tile
    } else {
      const int64_t dst_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + dst_byte0) & 15);
      IT* st = reinterpret_cast<IT*>(stage + mis);
      if (valid) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int rk = rks[pos0 + q];
          if (rk >= 0) st[lb * f.kept + rk] = (IT)bin_q(v[q]);
        }
      }
      __syncthreads();
      smem_to_tile(reinterpret_cast<unsigned char*>(indices) + dst_byte0, stage,
                   (int64_t)nvalid * f.kept * sizeof(IT), mis, t, NT);
      __syncthreads();
    }
  }
}

template <typename IT, int FK, typename TOut>
__global__ void __launch_bounds__(256, 2)
k_half3_decompress(const FastParams p, const void* __restrict__ maxima,
                   const IT* __restrict__ indices, TOut* __restrict__ out) {
  using namespace h3;
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);
  unsigned char* stage = reinterpret_cast<unsigned char*>(xs + BPC * BSP);
  const size_t stage_sz = ((size_t)BPC * f.kept * sizeof(IT) + 32 + 15) / 16 * 16;
  int16_t* rks = reinterpret_cast<int16_t*>(stage + stage_sz);
  if (!f.full_mask) {
    for (int i = threadIdx.x; i < BS; i += NT) rks[i] = (int16_t)f.rank[i];
    __syncthreads();
  }

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;
  const int hi = o >> 1, half = o & 1;
  const int key = lb & 7;
  double* blk = xs + lb * BSP;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const double rinv = 1.0 / rr;
  const double nsafe = 1.7976931348623157e308 / (rr * BS * 4.0);
  const int64_t s0 = f.stride[0], s1 = f.stride[1];

  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)BPC, f.nblocks - b0);

    const int64_t src_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
    const int mis = (int)(((uintptr_t)indices + src_byte0) & 15);
    tile_to_smem(stage, reinterpret_cast<const unsigned char*>(indices) + src_byte0,
                 (int64_t)nvalid * f.kept * sizeof(IT), mis, t, NT);
    __syncthreads();
    const IT* st = reinterpret_cast<const IT*>(stage + mis) + lb * f.kept;

    // ---- A': (ky = hi, kx in half): 8 kz x 4 kx, inverse axis 0
    double v[32];
#pragma unroll
    for (int kz = 0; kz < 8; ++kz)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int pos = kz * 64 + hi * 8 + half * 4 + j;
        const int rk = f.full_mask ? pos : rks[pos];
        v[kz * 4 + j] = (valid && rk >= 0) ? (double)st[rk] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) line8<4, true>(v + j, p.H);
#pragma unroll
    for (int z = 0; z < 8; ++z)
#pragma unroll
      for (int j = 0; j < 4; j += 2)
        st2(blk, z * 64 + hi * 8 + half * 4 + j, key, v[z * 4 + j], v[z * 4 + j + 1]);
    __syncthreads();

    // ---- B': (nz = hi, kx in half): 8 ky x 4 kx, inverse axis 1 in place
#pragma unroll
    for (int yy = 0; yy < 8; ++yy)
#pragma unroll
      for (int j = 0; j < 4; j += 2) {
        const double2 w = ld2(blk, hi * 64 + yy * 8 + half * 4 + j, key);
        v[yy * 4 + j] = w.x;
        v[yy * 4 + j + 1] = w.y;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) line8<4, true>(v + j, p.H);
#pragma unroll
    for (int yy = 0; yy < 8; ++yy)
#pragma unroll
      for (int j = 0; j < 4; j += 2)
        st2(blk, hi * 64 + yy * 8 + half * 4 + j, key, v[yy * 4 + j], v[yy * 4 + j + 1]);
    __syncthreads();

    // ---- C': (nz = hi, ny in half): 4 ny x 8 kx, inverse axis 2 -> rows
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int xx = 0; xx < 8; xx += 2) {
        const double2 w = ld2(blk, hi * 64 + (half * 4 + i) * 8 + xx, key);
        v[i * 8 + xx] = w.x;
        v[i * 8 + xx + 1] = w.y;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) line8<1, true>(v + i * 8, p.H);
    if (valid) {
      const double n = load_kind<FK>(maxima, b);
      const bool safe = (n >= 0x1p-900) && (n <= nsafe);
      if (safe) {
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = div_const(__dmul_rn(v[q], n), rr, rinv);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __ddiv_rn(__dmul_rn(v[q], n), rr);
      }
      int64_t gc[4] = {0, 0, 0, 0};
      block_coords<3>(f, b, gc);
      const int64_t z = gc[0] * E + hi, y0 = gc[1] * E + half * 4, x0 = gc[2] * E;
      if (z < f.shape[0]) {
        const bool xfull = x0 + E <= f.shape[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (y0 + i < f.shape[1]) {
            TOut* dst = out + z * s0 + (y0 + i) * s1 + x0;
            if (xfull && f.vec_dense) {
              store_row_vec<TOut, 8>(dst, v + i * 8);
            } else {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (x0 + k < f.shape[2])
                  dst[k] = (TOut)(sizeof(TOut) == 4 ? (double)__double2float_rn(v[i * 8 + k]) : v[i * 8 + k]);
            }
          }
        }
      }
    }
    __syncthreads();  // xs reused by the next tile
  }
}

// ----------------------------------------------------------------- launch --
template <typename TIn, int FK, typename IT>
static int launch_c(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s) {
  using namespace h3;
  FastParams p;
  if (!make_fast_params(g, BPC, x, sizeof(TIn), p)) {
    set_error("half3 compress: host matrices missing");
    return BZ_E_INVALID;
  }
  size_t smem = (size_t)BPC * BSP * 8 + (size_t)NT * 8 +
                (p.f.full_mask ? 0 : ((size_t)BPC * g.kept * sizeof(IT) + 16 + 15) / 16 * 16 + BS * 2);
  auto kern = k_half3_compress<TIn, FK, IT>;
  const int occ = occupancy((const void*)kern, NT, smem);
  const int64_t grid = std::min<int64_t>(p.f.ntiles, (int64_t)kSMs * std::max(occ, 1));
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, NT, smem, s>>>(p, reinterpret_cast<const TIn*>(x), maxima,
                                   reinterpret_cast<IT*>(indices));
  return check_launch("half3_compress");
}

template <typename IT, int FK, typename TOut>
static int launch_d(const Geo& g, const void* maxima, const void* indices, void* out,
                    cudaStream_t s) {
  using namespace h3;
  FastParams p;
  if (!make_fast_params(g, BPC, out, sizeof(TOut), p)) {
    set_error("half3 decompress: host matrices missing");
    return BZ_E_INVALID;
  }
  size_t smem = (size_t)BPC * BSP * 8 + ((size_t)BPC * g.kept * sizeof(IT) + 32 + 15) / 16 * 16 +
                (p.f.full_mask ? 0 : BS * 2);
  auto kern = k_half3_decompress<IT, FK, TOut>;
  const int occ = occupancy((const void*)kern, NT, smem);
  const int64_t grid = std::min<int64_t>(p.f.ntiles, (int64_t)kSMs * std::max(occ, 1));
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, NT, smem, s>>>(p, maxima, reinterpret_cast<const IT*>(indices),
                                   reinterpret_cast<TOut*>(out));
  return check_launch("half3_decompress");
}

int launch_half3_compress(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s) {
#define BZ_K(TIN, FKV)                                                                  \
  switch (g.index_kind) {                                                               \
    case BZ_I8: return launch_c<TIN, FKV, int8_t>(g, x, maxima, indices, s);            \
    case BZ_I16: return launch_c<TIN, FKV, int16_t>(g, x, maxima, indices, s);          \
    case BZ_I32: return launch_c<TIN, FKV, int32_t>(g, x, maxima, indices, s);          \
  }
  if (g.float_kind == BZ_F32) { BZ_K(float, BZ_F32) }
  if (g.float_kind == BZ_F64) { BZ_K(double, BZ_F64) }
#undef BZ_K
  set_error("half3 compress: unsupported configuration");
  return BZ_E_UNSUPPORTED;
}

int launch_half3_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                            int out_kind, cudaStream_t s) {
#define BZ_O(IT, FKV)                                                                      \
  if (out_kind == BZ_F64) return launch_d<IT, FKV, double>(g, maxima, indices, out, s);    \
  if (out_kind == BZ_F32) return launch_d<IT, FKV, float>(g, maxima, indices, out, s);
#define BZ_K(FKV)                              \
  switch (g.index_kind) {                      \
    case BZ_I8: { BZ_O(int8_t, FKV) break; }   \
    case BZ_I16: { BZ_O(int16_t, FKV) break; } \
    case BZ_I32: { BZ_O(int32_t, FKV) break; } \
  }
  if (g.float_kind == BZ_F32) { BZ_K(BZ_F32) }
  if (g.float_kind == BZ_F64) { BZ_K(BZ_F64) }
#undef BZ_K
#undef BZ_O
  set_error("half3 decompress: unsupported configuration");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
