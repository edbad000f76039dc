// bz_line3.cu -- fused compress / decompress for 3-D blocks (E^3, E = 4, 8):
// one transform LINE per thread.
//
// A CTA owns NB blocks (NB * E^2 = 256 threads).  Per tile:
//   axis 0: thread (y,x) reads its z-line straight from HBM (lanes = x, so a
//           warp touches whole 32-byte rows), runs the reference FMA chain in
//           registers and writes the E coefficients to the block's f64 tile
//           in shared memory;
//   axis 1: thread (kz,x) transforms its y-line in place in shared memory;
//   axis 2: thread (kz,ky) reads its contiguous x-line, transforms it, and
//           keeps the E coefficients in registers for the block maximum and
//           the binning, then stores its E indices (contiguous in the
//           compressed layout: positions kz*E^2 + ky*E + kx).
// Every value crosses shared memory only twice (32 B/element), registers
// stay low (two lines of E doubles), so many warps per SM hide latency.
// Decompress mirrors it: staged index tile -> axis 0 -> axis 1 -> axis 2 ->
// ((y*N)/r) -> contiguous output rows.
// The FMA chains are the reference's (bz_fast.cuh): results are bit-identical.
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

template <int E>
struct Line3 {
  static constexpr int L = E * E;      // lines per block per axis
  static constexpr int BS = E * E * E;
  static constexpr int NT = 256;
  static constexpr int NB = NT / L;    // blocks per tile
  // f64 tile: z-planes at stride ZS (= 8 mod 16 doubles for E=8, 4 mod 16
  // for E=4, so the planes a half-warp touches fall on distinct banks); rows
  // of E doubles whose 16-byte units are XOR-permuted by (y>>1), so eight
  // lanes reading eight different rows hit eight distinct bank groups
  static constexpr int ZS = E == 8 ? 72 : 20;
  static constexpr int PAD = E * ZS;   // doubles per block
};

template <int E>
__device__ __forceinline__ int tpos(int z, int y, int x) {
  return z * Line3<E>::ZS + y * E + ((((x >> 1) ^ ((y >> 1) & (E / 2 - 1)))) << 1) + (x & 1);
}

// reference FMA chain over a line held in registers
template <int E, bool INV>
__device__ __forceinline__ void line_fma(const double* in, double* out, const double (&H)[64]) {
#pragma unroll
  for (int k = 0; k < E; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < E; ++n) acc = __fma_rn(in[n], INV ? H[k * E + n] : H[n * E + k], acc);
    out[k] = acc;
  }
}

template <int E, typename TIn, int FK, typename IT>
__global__ void __launch_bounds__(256, 3)
k_line3_compress(const FastParams p, const TIn* __restrict__ x, void* __restrict__ maxima,
                 IT* __restrict__ indices) {
  using LC = Line3<E>;
  constexpr int L = LC::L, NB = LC::NB, NT = LC::NT, PAD = LC::PAD;
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* tile = reinterpret_cast<double*>(smem_raw);                       // NB * PAD
  unsigned long long* red = reinterpret_cast<unsigned long long*>(tile + NB * PAD);  // NT / 32
  unsigned char* stage = reinterpret_cast<unsigned char*>(red + NT / 32 + 2);

  const int t = threadIdx.x;
  const int lb = t / L;      // block slot in the tile
  const int l = t % L;       // line within the block
  const int hi = l / E, lo = l % E;
  double* blk = tile + lb * PAD;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const int64_t s0 = f.stride[0], s1 = f.stride[1];
  const int64_t ntiles = (f.nblocks + NB - 1) / NB;

  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t b0 = tl * NB;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;

    // ---- axis 0: z-line of (y = hi, x = lo) from HBM
    double in[E], out[E];
    {
      int64_t gc[4] = {0, 0, 0, 0};
      if (valid) block_coords<3>(f, b, gc);
      const int64_t z0 = gc[0] * E, y = gc[1] * E + hi, xx = gc[2] * E + lo;
      const bool ok = valid && y < f.shape[1] && xx < f.shape[2];
      const TIn* src = x + z0 * s0 + y * s1 + xx;
      const int zmax = (int)min((int64_t)E, f.shape[0] - z0);
#pragma unroll
      for (int z = 0; z < E; ++z) in[z] = (ok && z < zmax) ? widen(__ldcs(src + z * s0)) : 0.0;
    }
    line_fma<E, false>(in, out, p.H);
#pragma unroll
    for (int k = 0; k < E; ++k) blk[tpos<E>(k, hi, lo)] = out[k];  // C0[kz][y][x]
    __syncthreads();

    // ---- axis 1: y-line of (kz = hi, x = lo), in place
#pragma unroll
    for (int yy = 0; yy < E; ++yy) in[yy] = blk[tpos<E>(hi, yy, lo)];
    line_fma<E, false>(in, out, p.H);
#pragma unroll
    for (int k = 0; k < E; ++k) blk[tpos<E>(hi, k, lo)] = out[k];  // C1[kz][ky][x]
    __syncthreads();

    // ---- axis 2: x-line of (kz = hi, ky = lo), 16-byte units
#pragma unroll
    for (int xx = 0; xx < E; xx += 2) {
      const double2 w = *reinterpret_cast<const double2*>(blk + tpos<E>(hi, lo, xx));
      in[xx] = w.x;
      in[xx + 1] = w.y;
    }
    line_fma<E, false>(in, out, p.H);  // C[kz][ky][kx], positions l*E + kx

    // ---- block maximum of |C| over the L lines (NaN > inf > finite)
    unsigned long long key = 0;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const unsigned long long k2 = abs_key(out[k]);
      key = k2 > key ? k2 : key;
    }
    constexpr int W = L < 32 ? L : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o, W);
      key = k2 > key ? k2 : key;
    }
    if constexpr (L > 32) {
      if ((t & 31) == 0) red[t >> 5] = key;
      __syncthreads();
#pragma unroll
      for (int w = 0; w < L / 32; ++w) {
        const unsigned long long k2 = red[lb * (L / 32) + w];
        key = k2 > key ? k2 : key;
      }
    }
    const double mx = __longlong_as_double((long long)key);
    const double n = round_to_kind<FK>(mx);
    constexpr bool CLAMP = !(FK == BZ_F32 || FK == BZ_F64);
    const BinCtx bc = bin_ctx<CLAMP>(n, rr, mx);
    if (valid && l == 0) store_kind<FK>(maxima, b, n);

    // ---- bin the thread's E coefficients (exact reference rounding)
    int q[E];
    if constexpr (sizeof(IT) <= 2) {
            unsigned nacc = 0;
#pragma unroll
      for (int k = 0; k < E; ++k) q[k] = fast_index32<IT, CLAMP>(out[k], bc.R, (int)rr, nacc);
      if (nacc | !bc.fast) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          unsigned nr = 0;
          fast_index32<IT, CLAMP>(out[k], bc.R, (int)rr, nr);
          if (nr | !bc.fast) q[k] = (int)bin_exact_ctx(out[k], bc, rr, rr);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) {
        bool nr = false;
        q[k] = bc.fast ? fast_index<IT>(out[k], bc.R, rr, nr) : 0;
        if (nr || !bc.fast) q[k] = (int)bin_exact_ctx(out[k], bc, rr, rr);
      }
    }

    // ---- store (positions l*E .. l*E+E-1 of block b)
    if (f.full_mask) {
      if (valid) {
        IT* dst = indices + b * (int64_t)LC::BS + l * E;
        if constexpr (E * sizeof(IT) == 8) {
          uint2 w;
          if constexpr (sizeof(IT) == 1) {
            w.x = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
            w.y = __byte_perm(__byte_perm(q[4], q[5], 0x0040), __byte_perm(q[6], q[7], 0x0040), 0x5410);
          } else {
            w.x = __byte_perm(q[0], q[1], 0x5410);
            w.y = __byte_perm(q[2], q[3], 0x5410);
          }
          __stcs(reinterpret_cast<uint2*>(dst), w);
        } else if constexpr (E * sizeof(IT) == 16) {
          __stcs(reinterpret_cast<uint4*>(dst), pack16<IT>(q));
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) dst[k] = (IT)q[k];
        }
      }
      __syncthreads();  // tile smem reused by the next tile
    } else {
      const int nvalid = (int)min((int64_t)NB, f.nblocks - b0);
      const int64_t dst_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + dst_byte0) & 15);
      IT* st = reinterpret_cast<IT*>(stage + mis);
      if (valid) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int rk = f.rank[l * E + k];
          if (rk >= 0) st[lb * f.kept + rk] = (IT)q[k];
        }
      }
      __syncthreads();
      smem_to_tile(reinterpret_cast<unsigned char*>(indices) + dst_byte0, stage,
                   (int64_t)nvalid * f.kept * sizeof(IT), mis, t, NT);
      __syncthreads();
    }
  }
}

template <int E, typename IT, int FK, typename TOut>
__global__ void __launch_bounds__(256, 2)
k_line3_decompress(const FastParams p, const void* __restrict__ maxima,
                   const IT* __restrict__ indices, TOut* __restrict__ out) {
  using LC = Line3<E>;
  constexpr int L = LC::L, NB = LC::NB, NT = LC::NT, PAD = LC::PAD;
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* tile = reinterpret_cast<double*>(smem_raw);
  unsigned char* stage = reinterpret_cast<unsigned char*>(tile + NB * PAD);

  const int t = threadIdx.x;
  const int lb = t / L;
  const int l = t % L;
  const int hi = l / E, lo = l % E;
  double* blk = tile + lb * PAD;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const double rinv = 1.0 / rr;
  const double nsafe = 1.7976931348623157e308 / (rr * LC::BS * 4.0);
  const int64_t s0 = f.stride[0], s1 = f.stride[1];
  const int64_t ntiles = (f.nblocks + NB - 1) / NB;

  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t b0 = tl * NB;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)NB, f.nblocks - b0);

    // ---- stage the tile's indices (coalesced 16-byte vectors)
    const int64_t src_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
    const int mis = (int)(((uintptr_t)indices + src_byte0) & 15);
    tile_to_smem(stage, reinterpret_cast<const unsigned char*>(indices) + src_byte0,
                 (int64_t)nvalid * f.kept * sizeof(IT), mis, t, NT);
    __syncthreads();
    const IT* st = reinterpret_cast<const IT*>(stage + mis) + lb * f.kept;

    // ---- axis 0: kz-line of (ky = hi, kx = lo)
    double in[E], y[E];
#pragma unroll
    for (int kz = 0; kz < E; ++kz) {
      const int pos = kz * L + hi * E + lo;
      const int rk = f.full_mask ? pos : f.rank[pos];
      in[kz] = (valid && rk >= 0) ? (double)st[rk] : 0.0;
    }
    line_fma<E, true>(in, y, p.H);
#pragma unroll
    for (int nz = 0; nz < E; ++nz) blk[tpos<E>(nz, hi, lo)] = y[nz];  // Y0[nz][ky][kx]
    __syncthreads();

    // ---- axis 1: ky-line of (nz = hi, kx = lo), in place
#pragma unroll
    for (int ky = 0; ky < E; ++ky) in[ky] = blk[tpos<E>(hi, ky, lo)];
    line_fma<E, true>(in, y, p.H);
#pragma unroll
    for (int ny = 0; ny < E; ++ny) blk[tpos<E>(hi, ny, lo)] = y[ny];  // Y1[nz][ny][kx]
    __syncthreads();

    // ---- axis 2: kx-line of (nz = hi, ny = lo) -> output row
#pragma unroll
    for (int kx = 0; kx < E; kx += 2) {
      const double2 w = *reinterpret_cast<const double2*>(blk + tpos<E>(hi, lo, kx));
      in[kx] = w.x;
      in[kx + 1] = w.y;
    }
    line_fma<E, true>(in, y, p.H);
    if (valid) {
      const double n = load_kind<FK>(maxima, b);
      const bool safe = (n >= 0x1p-900) && (n <= nsafe);
      if (safe) {
#pragma unroll
        for (int k = 0; k < E; ++k) y[k] = div_const(__dmul_rn(y[k], n), rr, rinv);
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) y[k] = __ddiv_rn(__dmul_rn(y[k], n), rr);
      }
      int64_t gc[4] = {0, 0, 0, 0};
      block_coords<3>(f, b, gc);
      const int64_t z = gc[0] * E + hi, yy = gc[1] * E + lo, x0 = gc[2] * E;
      if (z < f.shape[0] && yy < f.shape[1]) {
        TOut* dst = out + z * s0 + yy * s1 + x0;
        if (x0 + E <= f.shape[2] && row_vectorizable<TOut>(E) && f.vec_dense) {
          if constexpr (row_vectorizable<TOut>(E)) store_row_vec<TOut, E>(dst, y);
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (x0 + k < f.shape[2]) dst[k] = (TOut)(sizeof(TOut) == 4 ? (double)__double2float_rn(y[k]) : y[k]);
        }
      }
    }
    __syncthreads();  // tile + stage reused by the next tile
  }
}

// ----------------------------------------------------------------- launch --
template <int E, typename TIn, int FK, typename IT>
static int launch_c(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s) {
  using LC = Line3<E>;
  FastParams p;
  if (!make_fast_params(g, LC::NB, x, sizeof(TIn), p)) {
    set_error("line3 compress: host matrices missing");
    return BZ_E_INVALID;
  }
  size_t smem = (size_t)LC::NB * LC::PAD * 8 + (LC::NT / 32 + 2) * 8 +
                (p.f.full_mask ? 0 : (size_t)LC::NB * g.kept * sizeof(IT) + 16);
  auto kern = k_line3_compress<E, TIn, FK, IT>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, LC::NT, smem);
  const int64_t ntiles = (g.nblocks + LC::NB - 1) / LC::NB;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)kSMs * std::max(occ, 1));
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, LC::NT, smem, s>>>(p, reinterpret_cast<const TIn*>(x), maxima,
                                       reinterpret_cast<IT*>(indices));
  return check_launch("line3_compress");
}

template <int E, typename IT, int FK, typename TOut>
static int launch_d(const Geo& g, const void* maxima, const void* indices, void* out,
                    cudaStream_t s) {
  using LC = Line3<E>;
  FastParams p;
  if (!make_fast_params(g, LC::NB, out, sizeof(TOut), p)) {
    set_error("line3 decompress: host matrices missing");
    return BZ_E_INVALID;
  }
  size_t smem = (size_t)LC::NB * LC::PAD * 8 + (size_t)LC::NB * g.kept * sizeof(IT) + 32;
  auto kern = k_line3_decompress<E, IT, FK, TOut>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, LC::NT, smem);
  const int64_t ntiles = (g.nblocks + LC::NB - 1) / LC::NB;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)kSMs * std::max(occ, 1));
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, LC::NT, smem, s>>>(p, maxima, reinterpret_cast<const IT*>(indices),
                                       reinterpret_cast<TOut*>(out));
  return check_launch("line3_decompress");
}

int launch_line3_compress(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s) {
  const int E = g.block[0];
#define BZ_K(EE, TIN, FKV)                                                                      \
  switch (g.index_kind) {                                                                       \
    case BZ_I8: return launch_c<EE, TIN, FKV, int8_t>(g, x, maxima, indices, s);                \
    case BZ_I16: return launch_c<EE, TIN, FKV, int16_t>(g, x, maxima, indices, s);              \
    case BZ_I32: return launch_c<EE, TIN, FKV, int32_t>(g, x, maxima, indices, s);              \
  }
  if (E == 8 && g.float_kind == BZ_F32) { BZ_K(8, float, BZ_F32) }
  if (E == 8 && g.float_kind == BZ_F64) { BZ_K(8, double, BZ_F64) }
  if (E == 4 && g.float_kind == BZ_F32) { BZ_K(4, float, BZ_F32) }
  if (E == 4 && g.float_kind == BZ_F64) { BZ_K(4, double, BZ_F64) }
#undef BZ_K
  set_error("line3 compress: unsupported configuration");
  return BZ_E_UNSUPPORTED;
}

int launch_line3_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                            int out_kind, cudaStream_t s) {
  const int E = g.block[0];
#define BZ_O(EE, IT, FKV)                                                                         \
  if (out_kind == BZ_F64) return launch_d<EE, IT, FKV, double>(g, maxima, indices, out, s);       \
  if (out_kind == BZ_F32) return launch_d<EE, IT, FKV, float>(g, maxima, indices, out, s);
#define BZ_K(EE, FKV)                              \
  switch (g.index_kind) {                          \
    case BZ_I8: { BZ_O(EE, int8_t, FKV) break; }   \
    case BZ_I16: { BZ_O(EE, int16_t, FKV) break; } \
    case BZ_I32: { BZ_O(EE, int32_t, FKV) break; } \
  }
  if (E == 8 && g.float_kind == BZ_F32) { BZ_K(8, BZ_F32) }
  if (E == 8 && g.float_kind == BZ_F64) { BZ_K(8, BZ_F64) }
  if (E == 4 && g.float_kind == BZ_F32) { BZ_K(4, BZ_F32) }
  if (E == 4 && g.float_kind == BZ_F64) { BZ_K(4, BZ_F64) }
#undef BZ_K
#undef BZ_O
  set_error("line3 decompress: unsupported configuration");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
