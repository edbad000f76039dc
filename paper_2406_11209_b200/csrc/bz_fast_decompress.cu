// bz_fast_decompress.cu -- fused decompress: indices -> inverse transform ->
// *N / r -> merge + crop, one pass (codec.py:364-384, arrays.py:181-190).
//
// Arithmetic is the reference's, step for step: the inverse transform runs on
// the raw integer indices as the same FMA chain dgemm uses (axis 0 first,
// bz_fast.cuh), then the block scale is applied as fl(fl(y * N) / r)
// (codec.py:377-379).  The division by the constant r uses Markstein's FMA
// correction (bz_common.cuh: div_const), which returns the correctly rounded
// quotient; blocks whose N could push y*N out of the normal range use IEEE
// division.  The f64 output is therefore bit-identical to the reference.
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

#include <cstdlib>

namespace bz {

template <typename IT, int N>
__device__ __forceinline__ void load_indices_vec(const IT* __restrict__ src, double* dst) {
  static_assert((N * sizeof(IT)) % 16 == 0, "whole 16-byte chunks");
#pragma unroll
  for (int c = 0; c < N * (int)sizeof(IT) / 16; ++c) {
    uint4 w = __ldcs(reinterpret_cast<const uint4*>(src) + c);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    constexpr int PER = 16 / sizeof(IT);
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      uint32_t word = ws[(e * sizeof(IT)) / 4];
      int sh = (e * sizeof(IT) * 8) % 32;
      int val;
      if constexpr (sizeof(IT) == 1) val = (int)(int8_t)(word >> sh);
      else if constexpr (sizeof(IT) == 2) val = (int)(int16_t)(word >> sh);
      else val = (int)word;
      dst[c * PER + e] = (double)val;
    }
  }
}

// raw 16-byte chunks of one block's indices (register prefetch), unpacked later
template <typename IT, int N>
struct RawIdx {
  static constexpr int C = (N * (int)sizeof(IT) + 15) / 16;
  uint4 w[C];
};

template <typename IT, int N>
__device__ __forceinline__ void load_raw(const IT* __restrict__ src, bool ok, bool v32,
                                         RawIdx<IT, N>& r) {
  constexpr int C = RawIdx<IT, N>::C;
  if constexpr (C % 2 == 0) {
    if (v32) {  // 256-bit loads
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        if (ok) ld_global_256(reinterpret_cast<const uint4*>(src) + c, r.w[c], r.w[c + 1]);
        else r.w[c] = r.w[c + 1] = make_uint4(0, 0, 0, 0);
      }
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
    r.w[c] = ok ? __ldcs(reinterpret_cast<const uint4*>(src) + c) : make_uint4(0, 0, 0, 0);
}

template <typename IT, int N>
__device__ __forceinline__ void unpack_raw(const RawIdx<IT, N>& r, double* dst) {
  constexpr int PER = 16 / sizeof(IT);
#pragma unroll
  for (int c = 0; c < RawIdx<IT, N>::C; ++c) {
    const uint32_t ws[4] = {r.w[c].x, r.w[c].y, r.w[c].z, r.w[c].w};
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const uint32_t word = ws[(e * sizeof(IT)) / 4];
      const int sh = (e * sizeof(IT) * 8) % 32;
      int val;
      if constexpr (sizeof(IT) == 1) val = (int)(int8_t)(word >> sh);
      else if constexpr (sizeof(IT) == 2) val = (int)(int16_t)(word >> sh);
      else val = (int)word;
      dst[c * PER + e] = (double)val;
    }
  }
}

template <int D, int E, typename IT, int FK, typename TOut>
__global__ void __launch_bounds__(Tile<D, E>::NT)
k_fast_decompress(const FastParams p, const void* __restrict__ maxima,
                  const IT* __restrict__ indices, TOut* __restrict__ out) {
  using TL = Tile<D, E>;
  constexpr int NIN = TL::NIN, BS = TL::BS, BPC = TL::BPC, NT = TL::NT;
  constexpr int LP = 0, LQ = D - 1;                   // first slice (holds axis 0)
  constexpr int SP = D >= 2 ? D - 2 : 0, SQ = D - 1;  // output slice
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);
  // two index-tile buffers: tile t+1 streams in (cp.async) while tile t computes
  const size_t stage_bytes = ((size_t)BPC * f.kept * sizeof(IT) + 16 + 15) / 16 * 16;
  unsigned char* stages = smem_raw + (TL::EXCH ? (size_t)BPC * BS * sizeof(double) : 0);

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;
  // rank table (position -> kept rank) in shared memory for pruned masks
  int16_t* rks = reinterpret_cast<int16_t*>(stages + 2 * stage_bytes);
  if (!f.full_mask) {
    for (int i = t; i < BS; i += NT) rks[i] = (int16_t)f.rank[i];
    __syncthreads();
  }
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const double rinv = 1.0 / rr;
  const double nsafe = 1.7976931348623157e308 / (rr * TL::BS * 4.0);
  const int swz = slot_swizzle(lb);
  double* blk = xs + lb * BS;
  const bool stage_in = TL::EXCH || !f.full_mask;

  // copy a tile's kept indices into stage buffer `buf` (body by cp.async)
  auto prefetch = [&](int64_t tile, int buf) {
    if (tile < f.ntiles) {
      const int64_t b0 = tile * BPC;
      const int nv = (int)min((int64_t)BPC, f.nblocks - b0);
      const int64_t byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int64_t nbytes = (int64_t)nv * f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + byte0) & 15);
      const unsigned char* g = reinterpret_cast<const unsigned char*>(indices) + byte0;
      unsigned char* st = stages + buf * stage_bytes;
      const int head = mis ? 16 - mis : 0;
      const int h = (int)min((int64_t)head, nbytes);
      for (int i = t; i < h; i += NT) st[mis + i] = g[i];
      const int64_t body = (nbytes - h) / 16;
      for (int64_t i = t; i < body; i += NT) cp_async16(st + mis + h + i * 16, g + h + i * 16);
      for (int64_t i = h + body * 16 + t; i < nbytes; i += NT) st[mis + i] = g[i];
    }
    cp_async_commit();
  };

  int buf = 0;
  if (stage_in) prefetch(blockIdx.x, 0);
  // whole-block direct loads (full mask, one thread per block): the next
  // tile's indices and maximum are fetched into registers before this tile's
  // transform runs, so loads overlap the FMA chain
  constexpr bool REGPF = (NIN * sizeof(IT)) % 16 == 0 && TL::TB == 1 && NIN <= 16;
  const bool idx32 = ((uintptr_t)indices % 32) == 0;
  RawIdx<IT, NIN> raw;
  double n_next = 0.0;
  auto reg_prefetch = [&](int64_t tile) {
    const int64_t bn = tile * BPC + lb;
    const bool ok = tile < f.ntiles && bn < f.nblocks;
    load_raw<IT, NIN>(indices + (ok ? bn : 0) * (int64_t)NIN, ok, idx32, raw);
    n_next = ok ? load_kind<FK>(maxima, bn) : 0.0;
  };
  if (REGPF && !stage_in) reg_prefetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x, buf ^= 1) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    double n_cur = 0.0;

    // ---- first slice (axis 0, axis D-1) at o, as f64 integers
    double v[NIN];
    if (stage_in) {
      cp_async_wait_all();
      __syncthreads();
      prefetch(tile + gridDim.x, buf ^ 1);
      const int64_t src_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + src_byte0) & 15);
      const IT* st = reinterpret_cast<const IT*>(stages + buf * stage_bytes + mis);
      const int base = D >= 2 ? slice_base<D, E, LP, LQ>(o) : 0;
#pragma unroll
      for (int i = 0; i < (D >= 2 ? E : 1); ++i)
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int pos = base + i * axis_stride<D, E>(LP) * (D >= 2) + j * axis_stride<D, E>(LQ);
          const int rk = f.full_mask ? pos : rks[pos];
          v[i * E + j] = (valid && rk >= 0) ? (double)st[lb * f.kept + rk] : 0.0;
        }
    } else if constexpr (REGPF) {
      unpack_raw<IT, NIN>(raw, v);
      n_cur = n_next;
      reg_prefetch(tile + gridDim.x);
    } else {
      if (valid) {
        if constexpr ((NIN * sizeof(IT)) % 16 == 0) {
          load_indices_vec<IT, NIN>(indices + b * (int64_t)NIN, v);
        } else {
#pragma unroll
          for (int q = 0; q < NIN; ++q) v[q] = (double)indices[b * (int64_t)NIN + q];
        }
      } else {
#pragma unroll
        for (int q = 0; q < NIN; ++q) v[q] = 0.0;
      }
    }

    // ---- inverse transform, axis 0 first (reference order)
    if constexpr (D == 1) {
      dense_line<E, 1, true>(v, p.H);
    } else if constexpr (D == 2) {
      slice_cols<E, true>(v, p.H);
      slice_rows<E, true>(v, p.H);
    } else if constexpr (D == 3) {
      slice_cols<E, true>(v, p.H);  // axis 0
      slice_store<D, E, 0, 2>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 1, 2>(blk, swz, o, v);
      slice_cols<E, true>(v, p.H);  // axis 1
      slice_rows<E, true>(v, p.H);  // axis 2
    } else {
      slice_cols<E, true>(v, p.H);  // axis 0
      slice_store<D, E, 0, 3>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 1, 2>(blk, swz, o, v);
      slice_cols<E, true>(v, p.H);  // axis 1
      slice_rows<E, true>(v, p.H);  // axis 2
      __syncthreads();
      slice_store<D, E, 1, 2>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 2, 3>(blk, swz, o, v);
      slice_rows<E, true>(v, p.H);  // axis 3
    }

    // ---- scale ((y * N) / r) and store the output slice (axis D-2 rows, D-1 cols)
    if (valid) {
      const double n = (REGPF && !stage_in) ? n_cur : load_kind<FK>(maxima, b);
      const bool safe = (n >= 0x1p-900) && (n <= nsafe);
      if (safe) {
#pragma unroll
        for (int q = 0; q < NIN; ++q) v[q] = div_const(__dmul_rn(v[q], n), rr, rinv);
      } else {
#pragma unroll
        for (int q = 0; q < NIN; ++q) v[q] = __ddiv_rn(__dmul_rn(v[q], n), rr);
      }
      if constexpr (sizeof(TOut) == 4) {
#pragma unroll
        for (int q = 0; q < NIN; ++q) v[q] = (double)__double2float_rn(v[q]);
      }
      int64_t gc[4] = {0, 0, 0, 0};
      int c[4];
      slice_coords<D, E, SP, SQ>(o, c);
      block_coords<D>(f, b, gc);
      bool interior, fixed_ok;
      int rows_ok = 0, cols_ok = 0;
      const int64_t off = dense_slice_origin<D, E, SP>(f, gc, c, interior, fixed_ok, rows_ok, cols_ok);
      constexpr int ROWS = D >= 2 ? E : 1;
      const int64_t rs = f.stride[SP];
      if (fixed_ok) {
        bool fast = false;
        if constexpr (row_vectorizable<TOut>(E)) fast = interior && f.vec_dense;
        if (fast) {
          if constexpr ((E * sizeof(TOut)) % 32 == 0) {
            if (f.vec32) {
#pragma unroll
              for (int r = 0; r < ROWS; ++r) store_row_vec32<TOut, E>(out + off + r * rs, v + r * E);
            } else {
#pragma unroll
              for (int r = 0; r < ROWS; ++r) store_row_vec<TOut, E>(out + off + r * rs, v + r * E);
            }
          } else if constexpr (row_vectorizable<TOut>(E)) {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) store_row_vec<TOut, E>(out + off + r * rs, v + r * E);
          }
        } else {
#pragma unroll
          for (int r = 0; r < ROWS; ++r)
#pragma unroll
            for (int cc = 0; cc < E; ++cc)
              if (r < rows_ok && cc < cols_ok) out[off + r * rs + cc] = (TOut)v[r * E + cc];
        }
      }
    }
    if (TL::EXCH) __syncthreads();  // exchange area reused by the next tile
  }
}

template <int D, int E, typename IT, int FK, typename TOut>
static int launch_one(const Geo& g, const void* maxima, const void* indices, void* out,
                      cudaStream_t s) {
  using TL = Tile<D, E>;
  FastParams p;
  if (!make_fast_params(g, TL::BPC, out, sizeof(TOut), p)) {
    set_error("fast decompress: host matrices missing");
    return BZ_E_INVALID;
  }
  size_t smem = (TL::EXCH ? (size_t)TL::BPC * TL::BS * sizeof(double) : 0) +
                ((TL::EXCH || !p.f.full_mask)
                     ? 2 * (((size_t)TL::BPC * g.kept * sizeof(IT) + 16 + 15) / 16 * 16) : 0) +
                (p.f.full_mask ? 0 : (size_t)TL::BS * 2 + 16);
  auto kern = k_fast_decompress<D, E, IT, FK, TOut>;
  const int occ = occupancy((const void*)kern, TL::NT, smem);
  int64_t grid = std::min<int64_t>(p.f.ntiles, (int64_t)kSMs * occ);
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, TL::NT, smem, s>>>(p, maxima, reinterpret_cast<const IT*>(indices),
                                       reinterpret_cast<TOut*>(out));
  return check_launch("fast_decompress");
}

template <int D, int E>
static int dispatch_kinds(const Geo& g, const void* maxima, const void* indices, void* out,
                          int out_kind, cudaStream_t s) {
#define BZ_OUT(IT, FKV)                                                                        \
  if (out_kind == BZ_F64) return launch_one<D, E, IT, FKV, double>(g, maxima, indices, out, s); \
  if (out_kind == BZ_F32) return launch_one<D, E, IT, FKV, float>(g, maxima, indices, out, s);
#define BZ_IDX(FKV)                              \
  switch (g.index_kind) {                        \
    case BZ_I8: { BZ_OUT(int8_t, FKV) break; }   \
    case BZ_I16: { BZ_OUT(int16_t, FKV) break; } \
    case BZ_I32: { BZ_OUT(int32_t, FKV) break; } \
  }
  if (g.float_kind == BZ_F32) { BZ_IDX(BZ_F32) }
  if (g.float_kind == BZ_F64) { BZ_IDX(BZ_F64) }
#undef BZ_IDX
#undef BZ_OUT
  set_error("fast decompress: unsupported kinds");
  return BZ_E_UNSUPPORTED;
}

bool fast_decompress_supported(const Geo& g, int out_kind) {
  if (out_kind != BZ_F64 && out_kind != BZ_F32) return false;
  return fast_supported(g, g.float_kind);
}

int launch_fast_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                           int out_kind, cudaStream_t s) {
  const int E = g.block[0];
  if (g.ndim == 3 && E == 8)
    return launch_half3_decompress(g, maxima, indices, out, out_kind, s);
#define BZ_CASE(DD, EE) \
  if (g.ndim == DD && E == EE) return dispatch_kinds<DD, EE>(g, maxima, indices, out, out_kind, s);
  BZ_CASE(1, 4) BZ_CASE(1, 8) BZ_CASE(2, 4) BZ_CASE(2, 8) BZ_CASE(3, 4) BZ_CASE(3, 8)
  BZ_CASE(4, 4)
#undef BZ_CASE
  set_error("fast decompress: unsupported block shape");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
