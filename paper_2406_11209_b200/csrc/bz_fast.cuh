// bz_fast.cuh -- shared pieces of the fused compress / decompress kernels.
//
// Bit-exact transform.  The reference's np.tensordot (OpenBLAS dgemm, kernel
// sizes <= 32) evaluates every coefficient as a sequential FMA chain
// acc = fma(x[n], H[n][k], acc), n ascending from acc = +0, one axis at a
// time, axis 0 first (transforms.py:118-126).  We evaluate exactly that chain,
// with the reference's own matrix entries carried as kernel parameters (DFMA
// constant-bank operands), so coefficients -- hence maxima, indices and
// decompressed values -- are bit-identical to the reference, not merely
// within a tolerance.  (Verified on every golden case, tests/golden.)
//
// Work decomposition for a block of E^D elements ("slices"):
//   a thread owns an E x E slice of two block axes (P, Q) at fixed
//   coordinates of the other D-2 axes; TB = E^(D-2) threads own a block.
//   Transforms along P or Q run in registers.  To reach another axis the
//   TB threads of a block exchange through shared memory in the block's
//   canonical (row-major) layout, XOR-swizzled by the block's slot so that
//   lanes of a warp (consecutive blocks) hit distinct banks.
//   D=2: one thread per block, slice (0,1).
//   D=3: load slice (0,2) | axis 0 | exchange -> (1,2) | axes 1, 2.
//   D=4: load slice (0,3) | axis 0 | exchange -> (1,2) | axes 1, 2 |
//        exchange -> (2,3) | axis 3.
// Threads are laid out t = o * BPC + lb (o = slice within block, lb = block
// slot), so consecutive lanes own consecutive blocks along the fastest grid
// axis and every dense row access is a run of contiguous 16-byte vectors.
#pragma once

#include <algorithm>

#include "bz_common.cuh"

namespace bz {

constexpr int ipow(int b, int e) { return e <= 0 ? 1 : b * ipow(b, e - 1); }

template <int D, int E>
struct Tile {
  static constexpr int TB = D >= 3 ? ipow(E, D - 2) : 1;  // threads per block
  static constexpr int NIN = D >= 2 ? E * E : E;          // values per thread
  static constexpr int BS = ipow(E, D);                   // block size
  static constexpr int NT = NIN >= 64 ? 128 : 256;        // threads per CTA
  static constexpr int BPC = NT / TB;                     // blocks per CTA tile
  static constexpr bool EXCH = D >= 3;
};

// n / d for 0 <= n < 2^31 by multiply-high (Granlund-Montgomery): 3
// instructions instead of a ~40-instruction integer division
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  f.s = s;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.s);
}

struct FastGeo {
  int64_t shape[4];
  int64_t grid[4];
  FastDiv gdiv[4];   // divisors = grid extents (valid when nblocks < 2^31)
  int32_t small;     // nblocks < 2^31: use the FastDiv path
  int64_t stride[4];
  int64_t nblocks;
  int64_t ntiles;
  int32_t kept;
  int32_t full_mask;
  int32_t vec_dense;  // 16-byte vector access legal on the dense side
  int32_t vec32;      // 32-byte (256-bit) access legal on the dense side
  const int32_t* rank;
};

struct FastParams {
  FastGeo f;
  double H[64];  // reference matrix entries [sample][basis] (E <= 8)
};

inline bool make_fast_params(const Geo& g, int bpc, const void* dense, int dense_bytes,
                             FastParams& p) {
  FastGeo& f = p.f;
  f = FastGeo{};
  for (int a = 0; a < g.ndim; ++a) {
    f.shape[a] = g.shape[a];
    f.grid[a] = g.grid[a];
    f.stride[a] = g.stride[a];
  }
  f.nblocks = g.nblocks;
  f.ntiles = (g.nblocks + bpc - 1) / bpc;
  f.small = g.nblocks < (1ll << 31);
  for (int a = 0; a < g.ndim; ++a)
    f.gdiv[a] = make_fastdiv((uint32_t)std::min<int64_t>(g.grid[a], 0x7fffffff));
  f.kept = g.kept;
  f.full_mask = g.kept == g.bsize;
  f.rank = g.rank;
  const int E = g.block[g.ndim - 1];
  bool ok = ((uintptr_t)dense % 16 == 0) && ((E * dense_bytes) % 16 == 0);
  for (int a = 0; a + 1 < g.ndim; ++a) ok = ok && ((g.stride[a] * dense_bytes) % 16 == 0);
  f.vec_dense = ok;
  bool ok32 = ((uintptr_t)dense % 32 == 0) && ((E * dense_bytes) % 32 == 0);
  for (int a = 0; a + 1 < g.ndim; ++a) ok32 = ok32 && ((g.stride[a] * dense_bytes) % 32 == 0);
  f.vec32 = ok32;
  if (!g.matrices_host) return false;
  for (int i = 0; i < E * E; ++i) p.H[i] = g.matrices_host[i];  // every axis uses the same E
  return true;
}

// ------------------------------------------------------------------ slices --
template <int D, int E>
__host__ __device__ constexpr int axis_stride(int a) { return ipow(E, D - 1 - a); }

// canonical position of slice element (0,0) for slice axes (P,Q) at fixed
// coordinates o (row-major over the other axes in ascending order)
template <int D, int E, int P, int Q>
__device__ __forceinline__ int slice_base(int o) {
  int pos = 0;
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    if (a != P && a != Q) {
      pos += (o % E) * axis_stride<D, E>(a);
      o /= E;
    }
  }
  return pos;
}

// fixed-axis coordinates of slice (P,Q) for thread o
template <int D, int E, int P, int Q>
__device__ __forceinline__ void slice_coords(int o, int (&c)[4]) {
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    if (a != P && a != Q) {
      c[a] = o % E;
      o /= E;
    } else {
      c[a] = 0;
    }
  }
}

// write slice (P,Q) of thread o into the block's canonical smem region.
// When Q is the last axis, element pairs (j, j+1) are adjacent and move as
// 16-byte accesses; the XOR swizzle then works on 16-byte units (`swz` is
// even), so 8 lanes with consecutive block slots hit 8 distinct bank groups.
template <int D, int E, int P, int Q>
__device__ __forceinline__ void slice_store(double* blk, int swz, int o, const double* v) {
  const int base = slice_base<D, E, P, Q>(o);
  if constexpr (Q == D - 1 && E % 2 == 0) {
#pragma unroll
    for (int i = 0; i < E; ++i)
#pragma unroll
      for (int j = 0; j < E; j += 2)
        *reinterpret_cast<double2*>(blk + ((base + i * axis_stride<D, E>(P) + j) ^ (swz & ~1))) =
            (swz & 1) ? make_double2(v[i * E + j + 1], v[i * E + j])
                      : make_double2(v[i * E + j], v[i * E + j + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i)
#pragma unroll
      for (int j = 0; j < E; ++j)
        blk[(base + i * axis_stride<D, E>(P) + j * axis_stride<D, E>(Q)) ^ swz] = v[i * E + j];
  }
}

template <int D, int E, int P, int Q>
__device__ __forceinline__ void slice_load(const double* blk, int swz, int o, double* v) {
  const int base = slice_base<D, E, P, Q>(o);
  if constexpr (Q == D - 1 && E % 2 == 0) {
#pragma unroll
    for (int i = 0; i < E; ++i)
#pragma unroll
      for (int j = 0; j < E; j += 2) {
        const double2 w =
            *reinterpret_cast<const double2*>(blk + ((base + i * axis_stride<D, E>(P) + j) ^ (swz & ~1)));
        v[i * E + j] = (swz & 1) ? w.y : w.x;
        v[i * E + j + 1] = (swz & 1) ? w.x : w.y;
      }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i)
#pragma unroll
      for (int j = 0; j < E; ++j)
        v[i * E + j] = blk[(base + i * axis_stride<D, E>(P) + j * axis_stride<D, E>(Q)) ^ swz];
  }
}

// swizzle key for block slot lb: bits 1-3 spread 16-byte units over the 8
// bank groups (conflict-free 128-bit phases of 8 lanes), bit 0 makes 16
// consecutive slots distinct for 64-bit accesses; 16-byte pair accesses
// apply bit 0 as an in-pair swap
__device__ __forceinline__ int slot_swizzle(int lb) { return ((lb & 7) << 1) | ((lb >> 3) & 1); }

// ------------------------------------------------- reference-exact lines --
// forward: C[k] = fma chain over n of x[n] * H[n][k];  inverse: y[n] = fma
// chain over k of C[k] * H[n][k]  (transforms.py:118-142 via dgemm order)
template <int E, int S, bool INV>
__device__ __forceinline__ void dense_line(double* v, const double (&H)[64]) {
  double in[E];
#pragma unroll
  for (int i = 0; i < E; ++i) in[i] = v[i * S];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < E; ++n) acc = __fma_rn(in[n], INV ? H[k * E + n] : H[n * E + k], acc);
    v[k * S] = acc;
  }
}

// slice columns (lines over i, the P axis) / rows (lines over j, the Q axis)
template <int E, bool INV>
__device__ __forceinline__ void slice_cols(double* v, const double (&H)[64]) {
#pragma unroll
  for (int j = 0; j < E; ++j) dense_line<E, E, INV>(v + j, H);
}
template <int E, bool INV>
__device__ __forceinline__ void slice_rows(double* v, const double (&H)[64]) {
#pragma unroll
  for (int i = 0; i < E; ++i) dense_line<E, 1, INV>(v + i * E, H);
}

// ------------------------------------------------ dense-side geometry ----
// block coordinates of block b
template <int D>
__device__ __forceinline__ void block_coords(const FastGeo& f, int64_t b, int64_t (&gc)[4]) {
  if (f.small) {
    uint32_t r = (uint32_t)b;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint32_t q = fdiv(r, f.gdiv[a]);
      gc[a] = r - q * f.gdiv[a].d;
      r = q;
    }
  } else {
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      gc[a] = b % f.grid[a];
      b /= f.grid[a];
    }
  }
}

// dense offset of slice (P, Q=D-1) element (0,0) at fixed coords c; whether
// the whole slice is inside the array; per-row / per-column validity limits
template <int D, int E, int P>
__device__ __forceinline__ int64_t dense_slice_origin(const FastGeo& f, const int64_t (&gc)[4],
                                                      const int (&c)[4], bool& interior,
                                                      bool& fixed_ok, int& rows_ok,
                                                      int& cols_ok) {
  int64_t off = 0;
  interior = true;
  fixed_ok = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int64_t c0 = gc[a] * E + c[a];
    off += c0 * f.stride[a];
    const int64_t room = f.shape[a] - gc[a] * E;  // valid coords along a within the block
    if (a == P || a == D - 1) {
      const int lim = room >= E ? E : (int)room;
      if (a == P && a != D - 1) rows_ok = lim;
      if (a == D - 1) cols_ok = lim;
      if (lim < E) interior = false;
    } else {
      if (c[a] >= room) fixed_ok = false;
    }
  }
  if (D == 1) rows_ok = 1;
  return off;
}

// ------------------------------------------------ vector row load / store --
template <typename T, int E>
__device__ __forceinline__ void load_row_vec(const T* __restrict__ src, double* dst) {
  constexpr int CH = 16 / sizeof(T);
  static_assert(E % CH == 0, "row must be a whole number of 16-byte chunks");
#pragma unroll
  for (int c = 0; c < E / CH; ++c) {
    uint4 w = __ldcs(reinterpret_cast<const uint4*>(src) + c);
    if constexpr (sizeof(T) == 4) {
      dst[c * 4 + 0] = (double)__uint_as_float(w.x);
      dst[c * 4 + 1] = (double)__uint_as_float(w.y);
      dst[c * 4 + 2] = (double)__uint_as_float(w.z);
      dst[c * 4 + 3] = (double)__uint_as_float(w.w);
    } else {
      dst[c * 2 + 0] = __hiloint2double((int)w.y, (int)w.x);
      dst[c * 2 + 1] = __hiloint2double((int)w.w, (int)w.z);
    }
  }
}

template <typename T, int E>
__device__ __forceinline__ void store_row_vec(T* __restrict__ dst, const double* src) {
  constexpr int CH = 16 / sizeof(T);
  static_assert(E % CH == 0, "row must be a whole number of 16-byte chunks");
#pragma unroll
  for (int c = 0; c < E / CH; ++c) {
    uint4 w;
    if constexpr (sizeof(T) == 4) {
      w.x = __float_as_uint((float)src[c * 4 + 0]);
      w.y = __float_as_uint((float)src[c * 4 + 1]);
      w.z = __float_as_uint((float)src[c * 4 + 2]);
      w.w = __float_as_uint((float)src[c * 4 + 3]);
    } else {
      w.x = (unsigned)__double2loint(src[c * 2 + 0]);
      w.y = (unsigned)__double2hiint(src[c * 2 + 0]);
      w.z = (unsigned)__double2loint(src[c * 2 + 1]);
      w.w = (unsigned)__double2hiint(src[c * 2 + 1]);
    }
    __stcs(reinterpret_cast<uint4*>(dst) + c, w);
  }
}

template <typename T>
__host__ __device__ constexpr bool row_vectorizable(int E) { return (E * (int)sizeof(T)) % 16 == 0; }

// 256-bit (32-byte) stores: one STG.E.256 per 32 bytes of a row
template <typename T, int E>
__device__ __forceinline__ void store_row_vec32(T* __restrict__ dst, const double* src) {
  static_assert((E * sizeof(T)) % 32 == 0, "row must be a whole number of 32-byte chunks");
#pragma unroll
  for (int c = 0; c < E * (int)sizeof(T) / 32; ++c) {
    if constexpr (sizeof(T) == 8) {
      asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(dst + c * 4), "d"(src[c * 4]),
                   "d"(src[c * 4 + 1]), "d"(src[c * 4 + 2]), "d"(src[c * 4 + 3])
                   : "memory");
    } else {
      asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(dst + c * 8),
                   "f"((float)src[c * 8]), "f"((float)src[c * 8 + 1]), "f"((float)src[c * 8 + 2]),
                   "f"((float)src[c * 8 + 3]), "f"((float)src[c * 8 + 4]), "f"((float)src[c * 8 + 5]),
                   "f"((float)src[c * 8 + 6]), "f"((float)src[c * 8 + 7])
                   : "memory");
    }
  }
}

// 256-bit load of 32 bytes (read-only path, no L1 allocation)
__device__ __forceinline__ void ld_global_256(const void* p, uint4& lo, uint4& hi) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z),
                 "=r"(hi.w)
               : "l"(p));
}

// ------------------------------------------------------------- cp.async --
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <typename T>
__device__ __forceinline__ void unpack_row(const uint4* src, double* dst, int units) {
  // units 16-byte chunks of T -> doubles
#pragma unroll
  for (int c = 0; c < units; ++c) {
    const uint4 w = src[c];
    if constexpr (sizeof(T) == 4) {
      dst[c * 4 + 0] = (double)__uint_as_float(w.x);
      dst[c * 4 + 1] = (double)__uint_as_float(w.y);
      dst[c * 4 + 2] = (double)__uint_as_float(w.z);
      dst[c * 4 + 3] = (double)__uint_as_float(w.w);
    } else {
      dst[c * 2 + 0] = __hiloint2double((int)w.y, (int)w.x);
      dst[c * 2 + 1] = __hiloint2double((int)w.w, (int)w.z);
    }
  }
}

// |x| as an ordered unsigned key: NaN > inf > finite
__device__ __forceinline__ unsigned long long abs_key(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

// copy `nbytes` of a contiguous global range to / from shared memory; the
// shared buffer is offset by `mis` = (global address mod 16) so that the
// body moves as aligned 16-byte vectors
__device__ __forceinline__ void tile_to_smem(unsigned char* st, const unsigned char* g,
                                             int64_t nbytes, int mis, int t, int nt) {
  const int head = mis ? 16 - mis : 0;
  const int h = (int)min((int64_t)head, nbytes);
  for (int i = t; i < h; i += nt) st[mis + i] = g[i];
  const int64_t body = (nbytes - h) / 16;
  for (int64_t i = t; i < body; i += nt)
    *reinterpret_cast<uint4*>(st + mis + h + i * 16) = __ldcs(reinterpret_cast<const uint4*>(g + h) + i);
  for (int64_t i = h + body * 16 + t; i < nbytes; i += nt) st[mis + i] = g[i];
}

__device__ __forceinline__ void smem_to_tile(unsigned char* g, const unsigned char* st,
                                             int64_t nbytes, int mis, int t, int nt) {
  const int head = mis ? 16 - mis : 0;
  const int h = (int)min((int64_t)head, nbytes);
  for (int i = t; i < h; i += nt) g[i] = st[mis + i];
  const int64_t body = (nbytes - h) / 16;
  for (int64_t i = t; i < body; i += nt)
    __stcs(reinterpret_cast<uint4*>(g + h) + i, *reinterpret_cast<const uint4*>(st + mis + h + i * 16));
  for (int64_t i = h + body * 16 + t; i < nbytes; i += nt) g[i] = st[mis + i];
}

// deterministic sum of every thread's red_acc into red_ws[1]: warp tree, CTA
// tree, the last CTA sums the CTA partials in index order (red_ws layout:
// [arrival counter, result, CTA partials]; the counter is re-armed)
__device__ __forceinline__ void red_finish(double red_acc, double* __restrict__ red_ws,
                                           double* __restrict__ out = nullptr) {
  for (int o = 16; o > 0; o >>= 1) red_acc += __shfl_xor_sync(0xffffffffu, red_acc, o);
  __shared__ double wsum[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = red_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += wsum[i];
    red_ws[2 + blockIdx.x] = s;
    last = ticket_arrive(reinterpret_cast<unsigned int*>(red_ws)) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)gridDim.x; ++i) s += __ldcg(red_ws + 2 + i);
    red_ws[1] = s;
    if (out) *out = s;
    *reinterpret_cast<unsigned int*>(red_ws) = 0u;  // re-arm
  }
}

}  // namespace bz
