// bz_fast.cuh -- shared pieces of the fused compress / decompress kernels.
//
// Work decomposition ("register planes"), for a block of E^D elements:
//   * D <= 2: one thread owns a whole block (E or E*E values in registers).
//   * D = 3, 4: TB = E^(D-2) threads own one block; thread o holds the E x E
//     plane of the two fastest axes at outer position o.  The fast-axis and
//     row transforms run in registers; one shared-memory exchange hands each
//     thread all outer positions of E*E/TB plane coefficients, and the outer
//     transform runs in registers again.  No f64 value touches shared memory
//     more than once per direction.
// Threads are laid out outer-major (t = o * BPC + lb), so consecutive lanes
// hold consecutive blocks along the fastest grid axis and every global row
// access is a run of contiguous 16-byte vectors.
#pragma once

#include "bz_common.cuh"
#include "bz_transforms.cuh"

namespace bz {

constexpr int ipow(int b, int e) { return e <= 0 ? 1 : b * ipow(b, e - 1); }

template <int D, int E>
struct Tile {
  static constexpr int TB = D >= 3 ? ipow(E, D - 2) : 1;  // threads per block
  static constexpr int NIN = D >= 2 ? E * E : E;          // values per thread
  static constexpr int M = NIN / TB;                      // plane positions per thread after exchange
  static constexpr int BS = ipow(E, D);                   // block size
  static constexpr int NT = NIN >= 64 ? 128 : 256;        // threads per CTA
  static constexpr int BPC = NT / TB;                     // blocks per CTA tile
  static constexpr bool EXCH = D >= 3;
};

struct FastGeo {
  int64_t shape[4];
  int64_t grid[4];
  int64_t stride[4];
  int64_t nblocks;
  int64_t ntiles;
  int32_t kept;
  int32_t full_mask;
  int32_t vec_in;    // 16-byte vector access legal on the dense side
  const int32_t* rank;
  const int32_t* kept_pos;
};

inline FastGeo make_fast_geo(const Geo& g, int bpc, const void* dense, int dense_bytes) {
  FastGeo f{};
  for (int a = 0; a < g.ndim; ++a) {
    f.shape[a] = g.shape[a];
    f.grid[a] = g.grid[a];
    f.stride[a] = g.stride[a];
  }
  f.nblocks = g.nblocks;
  f.ntiles = (g.nblocks + bpc - 1) / bpc;
  f.kept = g.kept;
  f.full_mask = g.kept == g.bsize;
  f.rank = g.rank;
  f.kept_pos = g.kept_pos;
  int E = g.block[g.ndim - 1];
  bool ok = ((uintptr_t)dense % 16 == 0) && ((E * dense_bytes) % 16 == 0);
  if (g.ndim >= 2) ok = ok && ((g.stride[g.ndim - 2] * dense_bytes) % 16 == 0);
  f.vec_in = ok;
  return f;
}

// decode block id -> block coordinates; returns the dense offset of the
// thread's plane origin (outer intra coords from o) and whether the plane
// lies fully inside the array.  `plane_valid` = false when the outer intra
// coordinate itself is padding (the plane is all zeros).
template <int D, int E>
__device__ __forceinline__ void plane_origin(const FastGeo& f, int64_t b, int o, int64_t& off,
                                             bool& interior, bool& plane_valid,
                                             int64_t (&gc)[4]) {
  int64_t rem = b;
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    gc[a] = rem % f.grid[a];
    rem /= f.grid[a];
  }
  off = 0;
  interior = true;
  plane_valid = true;
  // outer axes 0..D-3 carry the thread's intra coordinate
  int orem = o;
  int ncoord[4] = {0, 0, 0, 0};
#pragma unroll
  for (int a = D - 3; a >= 0; --a) {
    ncoord[a] = orem % E;
    orem /= E;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int64_t c0 = gc[a] * E;
    if (a < D - 2) {
      int64_t c = c0 + ncoord[a];
      if (c >= f.shape[a]) plane_valid = false;
      off += c * f.stride[a];
    } else {
      off += c0 * f.stride[a];
      if (c0 + E > f.shape[a]) interior = false;
    }
  }
}

// ------------------------------------------------ vector row load / store --
template <typename T, int E>
__device__ __forceinline__ void load_row_vec(const T* __restrict__ src, double* dst) {
  constexpr int CH = 16 / sizeof(T);
  static_assert(E % CH == 0, "row must be a whole number of 16-byte chunks");
#pragma unroll
  for (int c = 0; c < E / CH; ++c) {
    uint4 w = __ldg(reinterpret_cast<const uint4*>(src) + c);
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
constexpr bool row_vectorizable(int E) { return (E * (int)sizeof(T)) % 16 == 0; }

// |x| as an ordered unsigned key: NaN > inf > finite
__device__ __forceinline__ unsigned long long abs_key(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

}  // namespace bz
