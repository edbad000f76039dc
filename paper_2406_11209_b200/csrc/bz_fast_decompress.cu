// bz_fast_decompress.cu -- fused decompress: indices -> inverse transform ->
// *N / r -> merge + crop, one pass (codec.py:364-384, arrays.py:181-190).
//
// Arithmetic follows the reference order: the inverse transform runs on the
// raw integer indices and the block scale is applied after it as
// fl(fl(y * N) / r) (codec.py:377-379).  The division by the constant r uses
// Markstein's FMA correction (bz_common.cuh: div_const), which returns the
// correctly rounded quotient; blocks whose N could push y*N out of the normal
// range fall back to IEEE division.
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

template <typename IT, int N>
__device__ __forceinline__ void load_indices_vec(const IT* __restrict__ src, double* dst) {
  static_assert((N * sizeof(IT)) % 16 == 0, "whole 16-byte chunks");
#pragma unroll
  for (int c = 0; c < N * (int)sizeof(IT) / 16; ++c) {
    uint4 w = __ldg(reinterpret_cast<const uint4*>(src) + c);
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

template <int D, int E, int FAM, typename IT, int FK, typename TOut>
__global__ void __launch_bounds__(Tile<D, E>::NT)
k_fast_decompress(FastGeo f, const void* __restrict__ maxima, const IT* __restrict__ indices,
                  TOut* __restrict__ out) {
  using TL = Tile<D, E>;
  constexpr int NIN = TL::NIN, TB = TL::TB, M = TL::M, BPC = TL::BPC, NT = TL::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);
  unsigned char* stage = smem_raw;

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const double rinv = 1.0 / rr;
  const double nsafe = 1.7976931348623157e308 / (rr * TL::BS * 4.0);
  constexpr int SWZ = NIN >= 16 ? 15 : 0;
  const bool stage_in = TL::EXCH || !f.full_mask;

  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)BPC, f.nblocks - b0);

    // ---- gather this thread's coefficients (as f64 integers)
    double u[NIN];
    if (stage_in) {
      const int64_t src_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + src_byte0) & 15);
      const unsigned char* gsrc = reinterpret_cast<const unsigned char*>(indices) + src_byte0;
      const int64_t nbytes = (int64_t)nvalid * f.kept * sizeof(IT);
      const int head = mis ? 16 - mis : 0;
      const int h = (int)min((int64_t)head, nbytes);
      for (int i = t; i < h; i += NT) stage[mis + i] = gsrc[i];
      const int64_t body = (nbytes - h) / 16;
      for (int64_t i = t; i < body; i += NT)
        *reinterpret_cast<uint4*>(stage + mis + h + i * 16) =
            __ldg(reinterpret_cast<const uint4*>(gsrc + h) + i);
      for (int64_t i = h + body * 16 + t; i < nbytes; i += NT) stage[mis + i] = gsrc[i];
      __syncthreads();
      const IT* st = reinterpret_cast<const IT*>(stage + mis);
#pragma unroll
      for (int o2 = 0; o2 < TB; ++o2)
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int pos = TL::EXCH ? o2 * NIN + o * M + m : m;
          const int rk = f.full_mask ? pos : f.rank[pos];
          u[o2 * M + m] = (valid && rk >= 0) ? (double)st[lb * f.kept + rk] : 0.0;
        }
      __syncthreads();  // staging area becomes the exchange area
    } else {
      if (valid) {
        if constexpr ((NIN * sizeof(IT)) % 16 == 0) {
          load_indices_vec<IT, NIN>(indices + b * (int64_t)NIN, u);
        } else {
#pragma unroll
          for (int p = 0; p < NIN; ++p) u[p] = (double)indices[b * (int64_t)NIN + p];
        }
      } else {
#pragma unroll
        for (int p = 0; p < NIN; ++p) u[p] = 0.0;
      }
    }

    // ---- inverse outer transform + exchange back to planes
    double v[NIN];
    if constexpr (TL::EXCH) {
      if constexpr (D == 3) {
#pragma unroll
        for (int m = 0; m < M; ++m) iline<FAM, E, M>(u + m);
      } else {
        plane<FAM, E, true>(u);
      }
#pragma unroll
      for (int o2 = 0; o2 < TB; ++o2)
#pragma unroll
        for (int m = 0; m < M; ++m)
          xs[(lb * TB + o2) * NIN + ((o * M + m) ^ (lb & SWZ))] = u[o2 * M + m];
      __syncthreads();
      const int row = lb * TB + o;
#pragma unroll
      for (int p = 0; p < NIN; ++p) v[p] = xs[row * NIN + (p ^ (lb & SWZ))];
    } else {
#pragma unroll
      for (int p = 0; p < NIN; ++p) v[p] = u[p];
    }
    if constexpr (D == 1) iline<FAM, E, 1>(v);
    else plane<FAM, E, true>(v);

    // ---- scale: ((y * N) / r), reference order
    if (valid) {
      const double n = load_kind<FK>(maxima, b);
      const bool safe = (n >= 0x1p-900) && (n <= nsafe);
      if (safe) {
#pragma unroll
        for (int p = 0; p < NIN; ++p) v[p] = div_const(__dmul_rn(v[p], n), rr, rinv);
      } else {
#pragma unroll
        for (int p = 0; p < NIN; ++p) v[p] = __ddiv_rn(__dmul_rn(v[p], n), rr);
      }
      if constexpr (sizeof(TOut) == 4) {
#pragma unroll
        for (int p = 0; p < NIN; ++p) v[p] = (double)__double2float_rn(v[p]);
      }

      // ---- store the plane
      int64_t off = 0, gc[4];
      bool interior = false, pvalid = false;
      plane_origin<D, E>(f, b, o, off, interior, pvalid, gc);
      constexpr int ROWS = D >= 2 ? E : 1;
      constexpr int RA = D >= 2 ? D - 2 : 0;
      const int64_t rs = D >= 2 ? f.stride[RA] : 0;
      if (pvalid) {
        if (interior && row_vectorizable<TOut>(E) && f.vec_in) {
#pragma unroll
          for (int r = 0; r < ROWS; ++r) {
            if constexpr (row_vectorizable<TOut>(E)) store_row_vec<TOut, E>(out + off + r * rs, v + r * E);
          }
        } else {
#pragma unroll
          for (int r = 0; r < ROWS; ++r) {
#pragma unroll
            for (int cc = 0; cc < E; ++cc) {
              bool in = true;
              if (D >= 2) in = gc[RA] * E + r < f.shape[RA];
              in = in && (gc[D - 1] * E + cc < f.shape[D - 1]);
              if (in) out[off + r * rs + cc] = (TOut)v[r * E + cc];
            }
          }
        }
      }
    }
    if constexpr (TL::EXCH) __syncthreads();  // exchange area reused by the next tile
  }
}

template <int D, int E, int FAM, typename IT, int FK, typename TOut>
static int launch_one(const Geo& g, const void* maxima, const void* indices, void* out,
                      cudaStream_t s) {
  using TL = Tile<D, E>;
  FastGeo f = make_fast_geo(g, TL::BPC, out, sizeof(TOut));
  size_t smem = 0;
  if (TL::EXCH) smem = (size_t)TL::NT * TL::NIN * sizeof(double);
  if (TL::EXCH || !f.full_mask) smem = std::max(smem, (size_t)TL::BPC * g.kept * sizeof(IT) + 16);
  auto kern = k_fast_decompress<D, E, FAM, IT, FK, TOut>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TL::NT, smem);
  if (occ < 1) occ = 1;
  int64_t grid = std::min<int64_t>(f.ntiles, (int64_t)kSMs * occ);
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, TL::NT, smem, s>>>(f, maxima, reinterpret_cast<const IT*>(indices),
                                       reinterpret_cast<TOut*>(out));
  return check_launch("fast_decompress");
}

template <int D, int E, int FAM>
static int dispatch_kinds(const Geo& g, const void* maxima, const void* indices, void* out,
                          int out_kind, cudaStream_t s) {
#define BZ_OUT(IT, FKV)                                                                   \
  if (out_kind == BZ_F64) return launch_one<D, E, FAM, IT, FKV, double>(g, maxima, indices, out, s); \
  if (out_kind == BZ_F32) return launch_one<D, E, FAM, IT, FKV, float>(g, maxima, indices, out, s);
#define BZ_IDX(FKV)                                    \
  switch (g.index_kind) {                              \
    case BZ_I8: { BZ_OUT(int8_t, FKV) break; }         \
    case BZ_I16: { BZ_OUT(int16_t, FKV) break; }       \
    case BZ_I32: { BZ_OUT(int32_t, FKV) break; }       \
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
  const bool haar = g.transform == BZ_HAAR;
#define BZ_CASE(DD, EE)                                                                   \
  if (g.ndim == DD && E == EE)                                                            \
    return haar ? dispatch_kinds<DD, EE, HAAR>(g, maxima, indices, out, out_kind, s)      \
                : dispatch_kinds<DD, EE, DCT>(g, maxima, indices, out, out_kind, s);
  BZ_CASE(1, 4) BZ_CASE(1, 8) BZ_CASE(2, 4) BZ_CASE(2, 8) BZ_CASE(3, 4) BZ_CASE(3, 8)
  BZ_CASE(4, 4)
#undef BZ_CASE
  set_error("fast decompress: unsupported block shape");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
