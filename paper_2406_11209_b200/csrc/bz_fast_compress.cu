// bz_fast_compress.cu -- fused compress: load -> transform -> max -> bin -> prune -> store.
//
// One pass over HBM: each input element is read once (16-byte vectors), each
// index and maximum written once.  Replaces convert_precision/block/
// forward_transform/bin_coefficients/prune_and_flatten (codec.py:321-334).
//
// Binning: v = C * (r / N) is rounded once by an FMA against a magic
// constant 1.5*2^(52-K), which leaves v in K-bit fixed point in the low word;
// an integer shift gives round(v).  Coefficients whose fixed-point fraction
// lies within W units of one half redo the reference's exact
// rint(fl(C / N) * r) (codec.py:272-277), so the fast path rounds exactly as
// the reference would on the same coefficient.  Blocks whose maximum is not
// finite, whose stored maximum is 0 / tiny, or whose stored maximum rounds far
// below the true maximum are appended to a list and recomputed by the exact
// generic kernel (bz_generic.cu) in reference order.
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

// exact reference binning, out of line: reached for ~1e-5 of coefficients
__device__ __noinline__ int bin_exact_call(double c, double n, double r) {
  return (int)bin_exact(c, n, r, r);
}

template <typename IT>
__device__ __forceinline__ int bin_one(double c, double R, double n, double rr) {
  bool near = false;
  int q = fast_index<IT>(c, R, rr, near);
  if (near) q = bin_exact_call(c, n, rr);
  return q;
}

template <int D, int E, int FAM, typename TIn, int FK, typename IT>
__global__ void __launch_bounds__(Tile<D, E>::NT)
k_fast_compress(FastGeo f, const TIn* __restrict__ x, void* __restrict__ maxima,
                IT* __restrict__ indices, int32_t* special_count, int32_t* special_list) {
  using TL = Tile<D, E>;
  constexpr int NIN = TL::NIN, TB = TL::TB, M = TL::M, BPC = TL::BPC, NT = TL::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);  // exchange: NT*NIN doubles (EXCH only)
  unsigned long long* red = reinterpret_cast<unsigned long long*>(
      smem_raw + (TL::EXCH ? (size_t)NT * NIN * sizeof(double) : 0));  // NT keys
  unsigned char* stage = smem_raw;  // output staging, reuses the exchange area

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  constexpr int SWZ = NIN >= 16 ? 15 : 0;
  const bool stage_out = TL::EXCH || !f.full_mask;

  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)BPC, f.nblocks - b0);

    // ---- load the thread's plane (rows along axis D-2, columns along D-1)
    double v[NIN];
    {
      int64_t off = 0, gc[4];
      bool interior = false, pvalid = false;
      if (valid) plane_origin<D, E>(f, b, o, off, interior, pvalid, gc);
      constexpr int ROWS = D >= 2 ? E : 1;
      constexpr int RA = D >= 2 ? D - 2 : 0;  // row axis
      const int64_t rs = D >= 2 ? f.stride[RA] : 0;
      if (valid && pvalid && interior && row_vectorizable<TIn>(E) && f.vec_in) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          if constexpr (row_vectorizable<TIn>(E)) load_row_vec<TIn, E>(x + off + r * rs, v + r * E);
        }
      } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
#pragma unroll
          for (int cc = 0; cc < E; ++cc) {
            bool in = valid && pvalid;
            if (D >= 2) in = in && (gc[RA] * E + r < f.shape[RA]);
            in = in && (gc[D - 1] * E + cc < f.shape[D - 1]);
            v[r * E + cc] = in ? widen(x[off + r * rs + cc]) : 0.0;
          }
        }
      }
    }

    // ---- transform the plane in registers
    if constexpr (D == 1) fline<FAM, E, 1>(v);
    else plane<FAM, E, false>(v);

    // ---- exchange: each thread gets M plane positions for all TB outer positions
    double u[NIN];
    if constexpr (TL::EXCH) {
      const int row = lb * TB + o;
#pragma unroll
      for (int p = 0; p < NIN; ++p) xs[row * NIN + (p ^ (lb & SWZ))] = v[p];
      __syncthreads();
#pragma unroll
      for (int o2 = 0; o2 < TB; ++o2)
#pragma unroll
        for (int m = 0; m < M; ++m)
          u[o2 * M + m] = xs[(lb * TB + o2) * NIN + ((o * M + m) ^ (lb & SWZ))];
      // outer transform
      if constexpr (D == 3) {
#pragma unroll
        for (int m = 0; m < M; ++m) fline<FAM, E, M>(u + m);
      } else {
        plane<FAM, E, false>(u);
      }
    } else {
#pragma unroll
      for (int p = 0; p < NIN; ++p) u[p] = v[p];
    }

    // ---- block maximum of |C| (bit-pattern order: NaN > inf > finite)
    unsigned long long key = 0;
#pragma unroll
    for (int p = 0; p < NIN; ++p) {
      unsigned long long k2 = abs_key(u[p]);
      key = k2 > key ? k2 : key;
    }
    if constexpr (TB > 1) {
      red[lb * TB + o] = key;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < TB; ++j) {
        unsigned long long k2 = red[lb * TB + j];
        key = k2 > key ? k2 : key;
      }
    }
    const double mx = __longlong_as_double((long long)key);
    const double n = round_to_kind<FK>(mx);
    const bool special = !(mx <= 1.7976931348623157e308) || !(n >= 0x1p-1000) ||
                         (mx > n * 1.00390625);
    const double R = special ? 0.0 : __ddiv_rn(rr, n);

    // ---- bin + store (kept indices, row-major intrablock order)
    if (valid && o == 0) {
      store_kind<FK>(maxima, b, n);
      if (special) special_list[atomicAdd(special_count, 1)] = (int32_t)b;
    }
    if (!stage_out) {
      if (valid) {
        IT* dst = indices + b * (int64_t)NIN;
        if constexpr ((NIN * sizeof(IT)) % 16 == 0) {
          constexpr int PER = 16 / sizeof(IT);
#pragma unroll
          for (int c = 0; c < NIN / PER; ++c) {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int e = 0; e < PER; ++e) {
              const int qv = special ? 0 : bin_one<IT>(u[c * PER + e], R, n, rr);
              const uint32_t bits = (uint32_t)qv & (sizeof(IT) == 4 ? 0xffffffffu : ((1u << (8 * sizeof(IT))) - 1));
              w[(e * sizeof(IT)) / 4] |= bits << ((e * sizeof(IT) * 8) % 32);
            }
            __stcs(reinterpret_cast<uint4*>(dst) + c, make_uint4(w[0], w[1], w[2], w[3]));
          }
        } else {
#pragma unroll
          for (int p = 0; p < NIN; ++p) dst[p] = (IT)(special ? 0 : bin_one<IT>(u[p], R, n, rr));
        }
      }
    } else {
      // stage the tile's kept indices in shared memory (the exchange area is
      // free: every thread passed the max-reduction barrier), then stream out
      const int64_t dst_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + dst_byte0) & 15);
      IT* st = reinterpret_cast<IT*>(stage + mis);
      if (valid) {
#pragma unroll
        for (int o2 = 0; o2 < TB; ++o2)
#pragma unroll
          for (int m = 0; m < M; ++m) {
            const int pos = TL::EXCH ? o2 * NIN + o * M + m : m;
            const int rk = f.full_mask ? pos : f.rank[pos];
            if (rk >= 0) st[lb * f.kept + rk] = (IT)(special ? 0 : bin_one<IT>(u[o2 * M + m], R, n, rr));
          }
      }
      __syncthreads();
      const int64_t nbytes = (int64_t)nvalid * f.kept * sizeof(IT);
      unsigned char* gdst = reinterpret_cast<unsigned char*>(indices) + dst_byte0;
      const int head = mis ? 16 - mis : 0;
      const int h = (int)min((int64_t)head, nbytes);
      for (int i = t; i < h; i += NT) gdst[i] = stage[mis + i];
      const int64_t body = (nbytes - h) / 16;
      for (int64_t i = t; i < body; i += NT)
        __stcs(reinterpret_cast<uint4*>(gdst + h) + i,
               *reinterpret_cast<const uint4*>(stage + mis + h + i * 16));
      for (int64_t i = h + body * 16 + t; i < nbytes; i += NT) gdst[i] = stage[mis + i];
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------- dispatch --
template <int D, int E, int FAM, typename TIn, int FK, typename IT>
static int launch_one(const Geo& g, const void* x, void* maxima, void* indices, int32_t* cnt,
                      int32_t* list, cudaStream_t s) {
  using TL = Tile<D, E>;
  FastGeo f = make_fast_geo(g, TL::BPC, x, sizeof(TIn));
  size_t smem = TL::EXCH ? (size_t)TL::NT * TL::NIN * sizeof(double) + TL::NT * 8
                         : (f.full_mask ? 0 : (size_t)TL::BPC * g.kept * sizeof(IT) + 16);
  if (TL::EXCH) smem = std::max(smem, (size_t)TL::BPC * g.kept * sizeof(IT) + 16 + TL::NT * 8);
  auto kern = k_fast_compress<D, E, FAM, TIn, FK, IT>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TL::NT, smem);
  if (occ < 1) occ = 1;
  int64_t grid = std::min<int64_t>(f.ntiles, (int64_t)kSMs * occ);
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, TL::NT, smem, s>>>(f, reinterpret_cast<const TIn*>(x), maxima,
                                       reinterpret_cast<IT*>(indices), cnt, list);
  return check_launch("fast_compress");
}

template <int D, int E, int FAM>
static int dispatch_kinds(const Geo& g, const void* x, void* maxima, void* indices, int32_t* cnt,
                          int32_t* list, cudaStream_t s) {
#define BZ_IDX(TIN, FKV)                                                                      \
  switch (g.index_kind) {                                                                     \
    case BZ_I8: return launch_one<D, E, FAM, TIN, FKV, int8_t>(g, x, maxima, indices, cnt, list, s);   \
    case BZ_I16: return launch_one<D, E, FAM, TIN, FKV, int16_t>(g, x, maxima, indices, cnt, list, s); \
    case BZ_I32: return launch_one<D, E, FAM, TIN, FKV, int32_t>(g, x, maxima, indices, cnt, list, s); \
  }
  if (g.float_kind == BZ_F32) { BZ_IDX(float, BZ_F32) }
  if (g.float_kind == BZ_F64) { BZ_IDX(double, BZ_F64) }
#undef BZ_IDX
  set_error("fast compress: unsupported kinds");
  return BZ_E_UNSUPPORTED;
}

static bool uniform_block(const Geo& g, int& E) {
  E = g.block[0];
  for (int a = 1; a < g.ndim; ++a)
    if (g.block[a] != E) return false;
  return true;
}

bool fast_supported(const Geo& g, int x_kind) {
  int E;
  if (!uniform_block(g, E)) return false;
  if (x_kind != g.float_kind) return false;
  if (g.float_kind != BZ_F32 && g.float_kind != BZ_F64) return false;
  if (g.index_kind == BZ_I64) return false;
  if (g.ndim < 1 || g.ndim > 4) return false;
  if (g.bsize * 8 > 4096) return false;
  switch (g.ndim) {
    case 1: return E == 4 || E == 8;
    case 2: return E == 4 || E == 8;
    case 3: return E == 4 || E == 8;
    case 4: return E == 4;
  }
  return false;
}

int launch_fast_compress(const Geo& g, const void* x, void* maxima, void* indices,
                         int32_t* cnt, int32_t* list, cudaStream_t s) {
  int E;
  uniform_block(g, E);
  const bool haar = g.transform == BZ_HAAR;
#define BZ_CASE(DD, EE)                                                                     \
  if (g.ndim == DD && E == EE)                                                              \
    return haar ? dispatch_kinds<DD, EE, HAAR>(g, x, maxima, indices, cnt, list, s)         \
                : dispatch_kinds<DD, EE, DCT>(g, x, maxima, indices, cnt, list, s);
  BZ_CASE(1, 4) BZ_CASE(1, 8) BZ_CASE(2, 4) BZ_CASE(2, 8) BZ_CASE(3, 4) BZ_CASE(3, 8)
  BZ_CASE(4, 4)
#undef BZ_CASE
  set_error("fast compress: unsupported block shape");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
