// bz_fast_compress.cu -- fused compress: load -> transform -> max -> bin -> prune -> store.
//
// One pass over HBM: each input element is read once (16-byte vectors), each
// index and maximum written once.  Replaces convert_precision/block/
// forward_transform/bin_coefficients/prune_and_flatten (codec.py:321-334).
// The transform is the reference's own FMA chain (bz_fast.cuh), so the
// coefficients are bit-identical to the reference's.
//
// Binning: v = C * (r / N) is rounded once by an FMA against a magic
// constant 1.5*2^(52-K), leaving v in K-bit fixed point in the low word; an
// integer shift gives round(v).  Coefficients whose fixed-point fraction lies
// within W units of one half redo the reference's exact rint(fl(C / N) * r)
// (codec.py:272-277), so every index equals the reference's.  Blocks whose
// maximum is not finite, whose stored maximum is 0 / tiny, or whose stored
// maximum rounds far below the true maximum bin every coefficient with the
// exact reference arithmetic (their coefficients already are the reference's).
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

#include <cstdlib>

namespace bz {

// exact reference binning, out of line: reached for ~1e-5 of coefficients
// and for every coefficient of a "special" block
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

template <typename IT>
__device__ __forceinline__ uint32_t idx_bits(int q) {
  return (uint32_t)q & (sizeof(IT) == 4 ? 0xffffffffu : ((1u << (8 * sizeof(IT))) - 1));
}

// PREFETCH: stream the next tile's rows into a per-thread shared-memory stage
// with cp.async while the current tile computes.  Measured slower than direct
// 16-byte loads on B200 for these kernels (C2: 183 vs 121 us), so it is off.
template <int D, int E, typename TIn, int FK, typename IT, bool PREFETCH = false>
__global__ void __launch_bounds__(Tile<D, E>::NT)
k_fast_compress(const FastParams p, const TIn* __restrict__ x, void* __restrict__ maxima,
                IT* __restrict__ indices, IT* __restrict__ dc) {
  using TL = Tile<D, E>;
  constexpr int NIN = TL::NIN, TB = TL::TB, BS = TL::BS, BPC = TL::BPC, NT = TL::NT;
  constexpr int LP = 0, LQ = D - 1;  // loaded slice axes
  const FastGeo& f = p.f;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* xs = reinterpret_cast<double*>(smem_raw);                      // BPC*BS doubles
  unsigned long long* red = reinterpret_cast<unsigned long long*>(
      smem_raw + (TL::EXCH ? (size_t)BPC * BS * sizeof(double) : 0));   // NT keys
  unsigned char* stage = reinterpret_cast<unsigned char*>(red + (TB > 1 ? NT : 0));

  const int t = threadIdx.x;
  const int lb = t % BPC;
  const int o = t / BPC;
  const double rr = radius_f64(sizeof(IT) == 1 ? BZ_I8 : (sizeof(IT) == 2 ? BZ_I16 : BZ_I32));
  const int swz = slot_swizzle(lb);
  double* blk = xs + lb * BS;

  // per-thread private prefetch stage: the next tile's slice rows arrive by
  // cp.async while the current tile computes (interleaved by thread, so the
  // 16-byte reads are bank-conflict free)
  constexpr int ROWS = D >= 2 ? E : 1;
  constexpr bool VEC = row_vectorizable<TIn>(E);
  constexpr int RU = VEC ? E * (int)sizeof(TIn) / 16 : 1;  // 16-byte units per row
  const size_t stage_sz = f.full_mask ? 0 : ((size_t)BPC * f.kept * sizeof(IT) + 16 + 15) / 16 * 16;
  // rank table (position -> kept rank) in shared memory for pruned masks
  int16_t* rks = reinterpret_cast<int16_t*>(stage + stage_sz);
  if (!f.full_mask) {
    for (int i = threadIdx.x; i < BS; i += NT) rks[i] = (int16_t)f.rank[i];
    __syncthreads();
  }
  uint4* pstage = reinterpret_cast<uint4*>(stage + stage_sz + (f.full_mask ? 0 : ((size_t)BS * 2 + 15) / 16 * 16));
  int c[4];
  slice_coords<D, E, LP, LQ>(o, c);
  const int64_t rs = f.stride[0];

  // geometry of this thread's slice in `tile`; true when the slice is a run
  // of whole, aligned, in-bounds 16-byte rows
  auto geom = [&](int64_t tile, int64_t& off, bool& fixed_ok, int& rows_ok, int& cols_ok) {
    const int64_t b = tile * BPC + lb;
    off = 0;
    fixed_ok = false;
    rows_ok = cols_ok = 0;
    if (tile >= f.ntiles || b >= f.nblocks) return false;
    int64_t gc[4] = {0, 0, 0, 0};
    block_coords<D>(f, b, gc);
    bool interior;
    off = dense_slice_origin<D, E, LP>(f, gc, c, interior, fixed_ok, rows_ok, cols_ok);
    return VEC && fixed_ok && interior && f.vec_dense;
  };
  auto prefetch = [&](int64_t tile) {
    int64_t off;
    bool fok;
    int ro, co;
    const bool fast = PREFETCH && geom(tile, off, fok, ro, co);
    if (fast) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int u = 0; u < RU; ++u)
          cp_async16(pstage + (r * RU + u) * NT + t, x + off + r * rs + u * (16 / sizeof(TIn)));
    }
    cp_async_commit();
    return fast;
  };

  bool pf = prefetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < f.ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * BPC;
    const int64_t b = b0 + lb;
    const bool valid = b < f.nblocks;
    const int nvalid = (int)min((int64_t)BPC, f.nblocks - b0);

    // ---- slice (axis 0, axis D-1) at fixed coords o: from the stage, or
    //      direct guarded loads for partial / unaligned blocks
    double v[NIN];
    int64_t off0;
    bool fok0;
    int ro0, co0;
    const bool direct = !pf && geom(tile, off0, fok0, ro0, co0);
    if (direct) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        if constexpr (VEC) load_row_vec<TIn, E>(x + off0 + r * rs, v + r * E);
      }
    } else if (pf) {
      cp_async_wait_all();
      uint4 w[ROWS * RU];
#pragma unroll
      for (int k = 0; k < ROWS * RU; ++k) w[k] = pstage[k * NT + t];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) unpack_row<TIn>(w + r * RU, v + r * E, RU);
    } else {
      int64_t off;
      bool fok;
      int ro, co;
      geom(tile, off, fok, ro, co);
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int cc = 0; cc < E; ++cc)
          v[r * E + cc] = (valid && fok && r < ro && cc < co) ? widen(x[off + r * rs + cc]) : 0.0;
    }
    pf = prefetch(tile + gridDim.x);  // stage reads above have completed (values in use)

    // ---- forward transform, axis 0 first (reference order)
    if constexpr (D == 1) {
      dense_line<E, 1, false>(v, p.H);
    } else if constexpr (D == 2) {
      slice_cols<E, false>(v, p.H);  // axis 0
      slice_rows<E, false>(v, p.H);  // axis 1
    } else if constexpr (D == 3) {
      slice_cols<E, false>(v, p.H);  // axis 0
      slice_store<D, E, 0, 2>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 1, 2>(blk, swz, o, v);
      slice_cols<E, false>(v, p.H);  // axis 1
      slice_rows<E, false>(v, p.H);  // axis 2
    } else {
      slice_cols<E, false>(v, p.H);  // axis 0
      slice_store<D, E, 0, 3>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 1, 2>(blk, swz, o, v);
      slice_cols<E, false>(v, p.H);  // axis 1
      slice_rows<E, false>(v, p.H);  // axis 2
      __syncthreads();
      slice_store<D, E, 1, 2>(blk, swz, o, v);
      __syncthreads();
      slice_load<D, E, 2, 3>(blk, swz, o, v);
      slice_rows<E, false>(v, p.H);  // axis 3
    }
    // thread o now holds canonical positions [o*NIN, (o+1)*NIN) of block b

    // ---- block maximum of |C| (bit-pattern order: NaN > inf > finite)
    unsigned long long key = 0;
#pragma unroll
    for (int q = 0; q < NIN; ++q) {
      unsigned long long k2 = abs_key(v[q]);
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
    constexpr bool CLAMP = !(FK == BZ_F32 || FK == BZ_F64);
    const BinCtx bc = bin_ctx<CLAMP>(n, rr, mx);
    if (valid && o == 0) store_kind<FK>(maxima, b, n);
    // v <= r(1+2^-24) for F32/F64 maxima: rounding cannot exceed r
        const int ir = (int)rr;
    // exact reference index of coefficient q (near-half fraction / non-fast block)
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

    // ---- bin + store kept indices
    if (f.full_mask) {
      if (valid) {
        IT* dst = indices + b * (int64_t)BS + o * NIN;
        if constexpr ((NIN * sizeof(IT)) % 16 == 0 && sizeof(IT) <= 2) {
          constexpr int PER = 16 / sizeof(IT);
#pragma unroll
          for (int cch = 0; cch < NIN / PER; ++cch) {
            int q[PER];
            unsigned nacc = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) q[e] = fast_index32<IT, CLAMP>(v[cch * PER + e], bc.R, ir, nacc);
            if (nacc | !bc.fast) {  // rare: exact reference arithmetic where needed
#pragma unroll
              for (int e = 0; e < PER; ++e) q[e] = bin_q(v[cch * PER + e]);
            }
            __stcs(reinterpret_cast<uint4*>(dst) + cch, pack16<IT>(q));
            if (cch == 0 && o == 0 && dc) dc[b] = (IT)q[0];  // DC plane: position 0
          }
        } else if constexpr ((NIN * sizeof(IT)) % 16 == 0) {
          constexpr int PER = 16 / sizeof(IT);
#pragma unroll
          for (int cch = 0; cch < NIN / PER; ++cch) {
            int q[PER];
#pragma unroll
            for (int e = 0; e < PER; ++e) q[e] = bin_q(v[cch * PER + e]);
            __stcs(reinterpret_cast<uint4*>(dst) + cch, pack16<IT>(q));
            if (cch == 0 && o == 0 && dc) dc[b] = (IT)q[0];
          }
        } else {
#pragma unroll
          for (int q = 0; q < NIN; ++q) {
            const IT qv = (IT)bin_q(v[q]);
            dst[q] = qv;
            if (q == 0 && o == 0 && dc) dc[b] = qv;
          }
        }
      }
    } else {
      // pruned mask: stage the tile's kept indices, then stream them out
      const int64_t dst_byte0 = b0 * (int64_t)f.kept * sizeof(IT);
      const int mis = (int)(((uintptr_t)indices + dst_byte0) & 15);
      IT* st = reinterpret_cast<IT*>(stage + mis);
      if (valid) {
#pragma unroll
        for (int q = 0; q < NIN; ++q) {
          const int rk = rks[o * NIN + q];
          if (rk >= 0) {
            const IT qv = (IT)bin_q(v[q]);
            st[lb * f.kept + rk] = qv;
            if (q == 0 && o == 0 && dc) dc[b] = qv;  // position 0 (dc only when kept)
          }
        }
      }
      __syncthreads();
      smem_to_tile(reinterpret_cast<unsigned char*>(indices) + dst_byte0, stage,
                   (int64_t)nvalid * f.kept * sizeof(IT), mis, t, NT);
    }
    if constexpr (TL::EXCH || TB > 1) {
      __syncthreads();  // smem reused by the next tile
    } else {
      if (!f.full_mask) __syncthreads();
    }
  }
}

// ----------------------------------------------------------------- dispatch --
template <int D, int E, typename TIn, int FK, typename IT>
static int launch_one(const Geo& g, const void* x, void* maxima, void* indices, void* dc,
                      cudaStream_t s) {
  using TL = Tile<D, E>;
  FastParams p;
  if (!make_fast_params(g, TL::BPC, x, sizeof(TIn), p)) {
    set_error("fast compress: host matrices missing");
    return BZ_E_INVALID;
  }
  constexpr int ROWS = D >= 2 ? E : 1;
  constexpr int RU = row_vectorizable<TIn>(E) ? E * (int)sizeof(TIn) / 16 : 1;
  size_t smem = (TL::EXCH ? (size_t)TL::BPC * TL::BS * sizeof(double) : 0) +
                (TL::TB > 1 ? (size_t)TL::NT * 8 : 0) +
                (p.f.full_mask ? 0 : ((size_t)TL::BPC * g.kept * sizeof(IT) + 16 + 15) / 16 * 16 +
                                     ((size_t)TL::BS * 2 + 15) / 16 * 16) +
                0 * (size_t)TL::NT * ROWS * RU * 16;  // PREFETCH stage (disabled)
  auto kern = k_fast_compress<D, E, TIn, FK, IT>;
  const int occ = occupancy((const void*)kern, TL::NT, smem);
  int64_t grid = std::min<int64_t>(p.f.ntiles, (int64_t)kSMs * occ);
  if (grid < 1) return BZ_OK;
  kern<<<(int)grid, TL::NT, smem, s>>>(p, reinterpret_cast<const TIn*>(x), maxima,
                                       reinterpret_cast<IT*>(indices), reinterpret_cast<IT*>(dc));
  return check_launch("fast_compress");
}

template <int D, int E>
static int dispatch_kinds(const Geo& g, const void* x, void* maxima, void* indices, void* dc,
                          cudaStream_t s) {
#define BZ_IDX(TIN, FKV)                                                                          \
  switch (g.index_kind) {                                                                         \
    case BZ_I8: return launch_one<D, E, TIN, FKV, int8_t>(g, x, maxima, indices, dc, s);   \
    case BZ_I16: return launch_one<D, E, TIN, FKV, int16_t>(g, x, maxima, indices, dc, s); \
    case BZ_I32: return launch_one<D, E, TIN, FKV, int32_t>(g, x, maxima, indices, dc, s); \
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
  if (!g.matrices_host) return false;
  if (x_kind != g.float_kind) return false;
  if (g.float_kind != BZ_F32 && g.float_kind != BZ_F64) return false;
  if (g.index_kind == BZ_I64) return false;
  switch (g.ndim) {
    case 1: return E == 4 || E == 8;
    case 2: return E == 4 || E == 8;
    case 3: return E == 4 || E == 8;
    case 4: return E == 4;
  }
  return false;
}

int launch_fast_compress(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s,
                         void* dc, bool* dc_done) {
  int E;
  uniform_block(g, E);
  if (dc_done) *dc_done = false;
  if (g.ndim == 3 && E == 8)
    return launch_half3_compress(g, x, maxima, indices, s);
  if (dc_done) *dc_done = dc != nullptr;
#define BZ_CASE(DD, EE) \
  if (g.ndim == DD && E == EE) return dispatch_kinds<DD, EE>(g, x, maxima, indices, dc, s);
  BZ_CASE(1, 4) BZ_CASE(1, 8) BZ_CASE(2, 4) BZ_CASE(2, 8) BZ_CASE(3, 4) BZ_CASE(3, 8)
  BZ_CASE(4, 4)
#undef BZ_CASE
  set_error("fast compress: unsupported block shape");
  return BZ_E_UNSUPPORTED;
}

}  // namespace bz
