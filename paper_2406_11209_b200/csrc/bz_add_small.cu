// bz_add_small.cu -- add / subtract / add_scalar (and the fused subtract+l2
// of the time-series workflow) for int8 indices with float32 maxima and
// small blocks whose kept indices are not whole 16-byte vectors (the C5
// low-pass mask keeps K = 66), bit-exact with the reference
// (ops.py:178-215, codec.py:337-350 and 253-278; cli.py:240-243).
//
// A CTA stages tiles of TBS blocks -- both operands' indices and maxima --
// in shared memory with 16-byte cp.async copies, double buffered (the next
// tile streams in while this one computes); a group of G = 4 lanes owns a
// block, lane `sub` holding its coefficients k = sub + 4 j (j < CPL, CPL =
// ceil(K / 4) exactly, a template parameter: no dead slots), read from a
// per-lane shared address plus immediates.  Coefficients follow bz_add8.cu:
// fl(F N / r) = fma(F, t_hi, F * t_lo) for int8 F and float32 N (exact), the
// maximum is a compare-select chain, and the rebinning is the one-FMA 32-bit
// fixed point (kMagicH, bz_common.cuh) whose index is the high word's low
// byte.  A block with tiny / huge / non-finite maxima, an uncertain stored
// maximum or a coefficient within 2^-24 of a rounding half is recomputed by
// its group with the reference's IEEE operations.  Results go back through
// the staged tile (one contiguous 16-byte store stream); the RED variant
// instead sums the squared rebinned indices times N^2 (l2_norm of the
// difference) and writes no array.
#include "bz_common.cuh"
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

namespace {

// exact reference arithmetic for one block (rare): IEEE product, division,
// NaN-propagating maximum, exact binning; the group's 8 lanes cooperate
template <int G, int MODE, bool RED>
__device__ __noinline__ double small_block_exact(int kept, int sub, unsigned gmask,
                                                 const int8_t* pa, const int8_t* pb, double na,
                                                 double nb, int subtract, double shift,
                                                 int8_t* po, float* out_max, int64_t b) {
  const double r = 127.0;
  auto coeff = [&](int k) -> double {
    const double xa = __ddiv_rn(__dmul_rn((double)pa[k], na), r);
    if (MODE == 0) {
      const double fb = subtract ? -(double)pb[k] : (double)pb[k];
      return __dadd_rn(xa, __ddiv_rn(__dmul_rn(fb, nb), r));
    }
    return k == 0 ? __dadd_rn(xa, shift) : xa;
  };
  double m = 0.0;
  for (int k = sub; k < kept; k += G) m = nanmax_abs(m, coeff(k));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(gmask, m, o, G);
    m = (isnan(t) || isnan(m)) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, t);
  }
  const double n = round_to_kind<BZ_F32>(m);
  if (!RED && sub == 0) out_max[b] = (float)n;
  int sq = 0;
  for (int k = sub; k < kept; k += G) {
    const int q = (int)bin_exact(coeff(k), n, r, r);
    if (RED) sq += q * q;
    else po[k] = (int8_t)q;
  }
  return RED ? __fma_rn((double)sq * n, n, 0.0) : 0.0;
}
}  // namespace

// smem layout: two input buffers {a indices, b indices, a maxima, b maxima}
// of TB blocks each (the next tile streams in with cp.async while this one
// computes), one output tile
constexpr int TBS = 192;  // blocks per tile (a multiple of 16: TBS * K is a multiple of 16 for any K;
                          // measured at C5: 128 -> 386 us, 192 -> 369 us, 256 -> 380 us -- fewer CTA
                          // barriers per block vs 3 CTAs per SM of shared memory)

__host__ __device__ constexpr int64_t small_idx_bytes(int kept) { return (int64_t)TBS * kept; }
__host__ __device__ constexpr int64_t small_buf_bytes(int kept) {
  return 2 * small_idx_bytes(kept) + 2 * TBS * (int64_t)sizeof(float);
}

// stage tile `tile` into buffer `buf`: 16-byte cp.async chunks (all bases
// 16-byte aligned, TBS * K a multiple of 16); the ragged end of the last
// tile is copied synchronously byte by byte
template <int MODE>
__device__ __forceinline__ void small_prefetch(unsigned char* buf, int64_t tile, int64_t nblocks,
                                               int kept, const float* a_max, const int8_t* a_idx,
                                               const float* b_max, const int8_t* b_idx, int t) {
  const int64_t b0 = tile * TBS;
  const int nv = (int)min((int64_t)TBS, nblocks - b0);
  const int64_t nbytes = (int64_t)nv * kept;
  const int64_t IB = small_idx_bytes(kept);
  unsigned char* sa = buf;
  unsigned char* sb = buf + IB;
  float* sma = reinterpret_cast<float*>(buf + 2 * IB);
  float* smb = sma + TBS;
  const unsigned char* ga = reinterpret_cast<const unsigned char*>(a_idx) + b0 * (int64_t)kept;
  const unsigned char* gb = reinterpret_cast<const unsigned char*>(b_idx) + b0 * (int64_t)kept;
  const int64_t nvec = nbytes / 16;
  for (int64_t i = t; i < nvec; i += 256) {
    cp_async16(sa + i * 16, ga + i * 16);
    if (MODE == 0) cp_async16(sb + i * 16, gb + i * 16);
  }
  for (int64_t i = nvec * 16 + t; i < nbytes; i += 256) {
    sa[i] = ga[i];
    if (MODE == 0) sb[i] = gb[i];
  }
  const int mvec = nv / 4;  // 4 maxima per chunk (b0 is a multiple of 4)
  for (int i = t; i < mvec; i += 256) {
    cp_async16(sma + 4 * i, a_max + b0 + 4 * i);
    if (MODE == 0) cp_async16(smb + 4 * i, b_max + b0 + 4 * i);
  }
  for (int i = 4 * mvec + t; i < nv; i += 256) {
    sma[i] = a_max[b0 + i];
    if (MODE == 0) smb[i] = b_max[b0 + i];
  }
}

template <int G, int CPL, int MODE, bool RED>
__global__ void __launch_bounds__(256, CPL <= 24 ? 3 : 2)
k_add_small(int64_t nblocks, int kept, const float* __restrict__ a_max,
            const int8_t* __restrict__ a_idx, const float* __restrict__ b_max,
            const int8_t* __restrict__ b_idx, int subtract, double shift,
            float* __restrict__ out_max, int8_t* __restrict__ out_idx,
            int8_t* __restrict__ out_dc, double* __restrict__ red_ws,
            double* __restrict__ red_out) {
  constexpr double r = 127.0, rinv = 1.0 / 127.0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t IB = small_idx_bytes(kept), BB = (small_buf_bytes(kept) + 15) / 16 * 16;
  unsigned char* so = smem_raw + 2 * BB;
  const int t = threadIdx.x, lane = t & 31, sub = lane & (G - 1);
  const unsigned gmask = ((1u << G) - 1u) << (lane & (32 - G));
  const bool last_ok = sub + G * (CPL - 1) < kept;  // this lane's last slot holds a coefficient
  double red_acc = 0.0;
  const int64_t ntiles = (nblocks + TBS - 1) / TBS;
  int64_t tile = blockIdx.x;
  if (tile < ntiles)
    small_prefetch<MODE>(smem_raw, tile, nblocks, kept, a_max, a_idx, b_max, b_idx, t);
  cp_async_commit();
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    unsigned char* cur = smem_raw + (it & 1) * BB;
    const int64_t nxt = tile + gridDim.x;
    if (nxt < ntiles)
      small_prefetch<MODE>(smem_raw + ((it + 1) & 1) * BB, nxt, nblocks, kept, a_max, a_idx,
                           b_max, b_idx, t);
    cp_async_commit();
    cp_async_wait_1();
    __syncthreads();
    const int64_t b0 = tile * TBS;
    const int nv = (int)min((int64_t)TBS, nblocks - b0);
    const unsigned char* sa = cur;
    const unsigned char* sb = cur + IB;
    const float* sma = reinterpret_cast<const float*>(cur + 2 * IB);
    const float* smb = sma + TBS;
    // warp-uniform trip count: every lane of a warp runs every iteration (a
    // group past the tile's last block computes on stale shared bytes --
    // lb < TBS -- and stores nothing), so the group votes and shuffles are
    // full-warp (a partial-mask vote serialised the 8 groups of a warp:
    // WARPSYNC.EXCLUSIVE + 8 votes per block)
    for (int lw = (t / 32) * (32 / G); lw < nv; lw += 256 / G) {
      const int lb = lw + lane / G;
      const bool active = lb < nv;
      const int64_t b = b0 + lb;
      const int8_t* pa = reinterpret_cast<const int8_t*>(sa) + lb * kept;
      const int8_t* pb = reinterpret_cast<const int8_t*>(sb) + lb * kept;
      int8_t* po = reinterpret_cast<int8_t*>(so) + lb * kept;
      const double na = (double)sma[lb];
      const double nb = MODE == 0 ? (double)smb[lb] : 0.0;
      bool safe = na >= 0x1p-900 && na <= 0x1p+900;
      if (MODE == 0) safe = safe && nb >= 0x1p-900 && nb <= 0x1p+900;
      // t = N / r as t_hi + t_lo (bz_add8.cu)
      const double tha = div_const(na, r, rinv);
      const double tla = __fma_rn(-tha, r, na) * rinv;
      double thb = 0.0, tlb = 0.0;
      if (MODE == 0) {
        thb = div_const(nb, r, rinv);
        tlb = __fma_rn(-thb, r, nb) * rinv;
        if (subtract) { thb = -thb; tlb = -tlb; }
      }
      double c[CPL];
      double m2[2];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const bool ok = j < CPL - 1 || last_ok;
        const double fa = ok ? (double)(int)pa[sub + G * j] : 0.0;
        double cc = __fma_rn(fa, tha, fa * tla);
        if (MODE == 0) {
          const double fb = ok ? (double)(int)pb[sub + G * j] : 0.0;
          cc = __dadd_rn(cc, __fma_rn(fb, thb, fb * tlb));
        } else if (j == 0) {
          if (sub == 0) cc = __dadd_rn(cc, shift);
        }
        c[j] = cc;
        // slots past `kept` hold 0: they cannot raise the maximum (the chains
        // start from real elements -- see bz_dct8.cu)
        if (j < 2) m2[j] = cc;
        else m2[j & 1] = fabs(cc) > fabs(m2[j & 1]) ? cc : m2[j & 1];
      }
      double m = CPL > 1 ? (fabs(m2[1]) > fabs(m2[0]) ? fabs(m2[1]) : fabs(m2[0])) : fabs(m2[0]);
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, m, o, G);
        m = x > m ? x : m;
      }
      const double n = round_to_kind<BZ_F32>(m);
      const BinCtx bc = bin_ctx<false>(n, r, m);
      unsigned z = 0xffffffffu;
      unsigned hb[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const double d = __fma_rn(c[j], bc.R, kMagicH);
        hb[j] = (unsigned)__double2hiint(d);
        z = min(z, (unsigned)__double2loint(d));
      }
      const bool bad = active && (!safe || !bc.fast || !(m < 1.7976931348623157e308) || z < kNearHalf);
      const unsigned vote = __ballot_sync(0xffffffffu, bad) & gmask;
      if (!active) continue;  // (after the warp's last collective of the iteration)
      if (vote == 0u) {
        if (RED) {
          int sq = 0;
#pragma unroll
          for (int j = 0; j < CPL; ++j) {
            const int q = (int)(int8_t)hb[j];
            if (j < CPL - 1 || last_ok) sq += q * q;
          }
          red_acc = __fma_rn((double)sq * n, n, red_acc);  // (i N) N: overflow-safe
        } else {
          if (sub == 0) {
            out_max[b] = (float)n;
            if (out_dc) out_dc[b] = (int8_t)hb[0];  // DC plane: flat position 0
          }
#pragma unroll
          for (int j = 0; j < CPL; ++j)
            if (j < CPL - 1 || last_ok) po[sub + G * j] = (int8_t)hb[j];
        }
      } else {  // group-uniform: the exact path
        red_acc += small_block_exact<G, MODE, RED>(kept, sub, gmask, pa, pb, na, nb, subtract, shift,
                                                po, out_max, b);
        if (!RED) {
          __syncwarp(gmask);
          if (sub == 0 && out_dc) out_dc[b] = po[0];
        }
      }
    }
    __syncthreads();  // every read of `cur` and write of `so` done
    if (!RED) {  // the tile's rebinned indices: 16-byte stores (+ a ragged end)
      const int64_t nbytes = (int64_t)nv * kept;
      unsigned char* g = reinterpret_cast<unsigned char*>(out_idx) + b0 * (int64_t)kept;
      const int64_t nvec = nbytes / 16;
      for (int64_t i = t; i < nvec; i += 256)
        __stcs(reinterpret_cast<uint4*>(g) + i, *reinterpret_cast<const uint4*>(so + i * 16));
      for (int64_t i = nvec * 16 + t; i < nbytes; i += 256) g[i] = so[i];
      __syncthreads();  // `so` reused by the next tile
    }
  }
  cp_async_wait_all();
  if constexpr (RED) red_finish(red_acc, red_ws, red_out);
}

bool add_small_supported(const Geo& ga, const Geo& gb, int mode, const void* a_max,
                         const void* a_idx, const void* b_max, const void* b_idx,
                         const void* out_idx) {
  if (ga.index_kind != BZ_I8 || ga.float_kind != BZ_F32) return false;
  if (mode == 0 && (gb.float_kind != BZ_F32 || gb.index_kind != BZ_I8)) return false;
  // cp.async staging: every base 16-byte aligned
  const uintptr_t al = (uintptr_t)a_max | (uintptr_t)a_idx | (uintptr_t)out_idx |
                       (mode == 0 ? ((uintptr_t)b_max | (uintptr_t)b_idx) : 0);
  return ga.kept >= 1 && ga.kept <= 128 && ga.kept % 16 != 0 && !(al & 15) &&
         !getenv("BZC_B200_NO_ADD_SMALL");
}

static size_t small_smem(int kept) {
  return 2 * (size_t)((small_buf_bytes(kept) + 15) / 16 * 16) + (size_t)small_idx_bytes(kept);
}

template <int MODE, bool RED>
static int launch_small_m(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                          const void* b_idx, int subtract, double shift, void* out_max,
                          void* out_idx, void* out_dc, double* red_ws, double* red_out,
                          cudaStream_t s) {
  const int kept = ga.kept;
  const size_t smem = small_smem(kept);
  const int64_t ntiles = (ga.nblocks + TBS - 1) / TBS;
  // 4 lanes per block: the per-block work (scales, maximum, binning
  // context) is paid by fewer lanes (measured: C5 add 510 -> 479 us vs 8)
  const int cpl = (kept + 3) / 4;
#define BZ_SM(GV, C)                                                                               \
  case C: {                                                                                        \
    auto kern = k_add_small<GV, C, MODE, RED>;                                                     \
    const int occ = occupancy((const void*)kern, 256, smem);                                       \
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)kSMs * std::min(occ, 3))); \
    kern<<<g, 256, smem, s>>>(ga.nblocks, kept, (const float*)a_max, (const int8_t*)a_idx,         \
                              (const float*)b_max, (const int8_t*)b_idx, subtract, shift,          \
                              (float*)out_max, (int8_t*)out_idx, (int8_t*)out_dc, red_ws, red_out); \
    return check_launch(RED ? "subtract_l2_small" : "add_small");                                  \
  }
  {
    switch (cpl) {
      BZ_SM(4, 1) BZ_SM(4, 2) BZ_SM(4, 3) BZ_SM(4, 4) BZ_SM(4, 5) BZ_SM(4, 6) BZ_SM(4, 7) BZ_SM(4, 8)
      BZ_SM(4, 9) BZ_SM(4, 10) BZ_SM(4, 11) BZ_SM(4, 12) BZ_SM(4, 13) BZ_SM(4, 14) BZ_SM(4, 15) BZ_SM(4, 16)
      BZ_SM(4, 17) BZ_SM(4, 18) BZ_SM(4, 19) BZ_SM(4, 20) BZ_SM(4, 21) BZ_SM(4, 22) BZ_SM(4, 23) BZ_SM(4, 24)
      BZ_SM(4, 25) BZ_SM(4, 26) BZ_SM(4, 27) BZ_SM(4, 28) BZ_SM(4, 29) BZ_SM(4, 30) BZ_SM(4, 31) BZ_SM(4, 32)
    }
  }
#undef BZ_SM
  set_error("add_small: unsupported kept count");
  return BZ_E_UNSUPPORTED;
}

int launch_add_small(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                     const void* b_idx, int subtract, double shift, int mode, void* out_max,
                     void* out_idx, void* out_dc, cudaStream_t s) {
  if (ga.nblocks == 0) return BZ_OK;
  return mode == 0 ? launch_small_m<0, false>(ga, a_max, a_idx, b_max, b_idx, subtract, shift,
                                              out_max, out_idx, out_dc, nullptr, nullptr, s)
                   : launch_small_m<1, false>(ga, a_max, a_idx, b_max, b_idx, subtract, shift,
                                              out_max, out_idx, out_dc, nullptr, nullptr, s);
}

// l2_norm(subtract(a, b))^2 into red_ws[1] and *out (the subtract_l2
// workspace contract), written by the kernel's last CTA
int launch_subtract_l2_small(const Geo& ga, const void* a_max, const void* a_idx,
                             const void* b_max, const void* b_idx, double* red_ws, double* out,
                             cudaStream_t s) {
  return launch_small_m<0, true>(ga, a_max, a_idx, b_max, b_idx, 1, 0.0, nullptr, nullptr,
                                 nullptr, red_ws, out, s);
}

}  // namespace bz
