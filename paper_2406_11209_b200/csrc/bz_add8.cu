// bz_add8.cu -- add / subtract / add_scalar for int8 indices with float32
// maxima (the C3 / C4 chain, ops.py:178-215), bit-exact with the reference.
//
// The reference computes every coefficient as fl(fl(F * N) / r) (codec.py:
// 337-350), sums the two operands, takes the block maximum and rebins.  For
// int8 F and a float32 N the product F * N is exact (8 + 24 bits), so
// fl(F * N / r) = RN(F * t) with t = N / r.  With t_hi = RN(t) and
// t_lo = RN(t - t_hi) (the remainder is exact by FMA) the kernel evaluates
//     x = fma(F, t_hi, F * t_lo)
// -- two FP64 operations instead of a product and a correctly rounded
// division.  Exactness: F * t_hi + RN(F * t_lo) differs from F * t by less
// than 2^-98 |F t|, while F * t = F N / 127 is either representable or sits
// at least 2^-8 ulp away from every rounding boundary (its binary expansion
// beyond the significand is j/127 of an ulp, 2 having order 7 modulo 127,
// and a midpoint would need j/127 = 1/2).  So x equals the reference's
// fl(fl(F N) / r) bit for bit.  Subtract negates t_hi and t_lo (exact).
//
// Rebinning uses the 32-bit fixed point of bz_common.cuh (kMagicH: one FMA
// per coefficient); a block whose maxima are tiny / huge / zero / non-finite,
// whose stored maximum could round differently, or with a coefficient
// within one fixed-point unit of a rounding half, is recomputed by the
// group with the exact IEEE path (codec.py:253-278) right away.
#include "bz_common.cuh"
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

namespace bz {

namespace {

// exact per-block path (rare): IEEE product, division, NaN-propagating
// maximum and exact binning, GS lanes of the group cooperating
template <int GS, int MODE, bool RED = false>
__device__ __noinline__ double add8_block_exact(int64_t b, int kept, int sub, unsigned gmask,
                                              const float* __restrict__ a_max,
                                              const int8_t* __restrict__ a_idx,
                                              const float* __restrict__ b_max,
                                              const int8_t* __restrict__ b_idx, int subtract,
                                              double shift, float* __restrict__ out_max,
                                              int8_t* __restrict__ out_idx,
                                              int8_t* __restrict__ out_dc) {
  const double r = 127.0;
  const int64_t base = b * (int64_t)kept;
  const double na = (double)a_max[b];
  const double nb = MODE == 0 ? (double)b_max[b] : 0.0;
  auto coeff = [&](int k) -> double {
    const double xa = __ddiv_rn(__dmul_rn((double)a_idx[base + k], na), r);
    if (MODE == 0) {
      const double fb = subtract ? -(double)b_idx[base + k] : (double)b_idx[base + k];
      return __dadd_rn(xa, __ddiv_rn(__dmul_rn(fb, nb), r));
    }
    return k == 0 ? __dadd_rn(xa, shift) : xa;
  };
  double m = 0.0;
  for (int k = sub; k < kept; k += GS) m = nanmax_abs(m, coeff(k));
#pragma unroll
  for (int o = GS / 2; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(gmask, m, o, GS);
    m = (isnan(t) || isnan(m)) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, t);
  }
  const double n = round_to_kind<BZ_F32>(m);
  if (RED) {  // fused l2 of the rebinned difference: this lane's sum of squares
    int sq = 0;
    for (int k = sub; k < kept; k += GS) {
      const int q = (int)bin_exact(coeff(k), n, r, r);
      sq += q * q;
    }
    return __fma_rn((double)sq * n, n, 0.0);
  }
  if (sub == 0) out_max[b] = (float)n;
  for (int k = sub; k < kept; k += GS) out_idx[base + k] = (int8_t)bin_exact(coeff(k), n, r, r);
  if (out_dc && sub == 0) out_dc[b] = (int8_t)bin_exact(coeff(0), n, r, r);
  return 0.0;
}

}  // namespace

// GS lanes per block, NCH 16-byte chunks (16 indices) per lane; the next
// block's chunks and maxima are loaded while the current block computes.
// RED: the fused l2_norm(subtract(a, b)) of the time-series workflow
// (cli.py:240-243) -- the rebinned indices are squared and summed (dp4a)
// times N^2 instead of stored; the last CTA writes the sum to red_out.
template <int GS, int NCH, int MODE, bool RED = false>
__global__ void __launch_bounds__(256, NCH == 1 ? 3 : 2)
k_add8(int64_t nblocks, int kept, const float* __restrict__ a_max,
       const int8_t* __restrict__ a_idx, const float* __restrict__ b_max,
       const int8_t* __restrict__ b_idx, int subtract, double shift,
       float* __restrict__ out_max, int8_t* __restrict__ out_idx, int8_t* __restrict__ out_dc,
       double* __restrict__ red_ws = nullptr, double* __restrict__ red_out = nullptr) {
  double red_acc = 0.0;
  constexpr double r = 127.0, rinv = 1.0 / 127.0;
  constexpr int L = NCH * 16;
  const int lane = threadIdx.x & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GS;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / GS;

  uint4 pa[NCH], pb[NCH];
  float pna = 0.f, pnb = 0.f;
  auto fetch = [&](int64_t b) {
    if (b < nblocks) {
      const int64_t base = b * (int64_t)kept;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int k0 = (ch * GS + sub) * 16;
        pa[ch] = k0 < kept ? __ldcs(reinterpret_cast<const uint4*>(a_idx + base + k0))
                           : make_uint4(0, 0, 0, 0);
        pb[ch] = (MODE == 0 && k0 < kept)
                     ? __ldcs(reinterpret_cast<const uint4*>(b_idx + base + k0))
                     : make_uint4(0, 0, 0, 0);
      }
      pna = __ldcs(a_max + b);
      pnb = MODE == 0 ? __ldcs(b_max + b) : 0.f;
    }
  };
  fetch(group);

  // warp-uniform trip count (the warp's first group decides): every lane runs
  // every iteration, so the group maximum and vote below are full-warp
  // collectives; a group past the end computes on stale registers and stores
  // nothing (a partial-mask vote compiled to WARPSYNC.EXCLUSIVE, one vote per
  // group in turn)
  for (int64_t b = group; b - lane / GS < nblocks; b += ngroups) {
    const bool active = b < nblocks;
    const int64_t base = b * (int64_t)kept;
    uint4 ca[NCH], cb[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      ca[ch] = pa[ch];
      cb[ch] = pb[ch];
    }
    const double na = (double)pna, nb = (double)pnb;
    fetch(b + ngroups);

    bool safe = na >= 0x1p-900 && na <= 0x1p+900;
    if (MODE == 0) safe = safe && nb >= 0x1p-900 && nb <= 0x1p+900;
    // t = N / r as t_hi + t_lo (t_hi correctly rounded, remainder exact by FMA)
    const double tha = div_const(na, r, rinv);
    const double tla = __fma_rn(-tha, r, na) * rinv;
    double thb = 0.0, tlb = 0.0;
    if (MODE == 0) {
      thb = div_const(nb, r, rinv);
      tlb = __fma_rn(-thb, r, nb) * rinv;
      if (subtract) { thb = -thb; tlb = -tlb; }
    }
    double c[L];
    // block maximum in float32: RN32 is monotone, so the largest RN32(|c|)
    // is RN32(max |c|) -- exactly the stored maximum N (round_to_kind<F32>)
    // -- for one conversion and a 3-input FMNMX per coefficient instead of
    // a DSETP + 2 FSEL compare-select chain, and one 32-bit shuffle per
    // step; an N that is not a normal float goes to the exact path
    float mf[2] = {0.f, 0.f};
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const uint32_t wa[4] = {ca[ch].x, ca[ch].y, ca[ch].z, ca[ch].w};
      // operand b's bytes as unsigned (f + 128): its f64 values come from the
      // bias form 2^52 + (f + 128) - (2^52 + 128) on the FP64 pipe, which
      // keeps the 16-per-clock conversion unit at two operations per
      // coefficient (a's int8 -> f64 and the float32 maximum)
      const uint32_t wb[4] = {cb[ch].x ^ 0x80808080u, cb[ch].y ^ 0x80808080u,
                              cb[ch].z ^ 0x80808080u, cb[ch].w ^ 0x80808080u};
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const double fa = (double)(int)(int8_t)(wa[e >> 2] >> (8 * (e & 3)));
        double cc = __fma_rn(fa, tha, fa * tla);
        if (MODE == 0) {
          const double fb =
              __hiloint2double(0x43300000, (int)__byte_perm(wb[e >> 2], 0u, 0x4440 + (e & 3))) -
              4503599627370624.0;  // 2^52 + 128
          cc = __dadd_rn(cc, __fma_rn(fb, thb, fb * tlb));
        } else if (ch == 0 && e == 0) {
          if (sub == 0) cc = __dadd_rn(cc, shift);
        }
        c[ch * 16 + e] = cc;
        // chunks past `kept` hold zeros: they cannot raise the maximum
        mf[e & 1] = fmaxf(mf[e & 1], __double2float_rn(fabs(cc)));
      }
    }
    float nf = fmaxf(mf[0], mf[1]);
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) nf = fmaxf(nf, __shfl_xor_sync(0xffffffffu, nf, o, GS));
    const double n = (double)nf;
    const BinCtx bc = bin_ctx<false>(n, r, n);
    // 32-bit fixed point (kMagicH, bz_common.cuh): index = low byte of the
    // high word unless the fraction (low word) is within 2^-24 of one half
    unsigned z4[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    uint4 ov[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      unsigned y[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const double d = __fma_rn(c[ch * 16 + e], bc.R, kMagicH);
        y[e] = (unsigned)__double2hiint(d);
        z4[e & 3] = min(z4[e & 3], (unsigned)__double2loint(d));
      }
      unsigned wd[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        wd[k] = __byte_perm(__byte_perm(y[4 * k], y[4 * k + 1], 0x0040),
                            __byte_perm(y[4 * k + 2], y[4 * k + 3], 0x0040), 0x5410);
      ov[ch] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
    const bool near = min(min(z4[0], z4[1]), min(z4[2], z4[3])) < kNearHalf;
    const bool bad = !safe || !bc.fast || !(nf >= 1.17549435e-38f && nf <= 3.40282347e+38f);
    const bool any_bad = (__ballot_sync(0xffffffffu, active && (near || bad)) & gmask) != 0u;
    if (!active) continue;
    if (!any_bad) {
      if constexpr (RED) {
        int sq = 0;  // <= 32 * 127^2 per chunk: exact in int32
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int k0 = (ch * GS + sub) * 16;
          if (k0 < kept) {
            sq = __dp4a((int)ov[ch].x, (int)ov[ch].x, sq);
            sq = __dp4a((int)ov[ch].y, (int)ov[ch].y, sq);
            sq = __dp4a((int)ov[ch].z, (int)ov[ch].z, sq);
            sq = __dp4a((int)ov[ch].w, (int)ov[ch].w, sq);
          }
        }
        red_acc = __fma_rn((double)sq * n, n, red_acc);  // (i N) N: overflow-safe
      } else {
        if (sub == 0) {
          out_max[b] = (float)n;
          if (out_dc) out_dc[b] = (int8_t)ov[0].x;  // DC plane: flat position 0
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int k0 = (ch * GS + sub) * 16;
          if (k0 < kept) __stcs(reinterpret_cast<uint4*>(out_idx + base + k0), ov[ch]);
        }
      }
    } else {  // group-uniform: the exact path for this block
      red_acc += add8_block_exact<GS, MODE, RED>(b, kept, sub, gmask, a_max, a_idx, b_max, b_idx,
                                                 subtract, shift, out_max, out_idx, out_dc);
    }
  }
  if constexpr (RED) red_finish(red_acc, red_ws, red_out);
}

bool add8_supported(const Geo& ga, const Geo& gb, int mode, const void* a_idx, const void* b_idx,
                    const void* out_idx) {
  if (ga.index_kind != BZ_I8 || ga.float_kind != BZ_F32) return false;
  if (mode == 0 && gb.float_kind != BZ_F32) return false;
  if (ga.kept < 16 || ga.kept % 16 || ga.kept > 32 * 16 * 2) return false;
  const uintptr_t al = (uintptr_t)a_idx | (uintptr_t)out_idx | (mode == 0 ? (uintptr_t)b_idx : 0);
  return (al & 15) == 0;
}

// lanes per block: on large arrays, blocks of more than 256 kept give each
// lane two 16-byte chunks (GS = 16 at K = 512: the per-block work -- t_hi /
// t_lo, the 5-round shuffle maximum, bin_ctx -- is shared by twice the
// coefficients; C3 add 1.16 -> 1.03 ms, subtract+l2 1.19 -> 1.08 ms).
// Small arrays (C1: 32768 blocks, 34 vs 51 us) and smaller blocks keep one
// chunk per lane and 3 CTAs per SM.
static int add8_group(int vecs, int64_t nblocks) {
  int GS = 1;
  if (vecs > 16 && nblocks >= (int64_t{1} << 18)) {
    while (GS < 32 && 2 * GS < vecs) GS <<= 1;
  } else {
    while (GS < 32 && GS < vecs) GS <<= 1;
  }
  return GS;
}

int launch_add8(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                const void* b_idx, int subtract, double shift, int mode, void* out_max,
                void* out_idx, cudaStream_t s, void* out_dc) {
  const int vecs = ga.kept / 16;
  const int GS = add8_group(vecs, ga.nblocks);
  const int NCH = (vecs + GS - 1) / GS;  // 1 or 2
  const int grid = grid_for(ga.nblocks * GS, 256, NCH == 1 ? 3 : 2);
#define BZ_A8(G, N, M)                                                                        \
  k_add8<G, N, M><<<grid, 256, 0, s>>>(ga.nblocks, ga.kept, (const float*)a_max,              \
                                       (const int8_t*)a_idx, (const float*)b_max,             \
                                       (const int8_t*)b_idx, subtract, shift, (float*)out_max, \
                                       (int8_t*)out_idx, (int8_t*)out_dc)
#define BZ_A8M(G, N) \
  do { if (mode == 0) BZ_A8(G, N, 0); else BZ_A8(G, N, 1); } while (0)
#define BZ_A8G(G)             \
  case G:                     \
    if (NCH == 1) BZ_A8M(G, 1); \
    else BZ_A8M(G, 2);        \
    break;
  switch (GS) { BZ_A8G(1) BZ_A8G(2) BZ_A8G(4) BZ_A8G(8) BZ_A8G(16) BZ_A8G(32) }
#undef BZ_A8G
#undef BZ_A8M
#undef BZ_A8
  return check_launch("add8");
}

// l2_norm(subtract(a, b))^2 into red_ws[1] and *out (the subtract_l2
// workspace contract: at most 3 * kSMs CTAs)
int launch_subtract_l2_add8(const Geo& ga, const void* a_max, const void* a_idx,
                            const void* b_max, const void* b_idx, double* red_ws, double* out,
                            cudaStream_t s) {
  const int vecs = ga.kept / 16;
  const int GS = add8_group(vecs, ga.nblocks);
  const int NCH = (vecs + GS - 1) / GS;  // 1 or 2
  const int grid = grid_for(ga.nblocks * GS, 256, NCH == 1 ? 3 : 2);
#define BZ_R8(G, N)                                                                           \
  k_add8<G, N, 0, true><<<grid, 256, 0, s>>>(ga.nblocks, ga.kept, (const float*)a_max,        \
                                             (const int8_t*)a_idx, (const float*)b_max,       \
                                             (const int8_t*)b_idx, 1, 0.0, nullptr, nullptr,  \
                                             nullptr, red_ws, out)
#define BZ_R8G(G)                                   \
  case G:                                           \
    if (NCH == 1) BZ_R8(G, 1); else BZ_R8(G, 2);    \
    break;
  switch (GS) { BZ_R8G(1) BZ_R8G(2) BZ_R8G(4) BZ_R8G(8) BZ_R8G(16) BZ_R8G(32) }
#undef BZ_R8G
#undef BZ_R8
  return check_launch("subtract_l2_add8");
}

}  // namespace bz
