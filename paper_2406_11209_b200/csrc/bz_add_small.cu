// bz_add_small.cu -- add / subtract / add_scalar (and the fused subtract+l2
// of the time-series workflow) for int8 indices with float32 maxima and
// small blocks whose kept indices are not whole 16-byte vectors (the C5
// low-pass mask keeps K = 66), bit-exact with the reference
// (ops.py:178-215, codec.py:337-350 and 253-278; cli.py:240-243).
//
// A CTA stages tiles of TB blocks -- both operands' indices and maxima --
// in shared memory with 16-byte global accesses; a group of 8 lanes owns a
// block, lane `sub` holding its coefficients k = sub + 8 j (j < CPL, CPL =
// ceil(K / 8) exactly, a template parameter: no dead slots), read from a
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
constexpr int GSZ = 8;  // lanes per block

// exact reference arithmetic for one block (rare): IEEE product, division,
// NaN-propagating maximum, exact binning; the group's 8 lanes cooperate
template <int MODE, bool RED>
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
  for (int k = sub; k < kept; k += GSZ) m = nanmax_abs(m, coeff(k));
#pragma unroll
  for (int o = GSZ / 2; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(gmask, m, o, GSZ);
    m = (isnan(t) || isnan(m)) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, t);
  }
  const double n = round_to_kind<BZ_F32>(m);
  if (!RED && sub == 0) out_max[b] = (float)n;
  int sq = 0;
  for (int k = sub; k < kept; k += GSZ) {
    const int q = (int)bin_exact(coeff(k), n, r, r);
    if (RED) sq += q * q;
    else po[k] = (int8_t)q;
  }
  return RED ? __fma_rn((double)sq * n, n, 0.0) : 0.0;
}
}  // namespace

template <int CPL, int MODE, bool RED>
__global__ void __launch_bounds__(256, 3)
k_add_small(int64_t nblocks, int kept, int tb, const float* __restrict__ a_max,
            const int8_t* __restrict__ a_idx, const float* __restrict__ b_max,
            const int8_t* __restrict__ b_idx, int subtract, double shift,
            float* __restrict__ out_max, int8_t* __restrict__ out_idx,
            int8_t* __restrict__ out_dc, double* __restrict__ red_ws,
            double* __restrict__ red_out) {
  constexpr double r = 127.0, rinv = 1.0 / 127.0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t region = ((int64_t)tb * kept + 32 + 15) / 16 * 16;
  unsigned char* sa = smem_raw;
  unsigned char* sb = sa + region;
  unsigned char* so = sb + region;
  float* sma = reinterpret_cast<float*>(so + region);
  float* smb = sma + tb;
  const int t = threadIdx.x, lane = t & 31, sub = lane & (GSZ - 1);
  const unsigned gmask = 0xffu << (lane & 24);
  const bool last_ok = sub + GSZ * (CPL - 1) < kept;  // this lane's last slot holds a coefficient
  double red_acc = 0.0;
  const int64_t ntiles = (nblocks + tb - 1) / tb;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * tb;
    const int nv = (int)min((int64_t)tb, nblocks - b0);
    const int64_t byte0 = b0 * (int64_t)kept;
    const int64_t nbytes = (int64_t)nv * kept;
    const int misa = (int)(((uintptr_t)a_idx + byte0) & 15);
    const int misb = (int)(((uintptr_t)b_idx + byte0) & 15);
    const int miso = RED ? 0 : (int)(((uintptr_t)out_idx + byte0) & 15);
    for (int i = t; i < nv; i += 256) {
      sma[i] = __ldcs(a_max + b0 + i);
      if (MODE == 0) smb[i] = __ldcs(b_max + b0 + i);
    }
    tile_to_smem(sa, reinterpret_cast<const unsigned char*>(a_idx) + byte0, nbytes, misa, t, 256);
    if (MODE == 0)
      tile_to_smem(sb, reinterpret_cast<const unsigned char*>(b_idx) + byte0, nbytes, misb, t, 256);
    __syncthreads();
    for (int lb = t / GSZ; lb < nv; lb += 256 / GSZ) {
      const int64_t b = b0 + lb;
      const int8_t* pa = reinterpret_cast<const int8_t*>(sa + misa) + lb * kept;
      const int8_t* pb = reinterpret_cast<const int8_t*>(sb + misb) + lb * kept;
      int8_t* po = reinterpret_cast<int8_t*>(so + miso) + lb * kept;
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
        const double fa = ok ? (double)(int)pa[sub + GSZ * j] : 0.0;
        double cc = __fma_rn(fa, tha, fa * tla);
        if (MODE == 0) {
          const double fb = ok ? (double)(int)pb[sub + GSZ * j] : 0.0;
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
      for (int o = GSZ / 2; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(gmask, m, o, GSZ);
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
      const bool bad = !safe || !bc.fast || !(m < 1.7976931348623157e308) || z < kNearHalf;
      if ((__ballot_sync(gmask, bad) & gmask) == 0u) {
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
            if (j < CPL - 1 || last_ok) po[sub + GSZ * j] = (int8_t)hb[j];
        }
      } else {  // group-uniform: the exact path
        red_acc += small_block_exact<MODE, RED>(kept, sub, gmask, pa, pb, na, nb, subtract, shift,
                                                po, out_max, b);
        if (!RED) {
          __syncwarp(gmask);
          if (sub == 0 && out_dc) out_dc[b] = po[0];
        }
      }
    }
    __syncthreads();
    if (!RED)
      smem_to_tile(reinterpret_cast<unsigned char*>(out_idx) + byte0, so, nbytes, miso, t, 256);
    __syncthreads();  // tiles reused
  }
  if constexpr (RED) red_finish(red_acc, red_ws, red_out);
}

bool add_small_supported(const Geo& ga, const Geo& gb, int mode) {
  if (ga.index_kind != BZ_I8 || ga.float_kind != BZ_F32) return false;
  if (mode == 0 && (gb.float_kind != BZ_F32 || gb.index_kind != BZ_I8)) return false;
  return ga.kept >= 1 && ga.kept <= 16 * GSZ && ga.kept % 16 != 0 && !getenv("BZC_B200_NO_ADD_SMALL");
}

// tile of TB blocks: ~8 KB of indices per operand
static int small_tile(int kept) { return std::max(32, (8192 / kept) / 32 * 32); }

static size_t small_smem(int kept, int tb) {
  const size_t region = ((size_t)tb * kept + 32 + 15) / 16 * 16;
  return 3 * region + 2 * (size_t)tb * sizeof(float);
}

template <int MODE, bool RED>
static int launch_small_m(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                          const void* b_idx, int subtract, double shift, void* out_max,
                          void* out_idx, void* out_dc, double* red_ws, double* red_out,
                          cudaStream_t s) {
  const int kept = ga.kept;
  const int cpl = (kept + GSZ - 1) / GSZ;
  const int tb = small_tile(kept);
  const size_t smem = small_smem(kept, tb);
  const int64_t ntiles = (ga.nblocks + tb - 1) / tb;
#define BZ_SM(C)                                                                                   \
  case C: {                                                                                        \
    auto kern = k_add_small<C, MODE, RED>;                                                         \
    const int occ = occupancy((const void*)kern, 256, smem);                                       \
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)kSMs * std::min(occ, 3))); \
    kern<<<g, 256, smem, s>>>(ga.nblocks, kept, tb, (const float*)a_max, (const int8_t*)a_idx,     \
                              (const float*)b_max, (const int8_t*)b_idx, subtract, shift,          \
                              (float*)out_max, (int8_t*)out_idx, (int8_t*)out_dc, red_ws, red_out); \
    return check_launch(RED ? "subtract_l2_small" : "add_small");                                  \
  }
  switch (cpl) {
    BZ_SM(1) BZ_SM(2) BZ_SM(3) BZ_SM(4) BZ_SM(5) BZ_SM(6) BZ_SM(7) BZ_SM(8)
    BZ_SM(9) BZ_SM(10) BZ_SM(11) BZ_SM(12) BZ_SM(13) BZ_SM(14) BZ_SM(15) BZ_SM(16)
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
