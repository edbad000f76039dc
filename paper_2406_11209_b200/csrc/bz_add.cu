// bz_add.cu -- add / subtract / add_scalar in the compressed domain
// (ops.py:178-215, codec.py:337-350): one pass over the kept coefficients of
// both operands with the reference's exact f64 op order, block maximum,
// rebinning -- bit-exact with the reference.
#include "bz_common.cuh"
#include "bz_fast.cuh"
#include "bz_kernels.cuh"

#include <cstdlib>
#include <type_traits>

namespace bz {

// --------------------------------------------------------- add / rebinning --
// A group of GS lanes handles one block; each lane owns V = 16/sizeof(IT)
// consecutive kept coefficients per chunk (one 16-byte vector when the
// block's kept indices are a whole number of vectors).
template <typename IT>
using elem_t = typename std::conditional<sizeof(IT) == 8, long long, int>::type;

template <typename IT>
__device__ __forceinline__ void load_chunk(const IT* __restrict__ p, int64_t base, int k0, int kept,
                                           bool vec, elem_t<IT> (&out)[16 / sizeof(IT)]) {
  constexpr int V = 16 / sizeof(IT);
  if (vec && k0 + V <= kept) {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(p + base + k0));
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if constexpr (sizeof(IT) == 1) out[e] = (int8_t)(ws[e / 4] >> (8 * (e % 4)));
      else if constexpr (sizeof(IT) == 2) out[e] = (int16_t)(ws[e / 2] >> (16 * (e % 2)));
      else if constexpr (sizeof(IT) == 4) out[e] = (int32_t)ws[e];
      else out[e] = (long long)(((unsigned long long)ws[2 * e + 1] << 32) | ws[2 * e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) out[e] = (k0 + e < kept) ? (elem_t<IT>)p[base + k0 + e] : 0;
  }
}

// exact out-of-line paths (rare): IEEE division, exact binning
__device__ __noinline__ double spec_coeff_slow(double f, double n, double r) {
  return __ddiv_rn(__dmul_rn(f, n), r);
}
__device__ __noinline__ long long bin_exact_out(double c, double n, double r, double bound) {
  return bin_exact(c, n, r, bound);
}

// F*N exactly as the reference's fl(float(F) * N): for |F| < 2^31 the
// integer is widened with the 2^52+2^31 bias trick (an integer op + the FMA
// below) instead of the slow int->f64 conversion; when N has <= 31
// significant bits (every BF16/F16/F32 maximum), bias*N is exact and
// fma(biased, N, -bias*N) = RN(F*N) in one DFMA.
struct Scale {
  double n, nbias;  // N and -(2^52+2^31)*N (exact when narrow)
  bool narrow;      // N fits 31 significant bits
};
__device__ __forceinline__ Scale make_scale(double n, int fk) {
  Scale s;
  s.n = n;
  s.narrow = fk != BZ_F64;
  s.nbias = -(4503601774854144.0 * n);
  return s;
}
__device__ __forceinline__ double fn_product(int f, const Scale& s) {
  if (s.narrow) {
    const double biased = __hiloint2double(0x43300000, (int)((unsigned)f ^ 0x80000000u));
    return __fma_rn(biased, s.n, s.nbias);
  }
  // wide (F64) maxima: one int -> f64 conversion (the conversion unit has
  // room here) instead of the bias form's constant move, xor and DADD --
  // k_add at C2 is issue-bound
  return __dmul_rn((double)f, s.n);
}
__device__ __forceinline__ double fn_product(long long f, const Scale& s) {
  return __dmul_rn((double)f, s.n);
}

// element e of a 16-byte chunk (compile-time e)
template <typename IT>
__device__ __forceinline__ elem_t<IT> vec_elem(const uint4& w, int e) {
  const uint32_t x = (e * (int)sizeof(IT)) / 4 == 0 ? w.x : (e * (int)sizeof(IT)) / 4 == 1 ? w.y
                   : (e * (int)sizeof(IT)) / 4 == 2 ? w.z : w.w;
  if constexpr (sizeof(IT) == 1) return (int8_t)(x >> (8 * (e % 4)));
  else if constexpr (sizeof(IT) == 2) return (int16_t)(x >> (16 * (e % 2)));
  else if constexpr (sizeof(IT) == 4) return (int32_t)x;
  else {
    const uint32_t hi = (e * 8) / 4 + 1 == 1 ? w.y : w.w;
    return (long long)(((unsigned long long)hi << 32) | x);
  }
}

// one chunk (16 bytes) of a block's kept indices as integers
template <typename IT>
__device__ __forceinline__ void unpack_chunk(const uint4& w, elem_t<IT> (&out)[16 / sizeof(IT)]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int e = 0; e < 16 / (int)sizeof(IT); ++e) {
    if constexpr (sizeof(IT) == 1) out[e] = (int8_t)(ws[e / 4] >> (8 * (e % 4)));
    else if constexpr (sizeof(IT) == 2) out[e] = (int16_t)(ws[e / 2] >> (16 * (e % 2)));
    else if constexpr (sizeof(IT) == 4) out[e] = (int32_t)ws[e];
    else out[e] = (long long)(((unsigned long long)ws[2 * e + 1] << 32) | ws[2 * e]);
  }
}

// mode 0: a + (+/-)b     mode 1: a + shift at the first coefficient (add_scalar)
// A group of GS lanes handles one block; each lane keeps NCH chunks of V
// coefficients in registers (GS*NCH*V >= kept), so the block is read once.
// VEC: the kept indices of every block are whole 16-byte vectors -- the next
// block's vectors and maxima are loaded before the current block computes.
// FK >= 0: every maximum is of that kind (compile time); FK < 0: run-time
// kinds fk_a / fk_b / fk_out.  MODE is the run-time `mode` made constant.
template <int FK>
__device__ __forceinline__ double ld_max(const void* p, int64_t i, int fk) {
  if constexpr (FK >= 0) return load_kind<FK>(p, i);
  else return load_kind_rt(p, i, fk);
}
template <int FK>
__device__ __forceinline__ double rnd_max(double x, int fk) {
  if constexpr (FK >= 0) return round_to_kind<FK>(x);
  else return round_to_kind_rt(x, fk);
}
template <int FK>
__device__ __forceinline__ void st_max(void* p, int64_t i, double v, int fk) {
  if constexpr (FK >= 0) store_kind<FK>(p, i, v);
  else store_kind_rt(p, i, v, fk);
}

// RED: instead of storing the result, accumulate its squared L2 norm
// sum (q * N)^2 = sum_blocks N^2 * sum q^2 (exact integer block sums) and
// reduce it deterministically into red_ws[1] (the fused time-series step
// l2_norm(add(s[i+1], negate(s[i]))), cli.py:240-243, in one pass).
// CTAs per SM: 3 (85 registers) by default; the 16-bit two-chunk blocks (C2's
// 4x4 I16) hold 16 f64 coefficients plus the next block's 64 bytes in flight
// per lane, which at 85 registers spilled the prefetch registers (the spill
// store waited on the pending load): 2 CTAs, 128 registers.
template <typename IT, int NCH>
constexpr int add_ctas() { return (sizeof(IT) == 2 && NCH == 2) ? 2 : 3; }

template <typename IT, int GS, int NCH, bool VEC, int FK, int MODE, bool RED = false>
__global__ void __launch_bounds__(256, add_ctas<IT, NCH>())
k_add(int64_t nblocks, int kept, int fk_a, int fk_b, int fk_out,
      const void* __restrict__ a_max, const IT* __restrict__ a_idx,
      const void* __restrict__ b_max, const IT* __restrict__ b_idx, int subtract,
      double shift, int mode_rt, void* __restrict__ out_max, IT* __restrict__ out_idx,
      double* __restrict__ red_ws = nullptr, IT* __restrict__ out_dc = nullptr,
      double* __restrict__ red_out = nullptr) {
  double red_acc = 0.0;
  constexpr int mode = MODE;
  (void)mode_rt;
  constexpr int V = 16 / sizeof(IT);
  constexpr int L = NCH * V;  // coefficients per lane
  constexpr int IK = sizeof(IT) == 1 ? BZ_I8 : sizeof(IT) == 2 ? BZ_I16 : sizeof(IT) == 4 ? BZ_I32 : BZ_I64;
  const double r = radius_f64(IK), bound = clamp_bound_f64(IK);
  const double rinv = 1.0 / r;
  const int lane = threadIdx.x & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GS;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / GS;

  // software pipeline (VEC): registers for the next block's raw data
  uint4 pa[NCH], pb[NCH];
  double pna = 0.0, pnb = 0.0;
  auto fetch = [&](int64_t b) {
    if (b < nblocks) {
      const int64_t base = b * (int64_t)kept;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int k0 = (ch * GS + sub) * V;
        pa[ch] = k0 < kept ? __ldcs(reinterpret_cast<const uint4*>(a_idx + base + k0)) : make_uint4(0, 0, 0, 0);
        pb[ch] = (mode == 0 && k0 < kept) ? __ldcs(reinterpret_cast<const uint4*>(b_idx + base + k0))
                                          : make_uint4(0, 0, 0, 0);
      }
      pna = ld_max<FK>(a_max, b, fk_a);
      pnb = mode == 0 ? ld_max<FK>(b_max, b, fk_b) : 0.0;
    }
  };
  if (VEC) fetch(group);

  for (int64_t b = group; b < nblocks; b += ngroups) {
    const int64_t base = b * (int64_t)kept;
    double na, nb;
    uint4 ca[NCH], cb[NCH];
    if (VEC) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) { ca[ch] = pa[ch]; cb[ch] = pb[ch]; }
      na = pna;
      nb = pnb;
      fetch(b + ngroups);  // next block's loads are in flight during this block
    } else {
      na = ld_max<FK>(a_max, b, fk_a);
      nb = mode == 0 ? ld_max<FK>(b_max, b, fk_b) : 0.0;
    }
    const Scale sa = make_scale(na, FK >= 0 ? FK : fk_a), sb = make_scale(nb, FK >= 0 ? FK : fk_b);
    const bool safe = na >= 0x1p-900 && na <= 0x1p+900 &&
                      (mode != 0 || (nb >= 0x1p-900 && nb <= 0x1p+900));
    double c[L];
    unsigned long long key = 0;
    double mxd = 0.0;
    // block-uniform choice of the arithmetic: the common (safe) path has no
    // per-coefficient branch; unsafe maxima (tiny / huge) use IEEE division
    auto coeffs = [&](auto safe_tag) {
      constexpr bool SAFE = decltype(safe_tag)::value;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int k0 = (ch * GS + sub) * V;
        elem_t<IT> fa[V], fb[V];
        if (!VEC) {
          load_chunk<IT>(a_idx, base, k0, kept, false, fa);
          if (mode == 0) load_chunk<IT>(b_idx, base, k0, kept, false, fb);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (VEC) {  // extract on the fly (no unpacked copies held in registers)
            fa[e] = vec_elem<IT>(ca[ch], e);
            fb[e] = vec_elem<IT>(cb[ch], e);
          }
          double cc;
          if constexpr (SAFE) {
            const double xa = div_const(fn_product(fa[e], sa), r, rinv);
            if (mode == 0) {
              const elem_t<IT> fbv = subtract ? -fb[e] : fb[e];
              cc = __dadd_rn(xa, div_const(fn_product(fbv, sb), r, rinv));
            } else {
              cc = (k0 + e == 0) ? __dadd_rn(xa, shift) : xa;
            }
          } else {
            const double xa = spec_coeff_slow((double)fa[e], na, r);
            if (mode == 0) {
              const double fbv = subtract ? -(double)fb[e] : (double)fb[e];
              cc = __dadd_rn(xa, spec_coeff_slow(fbv, nb, r));
            } else {
              cc = (k0 + e == 0) ? __dadd_rn(xa, shift) : xa;
            }
          }
          c[ch * V + e] = cc;
          if (VEC ? (k0 < kept) : (k0 + e < kept)) {  // VEC: chunks are whole
            if constexpr (SAFE) {  // finite on the safe path: plain compare-select
              const double a = fabs(cc);
              mxd = a > mxd ? a : mxd;
            } else {  // NaN-propagating via the bit order
              const unsigned long long k2 = (unsigned long long)__double_as_longlong(cc) & 0x7fffffffffffffffull;
              key = k2 > key ? k2 : key;
            }
          }
        }
      }
      if constexpr (SAFE) key = (unsigned long long)__double_as_longlong(mxd);
    };
    if (safe) coeffs(std::true_type{});
    else coeffs(std::false_type{});
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(gmask, key, o, GS);
      key = k2 > key ? k2 : key;
    }
    const double mx = __longlong_as_double((long long)key);  // NaN-propagating via bit order
    const double n = rnd_max<FK>(mx, fk_out);
    if (!RED && sub == 0) st_max<FK>(out_max, b, n, fk_out);
    // 16-bit indices under F64 / F32 maxima (stored maximum within 2^-20 of
    // the true one: no clamp) bin through kMagicH (bz_common.cuh): the index
    // is the high word's low half, the low word the near-half test -- one
    // DFMA and a min per coefficient (C2: k_add is issue-bound)
    constexpr bool MAGIC16 = sizeof(IT) == 2 && (FK == BZ_F64 || FK == BZ_F32);
    const BinCtx bc = bin_ctx<!MAGIC16>(n, r, mx);
    long long red_sq = 0;  // RED: this lane's exact sum of q^2 over the block
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int k0 = (ch * GS + sub) * V;
      int q[V];
      if constexpr (MAGIC16) {
        unsigned z = 0xffffffffu;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const double d = __fma_rn(c[ch * V + e], bc.R, kMagicH);
          q[e] = (int)(short)__double2hiint(d);
          z = min(z, (unsigned)__double2loint(d));
        }
        if ((z < kNearHalf) | !bc.fast) {
#pragma unroll
          for (int e = 0; e < V; ++e) q[e] = (int)bin_exact_ctx(c[ch * V + e], bc, r, r);
        }
      } else if constexpr (sizeof(IT) <= 2) {
        unsigned nacc = 0;
#pragma unroll
        for (int e = 0; e < V; ++e) q[e] = fast_index32<IT, true>(c[ch * V + e], bc.R, (int)r, nacc);
        if (nacc | !bc.fast) {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            unsigned nr = 0;
            fast_index32<IT, true>(c[ch * V + e], bc.R, (int)r, nr);
            if (nr | !bc.fast) q[e] = (int)bin_exact_ctx(c[ch * V + e], bc, r, r);
          }
        }
      }
      long long q64[V];
      if constexpr (sizeof(IT) > 2) {
#pragma unroll
        for (int e = 0; e < V; ++e) {
          bool nr = false;
          if constexpr (sizeof(IT) == 4) q64[e] = bc.fast ? fast_index<int32_t>(c[ch * V + e], bc.R, r, nr) : 0;
          else q64[e] = 0;
          if (nr || !bc.fast || sizeof(IT) == 8) q64[e] = bin_exact_ctx(c[ch * V + e], bc, r, bound);
        }
      }
      if (!RED && out_dc && k0 == 0) {  // DC plane: flat position 0
        if constexpr (sizeof(IT) <= 2) out_dc[b] = (IT)q[0];
        else out_dc[b] = (IT)q64[0];
      }
      if constexpr (RED) {
        if constexpr (sizeof(IT) <= 2) {
#pragma unroll
          for (int e = 0; e < V; ++e)
            if (VEC ? (k0 < kept) : (k0 + e < kept)) red_sq += (long long)(q[e] * q[e]);
        }
      } else if (VEC && k0 < kept) {
        if constexpr (sizeof(IT) <= 2) {
          __stcs(reinterpret_cast<uint4*>(out_idx + base + k0), pack16<IT>(q));
        } else {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < V; ++e) {
            if constexpr (sizeof(IT) == 8) {
              w[2 * e] = (uint32_t)q64[e];
              w[2 * e + 1] = (uint32_t)((unsigned long long)q64[e] >> 32);
            } else {
              w[e] = (uint32_t)q64[e];
            }
          }
          __stcs(reinterpret_cast<uint4*>(out_idx + base + k0), make_uint4(w[0], w[1], w[2], w[3]));
        }
      } else if (!VEC) {
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (k0 + e < kept) {
            if constexpr (sizeof(IT) <= 2) out_idx[base + k0 + e] = (IT)q[e];
            else out_idx[base + k0 + e] = (IT)q64[e];
          }
        }
      }
    }
    if (RED) red_acc = __fma_rn((double)red_sq * n, n, red_acc);
  }
  if constexpr (RED) red_finish(red_acc, red_ws, red_out);
}

// --------------------------------------- staged add (unaligned blocks) --
// Blocks whose kept indices are not whole 16-byte vectors (e.g. C5's 66 int8
// indices) are moved as contiguous tiles of TB blocks through shared memory
// with 16-byte accesses (tile_to_smem / smem_to_tile); GS = 256/TB lanes per
// block then read their coefficients from shared memory.  Same exact
// arithmetic as k_add (codec.py:337-350, ops.py:178-204): the coefficient is
// recomputed in the binning pass instead of being kept in registers.
template <typename IT, int FK, int MODE>
__global__ void __launch_bounds__(256)
k_add_staged(int64_t nblocks, int kept, int tb, const void* __restrict__ a_max,
             const IT* __restrict__ a_idx, const void* __restrict__ b_max,
             const IT* __restrict__ b_idx, int subtract, double shift,
             void* __restrict__ out_max, IT* __restrict__ out_idx) {
  constexpr int IK = sizeof(IT) == 1 ? BZ_I8 : BZ_I16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const double r = radius_f64(IK), rinv = 1.0 / r;
  const int64_t tile_bytes = (int64_t)tb * kept * sizeof(IT);
  const int64_t region = (tile_bytes + 32 + 15) / 16 * 16;
  unsigned char* sa = smem_raw;
  unsigned char* sb = sa + region;
  unsigned char* so = sb + region;
  const int t = threadIdx.x;
  const int gs = 256 / tb;
  const int lb = t / gs, sub = t % gs;
  const unsigned gmask = gs == 32 ? 0xffffffffu : (((1u << gs) - 1) << ((t & 31) - sub));
  const int64_t ntiles = (nblocks + tb - 1) / tb;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * tb;
    const int nv = (int)min((int64_t)tb, nblocks - b0);
    const int64_t byte0 = b0 * (int64_t)kept * sizeof(IT);
    const int64_t nbytes = (int64_t)nv * kept * sizeof(IT);
    const int misa = (int)(((uintptr_t)a_idx + byte0) & 15);
    const int misb = (int)(((uintptr_t)b_idx + byte0) & 15);
    const int miso = (int)(((uintptr_t)out_idx + byte0) & 15);
    tile_to_smem(sa, reinterpret_cast<const unsigned char*>(a_idx) + byte0, nbytes, misa, t, 256);
    if (MODE == 0) tile_to_smem(sb, reinterpret_cast<const unsigned char*>(b_idx) + byte0, nbytes, misb, t, 256);
    const bool valid = lb < nv;
    const int64_t b = b0 + lb;
    const double na = valid ? load_kind<FK>(a_max, b) : 1.0;
    const double nb = (valid && MODE == 0) ? load_kind<FK>(b_max, b) : 1.0;
    __syncthreads();
    const IT* pa = reinterpret_cast<const IT*>(sa + misa) + (int64_t)lb * kept;
    const IT* pb = reinterpret_cast<const IT*>(sb + misb) + (int64_t)lb * kept;
    IT* po = reinterpret_cast<IT*>(so + miso) + (int64_t)lb * kept;
    const Scale sca = make_scale(na, FK), scb = make_scale(nb, FK);
    const bool safe = na >= 0x1p-900 && na <= 0x1p+900 &&
                      (MODE != 0 || (nb >= 0x1p-900 && nb <= 0x1p+900));
    auto coeff = [&](int k) -> double {
      const int fa = (int)pa[k];
      if (safe) {
        const double xa = div_const(fn_product(fa, sca), r, rinv);
        if (MODE == 0) {
          const int fb = subtract ? -(int)pb[k] : (int)pb[k];
          return __dadd_rn(xa, div_const(fn_product(fb, scb), r, rinv));
        }
        return k == 0 ? __dadd_rn(xa, shift) : xa;
      }
      const double xa = __ddiv_rn(__dmul_rn((double)fa, na), r);
      if (MODE == 0) {
        const double fb = subtract ? -(double)pb[k] : (double)pb[k];
        return __dadd_rn(xa, __ddiv_rn(__dmul_rn(fb, nb), r));
      }
      return k == 0 ? __dadd_rn(xa, shift) : xa;
    };
    // pass 1: block maximum (NaN-propagating by bit order)
    unsigned long long key = 0;
    if (valid)
#pragma unroll 4
      for (int k = sub; k < kept; k += gs) {
        const unsigned long long k2 = (unsigned long long)__double_as_longlong(coeff(k)) & 0x7fffffffffffffffull;
        key = k2 > key ? k2 : key;
      }
    for (int o = gs / 2; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(gmask, key, o, gs);
      key = k2 > key ? k2 : key;
    }
    const double mx = __longlong_as_double((long long)key);
    const double n = round_to_kind<FK>(mx);
    const BinCtx bc = bin_ctx(n, r, mx);
    // pass 2: bin into the output tile (the coefficient is recomputed)
    if (valid) {
      if (sub == 0) store_kind<FK>(out_max, b, n);
#pragma unroll 4
      for (int k = sub; k < kept; k += gs) {
        const double c = coeff(k);
        unsigned nr = 0;
        int q = fast_index32<IT, true>(c, bc.R, (int)r, nr);
        if (nr | !bc.fast) q = (int)bin_exact_ctx(c, bc, r, r);
        po[k] = (IT)q;
      }
    }
    __syncthreads();
    smem_to_tile(reinterpret_cast<unsigned char*>(out_idx) + byte0, so, nbytes, miso, t, 256);
    __syncthreads();  // tiles reused
  }
}

// ------------------------------------------ general add (any block size) --
// Blocks too large for the register-held layouts above (e.g. I64 indices
// with 8x8x8 full masks, I32 32x32 blocks): a warp per block, run-time float
// kinds, two passes over the block (the second re-reads through L1/L2), IEEE
// division and exact binning -- codec.py:337-350 / 253-278 verbatim.
template <typename IT, int MODE>
__global__ void __launch_bounds__(256)
k_add_general(int64_t nblocks, int kept, int fk_a, int fk_b, int fk_out,
              const void* __restrict__ a_max, const IT* __restrict__ a_idx,
              const void* __restrict__ b_max, const IT* __restrict__ b_idx, int subtract,
              double shift, void* __restrict__ out_max, IT* __restrict__ out_idx) {
  constexpr int IK = sizeof(IT) == 1 ? BZ_I8 : sizeof(IT) == 2 ? BZ_I16 : sizeof(IT) == 4 ? BZ_I32 : BZ_I64;
  const double r = radius_f64(IK), bound = clamp_bound_f64(IK);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nblocks; b += nwarps) {
    const int64_t base = b * (int64_t)kept;
    const double na = load_kind_rt(a_max, b, fk_a);
    const double nb = MODE == 0 ? load_kind_rt(b_max, b, fk_b) : 0.0;
    auto coeff = [&](int k) -> double {
      const double xa = __ddiv_rn(__dmul_rn((double)a_idx[base + k], na), r);
      if (MODE == 0) {
        const double fb = subtract ? -(double)b_idx[base + k] : (double)b_idx[base + k];
        return __dadd_rn(xa, __ddiv_rn(__dmul_rn(fb, nb), r));
      }
      return k == 0 ? __dadd_rn(xa, shift) : xa;
    };
    double m = 0.0;
    for (int k = lane; k < kept; k += 32) m = nanmax_abs(m, coeff(k));
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, m, o);
      m = (isnan(t) || isnan(m)) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, t);
    }
    const double n = round_to_kind_rt(m, fk_out);
    if (lane == 0) store_kind_rt(out_max, b, n, fk_out);
    for (int k = lane; k < kept; k += 32) out_idx[base + k] = (IT)bin_exact(coeff(k), n, r, bound);
  }
}

// Register-cached variant of the staged add: GS lanes per block (compile
// time), each lane keeps its CPL coefficients in registers so they are
// computed once; a tile of TB blocks' indices AND maxima is staged in shared
// memory, and the groups of the CTA walk the tile's blocks.
// RED: accumulate the result's squared L2 norm instead of storing it (the
// fused time-series step, as k_add<..., RED>).
template <typename IT, int FK, int MODE, int GS, int CPL, bool RED = false>
__global__ void __launch_bounds__(256, 3)
k_add_tiled(int64_t nblocks, int kept, int tb, const void* __restrict__ a_max,
            const IT* __restrict__ a_idx, const void* __restrict__ b_max,
            const IT* __restrict__ b_idx, int subtract, double shift,
            void* __restrict__ out_max, IT* __restrict__ out_idx,
            double* __restrict__ red_ws = nullptr, double* __restrict__ red_out = nullptr) {
  double red_acc = 0.0;
  constexpr int IK = sizeof(IT) == 1 ? BZ_I8 : BZ_I16;
  using MT = typename std::conditional<FK == BZ_F64, double, float>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const double r = radius_f64(IK), rinv = 1.0 / r;
  const int64_t region = ((int64_t)tb * kept * sizeof(IT) + 32 + 15) / 16 * 16;
  unsigned char* sa = smem_raw;
  unsigned char* sb = sa + region;
  unsigned char* so = sb + region;
  MT* sma = reinterpret_cast<MT*>(so + region);
  MT* smb = sma + tb;
  const int t = threadIdx.x;
  const int lane = t & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  const int64_t ntiles = (nblocks + tb - 1) / tb;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * tb;
    const int nv = (int)min((int64_t)tb, nblocks - b0);
    const int64_t byte0 = b0 * (int64_t)kept * sizeof(IT);
    const int64_t nbytes = (int64_t)nv * kept * sizeof(IT);
    const int misa = (int)(((uintptr_t)a_idx + byte0) & 15);
    const int misb = (int)(((uintptr_t)b_idx + byte0) & 15);
    const int miso = (int)(((uintptr_t)out_idx + byte0) & 15);
    for (int i = t; i < nv; i += 256) {
      sma[i] = reinterpret_cast<const MT*>(a_max)[b0 + i];
      if (MODE == 0) smb[i] = reinterpret_cast<const MT*>(b_max)[b0 + i];
    }
    tile_to_smem(sa, reinterpret_cast<const unsigned char*>(a_idx) + byte0, nbytes, misa, t, 256);
    if (MODE == 0) tile_to_smem(sb, reinterpret_cast<const unsigned char*>(b_idx) + byte0, nbytes, misb, t, 256);
    __syncthreads();
    for (int lb = t / GS; lb < nv; lb += 256 / GS) {
      const int64_t b = b0 + lb;
      const IT* pa = reinterpret_cast<const IT*>(sa + misa) + (int64_t)lb * kept;
      const IT* pb = reinterpret_cast<const IT*>(sb + misb) + (int64_t)lb * kept;
      IT* po = reinterpret_cast<IT*>(so + miso) + (int64_t)lb * kept;
      const double na = (double)sma[lb];
      const double nb = MODE == 0 ? (double)smb[lb] : 1.0;
      const Scale sca = make_scale(na, FK), scb = make_scale(nb, FK);
      const bool safe = na >= 0x1p-900 && na <= 0x1p+900 &&
                        (MODE != 0 || (nb >= 0x1p-900 && nb <= 0x1p+900));
      double c[CPL];
      unsigned long long key = 0;
      // narrow maxima (F32): F * N is exact and fl(F N / r) = fma(F, t_hi,
      // F * t_lo) with t = N / r split in two (bz_add8.cu has the proof)
      constexpr bool NARROW = FK != BZ_F64;
      double tha = 0.0, tla = 0.0, thb = 0.0, tlb = 0.0;
      if (NARROW) {
        tha = div_const(na, r, rinv);
        tla = __fma_rn(-tha, r, na) * rinv;
        if (MODE == 0) {
          thb = div_const(nb, r, rinv);
          tlb = __fma_rn(-thb, r, nb) * rinv;
          if (subtract) { thb = -thb; tlb = -tlb; }
        }
      }
      auto coeffs = [&](auto safe_tag) {
        constexpr bool SAFE = decltype(safe_tag)::value;
        double mxd = 0.0;
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int k = sub + j * GS;
          double cc = 0.0;
          if (k < kept) {
            const int fa = (int)pa[k];
            if constexpr (SAFE && NARROW) {
              const double fad = (double)fa;
              cc = __fma_rn(fad, tha, fad * tla);
              if (MODE == 0) {
                const double fbd = (double)(int)pb[k];
                cc = __dadd_rn(cc, __fma_rn(fbd, thb, fbd * tlb));
              } else if (k == 0) {
                cc = __dadd_rn(cc, shift);
              }
              const double a = fabs(cc);
              mxd = a > mxd ? a : mxd;
            } else if constexpr (SAFE) {
              const double xa = div_const(fn_product(fa, sca), r, rinv);
              if (MODE == 0) {
                const int fb = subtract ? -(int)pb[k] : (int)pb[k];
                cc = __dadd_rn(xa, div_const(fn_product(fb, scb), r, rinv));
              } else {
                cc = k == 0 ? __dadd_rn(xa, shift) : xa;
              }
              const double a = fabs(cc);
              mxd = a > mxd ? a : mxd;
            } else {
              const double xa = spec_coeff_slow((double)fa, na, r);
              if (MODE == 0) {
                const double fb = subtract ? -(double)pb[k] : (double)pb[k];
                cc = __dadd_rn(xa, spec_coeff_slow(fb, nb, r));
              } else {
                cc = k == 0 ? __dadd_rn(xa, shift) : xa;
              }
              const unsigned long long k2 = (unsigned long long)__double_as_longlong(cc) & 0x7fffffffffffffffull;
              key = k2 > key ? k2 : key;
            }
          }
          c[j] = cc;
        }
        if constexpr (SAFE) key = (unsigned long long)__double_as_longlong(mxd);
      };
      if (safe) coeffs(std::true_type{});
      else coeffs(std::false_type{});
#pragma unroll
      for (int o = GS / 2; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(gmask, key, o, GS);
        key = k2 > key ? k2 : key;
      }
      const double mx = __longlong_as_double((long long)key);
      const double n = round_to_kind<FK>(mx);
      const BinCtx bc = bin_ctx(n, r, mx);
      if (!RED && sub == 0) store_kind<FK>(out_max, b, n);
      int q[CPL];
      unsigned nacc = 0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) q[j] = fast_index32<IT, true>(c[j], bc.R, (int)r, nacc);
      if (nacc | !bc.fast) {
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          unsigned nr = 0;
          fast_index32<IT, true>(c[j], bc.R, (int)r, nr);
          if (nr | !bc.fast) q[j] = (int)bin_exact_ctx(c[j], bc, r, r);
        }
      }
      if constexpr (RED) {
        int sq = 0;  // exact: <= CPL * 32767^2 < 2^31 for CPL <= 2
        long long sq64 = 0;
#pragma unroll
        for (int j = 0; j < CPL; ++j)
          if (sub + j * GS < kept) {
            if constexpr (sizeof(IT) == 1) sq += q[j] * q[j];
            else sq64 += (long long)(q[j] * q[j]);
          }
        red_acc = __fma_rn((double)(sq64 + sq) * n, n, red_acc);
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j)
          if (sub + j * GS < kept) po[sub + j * GS] = (IT)q[j];
      }
    }
    __syncthreads();
    if (!RED) smem_to_tile(reinterpret_cast<unsigned char*>(out_idx) + byte0, so, nbytes, miso, t, 256);
    __syncthreads();  // tiles reused
  }
  if constexpr (RED) red_finish(red_acc, red_ws, red_out);
}

template <typename IT>
static int launch_add_t(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                        const void* b_max, const void* b_idx, int subtract, double shift,
                        int mode, void* out_max, void* out_idx, cudaStream_t s, void* out_dc,
                        bool& dc_done) {
  dc_done = true;  // every path below writes the DC plane itself, except the tiled / staged ones
  // int8 indices with float32 maxima, whole 16-byte chunks: bz_add8.cu
  if (sizeof(IT) == 1 && add8_supported(ga, gb, mode, a_idx, b_idx, out_idx) &&
      !getenv("BZC_B200_NO_ADD8"))
    return launch_add8(ga, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s,
                       out_dc);
  // int8 / float32 small unaligned blocks (the C5 low-pass mask): bz_add_small.cu
  if (sizeof(IT) == 1 && add_small_supported(ga, gb, mode, a_max, a_idx, b_max, b_idx, out_idx))
    return launch_add_small(ga, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max,
                            out_idx, out_dc, s);
  constexpr int V = 16 / sizeof(IT);
  const int kept = ga.kept;
  const int vecs = (kept + V - 1) / V;  // chunks per block
  // one lane per block for small blocks; otherwise spread over up to 32 lanes
  int GS = 1, NCH = 1;
  if (vecs <= 4) {
    NCH = vecs <= 1 ? 1 : (vecs <= 2 ? 2 : 4);
  } else {
    while (GS < 32 && GS < vecs) GS <<= 1;
    NCH = (vecs + GS - 1) / GS;
    if (NCH > 4) {  // too large to hold in registers: the general warp-per-block kernel
      dc_done = false;
      const int g = grid_for(ga.nblocks * 32, 256, 4);
      if (mode == 0)
        k_add_general<IT, 0><<<g, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind, gb.float_kind,
                                               ga.float_kind, a_max, (const IT*)a_idx, b_max,
                                               (const IT*)b_idx, subtract, shift, out_max,
                                               (IT*)out_idx);
      else
        k_add_general<IT, 1><<<g, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind, gb.float_kind,
                                               ga.float_kind, a_max, (const IT*)a_idx, b_max,
                                               (const IT*)b_idx, subtract, shift, out_max,
                                               (IT*)out_idx);
      return check_launch("add_general");
    }
    NCH = NCH <= 1 ? 1 : (NCH <= 2 ? 2 : 4);
  }
  const bool vec = ((kept * sizeof(IT)) % 16 == 0) &&
                   !(((uintptr_t)a_idx | (uintptr_t)out_idx | (mode == 0 ? (uintptr_t)b_idx : 0)) & 15);
  const int64_t threads = ga.nblocks * GS;
  // persistent: add_ctas<IT, NCH>() CTAs per SM
  const int grid = grid_for(threads, 256, (sizeof(IT) == 2 && NCH == 2) ? 2 : 3);
  const bool same_fk = ga.float_kind == gb.float_kind || mode != 0;
  // unaligned blocks of I8 / I16 indices: shared-memory staged tiles
  if constexpr (sizeof(IT) <= 2) {
    dc_done = false;
    const int64_t bpb = (int64_t)kept * sizeof(IT);
    if ((bpb % 16) != 0 && kept >= 8 && bpb <= 2048 && same_fk &&
        (ga.float_kind == BZ_F32 || ga.float_kind == BZ_F64)) {
      if (kept <= 512) {  // register-cached tiles
        const int gs = kept <= 128 ? 8 : 32;
        const int cpl = (kept + gs - 1) / gs;
        const int tbt = std::max(256 / gs, (int)(8192 / bpb) / (256 / gs) * (256 / gs));
        const size_t region = (size_t)((tbt * bpb + 32 + 15) / 16 * 16);
        const size_t smem = 3 * region + 2 * (size_t)tbt * (ga.float_kind == BZ_F64 ? 8 : 4);
        const int64_t ntiles = (ga.nblocks + tbt - 1) / tbt;
#define BZ_TT(F, M, G, C)                                                                           \
  {                                                                                                 \
    auto kern = k_add_tiled<IT, F, M, G, C>;                                                        \
    const int occ = occupancy((const void*)kern, 256, smem);                                        \
    const int g2 = (int)std::min<int64_t>(ntiles, (int64_t)kSMs * std::max(occ, 1));                \
    kern<<<g2, 256, smem, s>>>(ga.nblocks, kept, tbt, a_max, (const IT*)a_idx, b_max,               \
                               (const IT*)b_idx, subtract, shift, out_max, (IT*)out_idx, nullptr, nullptr); \
    return check_launch("add_tiled");                                                               \
  }
#define BZ_TC(F, M)                                                     \
  {                                                                     \
    if (gs == 8) {                                                      \
      if (cpl <= 4) BZ_TT(F, M, 8, 4) else if (cpl <= 8) BZ_TT(F, M, 8, 8) \
      else if (cpl <= 12) BZ_TT(F, M, 8, 12) else BZ_TT(F, M, 8, 16)      \
    } else {                                                            \
      if (cpl <= 8) BZ_TT(F, M, 32, 8) else BZ_TT(F, M, 32, 16)         \
    }                                                                   \
  }
        if (ga.float_kind == BZ_F64) { if (mode == 0) BZ_TC(BZ_F64, 0) else BZ_TC(BZ_F64, 1) }
        else { if (mode == 0) BZ_TC(BZ_F32, 0) else BZ_TC(BZ_F32, 1) }
#undef BZ_TC
#undef BZ_TT
      }
      int tb = 256;  // blocks per tile: about 8 KB of indices per operand
      while (tb > 8 && (int64_t)tb * bpb > 8192) tb >>= 1;
      const size_t region = (size_t)((tb * bpb + 32 + 15) / 16 * 16);
      const size_t smem = 3 * region;
      const int64_t ntiles = (ga.nblocks + tb - 1) / tb;
#define BZ_ST(F, M)                                                                                 \
  {                                                                                                 \
    auto kern = k_add_staged<IT, F, M>;                                                             \
    const int occ = occupancy((const void*)kern, 256, smem);                                        \
    const int g2 = (int)std::min<int64_t>(ntiles, (int64_t)kSMs * std::max(occ, 1));                \
    kern<<<g2, 256, smem, s>>>(ga.nblocks, kept, tb, a_max, (const IT*)a_idx, b_max,                \
                               (const IT*)b_idx, subtract, shift, out_max, (IT*)out_idx);           \
    return check_launch("add_staged");                                                              \
  }
      if (ga.float_kind == BZ_F64) { if (mode == 0) BZ_ST(BZ_F64, 0) else BZ_ST(BZ_F64, 1) }
      else { if (mode == 0) BZ_ST(BZ_F32, 0) else BZ_ST(BZ_F32, 1) }
#undef BZ_ST
    }
    dc_done = true;
  }
#define BZ_K(G, N, V, F, M)                                                                    \
  k_add<IT, G, N, V, F, M><<<grid, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind, gb.float_kind, \
                                               ga.float_kind, a_max, (const IT*)a_idx, b_max,  \
                                               (const IT*)b_idx, subtract, shift, mode,        \
                                               out_max, (IT*)out_idx, nullptr, (IT*)out_dc)
#define BZ_LAUNCH(G, N)                                                              \
  do {                                                                               \
    if (vec && same_fk && ga.float_kind == BZ_F64) {                                 \
      if (mode == 0) BZ_K(G, N, true, BZ_F64, 0); else BZ_K(G, N, true, BZ_F64, 1);  \
    } else if (vec && same_fk && ga.float_kind == BZ_F32) {                          \
      if (mode == 0) BZ_K(G, N, true, BZ_F32, 0); else BZ_K(G, N, true, BZ_F32, 1);  \
    } else if (vec) {                                                                \
      if (mode == 0) BZ_K(G, N, true, -1, 0); else BZ_K(G, N, true, -1, 1);          \
    } else {                                                                         \
      if (mode == 0) BZ_K(G, N, false, -1, 0); else BZ_K(G, N, false, -1, 1);        \
    }                                                                                \
  } while (0)
#define BZ_GS(G)                                   \
  case G:                                          \
    if (NCH == 1) BZ_LAUNCH(G, 1);                 \
    else if (NCH == 2) BZ_LAUNCH(G, 2);            \
    else BZ_LAUNCH(G, 4);                          \
    break;
  // GS is 1 (<= 4 chunks per block) or >= 8 (see above)
  switch (GS) { BZ_GS(1) BZ_GS(8) BZ_GS(16) BZ_GS(32) }
#undef BZ_GS
#undef BZ_LAUNCH
#undef BZ_K
  return check_launch("add");
}

// fused l2_norm(subtract(a, b)): the k_add RED variant; ws (zeroed once,
// re-armed by the kernel) holds [counter, result, CTA partials]; the sum of
// squares lands in ws[1] and is copied to `out`
__global__ void k_store_zero(double* out) { *out = 0.0; }

size_t subtract_l2_workspace() { return (size_t)(2 + kSMs * 3) * sizeof(double); }

template <typename IT>
static int launch_subtract_l2_t(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                                const void* b_max, const void* b_idx, double* ws, double* out,
                                cudaStream_t s) {
  constexpr int V = 16 / sizeof(IT);
  const int kept = ga.kept;
  const int vecs = (kept + V - 1) / V;
  int GS = 1, NCH = 1;
  if (vecs <= 4) {
    NCH = vecs <= 1 ? 1 : (vecs <= 2 ? 2 : 4);
  } else {
    while (GS < 32 && GS < vecs) GS <<= 1;
    NCH = (vecs + GS - 1) / GS;
    if (NCH > 4) return BZ_E_UNSUPPORTED;
    NCH = NCH <= 1 ? 1 : (NCH <= 2 ? 2 : 4);
  }
  const bool vec = ((kept * sizeof(IT)) % 16 == 0) && !(((uintptr_t)a_idx | (uintptr_t)b_idx) & 15);
  const int64_t bpb = (int64_t)kept * sizeof(IT);
  if (!vec && kept >= 8 && kept <= 512 && bpb <= 2048 && ga.float_kind == gb.float_kind &&
      (ga.float_kind == BZ_F32 || ga.float_kind == BZ_F64)) {
    // unaligned blocks: register-cached shared-memory tiles (k_add_tiled)
    const int gs = kept <= 128 ? 8 : 32;
    const int cpl = (kept + gs - 1) / gs;
    const int tbt = std::max(256 / gs, (int)(8192 / bpb) / (256 / gs) * (256 / gs));
    const size_t region = (size_t)((tbt * bpb + 32 + 15) / 16 * 16);
    const size_t smem = 3 * region + 2 * (size_t)tbt * (ga.float_kind == BZ_F64 ? 8 : 4);
    const int64_t ntiles = (ga.nblocks + tbt - 1) / tbt;
#define BZ_TT(F, G, C)                                                                              \
  {                                                                                                 \
    auto kern = k_add_tiled<IT, F, 0, G, C, true>;                                                  \
    const int occ = occupancy((const void*)kern, 256, smem);                                        \
    const int g2 = (int)std::min<int64_t>(ntiles, (int64_t)kSMs * std::min(std::max(occ, 1), 3));   \
    kern<<<g2, 256, smem, s>>>(ga.nblocks, kept, tbt, a_max, (const IT*)a_idx, b_max,               \
                               (const IT*)b_idx, 1, 0.0, nullptr, nullptr, ws, out);                \
  }
#define BZ_TC(F)                                                            \
  {                                                                         \
    if (gs == 8) {                                                          \
      if (cpl <= 4) BZ_TT(F, 8, 4) else if (cpl <= 8) BZ_TT(F, 8, 8)        \
      else if (cpl <= 12) BZ_TT(F, 8, 12) else BZ_TT(F, 8, 16)              \
    } else {                                                                \
      if (cpl <= 8) BZ_TT(F, 32, 8) else BZ_TT(F, 32, 16)                   \
    }                                                                       \
  }
    if (ga.float_kind == BZ_F64) BZ_TC(BZ_F64) else BZ_TC(BZ_F32)
#undef BZ_TC
#undef BZ_TT
    return check_launch("subtract_l2_tiled");
  }
  if (!vec || ga.float_kind != gb.float_kind ||
      (ga.float_kind != BZ_F32 && ga.float_kind != BZ_F64))
    return BZ_E_UNSUPPORTED;
  const int grid = grid_for(ga.nblocks * GS, 256, (sizeof(IT) == 2 && NCH == 2) ? 2 : 3);
#define BZ_R(G, N, F)                                                                          \
  k_add<IT, G, N, true, F, 0, true><<<grid, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind,       \
                                                         gb.float_kind, ga.float_kind, a_max,   \
                                                         (const IT*)a_idx, b_max,               \
                                                         (const IT*)b_idx, 1, 0.0, 0, nullptr,  \
                                                         nullptr, ws, nullptr, out)
#define BZ_RF(G, N) \
  do { if (ga.float_kind == BZ_F64) BZ_R(G, N, BZ_F64); else BZ_R(G, N, BZ_F32); } while (0)
#define BZ_RG(G)                               \
  case G:                                      \
    if (NCH == 1) BZ_RF(G, 1);                 \
    else if (NCH == 2) BZ_RF(G, 2);            \
    else BZ_RF(G, 4);                          \
    break;
  switch (GS) { BZ_RG(1) BZ_RG(8) BZ_RG(16) BZ_RG(32) default: return BZ_E_UNSUPPORTED; }
#undef BZ_RG
#undef BZ_RF
#undef BZ_R
  return check_launch("subtract_l2");
}

int launch_subtract_l2(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                       const void* b_max, const void* b_idx, double* out, void* ws,
                       size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < subtract_l2_workspace()) { set_error("subtract_l2: workspace too small"); return BZ_E_WORKSPACE; }
  if (ga.nblocks == 0 || ga.kept == 0) {  // out may be pinned host memory: a store, not a memset
    k_store_zero<<<1, 1, 0, s>>>(out);
    return check_launch("subtract_l2 empty");
  }
  double* w = reinterpret_cast<double*>(ws);
  if (add_small_supported(ga, gb, 0, a_max, a_idx, b_max, b_idx, nullptr))  // bz_add_small.cu
    return launch_subtract_l2_small(ga, a_max, a_idx, b_max, b_idx, w, out, s);
  if (add8_supported(ga, gb, 0, a_idx, b_idx, a_idx) && !getenv("BZC_B200_NO_ADD8"))  // bz_add8.cu
    return launch_subtract_l2_add8(ga, a_max, a_idx, b_max, b_idx, w, out, s);
  int rc = BZ_E_UNSUPPORTED;
  if (ga.index_kind == BZ_I8) rc = launch_subtract_l2_t<int8_t>(ga, gb, a_max, a_idx, b_max, b_idx, w, out, s);
  else if (ga.index_kind == BZ_I16) rc = launch_subtract_l2_t<int16_t>(ga, gb, a_max, a_idx, b_max, b_idx, w, out, s);
  if (rc == BZ_E_UNSUPPORTED) set_error("subtract_l2: configuration not fused (use add + moments)");
  return rc;
}

int launch_add(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
               const void* b_max, const void* b_idx, int subtract, double shift, int mode,
               void* out_max, void* out_idx, cudaStream_t s, void* out_dc) {
  if (ga.nblocks == 0) return BZ_OK;
  if (!ga.keeps_first) out_dc = nullptr;
  // the kernels write the DC plane themselves; the tiled / staged ones and the
  // warp-per-block general kernel are followed by a gather of first coefficients
  bool own = false;
  int rc;
  switch (ga.index_kind) {
    case BZ_I8: rc = launch_add_t<int8_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s, out_dc, own); break;
    case BZ_I16: rc = launch_add_t<int16_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s, out_dc, own); break;
    case BZ_I32: rc = launch_add_t<int32_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s, out_dc, own); break;
    default: rc = launch_add_t<int64_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s, out_dc, own); break;
  }
  if (rc || !out_dc || own) return rc;
  return launch_extract_dc(ga, out_idx, out_dc, s);
}

}  // namespace bz
