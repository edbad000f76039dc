// bz_ops.cu -- compressed-domain operators (ops.py:195-348).
//
//  negate / mul_scalar : elementwise over indices / maxima (ops.py:195-223)
//  add / subtract / add_scalar : one pass over the kept coefficients of both
//      operands with the reference's exact f64 op order, then rebinning
//      (ops.py:178-215, codec.py:337-350) -- bit-exact with the reference.
//  moments : one pass computing every partial sum dot / l2 / mean / variance /
//      covariance / cosine / ssim need (ops.py:226-348), exact integer
//      per-block sums, f64 across blocks, Chan-merged partial records.
#include "bz_common.cuh"
#include "bz_kernels.cuh"

#include <type_traits>

namespace bz {

// ------------------------------------------------------------------ negate --
// mode: -1 negate, 0 zero fill
template <typename IT>
__global__ void k_negate(const IT* __restrict__ in, IT* __restrict__ out, int64_t n, int mode) {
  const int64_t nvec = n * (int64_t)sizeof(IT) / 16;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4* vin = reinterpret_cast<const uint4*>(in);
  uint4* vout = reinterpret_cast<uint4*>(out);
  for (int64_t i = tid; i < nvec; i += stride) {
    uint4 w = mode ? __ldcs(vin + i) : make_uint4(0, 0, 0, 0);
    if (mode) {
      if constexpr (sizeof(IT) == 1) {
        w.x = __vneg4(w.x); w.y = __vneg4(w.y); w.z = __vneg4(w.z); w.w = __vneg4(w.w);
      } else if constexpr (sizeof(IT) == 2) {
        w.x = __vneg2(w.x); w.y = __vneg2(w.y); w.z = __vneg2(w.z); w.w = __vneg2(w.w);
      } else if constexpr (sizeof(IT) == 4) {
        w.x = -w.x; w.y = -w.y; w.z = -w.z; w.w = -w.w;
      } else {
        long long a = -(long long)(((unsigned long long)w.y << 32) | w.x);
        long long b = -(long long)(((unsigned long long)w.w << 32) | w.z);
        w.x = (unsigned)a; w.y = (unsigned)((unsigned long long)a >> 32);
        w.z = (unsigned)b; w.w = (unsigned)((unsigned long long)b >> 32);
      }
    }
    __stcs(vout + i, w);
  }
  for (int64_t i = nvec * (16 / sizeof(IT)) + tid; i < n; i += stride)
    out[i] = mode ? (IT)(-in[i]) : (IT)0;
}

int launch_negate_mode(int ik, const void* in, void* out, int64_t n, int mode, cudaStream_t s) {
  if (n <= 0) return BZ_OK;
  if (((uintptr_t)in | (uintptr_t)out) & 15) { set_error("negate: pointers must be 16-byte aligned"); return BZ_E_INVALID; }
  int64_t work = n * index_kind_bytes(ik) / 16 + 1;
  int grid = grid_for(work, 256, 8);
  switch (ik) {
    case BZ_I8: k_negate<int8_t><<<grid, 256, 0, s>>>((const int8_t*)in, (int8_t*)out, n, mode); break;
    case BZ_I16: k_negate<int16_t><<<grid, 256, 0, s>>>((const int16_t*)in, (int16_t*)out, n, mode); break;
    case BZ_I32: k_negate<int32_t><<<grid, 256, 0, s>>>((const int32_t*)in, (int32_t*)out, n, mode); break;
    default: k_negate<int64_t><<<grid, 256, 0, s>>>((const int64_t*)in, (int64_t*)out, n, mode); break;
  }
  return check_launch("negate");
}

int launch_negate(int ik, const void* in, void* out, int64_t n, cudaStream_t s) {
  return launch_negate_mode(ik, in, out, n, -1, s);
}

// -------------------------------------------------------------- mul_scalar --
// N' = RN_kind(N * |x|)  (ops.py:221)
__global__ void k_scale_maxima(const void* in, void* out, int fk, int64_t n, double ax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_kind_rt(out, i, round_to_kind_rt(__dmul_rn(load_kind_rt(in, i, fk), ax), fk), fk);
}

int launch_mul_scalar(const Geo& g, const void* maxima, const void* indices, double x,
                      void* maxima_out, void* indices_out, cudaStream_t s) {
  if (g.nblocks > 0) {
    k_scale_maxima<<<grid_for(g.nblocks, 256), 256, 0, s>>>(maxima, maxima_out, g.float_kind,
                                                            g.nblocks, fabs(x));
    int rc = check_launch("mul_scalar");
    if (rc) return rc;
  }
  if (indices_out) {
    int mode = x < 0 ? -1 : 0;  // x > 0 aliases; NaN and 0 -> sign 0 (ops.py:222)
    if (x > 0) { set_error("mul_scalar: indices_out must be NULL for x > 0"); return BZ_E_INVALID; }
    return launch_negate_mode(g.index_kind, indices, indices_out, g.nblocks * g.kept, mode, s);
  }
  return BZ_OK;
}

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
  const double biased = __hiloint2double(0x43300000, (int)((unsigned)f ^ 0x80000000u));
  if (s.narrow) return __fma_rn(biased, s.n, s.nbias);
  return __dmul_rn(biased - 4503601774854144.0, s.n);
}
__device__ __forceinline__ double fn_product(long long f, const Scale& s) {
  return __dmul_rn((double)f, s.n);
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
template <typename IT, int GS, int NCH, bool VEC>
__global__ void __launch_bounds__(256, 3)
k_add(int64_t nblocks, int kept, int fk_a, int fk_b, int fk_out,
      const void* __restrict__ a_max, const IT* __restrict__ a_idx,
      const void* __restrict__ b_max, const IT* __restrict__ b_idx, int subtract,
      double shift, int mode, void* __restrict__ out_max, IT* __restrict__ out_idx) {
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
      pna = load_kind_rt(a_max, b, fk_a);
      pnb = mode == 0 ? load_kind_rt(b_max, b, fk_b) : 0.0;
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
      na = load_kind_rt(a_max, b, fk_a);
      nb = mode == 0 ? load_kind_rt(b_max, b, fk_b) : 0.0;
    }
    const Scale sa = make_scale(na, fk_a), sb = make_scale(nb, fk_b);
    const bool safe = na >= 0x1p-900 && na <= 0x1p+900 &&
                      (mode != 0 || (nb >= 0x1p-900 && nb <= 0x1p+900));
    double c[L];
    unsigned long long key = 0;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int k0 = (ch * GS + sub) * V;
      elem_t<IT> fa[V], fb[V];
      if (VEC) {
        unpack_chunk<IT>(ca[ch], fa);
        unpack_chunk<IT>(cb[ch], fb);
      } else {
        load_chunk<IT>(a_idx, base, k0, kept, false, fa);
        if (mode == 0) load_chunk<IT>(b_idx, base, k0, kept, false, fb);
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double cc;
        if (safe) {
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
        if (k0 + e < kept) {
          const unsigned long long k2 = (unsigned long long)__double_as_longlong(cc) & 0x7fffffffffffffffull;
          key = k2 > key ? k2 : key;
        }
      }
    }
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(gmask, key, o, GS);
      key = k2 > key ? k2 : key;
    }
    const double mx = __longlong_as_double((long long)key);  // NaN-propagating via bit order
    const double n = round_to_kind_rt(mx, fk_out);
    if (sub == 0) store_kind_rt(out_max, b, n, fk_out);
    const BinCtx bc = bin_ctx(n, r, mx);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int k0 = (ch * GS + sub) * V;
      int q[V];
      if constexpr (sizeof(IT) <= 2) {
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
      if (VEC && k0 < kept) {
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
  }
}

template <typename IT>
static int launch_add_t(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                        const void* b_max, const void* b_idx, int subtract, double shift,
                        int mode, void* out_max, void* out_idx, cudaStream_t s) {
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
    if (NCH > 4) { set_error("add: kept block too large (%d indices)", kept); return BZ_E_UNSUPPORTED; }
    NCH = NCH <= 1 ? 1 : (NCH <= 2 ? 2 : 4);
  }
  const bool vec = ((kept * sizeof(IT)) % 16 == 0) &&
                   !(((uintptr_t)a_idx | (uintptr_t)out_idx | (mode == 0 ? (uintptr_t)b_idx : 0)) & 15);
  const int64_t threads = ga.nblocks * GS;
  const int grid = grid_for(threads, 256, 3);  // persistent: 3 CTAs per SM
#define BZ_LAUNCH(G, N)                                                                         \
  do {                                                                                          \
    if (vec)                                                                                    \
      k_add<IT, G, N, true><<<grid, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind, gb.float_kind, \
                                                ga.float_kind, a_max, (const IT*)a_idx, b_max,  \
                                                (const IT*)b_idx, subtract, shift, mode,        \
                                                out_max, (IT*)out_idx);                         \
    else                                                                                        \
      k_add<IT, G, N, false><<<grid, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind,               \
                                                 gb.float_kind, ga.float_kind, a_max,           \
                                                 (const IT*)a_idx, b_max, (const IT*)b_idx,     \
                                                 subtract, shift, mode, out_max, (IT*)out_idx); \
  } while (0)
#define BZ_GS(G)                                   \
  case G:                                          \
    if (NCH == 1) BZ_LAUNCH(G, 1);                 \
    else if (NCH == 2) BZ_LAUNCH(G, 2);            \
    else BZ_LAUNCH(G, 4);                          \
    break;
  switch (GS) { BZ_GS(1) BZ_GS(2) BZ_GS(4) BZ_GS(8) BZ_GS(16) BZ_GS(32) }
#undef BZ_GS
#undef BZ_LAUNCH
  return check_launch("add");
}

int launch_add(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
               const void* b_max, const void* b_idx, int subtract, double shift, int mode,
               void* out_max, void* out_idx, cudaStream_t s) {
  if (ga.nblocks == 0) return BZ_OK;
  switch (ga.index_kind) {
    case BZ_I8: return launch_add_t<int8_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s);
    case BZ_I16: return launch_add_t<int16_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s);
    case BZ_I32: return launch_add_t<int32_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s);
    default: return launch_add_t<int64_t>(ga, gb, a_max, a_idx, b_max, b_idx, subtract, shift, mode, out_max, out_idx, s);
  }
}

}  // namespace bz
