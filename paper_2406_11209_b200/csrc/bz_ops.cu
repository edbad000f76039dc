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
// Element access for a group of GS lanes handling one block, V elements per
// lane per chunk (V*sizeof(IT) == 16 when vectorised).
template <typename IT>
__device__ __forceinline__ void load_chunk(const IT* __restrict__ p, int64_t base, int k0, int kept,
                                           bool vec, long long (&out)[16 / sizeof(IT)]) {
  constexpr int V = 16 / sizeof(IT);
  if (vec && k0 + V <= kept) {
    uint4 w = __ldg(reinterpret_cast<const uint4*>(p + base + k0));
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < V; ++e) {
      uint32_t word = ws[(e * sizeof(IT)) / 4];
      int sh = (e * sizeof(IT) * 8) % 32;
      if constexpr (sizeof(IT) == 1) out[e] = (int8_t)(word >> sh);
      else if constexpr (sizeof(IT) == 2) out[e] = (int16_t)(word >> sh);
      else if constexpr (sizeof(IT) == 4) out[e] = (int32_t)word;
      else out[e] = (long long)(((unsigned long long)ws[2 * e + 1] << 32) | ws[2 * e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) out[e] = (k0 + e < kept) ? (long long)p[base + k0 + e] : 0;
  }
}

// fl(fl(F * N) / r): Markstein division when N keeps F*N in the normal range
__device__ __forceinline__ double spec_coeff(long long f, double n, double r, double rinv, bool safe) {
  double x = __dmul_rn((double)f, n);
  return safe ? div_const(x, r, rinv) : __ddiv_rn(x, r);
}

// mode 0: a + (+/-)b     mode 1: a + shift at the first coefficient (add_scalar)
template <typename IT, int GS>
__global__ void k_add(int64_t nblocks, int kept, int fk_a, int fk_b, int fk_out,
                      const void* __restrict__ a_max, const IT* __restrict__ a_idx,
                      const void* __restrict__ b_max, const IT* __restrict__ b_idx, int subtract,
                      double shift, int mode, void* __restrict__ out_max,
                      IT* __restrict__ out_idx, bool vec) {
  constexpr int V = 16 / sizeof(IT);
  constexpr int CH = GS * V;  // elements per chunk
  const double r = radius_f64(sizeof(IT) == 1 ? BZ_I8 : sizeof(IT) == 2 ? BZ_I16 : sizeof(IT) == 4 ? BZ_I32 : BZ_I64);
  const double rinv = 1.0 / r;
  const double bound = clamp_bound_f64(sizeof(IT) == 8 ? BZ_I64 : BZ_I32);
  using FB_T = typename std::conditional<sizeof(IT) == 8, int32_t, IT>::type;
  const int lane = threadIdx.x & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GS;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / GS;
  const int nchunks = (kept + CH - 1) / CH;
  const int64_t iters = (nblocks + ngroups - 1) / ngroups;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t b = group + it * ngroups;
    const bool valid = b < nblocks;
    const int64_t base = (valid ? b : 0) * (int64_t)kept;
    double na = 0.0, nb = 0.0;
    if (valid) {
      na = load_kind_rt(a_max, b, fk_a);
      if (mode == 0) nb = load_kind_rt(b_max, b, fk_b);
    }
    const bool safe_a = na >= 0x1p-900 && na <= 0x1p+900;
    const bool safe_b = nb >= 0x1p-900 && nb <= 0x1p+900;
    double c[V];
    unsigned long long key = 0;
    // pass 1 (and only pass when the block fits one chunk): coefficients + max
    for (int ch = 0; ch < nchunks; ++ch) {
      const int k0 = ch * CH + sub * V;
      long long fa[V], fb[V];
      load_chunk<IT>(a_idx, base, k0, valid ? kept : 0, vec, fa);
      if (mode == 0) load_chunk<IT>(b_idx, base, k0, valid ? kept : 0, vec, fb);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double ca = spec_coeff(fa[e], na, r, rinv, safe_a);
        double cc;
        if (mode == 0) {
          double cb = spec_coeff(subtract ? -fb[e] : fb[e], nb, r, rinv, safe_b);
          cc = __dadd_rn(ca, cb);
        } else {
          cc = (k0 + e == 0) ? __dadd_rn(ca, shift) : ca;
        }
        c[e] = cc;
        if (k0 + e < kept) {
          unsigned long long k2 = (unsigned long long)__double_as_longlong(cc) & 0x7fffffffffffffffull;
          key = k2 > key ? k2 : key;
        }
      }
    }
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) {
      unsigned long long k2 = __shfl_xor_sync(gmask, key, o, GS);
      key = k2 > key ? k2 : key;
    }
    const double mx = __longlong_as_double((long long)key);  // NaN-propagating via bit order
    const double n = round_to_kind_rt(mx, fk_out);
    if (valid && sub == 0) store_kind_rt(out_max, b, n, fk_out);
    // exact binning: fast path unless the block is special; near-half -> exact division
    const bool special = !(mx <= 1.7976931348623157e308) || !(n >= 0x1p-1000) || (mx > n * 1.00390625);
    const double R = special ? 0.0 : __ddiv_rn(r, n);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int k0 = ch * CH + sub * V;
      if (nchunks > 1) {  // recompute this chunk's coefficients
        long long fa[V], fb[V];
        load_chunk<IT>(a_idx, base, k0, valid ? kept : 0, vec, fa);
        if (mode == 0) load_chunk<IT>(b_idx, base, k0, valid ? kept : 0, vec, fb);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          double ca = spec_coeff(fa[e], na, r, rinv, safe_a);
          if (mode == 0) {
            double cb = spec_coeff(subtract ? -fb[e] : fb[e], nb, r, rinv, safe_b);
            c[e] = __dadd_rn(ca, cb);
          } else {
            c[e] = (k0 + e == 0) ? __dadd_rn(ca, shift) : ca;
          }
        }
      }
      long long q[V];
      if (special || sizeof(IT) == 8) {
#pragma unroll
        for (int e = 0; e < V; ++e) q[e] = bin_exact(c[e], n, r, bound);
      } else {
        bool near = false;
#pragma unroll
        for (int e = 0; e < V; ++e) q[e] = fast_index<FB_T>(c[e], R, r, near);
        if (near) {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            bool nr = false;
            fast_index<FB_T>(c[e], R, r, nr);
            if (nr) q[e] = bin_exact(c[e], n, r, r);
          }
        }
      }
      if (valid) {
        if (vec && k0 + V <= kept) {
          uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
          for (int e = 0; e < V; ++e) {
            if constexpr (sizeof(IT) == 8) {
              w[2 * e] = (uint32_t)q[e];
              w[2 * e + 1] = (uint32_t)((unsigned long long)q[e] >> 32);
            } else {
              uint32_t bits = (uint32_t)q[e] & (sizeof(IT) == 4 ? 0xffffffffu : ((1u << (8 * sizeof(IT))) - 1));
              w[(e * sizeof(IT)) / 4] |= bits << ((e * sizeof(IT) * 8) % 32);
            }
          }
          __stcs(reinterpret_cast<uint4*>(out_idx + base + k0), make_uint4(w[0], w[1], w[2], w[3]));
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e)
            if (k0 + e < kept) out_idx[base + k0 + e] = (IT)q[e];
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
  int GS = 1;
  while (GS < 32 && GS * V < kept) GS <<= 1;
  bool vec = ((kept * sizeof(IT)) % 16 == 0) && !(((uintptr_t)a_idx | (uintptr_t)out_idx |
                                                     (mode == 0 ? (uintptr_t)b_idx : 0)) & 15);
  int64_t threads = ga.nblocks * GS;
  int grid = grid_for(threads, 256, 8);
#define BZ_GS(G)                                                                              \
  case G:                                                                                     \
    k_add<IT, G><<<grid, 256, 0, s>>>(ga.nblocks, kept, ga.float_kind, gb.float_kind,         \
                                      ga.float_kind, a_max, (const IT*)a_idx, b_max,          \
                                      (const IT*)b_idx, subtract, shift, mode, out_max,       \
                                      (IT*)out_idx, vec);                                     \
    break;
  switch (GS) { BZ_GS(1) BZ_GS(2) BZ_GS(4) BZ_GS(8) BZ_GS(16) BZ_GS(32) }
#undef BZ_GS
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

// ----------------------------------------------------------------- moments --
struct Rec {
  double n, ma, mb, Mab, Maa, Mbb, Sab, Saa, Sbb;
};

__device__ __forceinline__ Rec rec_merge(const Rec& x, const Rec& y) {
  if (x.n == 0.0) return y;
  if (y.n == 0.0) return x;
  Rec r;
  r.n = x.n + y.n;
  const double da = y.ma - x.ma, db = y.mb - x.mb;
  const double wy = y.n / r.n, f = x.n * y.n / r.n;
  r.ma = x.ma + da * wy;
  r.mb = x.mb + db * wy;
  r.Mab = x.Mab + y.Mab + da * db * f;
  r.Maa = x.Maa + y.Maa + da * da * f;
  r.Mbb = x.Mbb + y.Mbb + db * db * f;
  r.Sab = x.Sab + y.Sab;
  r.Saa = x.Saa + y.Saa;
  r.Sbb = x.Sbb + y.Sbb;
  return r;
}

__device__ __forceinline__ Rec rec_shfl(const Rec& x, int o) {
  Rec y;
  y.n = __shfl_xor_sync(0xffffffffu, x.n, o);
  y.ma = __shfl_xor_sync(0xffffffffu, x.ma, o);
  y.mb = __shfl_xor_sync(0xffffffffu, x.mb, o);
  y.Mab = __shfl_xor_sync(0xffffffffu, x.Mab, o);
  y.Maa = __shfl_xor_sync(0xffffffffu, x.Maa, o);
  y.Mbb = __shfl_xor_sync(0xffffffffu, x.Mbb, o);
  y.Sab = __shfl_xor_sync(0xffffffffu, x.Sab, o);
  y.Saa = __shfl_xor_sync(0xffffffffu, x.Saa, o);
  y.Sbb = __shfl_xor_sync(0xffffffffu, x.Sbb, o);
  return y;
}

// integer block sums: exact for I8 (dp4a, int32) and I16 (int32 pairs -> int64)
template <typename IT>
struct Acc {
  long long ab = 0, aa = 0, bb = 0;
  double fab = 0, faa = 0, fbb = 0;  // I32 / I64: f64 products
};

template <typename IT>
__device__ __forceinline__ void acc_chunk(Acc<IT>& acc, const IT* pa, const IT* pb, int64_t base,
                                          int k0, int kept, bool vec, bool pair) {
  constexpr int V = 16 / sizeof(IT);
  if constexpr (sizeof(IT) == 1) {
    if (vec && k0 + V <= kept) {
      uint4 wa = __ldg(reinterpret_cast<const uint4*>(pa + base + k0));
      int sab = 0, saa = 0, sbb = 0;
      saa = __dp4a((int)wa.x, (int)wa.x, saa); saa = __dp4a((int)wa.y, (int)wa.y, saa);
      saa = __dp4a((int)wa.z, (int)wa.z, saa); saa = __dp4a((int)wa.w, (int)wa.w, saa);
      if (pair) {
        uint4 wb = __ldg(reinterpret_cast<const uint4*>(pb + base + k0));
        sab = __dp4a((int)wa.x, (int)wb.x, sab); sab = __dp4a((int)wa.y, (int)wb.y, sab);
        sab = __dp4a((int)wa.z, (int)wb.z, sab); sab = __dp4a((int)wa.w, (int)wb.w, sab);
        sbb = __dp4a((int)wb.x, (int)wb.x, sbb); sbb = __dp4a((int)wb.y, (int)wb.y, sbb);
        sbb = __dp4a((int)wb.z, (int)wb.z, sbb); sbb = __dp4a((int)wb.w, (int)wb.w, sbb);
      }
      acc.ab += sab; acc.aa += saa; acc.bb += sbb;
      return;
    }
  }
  if constexpr (sizeof(IT) == 2) {
    if (vec && k0 + V <= kept) {
      uint4 wa = __ldg(reinterpret_cast<const uint4*>(pa + base + k0));
      uint4 wb = pair ? __ldg(reinterpret_cast<const uint4*>(pb + base + k0)) : wa;
      const uint32_t xa[4] = {wa.x, wa.y, wa.z, wa.w}, xb[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        int a0 = (int)(int16_t)(xa[w] & 0xffff), a1 = (int)(int16_t)(xa[w] >> 16);
        int b0 = (int)(int16_t)(xb[w] & 0xffff), b1 = (int)(int16_t)(xb[w] >> 16);
        acc.aa += (long long)(a0 * a0 + a1 * a1);  // each pair < 2^31
        if (pair) {
          acc.ab += (long long)(a0 * b0) + (long long)(a1 * b1);
          acc.bb += (long long)(b0 * b0 + b1 * b1);
        }
      }
      return;
    }
  }
#pragma unroll
  for (int e = 0; e < V; ++e) {
    if (k0 + e < kept) {
      long long a = (long long)pa[base + k0 + e];
      long long b = pair ? (long long)pb[base + k0 + e] : a;
      if constexpr (sizeof(IT) <= 2) {
        acc.aa += a * a; acc.ab += a * b; acc.bb += b * b;
      } else {
        double da = (double)a, db = (double)b;
        acc.faa = __fma_rn(da, da, acc.faa);
        acc.fab = __fma_rn(da, db, acc.fab);
        acc.fbb = __fma_rn(db, db, acc.fbb);
      }
    }
  }
}

template <typename IT, int GS>
__global__ void __launch_bounds__(256)
k_moments(int64_t nblocks, int kept, int keeps_first, int fk_a, int fk_b,
          const void* __restrict__ a_max, const IT* __restrict__ a_idx,
          const void* __restrict__ b_max, const IT* __restrict__ b_idx, int pair, int dc_only,
          bool vec, double* __restrict__ cta_records) {
  constexpr int V = 16 / sizeof(IT);
  constexpr int CH = GS * V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GS;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / GS;
  const int nchunks = dc_only ? 0 : (kept + CH - 1) / CH;
  const IT* pb = pair ? b_idx : a_idx;

  // thread state (group leaders only): pivot-shifted DC sums + AC sums
  double cnt = 0, pa = 0, pbv = 0, sa = 0, sb = 0, sab = 0, saa = 0, sbb = 0;
  double Sab = 0, Saa = 0, Sbb = 0;
  const int64_t iters = (nblocks + ngroups - 1) / ngroups;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t b = group + it * ngroups;
    const bool valid = b < nblocks;
    const int64_t base = (valid ? b : 0) * (int64_t)kept;
    Acc<IT> acc;
    for (int ch = 0; ch < nchunks; ++ch)
      acc_chunk<IT>(acc, a_idx, pb, base, ch * CH + sub * V, valid ? kept : 0, vec, pair);
    if (nchunks > 0) {
#pragma unroll
      for (int o = GS / 2; o > 0; o >>= 1) {
        acc.ab += __shfl_xor_sync(gmask, acc.ab, o, GS);
        acc.aa += __shfl_xor_sync(gmask, acc.aa, o, GS);
        acc.bb += __shfl_xor_sync(gmask, acc.bb, o, GS);
        if constexpr (sizeof(IT) > 2) {
          acc.fab += __shfl_xor_sync(gmask, acc.fab, o, GS);
          acc.faa += __shfl_xor_sync(gmask, acc.faa, o, GS);
          acc.fbb += __shfl_xor_sync(gmask, acc.fbb, o, GS);
        }
      }
    }
    if (valid && sub == 0) {
      const double na = load_kind_rt(a_max, b, fk_a);
      const double nb = pair ? load_kind_rt(b_max, b, fk_b) : na;
      long long fa0 = 0, fb0 = 0;
      if (keeps_first && kept > 0) {
        fa0 = (long long)a_idx[base];
        fb0 = (long long)pb[base];
      }
      if (!dc_only && kept > 0) {
        double iab, iaa, ibb;
        if constexpr (sizeof(IT) <= 2) {
          iab = (double)(acc.ab - fa0 * fb0);
          iaa = (double)(acc.aa - fa0 * fa0);
          ibb = (double)(acc.bb - fb0 * fb0);
        } else {
          iab = acc.fab - (double)fa0 * (double)fb0;
          iaa = acc.faa - (double)fa0 * (double)fa0;
          ibb = acc.fbb - (double)fb0 * (double)fb0;
        }
        Sab += iab * (na * nb);
        Saa += iaa * (na * na);
        Sbb += ibb * (nb * nb);
      }
      if (keeps_first) {
        const double dca = (double)fa0 * na, dcb = (double)fb0 * nb;
        if (cnt == 0) { pa = dca; pbv = dcb; }
        const double xa = dca - pa, xb = dcb - pbv;
        sa += xa; sb += xb;
        sab = __fma_rn(xa, xb, sab);
        saa = __fma_rn(xa, xa, saa);
        sbb = __fma_rn(xb, xb, sbb);
      }
      cnt += 1.0;
    }
  }
  // thread state -> record
  Rec r;
  r.n = cnt;
  r.ma = cnt > 0 ? pa + sa / cnt : 0.0;
  r.mb = cnt > 0 ? pbv + sb / cnt : 0.0;
  r.Mab = cnt > 0 ? sab - sa * sb / cnt : 0.0;
  r.Maa = cnt > 0 ? saa - sa * sa / cnt : 0.0;
  r.Mbb = cnt > 0 ? sbb - sb * sb / cnt : 0.0;
  r.Sab = Sab; r.Saa = Saa; r.Sbb = Sbb;
  if (!keeps_first) { r.ma = r.mb = r.Mab = r.Maa = r.Mbb = 0.0; }
  // warp tree (fixed order), then CTA
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Rec y = rec_shfl(r, o);
    r = (lane & o) ? rec_merge(y, r) : rec_merge(r, y);
  }
  __shared__ Rec wrec[8];
  if (lane == 0) wrec[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    Rec t = wrec[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = rec_merge(t, wrec[w]);
    double* dst = cta_records + blockIdx.x * BZ_RECORD_DOUBLES;
    dst[0] = t.n; dst[1] = t.ma; dst[2] = t.mb; dst[3] = t.Mab; dst[4] = t.Maa;
    dst[5] = t.Mbb; dst[6] = t.Sab; dst[7] = t.Saa; dst[8] = t.Sbb;
  }
}

__global__ void k_moments_final(const double* __restrict__ cta_records, int ncta, int pair,
                                double* __restrict__ record) {
  if (threadIdx.x != 0) return;
  Rec t{};
  for (int i = 0; i < ncta; ++i) {
    const double* s = cta_records + i * BZ_RECORD_DOUBLES;
    Rec y{s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8]};
    t = rec_merge(t, y);
  }
  if (!pair) { t.mb = t.ma; t.Mab = t.Maa; t.Mbb = t.Maa; t.Sab = t.Saa; t.Sbb = t.Saa; }
  record[0] = t.n; record[1] = t.ma; record[2] = t.mb; record[3] = t.Mab; record[4] = t.Maa;
  record[5] = t.Mbb; record[6] = t.Sab; record[7] = t.Saa; record[8] = t.Sbb;
  for (int i = 9; i < BZ_RECORD_DOUBLES; ++i) record[i] = 0.0;
}

static int moments_grid(const Geo& g, int GS) {
  int64_t threads = std::max<int64_t>(g.nblocks * GS, 1);
  return grid_for(threads, 256, 4);
}

static int pick_gs(int kept, int esize, bool dc_only) {
  if (dc_only) return 1;
  const int V = 16 / esize;
  int GS = 1;
  while (GS < 32 && GS * V < kept) GS <<= 1;
  return GS;
}

size_t moments_workspace(const Geo& g) {
  return (size_t)kSMs * 4 * BZ_RECORD_DOUBLES * sizeof(double);
}

template <typename IT>
static int launch_moments_t(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                            const void* b_max, const void* b_idx, int pair, int dc_only,
                            double* record, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int GS = pick_gs(ga.kept, sizeof(IT), dc_only);
  const int grid = moments_grid(ga, GS);
  if (ws_bytes < (size_t)grid * BZ_RECORD_DOUBLES * sizeof(double)) {
    set_error("moments: workspace too small");
    return BZ_E_WORKSPACE;
  }
  bool vec = ((ga.kept * sizeof(IT)) % 16 == 0) &&
             !(((uintptr_t)a_idx | (pair ? (uintptr_t)b_idx : 0)) & 15);
  double* recs = (double*)ws;
#define BZ_GS(G)                                                                               \
  case G:                                                                                      \
    k_moments<IT, G><<<grid, 256, 0, s>>>(ga.nblocks, ga.kept, ga.keeps_first, ga.float_kind,  \
                                          gb.float_kind, a_max, (const IT*)a_idx, b_max,       \
                                          (const IT*)b_idx, pair, dc_only, vec, recs);         \
    break;
  switch (GS) { BZ_GS(1) BZ_GS(2) BZ_GS(4) BZ_GS(8) BZ_GS(16) BZ_GS(32) }
#undef BZ_GS
  int rc = check_launch("moments");
  if (rc) return rc;
  k_moments_final<<<1, 32, 0, s>>>(recs, grid, pair, record);
  return check_launch("moments_final");
}

int launch_moments(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                   const void* b_max, const void* b_idx, int pair, int dc_only, double* record,
                   void* ws, size_t ws_bytes, cudaStream_t s) {
  switch (ga.index_kind) {
    case BZ_I8: return launch_moments_t<int8_t>(ga, gb, a_max, a_idx, b_max, b_idx, pair, dc_only, record, ws, ws_bytes, s);
    case BZ_I16: return launch_moments_t<int16_t>(ga, gb, a_max, a_idx, b_max, b_idx, pair, dc_only, record, ws, ws_bytes, s);
    case BZ_I32: return launch_moments_t<int32_t>(ga, gb, a_max, a_idx, b_max, b_idx, pair, dc_only, record, ws, ws_bytes, s);
    default: return launch_moments_t<int64_t>(ga, gb, a_max, a_idx, b_max, b_idx, pair, dc_only, record, ws, ws_bytes, s);
  }
}

}  // namespace bz
