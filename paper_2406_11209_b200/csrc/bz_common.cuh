// bz_common.cuh -- shared device helpers for the B200 PyBlaz kernels.
//
// Kind traits, IEEE rounding into narrow float kinds (kinds.py:186-206),
// exact and fast binning (codec.py:253-278), descriptor helpers.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/bzc_b200.h"

namespace bz {

constexpr int kSMs = 148;  // B200

// ------------------------------------------------------------------ errors --
void set_error(const char* fmt, ...);
int check_launch(const char* what);
// Resident CTAs per SM for (kernel, threads, dynamic smem) on the current
// device, cached (the occupancy query and the smem attribute cost
// microseconds of host time per launch); raises the kernel's dynamic-smem
// limit to `smem` once per device when it exceeds 48 KB.
int occupancy(const void* kern, int threads, size_t smem);

// Arrival ticket of a last-CTA reduction: atomic add with acquire-release
// semantics at GPU scope.  The release orders this thread's earlier stores
// (its CTA's partial) before the increment; the acquire, followed by a
// CTA barrier, orders the last CTA's later reads of every partial after it.
// (__threadfence() is a sequentially consistent fence -- MEMBAR.SC.GPU --
// measured at several microseconds per CTA of a short reduction.)
__device__ __forceinline__ unsigned ticket_arrive(unsigned* counter) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
  return old;
}

// The last entry of a reduction record is its completion flag, stored after
// every other entry with a system-scope release: a host polling a record in
// pinned (mapped) memory reads the values once it sees 1.0 (bz_wait_record).
__device__ __forceinline__ void record_complete(double* record) {
  __threadfence_system();
  *reinterpret_cast<volatile double*>(record + BZ_RECORD_DOUBLES - 1) = 1.0;
}

// Fixed-point binning of the factored kernels.  With v = c * r / N and
// |v| < r + 1/2, d = fma(c, r / N, kMagicH) lies in [2^20, 2^21), where one
// unit of the last place is 2^-32, so d's significand holds
// 2^19 + v + 1/2 + 2^-24 rounded once to 32 fraction bits:
//   * high word, low byte: floor(v + 1/2 + 2^-24) mod 256 -- the int8 index
//     rint(v) (two's complement) unless v is within 2^-24 of a rounding half;
//   * low word: the 32-bit fraction of v + 1/2 + 2^-24; it is below
//     kNearHalf = 2^9 exactly when v lies within [-2^-24, 2^-24) of a half
//     (plus the 2^-33 rounding) -- such a block goes to the exact path.
// The constant needs 45 significant bits: exact.  (codec.py:272-277)
constexpr double kMagicH = 1.5 * 1048576.0 + 0.5 + 0x1p-24;
constexpr unsigned kNearHalf = 512u;

// ------------------------------------------------------------- kind traits --
template <int K> struct FloatKind;
template <> struct FloatKind<BZ_BF16> { using T = uint16_t; static constexpr int SIG = 7,  EMIN = -126,  EMAX = 127; };
template <> struct FloatKind<BZ_F16>  { using T = uint16_t; static constexpr int SIG = 10, EMIN = -14,   EMAX = 15; };
template <> struct FloatKind<BZ_F32>  { using T = float;    static constexpr int SIG = 23, EMIN = -126,  EMAX = 127; };
template <> struct FloatKind<BZ_F64>  { using T = double;   static constexpr int SIG = 52, EMIN = -1022, EMAX = 1023; };

inline int float_kind_bytes(int k) { return k == BZ_F64 ? 8 : (k == BZ_F32 ? 4 : 2); }
inline int index_kind_bytes(int k) { return 1 << k; }

template <int K> struct IndexKind;
template <> struct IndexKind<BZ_I8>  { using T = int8_t;  };
template <> struct IndexKind<BZ_I16> { using T = int16_t; };
template <> struct IndexKind<BZ_I32> { using T = int32_t; };
template <> struct IndexKind<BZ_I64> { using T = int64_t; };

// radius r = 2^(b-1)-1 as the reference's float(radius) (kinds.py:128-130; an
// i64 radius rounds to 2^63).  clamp bound = largest f64 <= r (kinds.py:137-147).
__host__ __device__ inline double radius_f64(int ik) {
  switch (ik) {
    case BZ_I8: return 127.0;
    case BZ_I16: return 32767.0;
    case BZ_I32: return 2147483647.0;
    default: return 9223372036854775808.0;
  }
}
__host__ __device__ inline double clamp_bound_f64(int ik) {
  return ik == BZ_I64 ? 9223372036854774784.0 : radius_f64(ik);
}

__device__ __forceinline__ double pow2(int k) {  // exact 2^k, -1022 <= k <= 1023
  return __hiloint2double((k + 1023) << 20, 0);
}

// IEEE round-to-nearest-even of a float64 into kind K, returned as float64.
// Same algorithm as kinds.py:193-206: quantum 2^(max(e-1,emin)-sig),
// rint(x/quantum)*quantum, overflow past max_finite -> signed inf.
template <int K>
__device__ __forceinline__ double round_to_kind(double x) {
  if constexpr (K == BZ_F64) {
    return x;
  } else if constexpr (K == BZ_F32) {
    return (double)__double2float_rn(x);  // cvt.rn.f32.f64 is IEEE RNE incl. subnormals/overflow
  } else {
    using FK = FloatKind<K>;
    if (!isfinite(x) || x == 0.0) return x;
    int e = ((__double2hiint(x) >> 20) & 0x7ff) - 1023;  // floor(log2|x|) for normal x
    int q = (e > FK::EMIN ? e : FK::EMIN) - FK::SIG;
    double r = rint(x * pow2(-q)) * pow2(q);
    const double maxf = (2.0 - 1.0 / (double)(1 << FK::SIG)) * pow2(FK::EMAX);
    if (fabs(r) > maxf) r = copysign(__longlong_as_double(0x7ff0000000000000ll), x);
    return r;
  }
}

__device__ __forceinline__ double round_to_kind_rt(double x, int k) {
  switch (k) {
    case BZ_BF16: return round_to_kind<BZ_BF16>(x);
    case BZ_F16: return round_to_kind<BZ_F16>(x);
    case BZ_F32: return round_to_kind<BZ_F32>(x);
    default: return x;
  }
}

// exact widening of stored values to f64
__device__ __forceinline__ double widen(float v) { return (double)v; }
__device__ __forceinline__ double widen(double v) { return v; }
template <int K>
__device__ __forceinline__ double load_kind(const void* p, int64_t i) {
  if constexpr (K == BZ_F64) return reinterpret_cast<const double*>(p)[i];
  else if constexpr (K == BZ_F32) return (double)reinterpret_cast<const float*>(p)[i];
  else if constexpr (K == BZ_F16) {
    __half h = __ushort_as_half(reinterpret_cast<const uint16_t*>(p)[i]);
    return (double)__half2float(h);
  } else {
    uint32_t b = (uint32_t)reinterpret_cast<const uint16_t*>(p)[i] << 16;
    return (double)__uint_as_float(b);
  }
}
// Predicated streaming loads that leave 0 when `pred` is false, without a
// select on the loaded value (a select -- or a register move -- of a pending
// load result waits for the load, which defeats a prefetch).
__device__ __forceinline__ uint32_t ld_cs_u32_or0(const void* p, bool pred) {
  uint32_t v;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b32 %0, 0;\n"
               " @q ld.global.cs.u32 %0, [%1];\n}\n"
               : "=r"(v) : "l"(p), "r"((int)pred) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_cs_u64_or0(const void* p, bool pred) {
  uint64_t v;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n"
               " @q ld.global.cs.u64 %0, [%1];\n}\n"
               : "=l"(v) : "l"(p), "r"((int)pred) : "memory");
  return v;
}

// widen one stored value (FloatKind<K>::T) to f64
template <int K>
__device__ __forceinline__ double widen_kind(typename FloatKind<K>::T v) {
  return load_kind<K>(&v, 0);
}
__device__ __forceinline__ double load_kind_rt(const void* p, int64_t i, int k) {
  switch (k) {
    case BZ_BF16: return load_kind<BZ_BF16>(p, i);
    case BZ_F16: return load_kind<BZ_F16>(p, i);
    case BZ_F32: return load_kind<BZ_F32>(p, i);
    default: return load_kind<BZ_F64>(p, i);
  }
}
// store a value ALREADY representable in kind K (exact narrowing)
template <int K>
__device__ __forceinline__ void store_kind(void* p, int64_t i, double v) {
  if constexpr (K == BZ_F64) reinterpret_cast<double*>(p)[i] = v;
  else if constexpr (K == BZ_F32) reinterpret_cast<float*>(p)[i] = (float)v;
  else if constexpr (K == BZ_F16) reinterpret_cast<uint16_t*>(p)[i] = __half_as_ushort(__double2half(v));
  else reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)(__float_as_uint((float)v) >> 16);
}
__device__ __forceinline__ void store_kind_rt(void* p, int64_t i, double v, int k) {
  switch (k) {
    case BZ_BF16: store_kind<BZ_BF16>(p, i, v); break;
    case BZ_F16: store_kind<BZ_F16>(p, i, v); break;
    case BZ_F32: store_kind<BZ_F32>(p, i, v); break;
    default: store_kind<BZ_F64>(p, i, v); break;
  }
}

__device__ __forceinline__ int64_t load_index_rt(const void* p, int64_t i, int ik) {
  switch (ik) {
    case BZ_I8: return reinterpret_cast<const int8_t*>(p)[i];
    case BZ_I16: return reinterpret_cast<const int16_t*>(p)[i];
    case BZ_I32: return reinterpret_cast<const int32_t*>(p)[i];
    default: return reinterpret_cast<const int64_t*>(p)[i];
  }
}
__device__ __forceinline__ void store_index_rt(void* p, int64_t i, int64_t v, int ik) {
  switch (ik) {
    case BZ_I8: reinterpret_cast<int8_t*>(p)[i] = (int8_t)v; break;
    case BZ_I16: reinterpret_cast<int16_t*>(p)[i] = (int16_t)v; break;
    case BZ_I32: reinterpret_cast<int32_t*>(p)[i] = (int32_t)v; break;
    default: reinterpret_cast<int64_t*>(p)[i] = v; break;
  }
}

// NaN-propagating max of |x| (np.max(np.abs(...)) semantics, codec.py:269)
__device__ __forceinline__ double nanmax_abs(double m, double x) {
  double a = fabs(x);
  if (isnan(a) || isnan(m)) return __longlong_as_double(0x7ff8000000000000ll);
  return a > m ? a : m;
}

// Exact reference binning of one coefficient (codec.py:272-278):
// q = C / N (IEEE), non-finite -> 0, clip(rint(q * r), +-bound).
__device__ __forceinline__ int64_t bin_exact(double c, double n, double r, double bound) {
  double q = __ddiv_rn(c, n);
  if (!isfinite(q)) q = 0.0;
  double v = rint(__dmul_rn(q, r));
  v = fmin(fmax(v, -bound), bound);
  return (int64_t)v;
}

// Correctly rounded x / r for a constant divisor r using Markstein's
// correction: q0 = x*y (y = RN(1/r)), e = x - q0*r exact by FMA,
// q = RN(q0 + e*y).  Valid for finite x with |x| not in the subnormal
// range (callers guarantee it per block; otherwise use __ddiv_rn).
__device__ __forceinline__ double div_const(double x, double r, double y) {
  double q0 = __dmul_rn(x, y);
  double e = __fma_rn(-q0, r, x);
  return __fma_rn(e, y, q0);
}

// Fast binning (see bz_fast_compress.cu): v = c * R, R = r / N, rounded once
// to K-bit fixed point by an FMA against 1.5*2^(52-K); |v| <= r(1+2^-8) keeps
// v*2^K inside the magic binade.  `near` flags fractions within W units of
// one half, which the caller recomputes exactly with bin_exact.
template <typename IT> struct FastBin;
template <> struct FastBin<int8_t>  { static constexpr int K = 24; static constexpr int W = 1; using Fix = int32_t; };
template <> struct FastBin<int16_t> { static constexpr int K = 15; static constexpr int W = 1; using Fix = int32_t; };
template <> struct FastBin<int32_t> { static constexpr int K = 19; static constexpr int W = 2; using Fix = int64_t; };

template <typename IT>
__device__ __forceinline__ int fast_index(double c, double R, double rr, bool& near) {
  using FB = FastBin<IT>;
  constexpr double MAGIC = 1.5 * (double)(1ll << (52 - FB::K));
  double t = __fma_rn(c, R, MAGIC);
  typename FB::Fix fx;
  if constexpr (sizeof(typename FB::Fix) == 4) {
    fx = (int32_t)__double2loint(t);
  } else {
    fx = (int64_t)(__double_as_longlong(t) & ((1ll << 52) - 1)) - (1ll << 51);
  }
  constexpr typename FB::Fix HALF = (typename FB::Fix)1 << (FB::K - 1);
  constexpr typename FB::Fix MASK = ((typename FB::Fix)1 << FB::K) - 1;
  typename FB::Fix frac = fx & MASK;
  near = near || ((frac - (HALF - FB::W)) >= 0 && (frac - (HALF - FB::W)) <= 2 * FB::W);
  long long idx = (long long)((fx + HALF) >> FB::K);
  long long ir = (long long)rr;
  idx = idx > ir ? ir : (idx < -ir ? -ir : idx);
  return (int)idx;
}

// 32-bit fixed-point variant for I8 / I16: no 64-bit integer ops; `nacc`
// collects a "near one half" flag; CLAMP only where the stored maximum can
// round far enough below the true maximum for |v| to reach r + 1/2.
template <typename IT, bool CLAMP>
__device__ __forceinline__ int fast_index32(double c, double R, int ir, unsigned& nacc) {
  using FB = FastBin<IT>;
  static_assert(sizeof(typename FB::Fix) == 4, "32-bit fixed point only");
  constexpr double MAGIC = 1.5 * (double)(1ll << (52 - FB::K));
  constexpr unsigned HALF = 1u << (FB::K - 1);
  constexpr unsigned MASK = (1u << FB::K) - 1;
  const int fx = __double2loint(__fma_rn(c, R, MAGIC));
  nacc |= (unsigned)((((unsigned)fx & MASK) - (HALF - FB::W)) <= 2u * FB::W);
  int idx = (fx + (int)HALF) >> FB::K;
  if (CLAMP) idx = min(max(idx, -ir), ir);
  return idx;
}

// Per-block binning context: everything the exact reference binning
// rint(fl(C / N) * r) (codec.py:272-277) needs, without IEEE division calls.
//  * N = 0, inf or NaN: every C / N is non-finite or 0 -> every index is 0.
//  * otherwise C / N = fl(C*s / (N*s)) with s a power of two lifting a tiny N
//    into the normal range, computed by Markstein's correction with the
//    correctly rounded reciprocal y = RN(1 / (N*s)).
//  * R ~ r / N feeds the fixed-point fast path (its error is covered by the
//    near-half window, so it need not be correctly rounded); mx is the true
//    block maximum the stored N was rounded from.
struct BinCtx {
  double R, ns, y, s;
  bool zero;  // all indices are 0
  bool fast;  // fast fixed-point path valid (N normal, not tiny)
};

// CLAMP = false callers (no index clamp in the fixed-point path) need |v| < r + 1/2,
// i.e. a stored maximum within 2^-20 of the true one (F32 normal / F64 maxima).
template <bool CLAMP = true>
__device__ __forceinline__ BinCtx bin_ctx(double n, double rr, double mx) {
  BinCtx b;
  b.zero = !(n > 0.0) || !(n <= 1.7976931348623157e308);
  b.s = n < 0x1p-900 ? 0x1p+600 : 1.0;
  b.ns = b.zero ? 1.0 : n * b.s;
  b.y = __drcp_rn(b.ns);
  b.R = rr * b.y * b.s;
  // fast path: |v| <= r(1+2^-8) keeps the fixed point in range (a stored
  // maximum rounded far below the true one -- narrow-kind subnormals -- is not)
  b.fast = !b.zero && n >= 0x1p-900 && mx <= n * (CLAMP ? 1.00390625 : 1.00000095367431640625);
  return b;
}

__device__ __forceinline__ long long bin_exact_ctx(double c, const BinCtx& b, double rr,
                                                   double bound) {
  if (b.zero) return 0;
  double q = div_const(c * b.s, b.ns, b.y);
  if (!isfinite(q)) q = 0.0;
  double v = rint(__dmul_rn(q, rr));
  v = fmin(fmax(v, -bound), bound);
  return (long long)v;
}

// pack 16 bytes of indices (I8: 16 values, I16: 8 values) with PRMT
template <typename IT>
__device__ __forceinline__ uint4 pack16(const int* q) {
  uint4 w;
  if constexpr (sizeof(IT) == 1) {
    unsigned o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned lo = __byte_perm((unsigned)q[4 * k], (unsigned)q[4 * k + 1], 0x0040);
      const unsigned hi = __byte_perm((unsigned)q[4 * k + 2], (unsigned)q[4 * k + 3], 0x0040);
      o[k] = __byte_perm(lo, hi, 0x5410);
    }
    w = make_uint4(o[0], o[1], o[2], o[3]);
  } else if constexpr (sizeof(IT) == 2) {
    w = make_uint4(__byte_perm((unsigned)q[0], (unsigned)q[1], 0x5410),
                   __byte_perm((unsigned)q[2], (unsigned)q[3], 0x5410),
                   __byte_perm((unsigned)q[4], (unsigned)q[5], 0x5410),
                   __byte_perm((unsigned)q[6], (unsigned)q[7], 0x5410));
  } else {
    w = make_uint4((unsigned)q[0], (unsigned)q[1], (unsigned)q[2], (unsigned)q[3]);
  }
  return w;
}

// ------------------------------------------------------------ descriptors --
struct Geo {  // device-side copy of the layout geometry
  int ndim;
  int64_t shape[BZ_MAX_DIMS];
  int32_t block[BZ_MAX_DIMS];
  int64_t grid[BZ_MAX_DIMS];
  int64_t stride[BZ_MAX_DIMS];   // dense element strides
  int64_t nblocks;
  int32_t bsize;                 // prod(block)
  int32_t kept;
  int32_t keeps_first;
  int32_t float_kind, index_kind, transform;
  const int32_t* kept_pos;
  const int32_t* rank;
  const double* matrices;
  const double* matrices_host;
  int32_t mat_off[BZ_MAX_DIMS];  // offset of axis a's matrix in `matrices`
};

inline Geo make_geo(const bz_layout* L) {
  Geo g{};
  g.ndim = L->ndim;
  int64_t s = 1;
  for (int a = L->ndim - 1; a >= 0; --a) { g.stride[a] = s; s *= L->shape[a]; }
  g.nblocks = 1;
  g.bsize = 1;
  int off = 0;
  for (int a = 0; a < L->ndim; ++a) {
    g.shape[a] = L->shape[a];
    g.block[a] = L->block[a];
    g.grid[a] = L->grid[a];
    g.nblocks *= L->grid[a];
    g.bsize *= L->block[a];
    g.mat_off[a] = off;
    off += L->block[a] * L->block[a];
  }
  g.kept = L->kept;
  g.keeps_first = L->keeps_first;
  g.float_kind = L->float_kind;
  g.index_kind = L->index_kind;
  g.transform = L->transform;
  g.kept_pos = L->kept_pos;
  g.rank = L->rank;
  g.matrices = L->matrices;
  g.matrices_host = L->matrices_host;
  return g;
}

inline int64_t dense_count(const bz_layout* L) {
  int64_t n = 1;
  for (int a = 0; a < L->ndim; ++a) n *= L->shape[a];
  return n;
}
inline int64_t block_count(const bz_layout* L) {
  int64_t n = 1;
  for (int a = 0; a < L->ndim; ++a) n *= L->grid[a];
  return n;
}
inline int block_size(const bz_layout* L) {
  int n = 1;
  for (int a = 0; a < L->ndim; ++a) n *= L->block[a];
  return n;
}

// dense offset of intrablock position `pos` (row-major) of block `b`, or -1 if padding
__device__ __forceinline__ int64_t element_offset(const Geo& g, int64_t b, int pos) {
  int64_t off = 0;
  for (int a = g.ndim - 1; a >= 0; --a) {
    int64_t gb = b % g.grid[a];
    b /= g.grid[a];
    int n = pos % g.block[a];
    pos /= g.block[a];
    int64_t c = gb * g.block[a] + n;
    if (c >= g.shape[a]) return -1;
    off += c * g.stride[a];
  }
  return off;
}

inline int grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t b = (work + threads - 1) / threads;
  int64_t cap = (int64_t)kSMs * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace bz
