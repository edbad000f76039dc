// bz_moments.cu -- one fused pass producing every partial sum the scalar
// reductions need (ops.py:226-348): dot, l2_norm, mean, variance,
// covariance, cosine_similarity and ssim all come from one record.
//
// Per block: exact integer sums  sum Fa*Fb, sum Fa^2, sum Fb^2  (dp4a for
// int8, int32 pairs -> int64 for int16, f64 for wider kinds), the first
// coefficients Fa0, Fb0 and the maxima.  Across blocks (f64):
//   S_xy += Nx*Ny*(sum Fx*Fy - Fx0*Fy0)       (AC part, plain sums)
//   DC_x  = Fx0*Nx, accumulated as pivot-shifted sums per thread and turned
//           into (n, mean, centred co-moment) records merged with Chan's
//           formulas (warp tree -> CTA -> one deterministic final tree).
// Streaming layout: the index arrays are read as a flat stream of 32-byte
// chunks (256-bit LDGs), U per operand in flight per thread, each scaled by
// its block's Na*Nb on the spot (see k_moments_stream).  Blocks smaller than
// one 16-byte vector are staged through shared memory and reduced one block
// per thread.
#include "bz_common.cuh"
#include "bz_kernels.cuh"
#include "bz_tma.cuh"

#include <type_traits>

namespace bz {

struct Rec {
  double n, ma, mb, Mab, Maa, Mbb, Sab, Saa, Sbb;
};

__device__ __forceinline__ Rec rec_zero() { return Rec{0, 0, 0, 0, 0, 0, 0, 0, 0}; }

__device__ __forceinline__ Rec rec_merge(const Rec& x, const Rec& y) {
  if (x.n == 0.0) {
    Rec r = y;
    r.Sab += x.Sab; r.Saa += x.Saa; r.Sbb += x.Sbb;
    return r;
  }
  if (y.n == 0.0) {
    Rec r = x;
    r.Sab += y.Sab; r.Saa += y.Saa; r.Sbb += y.Sbb;
    return r;
  }
  Rec r;
  r.n = x.n + y.n;
  const double inv = __drcp_rn(r.n);  // == 1.0 / n, without the division sequence
  const double da = y.ma - x.ma, db = y.mb - x.mb;
  const double wy = y.n * inv, f = x.n * y.n * inv;
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

// Pivot-shifted accumulator (no divisions on the per-block path).  Every
// thread of a CTA shifts the DC values by the same pivots (the DC values of
// one block of the CTA, set_pivot), so the threads' partials of a CTA are
// plain sums that merge by addition; CTA records merge with Chan's formulas.
struct MomState {
  double cnt = 0, pa = 0, pb = 0, sa = 0, sb = 0, sab = 0, saa = 0, sbb = 0;
  double Sab = 0, Saa = 0, Sbb = 0;

  // PAIR = false: only the a-terms are accumulated (finish() mirrors them)
  template <bool PAIR = true>
  __device__ __forceinline__ void add_block(double iab, double iaa, double ibb, double fa0,
                                            double fb0, double na, double nb, bool dc) {
    Saa = __fma_rn(iaa * na, na, Saa);  // (i*N)*N: an all-zero segment adds 0 even when N*N overflows
    if (PAIR) {
      Sab = __fma_rn(iab * na, nb, Sab);
      Sbb = __fma_rn(ibb * nb, nb, Sbb);
    }
    if (dc) {
      const double dca = fa0 * na;
      const double xa = dca - pa;
      sa += xa;
      saa = __fma_rn(xa, xa, saa);
      if (PAIR) {
        const double dcb = fb0 * nb;
        const double xb = dcb - pb;
        sb += xb;
        sab = __fma_rn(xa, xb, sab);
        sbb = __fma_rn(xb, xb, sbb);
      }
    }
    cnt += 1.0;
  }

  // AC part of one block segment (linear: segments may be added separately)
  template <bool PAIR = true>
  __device__ __forceinline__ void add_ac(double iab, double iaa, double ibb, double na, double nb) {
    Saa = __fma_rn(iaa * na, na, Saa);  // (i*N)*N: an all-zero segment adds 0 even when N*N overflows
    if (PAIR) {
      Sab = __fma_rn(iab * na, nb, Sab);
      Sbb = __fma_rn(ibb * nb, nb, Sbb);
    }
  }
  // once per block: its DC value (when the mask keeps it) and the block count
  template <bool PAIR = true>
  __device__ __forceinline__ void add_dc(double fa0, double fb0, double na, double nb, bool dc) {
    if (dc) {
      const double dca = fa0 * na;
      const double xa = dca - pa;
      sa += xa;
      saa = __fma_rn(xa, xa, saa);
      if (PAIR) {
        const double dcb = fb0 * nb;
        const double xb = dcb - pb;
        sb += xb;
        sab = __fma_rn(xa, xb, sab);
        sbb = __fma_rn(xb, xb, sbb);
      }
    }
    cnt += 1.0;
  }

  __device__ __forceinline__ void set_pivot(double a, double b) {
    pa = isfinite(a) ? a : 0.0;  // a non-finite pivot would poison every
    pb = isfinite(b) ? b : 0.0;  // difference; 0 keeps the reference's propagation
  }

  __device__ __forceinline__ Rec record(bool dc) const {
    Rec r = rec_zero();
    r.n = cnt;
    if (cnt > 0 && dc) {
      const double inv = __drcp_rn(cnt);
      r.ma = pa + sa * inv;
      r.mb = pb + sb * inv;
      r.Mab = sab - sa * sb * inv;
      r.Maa = saa - sa * sa * inv;
      r.Mbb = sbb - sb * sb * inv;
    }
    r.Sab = Sab; r.Saa = Saa; r.Sbb = Sbb;
    return r;
  }
};

// deterministic tree over the records of one CTA (warp tree, then warp 0)
__device__ __forceinline__ Rec cta_tree(Rec r) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Rec y = rec_shfl(r, o);
    r = (lane & o) ? rec_merge(y, r) : rec_merge(r, y);
  }
  __shared__ Rec wrec[32];
  __syncthreads();  // wrec may still be read by a previous call
  if (lane == 0) wrec[threadIdx.x >> 5] = r;
  __syncthreads();
  Rec t = rec_zero();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    t = lane < nw ? wrec[lane] : rec_zero();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Rec y = rec_shfl(t, o);
      t = (lane & o) ? rec_merge(y, t) : rec_merge(t, y);
    }
  }
  return t;  // valid in thread 0
}

__device__ __forceinline__ void store_rec(double* dst, const Rec& t) {
  dst[0] = t.n; dst[1] = t.ma; dst[2] = t.mb; dst[3] = t.Mab; dst[4] = t.Maa;
  dst[5] = t.Mbb; dst[6] = t.Sab; dst[7] = t.Saa; dst[8] = t.Sbb;
}

// Additive tree of N doubles over a CTA (fixed order: deterministic); the
// result is valid in every thread.
template <int N>
__device__ __forceinline__ void sum_tree(double (&v)[N], double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // sh may still be read by a previous call
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) sh[N * w + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = 0.0;
  for (int i = 0; i < nw; ++i)
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] += sh[N * i + k];
}

// The CTA's threads share one pivot: their partials add up (one additive
// tree); thread 0 turns the CTA's sums into a record and stores it; the last
// CTA to arrive (acquire-release ticket) Chan-merges all CTA records in CTA
// order -- deterministic -- writes the final record and re-arms the ticket.
// ws layout: [counter (16 B)][CTA records].
__device__ __forceinline__ void finish(const MomState& st, bool dc, double* __restrict__ ws,
                                       int pair, double* __restrict__ record) {
  unsigned int* counter = reinterpret_cast<unsigned int*>(ws);
  double* recs = ws + 2;
  __shared__ double sh[9 * 32];
  __shared__ bool last;
  double v[9] = {st.cnt, st.sa, st.sb, st.sab, st.saa, st.sbb, st.Sab, st.Saa, st.Sbb};
  sum_tree<9>(v, sh);
  if (threadIdx.x == 0) {
    MomState c = st;
    c.cnt = v[0]; c.sa = v[1]; c.sb = v[2]; c.sab = v[3]; c.saa = v[4]; c.sbb = v[5];
    c.Sab = v[6]; c.Saa = v[7]; c.Sbb = v[8];
    store_rec(recs + blockIdx.x * BZ_RECORD_DOUBLES, c.record(dc));
    last = ticket_arrive(counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  const int per = (gridDim.x + blockDim.x - 1) / blockDim.x;
  Rec m = rec_zero();
  for (int i = threadIdx.x * per; i < min((int)gridDim.x, (int)(threadIdx.x + 1) * per); ++i) {
    const double* s = recs + i * BZ_RECORD_DOUBLES;
    m = rec_merge(m, Rec{__ldcg(s), __ldcg(s + 1), __ldcg(s + 2), __ldcg(s + 3), __ldcg(s + 4),
                         __ldcg(s + 5), __ldcg(s + 6), __ldcg(s + 7), __ldcg(s + 8)});
  }
  Rec f = cta_tree(m);
  if (threadIdx.x == 0) {
    if (!pair) { f.mb = f.ma; f.Mab = f.Maa; f.Mbb = f.Maa; f.Sab = f.Saa; f.Sbb = f.Saa; }
    store_rec(record, f);
    for (int i = 9; i < BZ_RECORD_DOUBLES - 1; ++i) record[i] = 0.0;
    record_complete(record);
    *counter = 0u;  // re-arm for the next launch on this workspace
  }
}

// "Sums" mode (dot / l2, no DC moments): the partials are plain sums
// (block count, S_ab, S_aa, S_bb), merged by addition in a fixed order --
// the reference's own arithmetic (np.dot over the chunks), and a far shorter
// tail than the Chan merge of full records.
__device__ __forceinline__ void finish_sums(double n, double sab, double saa, double sbb,
                                            double* __restrict__ ws, int pair,
                                            double* __restrict__ record) {
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  double* parts = ws + 2;
  __shared__ double sh[4 * 32];
  __shared__ bool last;
  double v[4] = {n, sab, saa, sbb};
  sum_tree<4>(v, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) parts[4 * blockIdx.x + k] = v[k];
    last = ticket_arrive(counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = 0.0;
  const int per = (gridDim.x + blockDim.x - 1) / blockDim.x;
  for (int i = threadIdx.x * per; i < min((int)gridDim.x, (int)(threadIdx.x + 1) * per); ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += __ldcg(parts + 4 * i + k);
  sum_tree<4>(v, sh);
  if (threadIdx.x == 0) {
    record[0] = v[0];
    for (int i = 1; i < 6; ++i) record[i] = 0.0;
    record[6] = pair ? v[1] : v[2];
    record[7] = v[2];
    record[8] = pair ? v[3] : v[2];
    for (int i = 9; i < BZ_RECORD_DOUBLES - 1; ++i) record[i] = 0.0;
    record_complete(record);
    *counter = 0u;  // re-arm
  }
}

// --------------------------------------------------- streaming chunks --
// The index arrays are read as one contiguous stream of CW-byte chunks
// (CW = 32: one 256-bit LDG per chunk; 16 when the base is only 16-byte
// aligned), grid-strided so every load instruction of a warp covers a
// contiguous range, U chunks per operand in flight per thread together with
// the maxima they need (their addresses depend only on the position, so no
// load waits on another).  A chunk holds indices of at most two blocks
// (K >= V): block b for its first element and -- when the next block starts
// inside the chunk at p = K - off < V -- block b + 1 for the rest.  The AC
// sums are linear, so each segment's exact integer sum is scaled by its
// block's Na*Nb and accumulated per thread in f64: no per-block cross-lane
// reduction.  The chunk holding a block's first element also feeds that
// block's DC value into the pivot-shifted moments (MomState).
template <int NW>
struct Chunk {
  unsigned w[NW];
};

template <int NW>
__device__ __forceinline__ Chunk<NW> ld_chunk(const void* p) {
  Chunk<NW> c;
  if constexpr (NW == 8) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3]), "=r"(c.w[4]),
                   "=r"(c.w[5]), "=r"(c.w[6]), "=r"(c.w[7])
                 : "l"(p));
  } else {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p));
    c.w[0] = v.x; c.w[1] = v.y; c.w[2] = v.z; c.w[3] = v.w;
  }
  return c;
}

template <typename IT>
struct SegSums {
  // int8: a segment's products stay below 32 * 127^2 -- 32-bit integer sums
  // and conversions (no 64-bit multiply / I2F.S64 per chunk)
  using T = typename std::conditional<
      sizeof(IT) == 1, int,
      typename std::conditional<(sizeof(IT) <= 2), long long, double>::type>::type;
  T ab[2] = {0, 0}, aa[2] = {0, 0}, bb[2] = {0, 0};
};

// byte mask of word w for the elements [0, p_bytes) of a chunk
__device__ __forceinline__ unsigned word_mask(int p_bytes, int w) {
  const int m = p_bytes - 4 * w;
  return m >= 4 ? 0xffffffffu : (m <= 0 ? 0u : ((1u << (8 * m)) - 1u));
}

// exact sums of the chunk's elements [0, p) (segment 0) and [p, V) (segment 1)
template <typename IT, bool PAIR, int NW, bool SPAN = true>
__device__ __forceinline__ void seg_sums(SegSums<IT>& s, const Chunk<NW>& a, const Chunk<NW>& b,
                                         int p) {
  constexpr int V = NW * 4 / (int)sizeof(IT);
  if constexpr (sizeof(IT) == 1) {
    int a0 = 0, ab0 = 0, b0 = 0, a1 = 0, ab1 = 0, b1 = 0;
    // warp-uniform choice (the seam path is branch-free and also right for
    // p >= V, where its mask is all ones): no divergent double execution
    if (!SPAN || __all_sync(__activemask(), p >= V)) {  // no active lane at a block seam
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        a0 = __dp4a((int)a.w[w], (int)a.w[w], a0);
        if (PAIR) { ab0 = __dp4a((int)a.w[w], (int)b.w[w], ab0); b0 = __dp4a((int)b.w[w], (int)b.w[w], b0); }
      }
    } else {  // branch-free two-segment split (p >= V: the mask is all ones)
      // whole-chunk sums and segment-0 sums (x & m) * y; segment 1 is the
      // difference.  Word w's byte mask covers its bytes below p: the low
      // 8 (p - 4w) bits, clamped to [0, 32] -- one clamped funnel shift
      int ta = 0, tab = 0, tb = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const unsigned m = __funnelshift_lc(0xffffffffu, 0u, (unsigned)max(8 * p - 32 * w, 0));
        const int xa = (int)a.w[w], la = (int)(a.w[w] & m);
        ta = __dp4a(xa, xa, ta);
        a0 = __dp4a(la, xa, a0);
        if (PAIR) {
          const int xb = (int)b.w[w], lb = (int)(b.w[w] & m);
          tab = __dp4a(xa, xb, tab); tb = __dp4a(xb, xb, tb);
          ab0 = __dp4a(la, xb, ab0); b0 = __dp4a(lb, xb, b0);
        }
      }
      a1 = ta - a0;
      if (PAIR) { ab1 = tab - ab0; b1 = tb - b0; }
    }
    s.aa[0] = a0; s.ab[0] = ab0; s.bb[0] = b0;
    s.aa[1] = a1; s.ab[1] = ab1; s.bb[1] = b1;
  } else if constexpr (sizeof(IT) == 2) {
    // pairs of int16 products stay below 2^31 in int32
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int x0 = (int)(int16_t)(a.w[w] & 0xffff), x1 = (int)(int16_t)(a.w[w] >> 16);
      const int y0 = (int)(int16_t)(b.w[w] & 0xffff), y1 = (int)(int16_t)(b.w[w] >> 16);
      const bool h0 = 2 * w >= p, h1 = 2 * w + 1 >= p;
      const long long xx0 = x0 * x0, xx1 = x1 * x1;
      s.aa[0] += (h0 ? 0 : xx0) + (h1 ? 0 : xx1);
      s.aa[1] += (h0 ? xx0 : 0) + (h1 ? xx1 : 0);
      if (PAIR) {
        const long long xy0 = (long long)x0 * y0, xy1 = (long long)x1 * y1;
        const long long yy0 = y0 * y0, yy1 = y1 * y1;
        s.ab[0] += (h0 ? 0 : xy0) + (h1 ? 0 : xy1);
        s.ab[1] += (h0 ? xy0 : 0) + (h1 ? xy1 : 0);
        s.bb[0] += (h0 ? 0 : yy0) + (h1 ? 0 : yy1);
        s.bb[1] += (h0 ? yy0 : 0) + (h1 ? yy1 : 0);
      }
    }
  } else {
    constexpr int WPE = sizeof(IT) / 4;  // words per element
#pragma unroll
    for (int e = 0; e < V; ++e) {
      double da, db;
      if constexpr (WPE == 1) {
        da = (double)(int32_t)a.w[e];
        db = (double)(int32_t)b.w[e];
      } else {
        da = (double)(long long)(((unsigned long long)a.w[2 * e + 1] << 32) | a.w[2 * e]);
        db = (double)(long long)(((unsigned long long)b.w[2 * e + 1] << 32) | b.w[2 * e]);
      }
      const bool hi = e >= p;
      const double d0 = hi ? 0.0 : da, d1 = hi ? da : 0.0;
      s.aa[0] = __fma_rn(d0, d0, s.aa[0]); s.aa[1] = __fma_rn(d1, d1, s.aa[1]);
      if (PAIR) {
        const double e0 = hi ? 0.0 : db, e1 = hi ? db : 0.0;
        s.ab[0] = __fma_rn(d0, e0, s.ab[0]); s.ab[1] = __fma_rn(d1, e1, s.ab[1]);
        s.bb[0] = __fma_rn(e0, e0, s.bb[0]); s.bb[1] = __fma_rn(e1, e1, s.bb[1]);
      }
    }
  }
}

template <int NW>
__device__ __forceinline__ unsigned chunk_word(const Chunk<NW>& c, int i) {
  unsigned r = c.w[0];
#pragma unroll
  for (int k = 1; k < NW; ++k) r = i == k ? c.w[k] : r;
  return r;
}

template <typename IT, int NW>
__device__ __forceinline__ long long chunk_elem(const Chunk<NW>& c, int e) {
  if constexpr (sizeof(IT) == 1) {
    return (long long)(int8_t)((chunk_word(c, e >> 2) >> (8 * (e & 3))) & 0xff);
  } else if constexpr (sizeof(IT) == 2) {
    return (long long)(int16_t)((chunk_word(c, e >> 1) >> (16 * (e & 1))) & 0xffff);
  } else if constexpr (sizeof(IT) == 4) {
    return (long long)(int32_t)chunk_word(c, e);
  } else {
    return (long long)(((unsigned long long)chunk_word(c, 2 * e + 1) << 32) | chunk_word(c, 2 * e));
  }
}

template <int FK>
__device__ __forceinline__ double ld_max(const void* p, int64_t i, int fk) {
  if constexpr (FK >= 0) return load_kind<FK>(p, i);
  else return load_kind_rt(p, i, fk);
}

template <typename IT>
__device__ __forceinline__ typename SegSums<IT>::T sprod(long long x, long long y) {
  if constexpr (sizeof(IT) == 1) return (int)x * (int)y;
  else if constexpr (sizeof(IT) <= 2) return x * y;
  else return (double)x * (double)y;
}

// position (block, offset) of a chunk's first element, advanced incrementally
// (no per-chunk division): a step of `nth` chunks is qs blocks + rs elements
struct ChunkPos {
  int64_t b;
  int off;
  __device__ __forceinline__ void advance(int64_t qs, int rs, int kept) {
    b += qs;
    off += rs;
    if (off >= kept) { off -= kept; ++b; }
  }
};

// FK >= 0: both operands' maxima are of float kind FK (compile time);
// SPAN = false: K is a multiple of V, no chunk crosses a block boundary;
// DC = false: no DC moments at all (keeps_first == 0 or the "sums" mode)
template <typename IT, int NW, int U, bool PAIR, int FK, bool SPAN, bool DC = true>
__global__ void __launch_bounds__(256, (PAIR || sizeof(IT) > 2 || FK < 0) ? 2 : 3)
k_moments_stream(int64_t nblocks, int kept, int keeps_first, int fk_a, int fk_b,
                 const void* __restrict__ a_max, const IT* __restrict__ a_idx,
                 const void* __restrict__ b_max, const IT* __restrict__ b_idx,
                 double* __restrict__ ws, double* __restrict__ record) {
  constexpr int CW = NW * 4;
  constexpr int V = CW / (int)sizeof(IT);
  const int64_t total = nblocks * (int64_t)kept;
  const int64_t nchunks = total / V;  // whole chunks (tail below)
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool dc = DC && keeps_first != 0;
  MomState st;
  if (dc && nblocks > 0) {  // the CTA's pivots: the DC values of one of its blocks
    const int64_t pb_ = blockIdx.x % nblocks;
    const double pva = (double)a_idx[pb_ * kept] * (double)ld_max<FK>(a_max, pb_, fk_a);
    st.set_pivot(pva, PAIR ? (double)b_idx[pb_ * kept] * (double)ld_max<FK>(b_max, pb_, fk_b) : pva);
  }
  const unsigned char* ca = reinterpret_cast<const unsigned char*>(a_idx);
  const unsigned char* cb = reinterpret_cast<const unsigned char*>(b_idx);
  const int64_t qs = (nth * V) / kept;
  const int rs = (int)(nth * V - qs * kept);

  // f32 maxima stay 32-bit until used
  using MT = typename std::conditional<FK == BZ_F32, float, double>::type;
  struct Nm {
    MT a0, b0, a1, b1;
  };
  auto ldn = [&](const void* p, int64_t i, int fk) -> MT {
    if constexpr (FK == BZ_F32) return __ldg(reinterpret_cast<const float*>(p) + i);
    else return ld_max<FK>(p, i, fk);
  };
  auto load_n = [&](const ChunkPos& cp) {
    Nm n;
    n.a0 = ldn(a_max, cp.b, fk_a);
    n.b0 = PAIR ? ldn(b_max, cp.b, fk_b) : n.a0;
    n.a1 = n.b1 = 0;
    if (SPAN && kept - cp.off < V) {
      n.a1 = ldn(a_max, cp.b + 1, fk_a);
      n.b1 = PAIR ? ldn(b_max, cp.b + 1, fk_b) : n.a1;
    }
    return n;
  };
  auto consume = [&](const ChunkPos& cp, const Chunk<NW>& wa, const Chunk<NW>& wb, const Nm& n) {
    const int p = SPAN ? kept - cp.off : V;  // elements of block cp.b in this chunk = min(p, V)
    SegSums<IT> s;
    seg_sums<IT, PAIR, NW, SPAN>(s, wa, wb, p);
    if (cp.off == 0) {  // block b starts here: element 0 is its DC
      const long long x0 = chunk_elem<IT, NW>(wa, 0), y0 = PAIR ? chunk_elem<IT, NW>(wb, 0) : x0;
      if (dc) {
        s.aa[0] -= sprod<IT>(x0, x0);
        if (PAIR) { s.ab[0] -= sprod<IT>(x0, y0); s.bb[0] -= sprod<IT>(y0, y0); }
      }
      st.template add_dc<PAIR>((double)x0, (double)y0, (double)n.a0, (double)n.b0, dc);
    }
    st.template add_ac<PAIR>((double)s.ab[0], (double)s.aa[0], (double)s.bb[0], (double)n.a0,
                             (double)n.b0);
    if (SPAN && p < V) {  // block b + 1 starts at element p
      const long long x0 = chunk_elem<IT, NW>(wa, p), y0 = PAIR ? chunk_elem<IT, NW>(wb, p) : x0;
      if (dc) {
        s.aa[1] -= sprod<IT>(x0, x0);
        if (PAIR) { s.ab[1] -= sprod<IT>(x0, y0); s.bb[1] -= sprod<IT>(y0, y0); }
      }
      st.template add_dc<PAIR>((double)x0, (double)y0, (double)n.a1, (double)n.b1, dc);
      st.template add_ac<PAIR>((double)s.ab[1], (double)s.aa[1], (double)s.bb[1], (double)n.a1,
                               (double)n.b1);
    }
  };

  ChunkPos cp;
  {
    const int64_t e0 = tid * V;
    cp.b = e0 / kept;
    cp.off = (int)(e0 - cp.b * kept);
  }
  int64_t c = tid;
  for (; c + (U - 1) * nth < nchunks; c += U * nth) {
    Chunk<NW> wa[U], wb[U];
    ChunkPos ps[U];
    Nm nm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ps[u] = cp;
      cp.advance(qs, rs, kept);
      wa[u] = ld_chunk<NW>(ca + (c + u * nth) * CW);
      wb[u] = PAIR ? ld_chunk<NW>(cb + (c + u * nth) * CW) : wa[u];
      nm[u] = load_n(ps[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) consume(ps[u], wa[u], wb[u], nm[u]);
  }
  for (; c < nchunks; c += nth) {
    const Chunk<NW> wa = ld_chunk<NW>(ca + c * CW);
    const Chunk<NW> wb = PAIR ? ld_chunk<NW>(cb + c * CW) : wa;
    consume(cp, wa, wb, load_n(cp));
    cp.advance(qs, rs, kept);
  }
  // trailing partial chunk (nblocks*kept not a multiple of V): one thread, scalar
  if (tid == 0 && nchunks * V < total) {
    for (int64_t e = nchunks * V; e < total; ++e) {
      const int64_t b = e / kept;
      const int pos = (int)(e - b * kept);
      const long long x = (long long)a_idx[e], y = PAIR ? (long long)b_idx[e] : x;
      const double na = ld_max<FK>(a_max, b, fk_a), nb = PAIR ? ld_max<FK>(b_max, b, fk_b) : na;
      if (pos == 0) {
        st.template add_dc<PAIR>((double)x, (double)y, na, nb, dc);
        if (dc) continue;
      }
      st.template add_ac<PAIR>((double)sprod<IT>(x, y), (double)sprod<IT>(x, x),
                               (double)sprod<IT>(y, y), na, nb);
    }
  }
  if constexpr (DC) finish(st, dc, ws, PAIR, record);
  else finish_sums(st.cnt, st.Sab, st.Saa, st.Sbb, ws, PAIR, record);
}

// ---------------------------------- unaligned blocks: staged, one per thread --
template <typename IT, bool PAIR>
__global__ void __launch_bounds__(256)
k_moments_staged(int64_t nblocks, int kept, int keeps_first, int fk_a, int fk_b,
                 const void* __restrict__ a_max, const IT* __restrict__ a_idx,
                 const void* __restrict__ b_max, const IT* __restrict__ b_idx,
                 double* __restrict__ ws, double* __restrict__ record) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = blockDim.x;
  const int64_t tile_bytes = (int64_t)T * kept * sizeof(IT);
  unsigned char* sa = smem_raw;
  unsigned char* sb = smem_raw + ((tile_bytes + 32 + 15) / 16) * 16;
  const bool dc = keeps_first != 0;
  MomState st;
  if (dc && nblocks > 0 && kept > 0) {  // the CTA's pivots (see MomState)
    const int64_t pb_ = blockIdx.x % nblocks;
    const double pva = (double)a_idx[pb_ * kept] * load_kind_rt(a_max, pb_, fk_a);
    st.set_pivot(pva, PAIR ? (double)b_idx[pb_ * kept] * load_kind_rt(b_max, pb_, fk_b) : pva);
  }
  const int64_t ntiles = (nblocks + T - 1) / T;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * T;
    const int nvalid = (int)min((int64_t)T, nblocks - b0);
    const int64_t byte0 = b0 * (int64_t)kept * sizeof(IT);
    const int64_t nbytes = (int64_t)nvalid * kept * sizeof(IT);
    const int misa = (int)(((uintptr_t)a_idx + byte0) & 15);
    const int misb = (int)(((uintptr_t)b_idx + byte0) & 15);
    // coalesced 16-byte staging (same helper logic as the fused kernels)
    {
      const unsigned char* g = reinterpret_cast<const unsigned char*>(a_idx) + byte0;
      const int head = misa ? 16 - misa : 0;
      const int h = (int)min((int64_t)head, nbytes);
      for (int i = threadIdx.x; i < h; i += T) sa[misa + i] = g[i];
      const int64_t body = (nbytes - h) / 16;
      for (int64_t i = threadIdx.x; i < body; i += T)
        *reinterpret_cast<uint4*>(sa + misa + h + i * 16) = __ldcs(reinterpret_cast<const uint4*>(g + h) + i);
      for (int64_t i = h + body * 16 + threadIdx.x; i < nbytes; i += T) sa[misa + i] = g[i];
    }
    if (PAIR) {
      const unsigned char* g = reinterpret_cast<const unsigned char*>(b_idx) + byte0;
      const int head = misb ? 16 - misb : 0;
      const int h = (int)min((int64_t)head, nbytes);
      for (int i = threadIdx.x; i < h; i += T) sb[misb + i] = g[i];
      const int64_t body = (nbytes - h) / 16;
      for (int64_t i = threadIdx.x; i < body; i += T)
        *reinterpret_cast<uint4*>(sb + misb + h + i * 16) = __ldcs(reinterpret_cast<const uint4*>(g + h) + i);
      for (int64_t i = h + body * 16 + threadIdx.x; i < nbytes; i += T) sb[misb + i] = g[i];
    }
    __syncthreads();
    if (threadIdx.x < nvalid) {
      const int64_t b = b0 + threadIdx.x;
      const IT* pa = reinterpret_cast<const IT*>(sa + misa) + threadIdx.x * kept;
      const IT* pb = PAIR ? reinterpret_cast<const IT*>(sb + misb) + threadIdx.x * kept : pa;
      long long ab = 0, aa = 0, bbs = 0;
      double fab = 0, faa = 0, fbb = 0;
      for (int k = 0; k < kept; ++k) {
        const long long x = (long long)pa[k], y = (long long)pb[k];
        if constexpr (sizeof(IT) <= 2) {
          aa += x * x; ab += x * y; bbs += y * y;
        } else {
          faa = __fma_rn((double)x, (double)x, faa);
          fab = __fma_rn((double)x, (double)y, fab);
          fbb = __fma_rn((double)y, (double)y, fbb);
        }
      }
      const double fa0 = kept ? (double)pa[0] : 0.0, fb0 = kept ? (double)pb[0] : 0.0;
      const bool d = dc && kept > 0;
      double iab, iaa, ibb;
      if constexpr (sizeof(IT) <= 2) {
        const long long a0 = (long long)fa0, c0 = (long long)fb0;
        iab = (double)(ab - (d ? a0 * c0 : 0));
        iaa = (double)(aa - (d ? a0 * a0 : 0));
        ibb = (double)(bbs - (d ? c0 * c0 : 0));
      } else {
        iab = fab - (d ? fa0 * fb0 : 0.0);
        iaa = faa - (d ? fa0 * fa0 : 0.0);
        ibb = fbb - (d ? fb0 * fb0 : 0.0);
      }
      const double na = load_kind_rt(a_max, b, fk_a);
      const double nb = PAIR ? load_kind_rt(b_max, b, fk_b) : na;
      st.add_block<PAIR>(iab, iaa, ibb, fa0, fb0, na, nb, d);
    }
    __syncthreads();
  }
  finish(st, dc, ws, PAIR, record);
}

// ------------------------------------------------- first coefficients only --
template <typename IT, int U, bool PAIR>
__global__ void __launch_bounds__(256, 2)
k_moments_dc(int64_t nblocks, int64_t kept, int fk_a, int fk_b, const void* __restrict__ a_max,
             const IT* __restrict__ a_idx, const void* __restrict__ b_max,
             const IT* __restrict__ b_idx, double* __restrict__ ws,
             double* __restrict__ record) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  MomState st;
  if (nblocks > 0) {  // the CTA's pivots (see MomState)
    const int64_t pb_ = blockIdx.x % nblocks;
    const double pva = (double)a_idx[pb_ * kept] * load_kind_rt(a_max, pb_, fk_a);
    st.set_pivot(pva, PAIR ? (double)b_idx[pb_ * kept] * load_kind_rt(b_max, pb_, fk_b) : pva);
  }
  for (int64_t bb = tid; bb < nblocks; bb += nth * U) {
    double fa[U], fb[U], na[U], nb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = bb + u * nth;
      const bool ok = b < nblocks;
      fa[u] = ok ? (double)__ldcs(a_idx + b * kept) : 0.0;
      na[u] = ok ? load_kind_rt(a_max, b, fk_a) : 0.0;
      fb[u] = (ok && PAIR) ? (double)__ldcs(b_idx + b * kept) : fa[u];
      nb[u] = (ok && PAIR) ? load_kind_rt(b_max, b, fk_b) : na[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (bb + u * nth < nblocks) st.add_block<PAIR>(0, 0, 0, fa[u], fb[u], na[u], nb[u], true);
  }
  finish(st, true, ws, PAIR, record);
}

// DC plane (mean, ops.py:244-257): each thread owns runs of 16 consecutive
// blocks -- their first coefficients arrive as 16-byte vectors (one per
// 16 / sizeof(IT) blocks) and the float32 / float64 maxima as 16-byte
// vectors too, U runs in flight per thread and one wave of CTAs, so the
// B*(idx+f) bytes stream at full width.  Every DC value x = F0*N is shifted
// by one global pivot p (block 0's value, which every thread loads), so a
// partial is just (count, sum(x-p), sum((x-p)^2)) and partials merge by
// plain addition -- a three-double tree instead of a Chan merge of the full
// record.  The last CTA adds the CTA partials in index order
// (deterministic) and writes the record's entries 0-5 (n, mean, M):
// mean = p + S1/n, M = S2 - S1^2/n.
__device__ __forceinline__ void sum3_tree(double& c, double& s1, double& s2, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // sh may still be read by a previous call
  if (lane == 0) { sh[3 * w] = c; sh[3 * w + 1] = s1; sh[3 * w + 2] = s2; }
  __syncthreads();
  c = s1 = s2 = 0.0;
  for (int i = 0; i < nw; ++i) { c += sh[3 * i]; s1 += sh[3 * i + 1]; s2 += sh[3 * i + 2]; }
}

template <typename IT, int FK, int U>
__global__ void __launch_bounds__(256)
k_moments_plane(int64_t nblocks, const void* __restrict__ maxima, const IT* __restrict__ dc,
                double* __restrict__ ws, double* __restrict__ record) {
  constexpr int RUN = 16;
  constexpr int DCV = RUN * (int)sizeof(IT) / 16;                        // dc vectors per run
  constexpr int MXV = FK == BZ_F64 ? 8 : (FK == BZ_F32 ? 4 : 2);        // maxima vectors per run
  const int64_t nruns = nblocks / RUN;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const double p = nblocks > 0 ? (double)dc[0] * load_kind<FK>(maxima, 0) : 0.0;  // pivot
  double c = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r0 < nruns; r0 += nth * U) {
    uint4 dv[U][DCV], mv[U][MXV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * nth;
      const bool ok = r < nruns;
      const uint4* dsrc = reinterpret_cast<const uint4*>(dc + r * RUN);
      const uint4* msrc = reinterpret_cast<const uint4*>(
          reinterpret_cast<const unsigned char*>(maxima) + r * (16 * MXV));
#pragma unroll
      for (int k = 0; k < DCV; ++k) dv[u][k] = ok ? __ldcs(dsrc + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < MXV; ++k) mv[u][k] = ok ? __ldcs(msrc + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r0 + u * nth >= nruns) break;
      const IT* f0 = reinterpret_cast<const IT*>(dv[u]);
      double a1 = 0.0, a2 = 0.0;  // two chains per run (latency)
#pragma unroll
      for (int e = 0; e < RUN; ++e) {
        double n;
        if constexpr (FK == BZ_F64) n = reinterpret_cast<const double*>(mv[u])[e];
        else if constexpr (FK == BZ_F32) n = (double)reinterpret_cast<const float*>(mv[u])[e];
        else n = load_kind<FK>(mv[u], e);
        const double x = __fma_rn((double)f0[e], n, -p);  // F0*N is exact in f64 only for
        a1 += x;                                          // narrow kinds; fma keeps one rounding
        a2 = __fma_rn(x, x, a2);
      }
      c += (double)RUN;
      s1 += a1;
      s2 += a2;
    }
  }
  // tail blocks (fewer than one run)
  for (int64_t b = nruns * RUN + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += nth) {
    const double x = __fma_rn((double)dc[b], load_kind<FK>(maxima, b), -p);
    c += 1.0;
    s1 += x;
    s2 = __fma_rn(x, x, s2);
  }
  __shared__ double sh[3 * 32];
  __shared__ bool last;
  sum3_tree(c, s1, s2, sh);
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  double* parts = ws + 2;
  if (threadIdx.x == 0) {
    parts[3 * blockIdx.x] = c;
    parts[3 * blockIdx.x + 1] = s1;
    parts[3 * blockIdx.x + 2] = s2;
    last = ticket_arrive(counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  c = s1 = s2 = 0.0;
  const int per = (gridDim.x + blockDim.x - 1) / blockDim.x;
  for (int i = threadIdx.x * per; i < min((int)gridDim.x, (int)(threadIdx.x + 1) * per); ++i) {
    c += __ldcg(parts + 3 * i);
    s1 += __ldcg(parts + 3 * i + 1);
    s2 += __ldcg(parts + 3 * i + 2);
  }
  sum3_tree(c, s1, s2, sh);
  if (threadIdx.x == 0) {
    const double ma = c > 0.0 ? p + s1 / c : 0.0;
    const double m2 = c > 0.0 ? s2 - s1 * (s1 / c) : 0.0;
    record[0] = c;
    record[1] = ma; record[2] = ma;
    record[3] = m2; record[4] = m2; record[5] = m2;
    for (int i = 6; i < BZ_RECORD_DOUBLES - 1; ++i) record[i] = 0.0;
    record_complete(record);
    *counter = 0u;  // re-arm
  }
}

// The same reduction with the plane streamed by bulk copies: one CTA per SM
// owns a contiguous range of blocks (a multiple of 16) and pulls it through
// a ring of PST shared-memory stages (CB blocks of maxima + CB first
// coefficients each, one mbarrier per stage), so every SM keeps PST * CB *
// (f + idx) bytes in flight from the first cycle instead of the registers'
// worth; the threads fold each landed stage into (count, sum(x-p),
// sum((x-p)^2)) and thread 0 refills it.  Block order of the folds and the
// CTA merge is fixed, so the result is deterministic.  Measured (CUDA graph):
// fewer, larger stages win (per-stage cost ~0.3 us), and more threads per
// CTA lose; used for float64 maxima only (see launch_plane_t).
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
namespace plb {
constexpr int NT = 256, CB = 4096, PST = 4;
template <typename IT, int FK>
constexpr size_t smem_bytes() {
  return 64 + (size_t)PST * CB * (sizeof(IT) + (FK == BZ_F64 ? 8 : FK == BZ_F32 ? 4 : 2));
}
}  // namespace plb

template <typename IT, int FK, int CB, int PST, int NT>
__global__ void __launch_bounds__(NT)
k_moments_plane_bulk(int64_t nblocks, const void* __restrict__ maxima, const IT* __restrict__ dc,
                     double* __restrict__ ws, double* __restrict__ record) {
  constexpr int FB = FK == BZ_F64 ? 8 : FK == BZ_F32 ? 4 : 2;
  constexpr int SB = CB * (FB + (int)sizeof(IT));  // stage bytes
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t bar0 = tma::smem_u32(smem_raw);
  unsigned char* st0 = smem_raw + 64;
  const int t = threadIdx.x;
  // this CTA's range [lo, hi), 16-block aligned (16-byte aligned copies)
  const int64_t nruns = nblocks / 16;
  const int64_t per = (nruns + gridDim.x - 1) / gridDim.x * 16;
  const int64_t lo = imin64((int64_t)blockIdx.x * per, nruns * 16);
  const int64_t hi = imin64(lo + per, nruns * 16);
  const int nch = (int)((hi - lo + CB - 1) / CB);
  auto issue = [&](int ch) {  // thread 0
    const int st = ch % PST;
    const int64_t b = lo + (int64_t)ch * CB;
    const uint32_t nb = (uint32_t)imin64(CB, hi - b);
    const uint32_t dst = tma::smem_u32(st0 + st * SB);
    tma::mbar_arrive_expect_tx(bar0 + 8 * st, nb * (FB + (uint32_t)sizeof(IT)));
    tma::bulk_g2s(dst, reinterpret_cast<const unsigned char*>(maxima) + b * FB, nb * FB, bar0 + 8 * st);
    tma::bulk_g2s(dst + CB * FB, dc + b, nb * (uint32_t)sizeof(IT), bar0 + 8 * st);
  };
  if (t == 0) {
    for (int i = 0; i < PST; ++i) tma::mbar_init(bar0 + 8 * i, 1);
    tma::fence_mbar_init();
    for (int ch = 0; ch < min(nch, PST); ++ch) issue(ch);
  }
  const double p = nblocks > 0 ? (double)dc[0] * load_kind<FK>(maxima, 0) : 0.0;  // pivot
  __syncthreads();
  double c = 0.0, s1 = 0.0, s2 = 0.0, s1b = 0.0, s2b = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % PST;
    tma::mbar_wait_spin(bar0 + 8 * st, (uint32_t)(ch / PST) & 1u);
    const unsigned char* sm = st0 + st * SB;
    const IT* f0 = reinterpret_cast<const IT*>(sm + CB * FB);
    const int nb = (int)imin64(CB, hi - (lo + (int64_t)ch * CB));
#pragma unroll 4
    for (int i = t; i < nb; i += NT) {
      const double x = __fma_rn((double)f0[i], load_kind<FK>(sm, i), -p);
      if (i & NT) { s1b += x; s2b = __fma_rn(x, x, s2b); }  // two chains (latency)
      else { s1 += x; s2 = __fma_rn(x, x, s2); }
    }
    c += (double)nb;  // every thread counts the stage; divided out below
    __syncthreads();  // every thread done with this stage
    if (t == 0 && ch + PST < nch) issue(ch + PST);
  }
  c = t == 0 ? c : 0.0;
  s1 += s1b;
  s2 += s2b;
  // tail blocks (fewer than 16), by the last CTA's threads
  if (blockIdx.x == gridDim.x - 1)
    for (int64_t b = nruns * 16 + t; b < nblocks; b += NT) {
      const double x = __fma_rn((double)dc[b], load_kind<FK>(maxima, b), -p);
      c += 1.0;
      s1 += x;
      s2 = __fma_rn(x, x, s2);
    }
  __shared__ double sh[3 * 32];
  __shared__ bool last;
  sum3_tree(c, s1, s2, sh);
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  double* parts = ws + 2;
  if (t == 0) {
    parts[3 * blockIdx.x] = c;
    parts[3 * blockIdx.x + 1] = s1;
    parts[3 * blockIdx.x + 2] = s2;
    last = ticket_arrive(counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  c = s1 = s2 = 0.0;
  const int pc = (gridDim.x + NT - 1) / NT;
  for (int i = t * pc; i < min((int)gridDim.x, (t + 1) * pc); ++i) {
    c += __ldcg(parts + 3 * i);
    s1 += __ldcg(parts + 3 * i + 1);
    s2 += __ldcg(parts + 3 * i + 2);
  }
  sum3_tree(c, s1, s2, sh);
  if (t == 0) {
    const double ma = c > 0.0 ? p + s1 / c : 0.0;
    const double m2 = c > 0.0 ? s2 - s1 * (s1 / c) : 0.0;
    record[0] = c;
    record[1] = ma; record[2] = ma;
    record[3] = m2; record[4] = m2; record[5] = m2;
    for (int i = 6; i < BZ_RECORD_DOUBLES - 1; ++i) record[i] = 0.0;
    record_complete(record);
    *counter = 0u;  // re-arm
  }
}

// ---------------------------------------------------------------- launch --
// The workspace must be zero on first use (the kernels re-arm the counter).
static constexpr int kMaxCTAs = kSMs * 8;

size_t moments_workspace(const Geo& g) {
  (void)g;
  return 16 + (size_t)kMaxCTAs * BZ_RECORD_DOUBLES * sizeof(double);
}

template <typename K>
static int persistent_grid(K kern, int threads, size_t smem, int64_t work_ctas) {
  const int occ = std::max(1, std::min(occupancy((const void*)kern, threads, smem), kMaxCTAs / kSMs));
  return (int)std::max<int64_t>(1, std::min<int64_t>(work_ctas, (int64_t)kSMs * occ));
}

template <typename IT, bool PAIR>
static int launch_typed(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                        const void* b_max, const void* b_idx, int dc_only, double* ws,
                        double* record, cudaStream_t s) {
  const int64_t B = ga.nblocks;
  const int kept = ga.kept;
  // dc_only == 2 ("sums"): no DC moments -- every kept position, the first
  // included, goes into S_* (the record of a mask without the first
  // coefficient); dot / l2 need nothing else
  const int kf = dc_only == 2 ? 0 : ga.keeps_first;
  if (dc_only == 1 && kept > 0) {
    constexpr int U = 8;
    auto kern = k_moments_dc<IT, U, PAIR>;
    const int grid = persistent_grid(kern, 256, 0, (B + 256 * U - 1) / (256 * U));
    kern<<<grid, 256, 0, s>>>(B, (int64_t)kept, ga.float_kind, gb.float_kind, a_max,
                              (const IT*)a_idx, b_max, (const IT*)b_idx, ws, record);
    return check_launch("moments_dc");
  }
  const uintptr_t base = (uintptr_t)a_idx | (PAIR ? (uintptr_t)b_idx : 0);
  // 32-byte chunks (256-bit loads) when aligned; 16-byte otherwise and for 32/64-bit kinds
  const int nw = (sizeof(IT) <= 2 && kept >= 32 / (int)sizeof(IT) && !(base & 31)) ? 8 : 4;
  if (kept >= 16 / (int)sizeof(IT) && !(base & 15)) {
    constexpr int U = PAIR ? 4 : 8;
    const int64_t chunks = B * (int64_t)kept * sizeof(IT) / (4 * nw);
    const int fk = ga.float_kind == gb.float_kind ? ga.float_kind : -1;
#define BZ_MS(NWV, FKV, SP)                                                                      \
  {                                                                                              \
    constexpr int UU = NWV == 8 ? U / 2 : U;                                                     \
    auto kern = kf ? k_moments_stream<IT, NWV, UU, PAIR, FKV, SP, true>                          \
                   : k_moments_stream<IT, NWV, UU, PAIR, FKV, SP, false>;                        \
    const int grid = persistent_grid(kern, 256, 0, (chunks + 256 * UU - 1) / (256 * UU));       \
    kern<<<grid, 256, 0, s>>>(B, kept, kf, ga.float_kind, gb.float_kind, a_max,                  \
                              (const IT*)a_idx, b_max, (const IT*)b_idx, ws, record);            \
    return check_launch("moments_stream");                                                       \
  }
#define BZ_NW(FKV, SPV)                                             \
  if (nw == 8) { BZ_MS(8, FKV, SPV) } else { BZ_MS(4, FKV, SPV) }
    if constexpr (sizeof(IT) <= 2) {
      const bool span8 = kept % (32 / (int)sizeof(IT)) != 0, span4 = kept % (16 / (int)sizeof(IT)) != 0;
      const bool span = nw == 8 ? span8 : span4;
      if (fk == BZ_F32) { if (span) { BZ_NW(BZ_F32, true) } else { BZ_NW(BZ_F32, false) } }
      if (fk == BZ_F64) { if (span) { BZ_NW(BZ_F64, true) } else { BZ_NW(BZ_F64, false) } }
      BZ_NW(-1, true)
    } else {
      BZ_MS(4, -1, true)
    }
#undef BZ_NW
#undef BZ_MS
  }
  // unaligned (or empty) blocks: stage tiles of 256 blocks in shared memory
  const size_t tile = (size_t)256 * kept * sizeof(IT);
  const size_t smem = 2 * (((tile + 32 + 15) / 16) * 16);
  if (smem > 200 * 1024) { set_error("moments: kept block too large to stage"); return BZ_E_UNSUPPORTED; }
  auto kern = k_moments_staged<IT, PAIR>;
  const int grid = persistent_grid(kern, 256, smem, (B + 255) / 256);  // sets the smem limit
  kern<<<grid, 256, smem, s>>>(B, kept, kf, ga.float_kind, gb.float_kind, a_max,
                               (const IT*)a_idx, b_max, (const IT*)b_idx, ws, record);
  return check_launch("moments_staged");
}

template <typename IT>
static int launch_moments_t(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                            const void* b_max, const void* b_idx, int pair, int dc_only,
                            double* record, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < moments_workspace(ga)) { set_error("moments: workspace too small"); return BZ_E_WORKSPACE; }
  double* w = (double*)ws;
  return pair ? launch_typed<IT, true>(ga, gb, a_max, a_idx, b_max, b_idx, dc_only, w, record, s)
              : launch_typed<IT, false>(ga, gb, a_max, a_idx, b_max, b_idx, dc_only, w, record, s);
}

// mean from the DC plane (k_moments_plane when the plane and maxima are
// 16-byte aligned; otherwise the dc_only gather kernel with stride 1)
template <typename IT>
static int launch_plane_t(const Geo& g, const void* maxima, const void* dc, double* ws,
                          double* record, cudaStream_t s) {
  // float64 maxima (10-16 bytes per block): bulk-copied stages (C2 plane
  // 14.7 -> 9.8 us in a CUDA graph); narrower maxima stream faster through
  // the register kernel below (C3 7.2 vs 7.9 us, C5 8.5 vs 10.0 us)
  if (g.float_kind == BZ_F64 && sizeof(IT) <= 4 && !(((uintptr_t)maxima | (uintptr_t)dc) & 15) &&
      g.nblocks >= 16 * 256) {
    auto kern = k_moments_plane_bulk<IT, BZ_F64, plb::CB, plb::PST, plb::NT>;
    constexpr size_t smem = plb::smem_bytes<IT, BZ_F64>();
    (void)occupancy((const void*)kern, plb::NT, smem);  // sets the smem attribute once
    const int grid = (int)std::min<int64_t>(kSMs, (g.nblocks / 16 + 255) / 256);
    kern<<<grid, plb::NT, smem, s>>>(g.nblocks, maxima, (const IT*)dc, ws, record);
    return check_launch("moments_plane_bulk");
  }
  if (!(((uintptr_t)maxima | (uintptr_t)dc) & 15)) {
    const int64_t runs = g.nblocks / 16;
    constexpr int U = 2;
#define BZ_PL(FKV)                                                                             \
  {                                                                                            \
    auto kern = k_moments_plane<IT, FKV, U>;                                                   \
    const int grid = persistent_grid(kern, 256, 0, (runs + 256 * U - 1) / (256 * U));          \
    kern<<<grid, 256, 0, s>>>(g.nblocks, maxima, (const IT*)dc, ws, record);                   \
    return check_launch("moments_plane");                                                      \
  }
    switch (g.float_kind) {
      case BZ_F64: { BZ_PL(BZ_F64) }
      case BZ_F32: { BZ_PL(BZ_F32) }
      case BZ_F16: { BZ_PL(BZ_F16) }
      default: { BZ_PL(BZ_BF16) }
    }
#undef BZ_PL
  }
  constexpr int U = 8;
  auto kern = k_moments_dc<IT, U, false>;
  const int grid = persistent_grid(kern, 256, 0, (g.nblocks + 256 * U - 1) / (256 * U));
  kern<<<grid, 256, 0, s>>>(g.nblocks, (int64_t)1, g.float_kind, g.float_kind, maxima,
                            (const IT*)dc, maxima, (const IT*)dc, ws, record);
  return check_launch("moments_plane");
}

int launch_moments_plane(const Geo& g, const void* maxima, const void* dc, double* record,
                         void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < moments_workspace(g)) { set_error("moments: workspace too small"); return BZ_E_WORKSPACE; }
  if (!g.keeps_first || g.kept == 0) { set_error("moments_plane: mask drops the first coefficient"); return BZ_E_INVALID; }
  double* w = (double*)ws;
  switch (g.index_kind) {
    case BZ_I8: return launch_plane_t<int8_t>(g, maxima, dc, w, record, s);
    case BZ_I16: return launch_plane_t<int16_t>(g, maxima, dc, w, record, s);
    case BZ_I32: return launch_plane_t<int32_t>(g, maxima, dc, w, record, s);
    default: return launch_plane_t<int64_t>(g, maxima, dc, w, record, s);
  }
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
