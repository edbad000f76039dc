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
// Streaming layout: GS lanes share a block, each loading 16-byte vectors;
// every group works on U consecutive blocks per iteration so U*16 bytes per
// lane and operand are in flight.  Blocks whose kept indices are not a whole
// number of 16-byte vectors (e.g. C5's 66-byte blocks) are staged through
// shared memory in coalesced tiles and reduced one block per thread.
#include "bz_common.cuh"
#include "bz_kernels.cuh"

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
  const double inv = 1.0 / r.n;
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

// pivot-shifted per-thread accumulator (no divisions on the per-block path)
struct MomState {
  double cnt = 0, pa = 0, pb = 0, sa = 0, sb = 0, sab = 0, saa = 0, sbb = 0;
  double Sab = 0, Saa = 0, Sbb = 0;

  // PAIR = false: only the a-terms are accumulated (finish() mirrors them)
  template <bool PAIR = true>
  __device__ __forceinline__ void add_block(double iab, double iaa, double ibb, double fa0,
                                            double fb0, double na, double nb, bool dc) {
    Saa = __fma_rn(iaa, na * na, Saa);
    if (PAIR) {
      Sab = __fma_rn(iab, na * nb, Sab);
      Sbb = __fma_rn(ibb, nb * nb, Sbb);
    }
    if (dc) {
      const double dca = fa0 * na;
      if (cnt == 0.0) pa = dca;
      const double xa = dca - pa;
      sa += xa;
      saa = __fma_rn(xa, xa, saa);
      if (PAIR) {
        const double dcb = fb0 * nb;
        if (cnt == 0.0) pb = dcb;
        const double xb = dcb - pb;
        sb += xb;
        sab = __fma_rn(xa, xb, sab);
        sbb = __fma_rn(xb, xb, sbb);
      }
    }
    cnt += 1.0;
  }

  __device__ __forceinline__ Rec record(bool dc) const {
    Rec r = rec_zero();
    r.n = cnt;
    if (cnt > 0 && dc) {
      const double inv = 1.0 / cnt;
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

// Every CTA stores its record; the last CTA to finish (atomic ticket) merges
// all of them in CTA order -- deterministic -- writes the final record and
// re-arms the ticket counter.  ws layout: [counter (16 B)][CTA records].
__device__ __forceinline__ void finish(Rec r, double* __restrict__ ws, int pair,
                                       double* __restrict__ record) {
  unsigned int* counter = reinterpret_cast<unsigned int*>(ws);
  double* recs = ws + 2;
  Rec t = cta_tree(r);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    store_rec(recs + blockIdx.x * BZ_RECORD_DOUBLES, t);
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
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
    for (int i = 9; i < BZ_RECORD_DOUBLES; ++i) record[i] = 0.0;
    *counter = 0u;  // re-arm for the next launch on this workspace
  }
}

// ------------------------------------------------ integer block partials --
template <typename IT>
struct Part {  // exact per-lane partial sums of one block (f64 for 32/64-bit kinds)
  using T = typename std::conditional<(sizeof(IT) <= 2), long long, double>::type;
  T ab = 0, aa = 0, bb = 0;
};

template <typename IT, bool PAIR>
__device__ __forceinline__ void part_vec(Part<IT>& p, const uint4& wa, const uint4& wb) {
  if constexpr (sizeof(IT) == 1) {
    int saa = 0, sab = 0, sbb = 0;
    saa = __dp4a((int)wa.x, (int)wa.x, saa); saa = __dp4a((int)wa.y, (int)wa.y, saa);
    saa = __dp4a((int)wa.z, (int)wa.z, saa); saa = __dp4a((int)wa.w, (int)wa.w, saa);
    if (PAIR) {
      sab = __dp4a((int)wa.x, (int)wb.x, sab); sab = __dp4a((int)wa.y, (int)wb.y, sab);
      sab = __dp4a((int)wa.z, (int)wb.z, sab); sab = __dp4a((int)wa.w, (int)wb.w, sab);
      sbb = __dp4a((int)wb.x, (int)wb.x, sbb); sbb = __dp4a((int)wb.y, (int)wb.y, sbb);
      sbb = __dp4a((int)wb.z, (int)wb.z, sbb); sbb = __dp4a((int)wb.w, (int)wb.w, sbb);
    }
    p.aa += saa; p.ab += sab; p.bb += sbb;
  } else if constexpr (sizeof(IT) == 2) {
    const uint32_t xa[4] = {wa.x, wa.y, wa.z, wa.w}, xb[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int a0 = (int)(int16_t)(xa[w] & 0xffff), a1 = (int)(int16_t)(xa[w] >> 16);
      p.aa += (long long)(a0 * a0 + a1 * a1);  // < 2^31 per pair
      if (PAIR) {
        const int b0 = (int)(int16_t)(xb[w] & 0xffff), b1 = (int)(int16_t)(xb[w] >> 16);
        p.ab += (long long)(a0 * b0) + (long long)(a1 * b1);
        p.bb += (long long)(b0 * b0 + b1 * b1);
      }
    }
  } else if constexpr (sizeof(IT) == 4) {
    const int32_t xa[4] = {(int32_t)wa.x, (int32_t)wa.y, (int32_t)wa.z, (int32_t)wa.w};
    const int32_t xb[4] = {(int32_t)wb.x, (int32_t)wb.y, (int32_t)wb.z, (int32_t)wb.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const double da = (double)xa[w], db = (double)xb[w];
      p.aa = __fma_rn(da, da, p.aa);
      if (PAIR) { p.ab = __fma_rn(da, db, p.ab); p.bb = __fma_rn(db, db, p.bb); }
    }
  } else {
    const long long a0 = (long long)(((unsigned long long)wa.y << 32) | wa.x);
    const long long a1 = (long long)(((unsigned long long)wa.w << 32) | wa.z);
    const long long b0 = (long long)(((unsigned long long)wb.y << 32) | wb.x);
    const long long b1 = (long long)(((unsigned long long)wb.w << 32) | wb.z);
    p.aa = __fma_rn((double)a0, (double)a0, p.aa);
    p.aa = __fma_rn((double)a1, (double)a1, p.aa);
    if (PAIR) {
      p.ab = __fma_rn((double)a0, (double)b0, p.ab);
      p.ab = __fma_rn((double)a1, (double)b1, p.ab);
      p.bb = __fma_rn((double)b0, (double)b0, p.bb);
      p.bb = __fma_rn((double)b1, (double)b1, p.bb);
    }
  }
}

template <typename IT>
__device__ __forceinline__ long long first_elem(const uint4& w) {
  if constexpr (sizeof(IT) == 1) return (long long)(int8_t)(w.x & 0xff);
  else if constexpr (sizeof(IT) == 2) return (long long)(int16_t)(w.x & 0xffff);
  else if constexpr (sizeof(IT) == 4) return (long long)(int32_t)w.x;
  else return (long long)(((unsigned long long)w.y << 32) | w.x);
}

template <typename IT, bool PAIR>
__device__ __forceinline__ void part_reduce(Part<IT>& p, unsigned mask, int width) {
  for (int o = width / 2; o > 0; o >>= 1) {
    p.aa += __shfl_xor_sync(mask, p.aa, o, width);
    if (PAIR) {
      p.ab += __shfl_xor_sync(mask, p.ab, o, width);
      p.bb += __shfl_xor_sync(mask, p.bb, o, width);
    }
  }
}

template <typename IT>
__device__ __forceinline__ void part_values(const Part<IT>& p, double fa0, double fb0, bool dc,
                                            double& iab, double& iaa, double& ibb) {
  if constexpr (sizeof(IT) <= 2) {
    const long long a0 = (long long)fa0, b0 = (long long)fb0;
    iab = (double)(p.ab - (dc ? a0 * b0 : 0));
    iaa = (double)(p.aa - (dc ? a0 * a0 : 0));
    ibb = (double)(p.bb - (dc ? b0 * b0 : 0));
  } else {
    iab = p.ab - (dc ? fa0 * fb0 : 0.0);
    iaa = p.aa - (dc ? fa0 * fa0 : 0.0);
    ibb = p.bb - (dc ? fb0 * fb0 : 0.0);
  }
}

// ------------------------------------------- aligned blocks, vector loads --
// K*sizeof(IT) is a multiple of 16.  GS lanes per block, each loading NCH
// 16-byte chunks per block (NCH = 0: run-time count), U blocks per group per
// iteration; every chunk of an iteration is loaded before any is consumed so
// a thread keeps U*NCH*16 bytes (per operand) in flight.
template <typename IT, int GS, int NCH, int U, bool PAIR>
__global__ void __launch_bounds__(256, 2)
k_moments_vec(int64_t nblocks, int kept, int keeps_first, int fk_a, int fk_b,
              const void* __restrict__ a_max, const IT* __restrict__ a_idx,
              const void* __restrict__ b_max, const IT* __restrict__ b_idx,
              double* __restrict__ ws, double* __restrict__ record) {
  constexpr int V = 16 / sizeof(IT);
  constexpr int NC = NCH > 0 ? NCH : 1;  // chunks held per (u) at once
  const int lane = threadIdx.x & 31;
  const int sub = lane % GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1) << (lane - sub));
  constexpr int GPW = 32 / GS;  // groups per warp
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int gw = lane / GS;       // group within the warp
  const int nch = NCH > 0 ? NCH : kept / (GS * V);  // chunks per lane per block
  const bool dc = keeps_first != 0;
  MomState st;
  using F0 = typename std::conditional<sizeof(IT) == 8, long long, int>::type;
  // the warp owns U*GPW consecutive blocks per iteration; block of (u, group)
  // is base + u*GPW + gw, so every load instruction covers a contiguous range
  for (int64_t base = warp * (U * GPW); base < nblocks; base += nwarps * (U * GPW)) {
    const int64_t bb = base + gw;  // block for u is bb + u*GPW
    double na[U], nb[U];
    Part<IT> p[U];
    F0 f0a[U], f0b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      na[u] = nb[u] = 0.0;
      f0a[u] = f0b[u] = 0;
      if (sub == 0 && bb + u * GPW < nblocks) {
        na[u] = load_kind_rt(a_max, bb + u * GPW, fk_a);
        nb[u] = PAIR ? load_kind_rt(b_max, bb + u * GPW, fk_b) : na[u];
      }
    }
    for (int c0 = 0; c0 < nch; c0 += NC) {
      uint4 wa[U][NC], wb[U][NC];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = bb + u * GPW < nblocks;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int64_t off = (bb + u * GPW) * (int64_t)kept + (int64_t)((c0 + c) * GS + sub) * V;
          wa[u][c] = ok ? __ldcs(reinterpret_cast<const uint4*>(a_idx + off)) : make_uint4(0, 0, 0, 0);
          wb[u][c] = (PAIR && ok) ? __ldcs(reinterpret_cast<const uint4*>(b_idx + off)) : wa[u][c];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int c = 0; c < NC; ++c) part_vec<IT, PAIR>(p[u], wa[u][c], wb[u][c]);
        if (c0 == 0 && sub == 0) {
          f0a[u] = (F0)first_elem<IT>(wa[u][0]);
          f0b[u] = (F0)first_elem<IT>(wb[u][0]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      part_reduce<IT, PAIR>(p[u], gmask, GS);
      if (sub == 0 && bb + u * GPW < nblocks) {
        double iab, iaa, ibb;
        part_values<IT>(p[u], (double)f0a[u], (double)f0b[u], dc, iab, iaa, ibb);
        st.add_block<PAIR>(iab, iaa, ibb, (double)f0a[u], (double)f0b[u], na[u], nb[u], dc);
      }
    }
  }
  finish(st.record(dc), ws, PAIR, record);
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
  finish(st.record(dc), ws, PAIR, record);
}

// ------------------------------------------------- first coefficients only --
template <typename IT, int U, bool PAIR>
__global__ void __launch_bounds__(256, 2)
k_moments_dc(int64_t nblocks, int kept, int fk_a, int fk_b, const void* __restrict__ a_max,
             const IT* __restrict__ a_idx, const void* __restrict__ b_max,
             const IT* __restrict__ b_idx, double* __restrict__ ws,
             double* __restrict__ record) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  MomState st;
  for (int64_t bb = tid; bb < nblocks; bb += nth * U) {
    double fa[U], fb[U], na[U], nb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = bb + u * nth;
      const bool ok = b < nblocks;
      fa[u] = ok ? (double)__ldcs(a_idx + b * (int64_t)kept) : 0.0;
      na[u] = ok ? load_kind_rt(a_max, b, fk_a) : 0.0;
      fb[u] = (ok && PAIR) ? (double)__ldcs(b_idx + b * (int64_t)kept) : fa[u];
      nb[u] = (ok && PAIR) ? load_kind_rt(b_max, b, fk_b) : na[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (bb + u * nth < nblocks) st.add_block<PAIR>(0, 0, 0, fa[u], fb[u], na[u], nb[u], true);
  }
  finish(st.record(true), ws, PAIR, record);
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
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  occ = std::max(1, std::min(occ, kMaxCTAs / kSMs));
  return (int)std::max<int64_t>(1, std::min<int64_t>(work_ctas, (int64_t)kSMs * occ));
}

template <typename IT, bool PAIR>
static int launch_typed(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                        const void* b_max, const void* b_idx, int dc_only, double* ws,
                        double* record, cudaStream_t s) {
  constexpr int V = 16 / sizeof(IT);
  const int64_t B = ga.nblocks;
  const int kept = ga.kept;
  if (dc_only && kept > 0) {
    constexpr int U = 8;
    auto kern = k_moments_dc<IT, U, PAIR>;
    const int grid = persistent_grid(kern, 256, 0, (B + 256 * U - 1) / (256 * U));
    kern<<<grid, 256, 0, s>>>(B, kept, ga.float_kind, gb.float_kind, a_max, (const IT*)a_idx,
                              b_max, (const IT*)b_idx, ws, record);
    return check_launch("moments_dc");
  }
  const bool aligned = kept > 0 && (kept * sizeof(IT)) % 16 == 0 &&
                       !(((uintptr_t)a_idx | (PAIR ? (uintptr_t)b_idx : 0)) & 15);
  if (aligned) {
    const int vecs = kept / V;  // 16-byte chunks per block
    // lanes of a group read consecutive chunks: GS = largest power of two
    // <= 32 dividing the chunk count, each lane NCH = vecs / GS chunks
    int GS = 1;
    while (GS < 32 && vecs % (2 * GS) == 0) GS <<= 1;
    const int nch = vecs / GS;
    const int NCHs = nch == 1 ? 1 : nch == 2 ? 2 : nch == 4 ? 4 : 0;
#define BZ_MV(G, N)                                                                       \
  {                                                                                       \
    constexpr int U = N == 0 ? 1 : std::max(1, (PAIR ? 2 : 8) / (N * (sizeof(IT) >= 4 ? 2 : 1))); \
    auto kern = k_moments_vec<IT, G, N, U, PAIR>;                                         \
    const int64_t work = (B * G + 256 * U - 1) / (256 * U);                               \
    const int grid = persistent_grid(kern, 256, 0, work);                                 \
    kern<<<grid, 256, 0, s>>>(B, kept, ga.keeps_first, ga.float_kind, gb.float_kind, a_max, \
                              (const IT*)a_idx, b_max, (const IT*)b_idx, ws, record);       \
  }
#define BZ_GS(G)                                                   \
  case G:                                                          \
    switch (NCHs) {                                                \
      case 1: BZ_MV(G, 1) break;                                   \
      case 2: BZ_MV(G, 2) break;                                   \
      case 4: BZ_MV(G, 4) break;                                   \
      default: BZ_MV(G, 0) break;                                  \
    }                                                              \
    break;
    switch (GS) { BZ_GS(1) BZ_GS(2) BZ_GS(4) BZ_GS(8) BZ_GS(16) BZ_GS(32) }
#undef BZ_GS
#undef BZ_MV
    return check_launch("moments_vec");
  }
  // unaligned (or empty) blocks: stage tiles of 256 blocks in shared memory
  const size_t tile = (size_t)256 * kept * sizeof(IT);
  const size_t smem = 2 * (((tile + 32 + 15) / 16) * 16);
  if (smem > 200 * 1024) { set_error("moments: kept block too large to stage"); return BZ_E_UNSUPPORTED; }
  auto kern = k_moments_staged<IT, PAIR>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, 256, smem, (B + 255) / 256);
  kern<<<grid, 256, smem, s>>>(B, kept, ga.keeps_first, ga.float_kind, gb.float_kind, a_max,
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
