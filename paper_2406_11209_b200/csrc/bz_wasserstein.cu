// bz_wasserstein.cu -- block means and the approximate Wasserstein distance
// (ops.py:351-384) on the device, no host round trip:
//
//   pa, pb = block_means(a), block_means(b)      F0*N/r/sqrt(bsize), IEEE order
//   p <- softmax(p) if |sum p - 1| > tol          exp(p - max p) / sum
//   d = |sort(pa) - sort(pb)|                     LSD radix sort, 8 x 8 bits
//   W = (sum d^order / n)^(1/order)
//
// Reductions are two-stage and deterministic (fixed grid, partials summed in
// CTA order).  The sort is a stable LSD radix sort of order-preserving 64-bit
// keys: per pass a tile histogram, one exclusive scan, and a stable scatter
// that ranks keys round by round (warp match + per-warp digit counts).
#include "bz_common.cuh"
#include "bz_kernels.cuh"

#include <utility>

namespace bz {

namespace ws_ {
constexpr int RT = 256;           // threads per CTA = keys per round
constexpr int MAX_ROUNDS = 16;    // rounds per tile (fewer for small sorts: more CTAs)
constexpr int RED_CTAS = 296;     // partial-sum CTAs (fixed: deterministic)
}  // namespace ws_

// ------------------------------------------------------------ block means --
// `stride` = kept (the K-strided first coefficients of the indices) or 1 (the
// DC plane: indices[..., 0] stored contiguously by the producing kernel)
template <typename IT>
__global__ void k_block_means(int64_t nblocks, int64_t stride, const void* __restrict__ maxima,
                              int fk, const IT* __restrict__ indices, double r, double scale,
                              double* __restrict__ out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    const double f = (double)indices[b * stride];
    const double n = load_kind_rt(maxima, b, fk);
    // firsts = F0 * N; firsts /= r (ops.py:172-175); / block_mean_scale (ops.py:358)
    out[b] = __ddiv_rn(__ddiv_rn(__dmul_rn(f, n), r), scale);
  }
}

// ------------------------------------------- deterministic sum / max pass --
// partial[c] = {sum a, max a, sum b, max b} over a fixed grid-stride slice
__global__ void k_sum_max_partial(const double* __restrict__ a, const double* __restrict__ b,
                                  int64_t n, double* __restrict__ partial) {
  double sa = 0.0, sb = 0.0, ma = -INFINITY, mb = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    sa += x;
    sb += y;
    ma = fmax(ma, x);
    mb = fmax(mb, y);
  }
  __shared__ double s[4][ws_::RT];
  s[0][threadIdx.x] = sa; s[1][threadIdx.x] = ma; s[2][threadIdx.x] = sb; s[3][threadIdx.x] = mb;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s[0][threadIdx.x] += s[0][threadIdx.x + o];
      s[1][threadIdx.x] = fmax(s[1][threadIdx.x], s[1][threadIdx.x + o]);
      s[2][threadIdx.x] += s[2][threadIdx.x + o];
      s[3][threadIdx.x] = fmax(s[3][threadIdx.x], s[3][threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) partial[blockIdx.x * 4 + k] = s[k][0];
}

// one CTA, one warp per statistic: stats = {sum a, max a, sum b, max b}.
// Lane l sums partials l, l+32, ... in order, then a fixed xor tree: the same
// bits every run (the single-thread sequential loop was a 300-deep chain of
// dependent L2 loads, ~40 us)
__global__ void k_sum_max_final(const double* __restrict__ partial, int nparts,
                                double* __restrict__ stats) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= 4) return;
  double v = (k & 1) ? -INFINITY : 0.0;
  for (int i = lane; i < nparts; i += 32) {
    const double x = partial[i * 4 + k];
    v = (k & 1) ? fmax(v, x) : v + x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, v, o);
    v = (k & 1) ? fmax(v, y) : v + y;
  }
  if (lane == 0) stats[k] = v;
}

// softmax step 1 (ops.py:351-353): x <- exp(x - max) where |sum - 1| > tol
__global__ void k_softmax_exp(double* __restrict__ a, double* __restrict__ b, int64_t n,
                              const double* __restrict__ stats, double tol,
                              int* __restrict__ flags) {
  const bool fa = fabs(stats[0] - 1.0) > tol, fb = fabs(stats[2] - 1.0) > tol;
  if (blockIdx.x == 0 && threadIdx.x == 0) { flags[0] = fa; flags[1] = fb; }
  const double ma = stats[1], mb = stats[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (fa) a[i] = exp(a[i] - ma);
    if (fb) b[i] = exp(b[i] - mb);
  }
}

// ------------------------------------------------------------ radix sort --
__device__ __forceinline__ unsigned long long key_of(double x) {
  // order-preserving: negative -> ~u, otherwise u | sign.  The xor is inline
  // PTX: written in C, nvcc turned `u | sign` of a computed double into the
  // floating-point -|x| (DADD), which rewrites NaN payloads (a NaN then
  // sorts below the positives instead of last)
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  const unsigned long long m = (unsigned long long)((long long)u >> 63) | 0x8000000000000000ull;
  unsigned long long k;
  asm("xor.b64 %0, %1, %2;" : "=l"(k) : "l"(u), "l"(m));
  return k;
}
__device__ __forceinline__ double value_of(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// softmax step 2: x <- x / sum x (stats recomputed after step 1), written
// straight out as the sort keys (the keys replace the values in place)
__global__ void k_softmax_div_keys(double* __restrict__ a, double* __restrict__ b, int64_t n,
                                   const double* __restrict__ stats, const int* __restrict__ flags) {
  const bool fa = flags[0], fb = flags[1];
  const double sa = stats[0], sb = stats[2];
  unsigned long long* ka = reinterpret_cast<unsigned long long*>(a);
  unsigned long long* kb = reinterpret_cast<unsigned long long*>(b);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    ka[i] = key_of(fa ? __ddiv_rn(x, sa) : x);
    kb[i] = key_of(fb ? __ddiv_rn(y, sb) : y);
  }
}

// Both distributions are sorted by the same launches: blockIdx.y selects the
// array (keys / histogram / chunk sums of array y).
// hist[y][d * ntiles + tile]
__global__ void __launch_bounds__(ws_::RT)
k_radix_hist(const unsigned long long* __restrict__ keys0, const unsigned long long* __restrict__ keys1,
             int64_t n, int shift, unsigned int* __restrict__ hist, int ntiles, int rounds) {
  const unsigned long long* __restrict__ keys = blockIdx.y ? keys1 : keys0;
  hist += (int64_t)blockIdx.y * 256 * ntiles;
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * ws_::RT * rounds;
  // every round's key is loaded before the first is counted: one DRAM latency
  // per tile instead of one per round
  unsigned long long k[ws_::MAX_ROUNDS];
#pragma unroll
  for (int rr = 0; rr < ws_::MAX_ROUNDS; ++rr) {
    const int64_t i = base + rr * ws_::RT + threadIdx.x;
    k[rr] = (rr < rounds && i < n) ? __ldcs(keys + i) : ~0ull;
  }
#pragma unroll
  for (int rr = 0; rr < ws_::MAX_ROUNDS; ++rr) {
    const int64_t i = base + rr * ws_::RT + threadIdx.x;
    if (rr < rounds && i < n) atomicAdd(&h[(unsigned)(k[rr] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of m entries in place: three phases over chunks of SCH
// entries (chunk sums, a scan of the chunk sums, chunk scans with their
// offsets); 1024 threads x 4 consecutive entries per chunk
constexpr int SCH = 4096;

// exclusive scan of one value per thread over a CTA of 1024 threads; *total
// receives the CTA sum
__device__ __forceinline__ unsigned cta_exclusive_scan(unsigned x, unsigned* total) {
  __shared__ unsigned wsum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // wsum reuse across calls
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  *total = wsum[31];
  return (w ? wsum[w - 1] : 0u) + inc - x;
}

__device__ __forceinline__ void load4(const unsigned* v, int64_t i, int64_t m, unsigned (&x)[4]) {
  if (i + 4 <= m) {
    const uint4 q = *reinterpret_cast<const uint4*>(v + i);
    x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = i + k < m ? v[i + k] : 0u;
  }
}

__global__ void __launch_bounds__(1024) k_scan_reduce(const unsigned* __restrict__ v, int64_t m,
                                                      unsigned* __restrict__ csum) {
  v += (int64_t)blockIdx.y * m;
  csum += (int64_t)blockIdx.y * gridDim.x;
  unsigned x[4];
  load4(v, (int64_t)blockIdx.x * SCH + 4 * threadIdx.x, m, x);
  unsigned total;
  cta_exclusive_scan(x[0] + x[1] + x[2] + x[3], &total);
  if (threadIdx.x == 0) csum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(unsigned* __restrict__ csum, int nc) {
  csum += (int64_t)blockIdx.x * nc;  // one CTA per array
  unsigned carry = 0;
  for (int base = 0; base < nc; base += 1024) {
    const int i = base + threadIdx.x;
    const unsigned x = i < nc ? csum[i] : 0u;
    unsigned total;
    const unsigned e = cta_exclusive_scan(x, &total);
    if (i < nc) csum[i] = carry + e;
    carry += total;
  }
}

__global__ void __launch_bounds__(1024) k_scan_down(unsigned* __restrict__ v, int64_t m,
                                                    const unsigned* __restrict__ csum) {
  v += (int64_t)blockIdx.y * m;
  if (csum) csum += (int64_t)blockIdx.y * gridDim.x;
  const int64_t i = (int64_t)blockIdx.x * SCH + 4 * threadIdx.x;
  unsigned x[4];
  load4(v, i, m, x);
  unsigned total;
  const unsigned off = csum ? csum[blockIdx.x] : 0u;  // one chunk: no chunk sums
  unsigned run = off + cta_exclusive_scan(x[0] + x[1] + x[2] + x[3], &total);
  unsigned y[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { y[k] = run; run += x[k]; }
  if (i + 4 <= m) {
    *reinterpret_cast<uint4*>(v + i) = make_uint4(y[0], y[1], y[2], y[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k < m) v[i + k] = y[k];
  }
}

// lanes of the warp holding the same 8-bit digit (bit-sliced ballots: eight
// votes instead of a MATCH.ANY); d >= 256 marks an invalid lane, which then
// matches only other invalid lanes
__device__ __forceinline__ unsigned digit_peers(unsigned d) {
  unsigned m = __ballot_sync(0xffffffffu, d < 256u);
  if (d >= 256u) m = ~m;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? v : ~v;
  }
  return m;
}

// stable scatter: keys of tile `blockIdx.x` to their global positions.  Warp
// w owns the tile's keys [w*32*rounds, (w+1)*32*rounds) (its rounds of 32
// consecutive keys, held in registers); pass 1 counts each warp's digits,
// one CTA-wide exclusive scan over the warps turns the counts into per-warp
// running positions, pass 2 writes every round's keys at position + rank
// among equal digits (bit-sliced votes).  Two CTA barriers per tile (the
// per-round CTA-wide ranking used three per 256 keys: C3 47 -> 43 us per
// pass; a variant that sorts the tile in shared memory first and writes
// digit runs measured 47 us -- the scattered 8-byte stores are not the limit).
__global__ void __launch_bounds__(ws_::RT)
k_radix_scatter(const unsigned long long* __restrict__ in0, const unsigned long long* __restrict__ in1,
                unsigned long long* __restrict__ out0, unsigned long long* __restrict__ out1,
                int64_t n, int shift, const unsigned int* __restrict__ offsets, int ntiles,
                int rounds) {
  const unsigned long long* __restrict__ in = blockIdx.y ? in1 : in0;
  unsigned long long* __restrict__ out = blockIdx.y ? out1 : out0;
  offsets += (int64_t)blockIdx.y * 256 * ntiles;
  constexpr int NW = ws_::RT / 32;
  __shared__ unsigned int cnt[NW][256];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int k = 0; k < NW; ++k) cnt[k][t] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * ws_::RT * rounds + (int64_t)w * 32 * rounds;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long kr[ws_::MAX_ROUNDS];
#pragma unroll
  for (int rr = 0; rr < ws_::MAX_ROUNDS; ++rr) {
    const int64_t i = wbase + rr * 32 + lane;
    kr[rr] = (rr < rounds && i < n) ? __ldcs(in + i) : 0ull;
  }
#pragma unroll
  for (int rr = 0; rr < ws_::MAX_ROUNDS; ++rr) {
    if (rr >= rounds) break;
    const bool valid = wbase + rr * 32 + lane < n;
    const unsigned d = valid ? ((unsigned)(kr[rr] >> shift) & 255u) : 256u;
    const unsigned peers = digit_peers(d);
    if (valid && (peers & lt) == 0u) cnt[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  unsigned run = offsets[(int64_t)t * ntiles + blockIdx.x];  // thread t = digit t
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    const unsigned c = cnt[k][t];
    cnt[k][t] = run;
    run += c;
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < ws_::MAX_ROUNDS; ++rr) {
    if (rr >= rounds) break;
    const bool valid = wbase + rr * 32 + lane < n;
    const unsigned d = valid ? ((unsigned)(kr[rr] >> shift) & 255u) : 256u;
    const unsigned peers = digit_peers(d);
    const unsigned pos = valid ? cnt[w][d] : 0u;
    if (valid) out[pos + __popc(peers & lt)] = kr[rr];
    __syncwarp();
    if (valid && (peers & lt) == 0u) cnt[w][d] = pos + __popc(peers);
    __syncwarp();
  }
}

// ------------------------------------------------ order-p distance terms --
__global__ void k_diff_pow_partial(const unsigned long long* __restrict__ ka,
                                   const unsigned long long* __restrict__ kb, int64_t n, double p,
                                   double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dlt = fabs(value_of(ka[i]) - value_of(kb[i]));
    s += p == 1.0 ? dlt : (p == 2.0 ? dlt * dlt : pow(dlt, p));
  }
  __shared__ double sh[ws_::RT];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// one warp: lane-strided partial sums in order, fixed xor tree
__global__ void k_diff_pow_final(const double* __restrict__ partial, int nparts, int64_t n,
                                 double p, double* __restrict__ result) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < nparts; i += 32) s += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) {
    const double m = s / (double)n;
    result[0] = p == 1.0 ? m : pow(m, 1.0 / p);
  }
}

// ---------------------------------------------------------------- launch --
// rounds per tile: enough tiles for two CTAs per SM, at most MAX_ROUNDS
static int rounds_of(int64_t n) {
  return (int)std::min<int64_t>(ws_::MAX_ROUNDS, std::max<int64_t>(1, n / ((int64_t)ws_::RT * 2 * kSMs)));
}
static int64_t ntiles_of(int64_t n) {
  const int64_t tile = (int64_t)ws_::RT * rounds_of(n);
  return (n + tile - 1) / tile;
}

size_t wasserstein_workspace(int64_t nblocks) {
  const int64_t nt = ntiles_of(nblocks);
  return 256 + (size_t)nblocks * 8 * 4        // pa, pb, two key buffers
         + 2 * ((size_t)256 * nt * 4 + 256)         // histograms / offsets, per array
         + 2 * ((size_t)256 * nt / SCH + 1) * 4 + 256  // chunk sums of the scans
         + (size_t)ws_::RED_CTAS * 4 * 8 + 256;
}

int launch_block_means(const Geo& g, const void* maxima, const void* indices, double* out,
                       cudaStream_t s, bool dc_plane) {
  const double r = radius_f64(g.index_kind), scale = sqrt((double)g.bsize);
  const int64_t stride = dc_plane ? 1 : g.kept;
  const int grid = grid_for(g.nblocks, 256, 8);
  switch (g.index_kind) {
    case BZ_I8: k_block_means<int8_t><<<grid, 256, 0, s>>>(g.nblocks, stride, maxima, g.float_kind, (const int8_t*)indices, r, scale, out); break;
    case BZ_I16: k_block_means<int16_t><<<grid, 256, 0, s>>>(g.nblocks, stride, maxima, g.float_kind, (const int16_t*)indices, r, scale, out); break;
    case BZ_I32: k_block_means<int32_t><<<grid, 256, 0, s>>>(g.nblocks, stride, maxima, g.float_kind, (const int32_t*)indices, r, scale, out); break;
    default: k_block_means<int64_t><<<grid, 256, 0, s>>>(g.nblocks, stride, maxima, g.float_kind, (const int64_t*)indices, r, scale, out); break;
  }
  return check_launch("block_means");
}

// sorts ka and kb (n keys each) together; the results end in ka / kb
static int radix_sort2(unsigned long long* ka, unsigned long long* kb, unsigned long long* ta,
                       unsigned long long* tb, int64_t n, unsigned int* hist, unsigned int* csum,
                       cudaStream_t s) {
  const int nt = (int)ntiles_of(n), rounds = rounds_of(n);
  const int64_t m = (int64_t)256 * nt;
  const int nc = (int)((m + SCH - 1) / SCH);
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 8 * pass;
    k_radix_hist<<<dim3(nt, 2), ws_::RT, 0, s>>>(ka, kb, n, shift, hist, nt, rounds);
    if (nc > 1) {
      k_scan_reduce<<<dim3(nc, 2), 1024, 0, s>>>(hist, m, csum);
      k_scan_top<<<2, 1024, 0, s>>>(csum, nc);
    }
    k_scan_down<<<dim3(nc, 2), 1024, 0, s>>>(hist, m, nc > 1 ? csum : nullptr);
    k_radix_scatter<<<dim3(nt, 2), ws_::RT, 0, s>>>(ka, kb, ta, tb, n, shift, hist, nt, rounds);
    if (int rc = check_launch("radix pass")) return rc;
    std::swap(ka, ta);  // 8 passes: the results end in the original buffers
    std::swap(kb, tb);
  }
  return BZ_OK;
}

int launch_approx_wasserstein(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                              const void* b_max, const void* b_idx, double order, double tol,
                              double* result, void* ws, size_t ws_bytes, cudaStream_t s,
                              const void* a_dc, const void* b_dc) {
  const int64_t n = ga.nblocks;
  if (ws_bytes < wasserstein_workspace(n)) { set_error("approx_wasserstein: workspace too small"); return BZ_E_WORKSPACE; }
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  auto take = [&](size_t bytes) { unsigned char* q = p; p += (bytes + 255) / 256 * 256; return q; };
  double* pa = reinterpret_cast<double*>(take(n * 8));
  double* pb = reinterpret_cast<double*>(take(n * 8));
  unsigned long long* ka = reinterpret_cast<unsigned long long*>(pa);  // keys replace values
  unsigned long long* kb = reinterpret_cast<unsigned long long*>(pb);
  unsigned long long* t1 = reinterpret_cast<unsigned long long*>(take(n * 8));
  unsigned long long* t2 = reinterpret_cast<unsigned long long*>(take(n * 8));
  unsigned int* hist = reinterpret_cast<unsigned int*>(take(2 * (size_t)256 * ntiles_of(n) * 4));
  unsigned int* csum = reinterpret_cast<unsigned int*>(take(2 * ((size_t)256 * ntiles_of(n) / SCH + 1) * 4));
  double* partial = reinterpret_cast<double*>(take((size_t)ws_::RED_CTAS * 4 * 8));
  double* stats = reinterpret_cast<double*>(take(64));
  int* flags = reinterpret_cast<int*>(stats + 4);
  if (n == 0) {  // mean over no blocks: NaN, as the reference's 0/0
    k_diff_pow_final<<<1, 32, 0, s>>>(partial, 0, 0, order, result);
    return check_launch("wasserstein empty");
  }
  if (int rc = launch_block_means(ga, a_max, a_dc ? a_dc : a_idx, pa, s, a_dc != nullptr)) return rc;
  if (int rc = launch_block_means(gb, b_max, b_dc ? b_dc : b_idx, pb, s, b_dc != nullptr)) return rc;
  const int g = grid_for(n, ws_::RT, 8);
  k_sum_max_partial<<<ws_::RED_CTAS, ws_::RT, 0, s>>>(pa, pb, n, partial);
  k_sum_max_final<<<1, 128, 0, s>>>(partial, ws_::RED_CTAS, stats);
  k_softmax_exp<<<g, ws_::RT, 0, s>>>(pa, pb, n, stats, tol, flags);
  k_sum_max_partial<<<ws_::RED_CTAS, ws_::RT, 0, s>>>(pa, pb, n, partial);
  k_sum_max_final<<<1, 128, 0, s>>>(partial, ws_::RED_CTAS, stats);
  k_softmax_div_keys<<<g, ws_::RT, 0, s>>>(pa, pb, n, stats, flags);
  if (int rc = check_launch("wasserstein prep")) return rc;
  if (int rc = radix_sort2(ka, kb, t1, t2, n, hist, csum, s)) return rc;
  k_diff_pow_partial<<<ws_::RED_CTAS, ws_::RT, 0, s>>>(ka, kb, n, order, partial);
  k_diff_pow_final<<<1, 32, 0, s>>>(partial, ws_::RED_CTAS, n, order, result);
  return check_launch("wasserstein distance");
}

}  // namespace bz
