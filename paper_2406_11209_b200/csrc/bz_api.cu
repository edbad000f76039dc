// bz_api.cu -- extern "C" entry points (include/bzc_b200.h).
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bz_common.cuh"
#include "bz_kernels.cuh"

namespace bz {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return BZ_E_CUDA;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BZ_OK;
}

int occupancy(const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> occ_cache;
  static std::map<std::pair<int, const void*>, size_t> smem_attr;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kern, threads, smem);
  std::lock_guard<std::mutex> lk(mu);
  auto it = occ_cache.find(key);
  if (it != occ_cache.end()) return it->second;
  if (smem > 48 * 1024) {
    size_t& cur = smem_attr[{dev, kern}];
    if (smem > cur) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cur = smem;
    }
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  occ = occ < 1 ? 1 : occ;
  occ_cache[key] = occ;
  return occ;
}

static int validate(const bz_layout* L) {
  if (!L || L->ndim < 1 || L->ndim > BZ_MAX_DIMS) { set_error("layout: ndim out of range"); return BZ_E_INVALID; }
  if (L->float_kind < 0 || L->float_kind > 3 || L->index_kind < 0 || L->index_kind > 3) { set_error("layout: bad kind"); return BZ_E_INVALID; }
  int bs = 1;
  for (int a = 0; a < L->ndim; ++a) {
    if (L->block[a] < 1 || (L->block[a] & (L->block[a] - 1))) { set_error("layout: block extents must be powers of two"); return BZ_E_INVALID; }
    if (L->shape[a] < 1) { set_error("layout: zero extent"); return BZ_E_INVALID; }
    if (L->grid[a] != (L->shape[a] + L->block[a] - 1) / L->block[a]) { set_error("layout: grid != ceil(shape/block)"); return BZ_E_INVALID; }
    bs *= L->block[a];
  }
  if (L->kept < 0 || L->kept > bs) { set_error("layout: kept out of range"); return BZ_E_INVALID; }
  if (L->kept > 0 && (!L->kept_pos || !L->rank)) { set_error("layout: mask tables missing"); return BZ_E_INVALID; }
  return BZ_OK;
}

// BZC_B200_FORCE_GENERIC=1 routes compress/decompress through the exact
// generic kernels (testing: fast vs generic agreement)
static bool force_generic() {
  const char* v = getenv("BZC_B200_FORCE_GENERIC");
  return v && v[0] == '1';
}

static int need_matrices(const bz_layout* L) {
  if (!L->matrices) { set_error("layout: transform matrices missing"); return BZ_E_INVALID; }
  return BZ_OK;
}

// two operands walked block by block together: same block count, kept
// count, first-coefficient flag and index kind (a C caller passing layouts
// of different grids would otherwise read past b's buffers)
static int check_pair(const bz_layout* La, const bz_layout* Lb, const char* what,
                      bool same_index_kind) {
  if (block_count(La) != block_count(Lb)) { set_error("%s: block counts differ", what); return BZ_E_INVALID; }
  if (La->kept != Lb->kept || La->keeps_first != Lb->keeps_first) { set_error("%s: masks differ", what); return BZ_E_INVALID; }
  if (same_index_kind && La->index_kind != Lb->index_kind) { set_error("%s: index kinds differ (convert first)", what); return BZ_E_INVALID; }
  return BZ_OK;
}

}  // namespace bz

using namespace bz;

#define S(stream) reinterpret_cast<cudaStream_t>(stream)

extern "C" {

int bz_version(void) { return 10000; }
long long bz_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
const char* bz_last_error(void) { return g_err; }

int bz_stream_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) {
    set_error("stream sync: %s", cudaGetErrorString(e));
    return BZ_E_CUDA;
  }
  return BZ_OK;
}

int bz_wait_record(const double* record, void* stream) {
  const volatile double* flag = record + BZ_RECORD_DOUBLES - 1;
  for (unsigned spin = 1;; ++spin) {
    if (*flag == 1.0) return BZ_OK;
    if ((spin & 1023u) == 0) {  // every ~1k polls: has the stream finished or failed?
      cudaError_t e = cudaStreamQuery(S(stream));
      if (e == cudaSuccess) {
        if (*flag == 1.0) return BZ_OK;
        set_error("wait_record: stream idle but the record is not complete");
        return BZ_E_INVALID;
      }
      if (e != cudaErrorNotReady) {
        set_error("wait_record: %s", cudaGetErrorString(e));
        return BZ_E_CUDA;
      }
    }
  }
}

int bz_fast_path(const bz_layout* L) {
  if (validate(L)) return 0;
  Geo g = make_geo(L);
  return fast_supported(g, L->float_kind) ? 1 : 0;
}

// workspace for compress: the generic kernel's global scratch (very large
// blocks only) or a pre-rounded copy of the input when its kind differs from
// the float kind and the fused kernel handles the layout.
size_t bz_compress_workspace(const bz_layout* L) {
  if (validate(L)) return 0;
  Geo g = make_geo(L);
  size_t generic = exact_compress_workspace(g, g.nblocks);
  size_t convert = (size_t)dense_count(L) * float_kind_bytes(L->float_kind) + 256;
  return std::max(std::max(generic, convert),
                  std::max(dct8_compress_workspace(g), dct4_compress_workspace(g))) + 256;
}

static int compress_body(const bz_layout* L, const Geo& g, const void* x, int x_kind,
                         void* maxima, void* indices, void* dc, bool& dc_done, void* ws,
                         size_t ws_bytes, cudaStream_t s);

int bz_compress(const bz_layout* L, const void* x, int x_kind, void* maxima, void* indices,
                void* dc, void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(L)) return rc;
  if (int rc = need_matrices(L)) return rc;
  Geo g = make_geo(L);
  if (g.nblocks == 0) return BZ_OK;
  if (!g.keeps_first || g.kept == 0) dc = nullptr;
  bool dc_done = false;
  if (int rc = compress_body(L, g, x, x_kind, maxima, indices, dc, dc_done, ws, ws_bytes, S(stream)))
    return rc;
  return (dc && !dc_done) ? launch_extract_dc(g, indices, dc, S(stream)) : BZ_OK;
}

// dc_done: the kernel wrote the DC plane itself (factored and generic paths)
static int compress_body(const bz_layout* L, const Geo& g, const void* x, int x_kind,
                         void* maxima, void* indices, void* dc, bool& dc_done, void* ws,
                         size_t ws_bytes, cudaStream_t s) {
  // input of another kind: convert_precision first (arrays.py:147-153)
  if (x_kind != L->float_kind && !force_generic() && fast_supported(g, L->float_kind)) {
    size_t need = (size_t)dense_count(L) * float_kind_bytes(L->float_kind);
    if (!ws || ws_bytes < need) { set_error("compress: workspace too small for conversion"); return BZ_E_WORKSPACE; }
    if (int rc = launch_round_to_kind(x, x_kind, ws, L->float_kind, dense_count(L), nullptr, s)) return rc;
    return launch_fast_compress(g, ws, maxima, indices, s, dc, &dc_done);
  }
  if (!force_generic() && dct8_compress_supported(g, x_kind) && ws &&
      ws_bytes >= dct8_compress_workspace(g)) {
    dc_done = true;
    return launch_dct8_compress(g, x, maxima, indices, ws, ws_bytes, s, dc);
  }
  if (!force_generic() && dct4_compress_supported(g, x_kind) && ws &&
      ws_bytes >= dct4_compress_workspace(g)) {
    dc_done = true;
    return launch_dct4_compress(g, x, maxima, indices, ws, ws_bytes, s, dc);
  }
  if (!force_generic() && fast_supported(g, x_kind))
    return launch_fast_compress(g, x, maxima, indices, s, dc, &dc_done);
  dc_done = true;
  return launch_exact_compress(g, x, x_kind, maxima, indices, nullptr, nullptr, g.nblocks, ws,
                               ws_bytes, s, dc);
}

size_t bz_decompress_workspace(const bz_layout* L) {
  if (validate(L)) return 0;
  Geo g = make_geo(L);
  return exact_compress_workspace(g, g.nblocks) + 256;
}

int bz_decompress(const bz_layout* L, const void* maxima, const void* indices, void* out,
                  int out_kind, void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(L)) return rc;
  if (int rc = need_matrices(L)) return rc;
  Geo g = make_geo(L);
  if (g.nblocks == 0) return BZ_OK;
  if (!force_generic() && dct8_supported(g) && (out_kind == BZ_F64 || out_kind == BZ_F32) &&
      g.index_kind != BZ_I64)
    return launch_dct8_decompress(g, maxima, indices, out, out_kind, S(stream));
  if (!force_generic() && dct4_supported(g) && (out_kind == BZ_F64 || out_kind == BZ_F32) &&
      (g.index_kind == BZ_I8 || g.index_kind == BZ_I16))
    return launch_dct4_decompress(g, maxima, indices, out, out_kind, S(stream));
  if (!force_generic() && fast_decompress_supported(g, out_kind))
    return launch_fast_decompress(g, maxima, indices, out, out_kind, S(stream));
  return launch_exact_decompress(g, maxima, indices, out, out_kind, ws, ws_bytes, S(stream));
}

int bz_negate(int index_kind, const void* in, void* out, int64_t count, void* stream) {
  if (index_kind < 0 || index_kind > 3) { set_error("negate: bad index kind"); return BZ_E_INVALID; }
  return launch_negate(index_kind, in, out, count, S(stream));
}

int bz_mul_scalar(const bz_layout* L, const void* maxima, const void* indices, const void* dc,
                  double x, void* maxima_out, void* indices_out, void* dc_out, void* stream) {
  if (int rc = validate(L)) return rc;
  Geo g = make_geo(L);
  if (int rc = launch_mul_scalar(g, maxima, indices, x, maxima_out, indices_out, S(stream))) return rc;
  if (dc && dc_out && !(x > 0)) {  // the plane follows the indices' sign change
    Geo gp = g;
    gp.kept = 1;
    return launch_mul_scalar_indices(gp, dc, x, dc_out, S(stream));
  }
  return BZ_OK;
}

int bz_add(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
           const void* b_max, const void* b_idx, int subtract, void* out_max, void* out_idx,
           void* out_dc, void* stream) {
  if (int rc = validate(La)) return rc;
  if (int rc = validate(Lb)) return rc;
  if (int rc = check_pair(La, Lb, "add", true)) return rc;
  return launch_add(make_geo(La), make_geo(Lb), a_max, a_idx, b_max, b_idx, subtract, 0.0, 0,
                    out_max, out_idx, S(stream), out_dc);
}

int bz_extract_dc(const bz_layout* L, const void* indices, void* dc, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_extract_dc(make_geo(L), indices, dc, S(stream));
}

size_t bz_subtract_l2_workspace(void) { return subtract_l2_workspace(); }

int bz_subtract_l2(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
                   const void* b_max, const void* b_idx, double* out, void* ws, size_t ws_bytes,
                   void* stream) {
  if (int rc = validate(La)) return rc;
  if (int rc = validate(Lb)) return rc;
  if (int rc = check_pair(La, Lb, "subtract_l2", true)) return rc;
  return launch_subtract_l2(make_geo(La), make_geo(Lb), a_max, a_idx, b_max, b_idx, out, ws,
                            ws_bytes, S(stream));
}

int bz_add_scalar(const bz_layout* L, const void* maxima, const void* indices, double shift,
                  void* out_max, void* out_idx, void* out_dc, void* stream) {
  if (int rc = validate(L)) return rc;
  if (!L->keeps_first) { set_error("add_scalar: mask drops the first coefficient"); return BZ_E_INVALID; }
  Geo g = make_geo(L);
  return launch_add(g, g, maxima, indices, nullptr, nullptr, 0, shift, 1, out_max, out_idx,
                    S(stream), out_dc);
}

size_t bz_moments_workspace(const bz_layout* L) {
  if (validate(L)) return 0;
  return moments_workspace(make_geo(L));
}

int bz_moments(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
               const void* b_max, const void* b_idx, int pair, int dc_only, double* record,
               void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(La)) return rc;
  const bz_layout* lb = pair ? Lb : La;
  if (pair) {
    if (int rc = validate(Lb)) return rc;
    if (int rc = check_pair(La, Lb, "moments", true)) return rc;
  }
  return launch_moments(make_geo(La), make_geo(lb), a_max, a_idx, pair ? b_max : a_max,
                        pair ? b_idx : a_idx, pair, dc_only, record, ws, ws_bytes, S(stream));
}

int bz_moments_dc(const bz_layout* L, const void* maxima, const void* dc, double* record,
                  void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_moments_plane(make_geo(L), maxima, dc, record, ws, ws_bytes, S(stream));
}

int bz_round_to_kind(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                     int32_t* mismatch, void* stream) {
  return launch_round_to_kind(in, in_kind, out, out_kind, n, mismatch, S(stream));
}

int bz_gradient(int ndim, const int64_t* shape, int kind, void* out, void* stream) {
  if (ndim < 1 || ndim > BZ_MAX_DIMS) { set_error("gradient: bad ndim"); return BZ_E_INVALID; }
  return launch_gradient(ndim, shape, kind, out, S(stream));
}

int bz_block(const bz_layout* L, const void* x, int x_kind, double* blocks, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_block(make_geo(L), x, x_kind, blocks, S(stream));
}

int bz_unblock(const bz_layout* L, const double* blocks, void* out, int out_kind, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_unblock(make_geo(L), blocks, out, out_kind, S(stream));
}

int bz_transform(const bz_layout* L, const double* in, double* out, int inverse, void* ws,
                 size_t ws_bytes, void* stream) {
  if (int rc = validate(L)) return rc;
  if (int rc = need_matrices(L)) return rc;
  return launch_transform(make_geo(L), in, out, inverse, ws, ws_bytes, S(stream));
}

int bz_bin(const bz_layout* L, const double* coeffs, void* maxima, void* full, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_bin(make_geo(L), coeffs, maxima, full, S(stream));
}

int bz_prune(const bz_layout* L, const void* full, void* flat, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_prune(make_geo(L), full, flat, S(stream));
}

int bz_unflatten(const bz_layout* L, const void* flat, void* full, void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_unflatten(make_geo(L), flat, full, S(stream));
}

int bz_specified(const bz_layout* L, const void* maxima, const void* flat, double* out,
                 void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_specified(make_geo(L), maxima, flat, out, S(stream));
}

int bz_fill_random(void* out, int kind, int64_t n, int64_t offset, uint64_t seed, int dist,
                   void* stream) {
  return launch_fill_random(out, kind, n, offset, seed, dist, S(stream));
}

int bz_convert_indices(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                       void* stream) {
  return launch_convert_indices(in, in_kind, out, out_kind, n, S(stream));
}

int bz_block_means(const bz_layout* L, const void* maxima, const void* indices, double* out,
                   void* stream) {
  if (int rc = validate(L)) return rc;
  if (L->kept == 0 || !L->keeps_first) { set_error("block_means: mask drops the first coefficient"); return BZ_E_INVALID; }
  return launch_block_means(make_geo(L), maxima, indices, out, S(stream));
}

int bz_block_means_dc(const bz_layout* L, const void* maxima, const void* dc, double* out,
                      void* stream) {
  if (int rc = validate(L)) return rc;
  if (L->kept == 0 || !L->keeps_first) { set_error("block_means: mask drops the first coefficient"); return BZ_E_INVALID; }
  return launch_block_means(make_geo(L), maxima, dc, out, S(stream), true);
}

size_t bz_wasserstein_workspace(const bz_layout* L) {
  if (validate(L)) return 0;
  return wasserstein_workspace(block_count(L));
}

int bz_approx_wasserstein(const bz_layout* La, const bz_layout* Lb, const void* a_max,
                          const void* a_idx, const void* b_max, const void* b_idx, double order,
                          double tol, double* result, void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(La)) return rc;
  if (int rc = validate(Lb)) return rc;
  if (block_count(La) != block_count(Lb)) { set_error("approx_wasserstein: block counts differ"); return BZ_E_INVALID; }
  if (!La->keeps_first || !Lb->keeps_first || La->kept == 0 || Lb->kept == 0) { set_error("approx_wasserstein: mask drops the first coefficient"); return BZ_E_INVALID; }
  return launch_approx_wasserstein(make_geo(La), make_geo(Lb), a_max, a_idx, b_max, b_idx, order,
                                   tol, result, ws, ws_bytes, S(stream));
}

int bz_approx_wasserstein_dc(const bz_layout* La, const bz_layout* Lb, const void* a_max,
                             const void* a_idx, const void* a_dc, const void* b_max,
                             const void* b_idx, const void* b_dc, double order, double tol,
                             double* result, void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(La)) return rc;
  if (int rc = validate(Lb)) return rc;
  if (block_count(La) != block_count(Lb)) { set_error("approx_wasserstein: block counts differ"); return BZ_E_INVALID; }
  if (!La->keeps_first || !Lb->keeps_first || La->kept == 0 || Lb->kept == 0) { set_error("approx_wasserstein: mask drops the first coefficient"); return BZ_E_INVALID; }
  return launch_approx_wasserstein(make_geo(La), make_geo(Lb), a_max, a_idx, b_max, b_idx, order,
                                   tol, result, ws, ws_bytes, S(stream), a_dc, b_dc);
}

int bz_error_bounds(const bz_layout* L, const void* maxima, const void* indices,
                    const double* coeffs, double* bin_bound, double* loose_linf, double* l2_coeff,
                    void* stream) {
  if (int rc = validate(L)) return rc;
  return launch_error_bounds(make_geo(L), maxima, indices, coeffs, bin_bound, loose_linf, l2_coeff,
                             S(stream));
}

int bz_block_diff(int64_t nblocks, int bsize, const double* x, const double* y, double* l2sq,
                  double* maxabs, void* stream) {
  if (nblocks < 0 || bsize < 1) { set_error("block_diff: bad sizes"); return BZ_E_INVALID; }
  return launch_block_diff(nblocks, bsize, x, y, l2sq, maxabs, S(stream));
}

int bz_stream_pack(const void* maxima, int64_t max_bytes, const void* indices, int64_t idx_bytes,
                   int64_t bit_offset, uint32_t head_word, void* out, int64_t out_words,
                   void* stream) {
  return launch_stream_pack(maxima, max_bytes, indices, idx_bytes, bit_offset, head_word, out,
                            out_words, S(stream));
}

int bz_stream_unpack(const void* in, int64_t in_words, int64_t bit_offset, void* maxima,
                     int64_t max_bytes, void* indices, int64_t idx_bytes, void* stream) {
  return launch_stream_unpack(in, in_words, bit_offset, maxima, max_bytes, indices, idx_bytes,
                              S(stream));
}

}  // extern "C"
