/*
 * bzc_b200.h -- C ABI of the B200 (sm_100a) PyBlaz hot path.
 *
 * The reference (arXiv 2406.11209, /root/reference/pkg/src/bzc) is pure
 * Python; its "operator API" is the module-level function set re-exported by
 * bzc/__init__.py:12-63.  Every entry point below replaces the numeric body of
 * one of those functions; the Python package paper_2406_11209_b200 keeps the
 * reference's names, signatures, validation and exceptions and calls these
 * through ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All data pointers are DEVICE pointers
 *    (cudaMalloc / torch CUDA tensors) unless noted; the library never
 *    allocates or frees device memory: callers pass workspaces sized by the
 *    *_workspace() queries.
 *  - Every call is asynchronous on the given stream and reentrant.
 *  - Return 0 on success; negative on error (BZ_E_*), with a thread-local
 *    message from bz_last_error().  Validation that the reference performs
 *    (codec.py:143-155, 197-218; ops.py:100-124) happens in Python BEFORE
 *    these calls, with the reference's exception types.
 */
#ifndef BZC_B200_H
#define BZC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BZ_MAX_DIMS 8
#define BZ_RECORD_DOUBLES 16

/* FloatKind.code (kinds.py:70-76) */
enum { BZ_BF16 = 0, BZ_F16 = 1, BZ_F32 = 2, BZ_F64 = 3 };
/* IndexKind.code (kinds.py:150-156) */
enum { BZ_I8 = 0, BZ_I16 = 1, BZ_I32 = 2, BZ_I64 = 3 };
/* TransformFamily.code (transforms.py:41-46) */
enum { BZ_DCT = 0, BZ_HAAR = 1 };

enum {
  BZ_OK = 0,
  BZ_E_INVALID = -1,     /* bad descriptor / argument */
  BZ_E_UNSUPPORTED = -2, /* configuration not handled */
  BZ_E_CUDA = -3,        /* CUDA launch/runtime error */
  BZ_E_WORKSPACE = -4    /* workspace too small */
};

/*
 * Layout of one compressed array (CodecSettings + original shape,
 * codec.py:133-250).  `shape` is the dense extent of THIS array (a shard's
 * slab in block-sharded use); `grid` = ceil(shape / block).
 * kept_pos / rank / matrices are small device tables built once per settings
 * by the caller:
 *   kept_pos[K]       row-major intrablock positions kept by the mask (codec.py:89-92)
 *   rank[prod(block)] position -> rank in kept_pos, -1 if pruned
 *   matrices          per-axis transform entries [sample][basis], axis 0 first,
 *                     each block[a]*block[a] doubles (transforms.py:67-98)
 *   matrices_host     the same entries in host memory (optional; the fused
 *                     kernels carry them as kernel parameters)
 */
typedef struct bz_layout {
  int32_t ndim;
  int32_t float_kind;
  int32_t index_kind;
  int32_t transform;
  int64_t shape[BZ_MAX_DIMS];
  int32_t block[BZ_MAX_DIMS];
  int64_t grid[BZ_MAX_DIMS];
  int32_t kept;
  int32_t keeps_first;
  const int32_t* kept_pos;
  const int32_t* rank;
  const double* matrices;
  const double* matrices_host;
} bz_layout;

/* Library identification / diagnostics. */
int bz_version(void);
const char* bz_last_error(void);
/* Number of kernels this library has launched in the process (benchmarks). */
long long bz_launch_count(void);
/* Which compress kernel a layout dispatches to: 1 = fused fast path, 0 = generic. */
int bz_fast_path(const bz_layout* L);
/* Wait for `stream` (the one host synchronisation of a scalar reduction);
 * BZ_E_CUDA on an asynchronous launch error.                                */
int bz_stream_sync(void* stream);
/* Wait until a reduction record in pinned host memory is complete: spins on
 * its completion flag record[BZ_RECORD_DOUBLES-1] (the caller zeroes it
 * before the launch; the kernel stores 1.0 last), checking the stream every
 * ~1k polls so a failed launch returns BZ_E_CUDA instead of hanging.       */
int bz_wait_record(const double* record, void* stream);

/* ---- codec: compress / decompress (codec.py:321-334, 364-384) ---------- */
/* x: dense row-major values of kind x_kind (already exactly representable in
 * it).  Outputs: maxima[grid] in float_kind storage, indices[grid][K].
 * dc (optional, may be NULL; ignored when the mask drops the first
 * coefficient): the DC plane dc[b] = indices[b][0], contiguous, in the index
 * kind -- what mean reads (bz_moments_dc) instead of a stride-K gather.     */
size_t bz_compress_workspace(const bz_layout* L);
int bz_compress(const bz_layout* L, const void* x, int x_kind, void* maxima,
                void* indices, void* dc, void* workspace, size_t workspace_bytes,
                void* stream);

/* out: dense row-major values of out_kind (BZ_F64 = reference semantics,
 * codec.py:367; narrower kinds round the f64 result once).                  */
size_t bz_decompress_workspace(const bz_layout* L);
int bz_decompress(const bz_layout* L, const void* maxima, const void* indices,
                  void* out, int out_kind, void* workspace, size_t workspace_bytes,
                  void* stream);

/* ---- compressed-domain elementwise ops (ops.py:195-223) ---------------- */
/* negate: out = -in over `count` indices (ops.py:195-197). */
int bz_negate(int index_kind, const void* in, void* out, int64_t count, void* stream);
/* mul_scalar: maxima_out = RN_kind(maxima * |x|); indices_out = indices * sign(x)
 * (ops.py:218-223).  indices_out may be NULL when x > 0 (indices aliased).
 * dc / dc_out (optional DC planes): dc_out = dc * sign(x) when x <= 0 or NaN
 * (NULL when x > 0: the plane is aliased like the indices).                  */
int bz_mul_scalar(const bz_layout* L, const void* maxima, const void* indices, const void* dc,
                  double x, void* maxima_out, void* indices_out, void* dc_out, void* stream);
/* add / subtract with rebinning under La's kinds (ops.py:178-204; subtract =
 * add(a, negate(b)), cli.py:242).  Bit-exact with the reference.            */
/* out_dc (optional): the result's DC plane (see bz_compress).             */
int bz_add(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
           const void* b_max, const void* b_idx, int subtract, void* out_max,
           void* out_idx, void* out_dc, void* stream);
/* add_scalar: shift each block's first coefficient by shift = x*sqrt(prod i)
 * then rebin (ops.py:207-215). */
int bz_add_scalar(const bz_layout* L, const void* maxima, const void* indices, double shift,
                  void* out_max, void* out_idx, void* out_dc, void* stream);
/* DC plane of an existing array (dc[b] = indices[b][0]; stride-K gather). */
int bz_extract_dc(const bz_layout* L, const void* indices, void* dc, void* stream);

/* ---- reductions (ops.py:226-348) ---------------------------------------
 * Produce one partial record of BZ_RECORD_DOUBLES doubles (device) for the
 * blocks of this array/shard:
 *   [0] n        number of blocks
 *   [1] mean_a   mean over blocks of DCa = Fa[0]*Na   (r not divided)
 *   [2] mean_b
 *   [3] M_ab     sum over blocks (DCa-mean_a)(DCb-mean_b)
 *   [4] M_aa     [5] M_bb
 *   [6] S_ab     sum over blocks Na*Nb*sum_{kept k != first} Fa_k*Fb_k
 *   [7] S_aa     [8] S_bb
 *   [15] 1.0, stored last: the completion flag (bz_wait_record)
 * When the mask drops the first coefficient, entries 1-5 are 0 and S_* run
 * over every kept position.  Records of shards merge with Chan's formulas.
 * `pair` = 0 reads only a (b ignored; *_b and *_ab mirror a).
 * dc_only = 1 computes entries 0-5 from the first coefficient only (mean).
 * dc_only = 2 ("sums", dot / l2): entries 1-5 are 0 and S_* run over every
 * kept position, the first included -- no per-block DC moments.
 * The workspace must be zero-filled before its first use; the kernels leave
 * it re-armed, so a caller keeps one workspace per stream.                  */
size_t bz_moments_workspace(const bz_layout* L);
int bz_moments(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
               const void* b_max, const void* b_idx, int pair, int dc_only, double* record,
               void* workspace, size_t workspace_bytes, void* stream);
/* The dc_only = 1 record (mean, ops.py:244-257) from the DC plane: reads
 * B*(idx+f) contiguous bytes; bit-identical to bz_moments(dc_only = 1).
 * Same workspace contract as bz_moments.                                    */
int bz_moments_dc(const bz_layout* L, const void* maxima, const void* dc, double* record,
                  void* workspace, size_t workspace_bytes, void* stream);

/* ---- building blocks of the API (arrays.py, transforms.py, codec.py) --- */
/* round_to_kind / convert_precision (kinds.py:186-206, arrays.py:147-153):
 * out[i] = RN_out_kind(in[i]).  If mismatch != NULL, atomically sets
 * *mismatch = 1 when any value changed (DenseArray representability check,
 * arrays.py:81-86; NaN == NaN).                                             */
int bz_round_to_kind(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                     int32_t* mismatch, void* stream);
/* gradient_array values (arrays.py:193-208) rounded into kind. */
int bz_gradient(int ndim, const int64_t* shape /*host*/, int kind, void* out, void* stream);
/* block (arrays.py:156-178): dense x -> blocks[grid][block] (f64), zero padded. */
int bz_block(const bz_layout* L, const void* x, int x_kind, double* blocks, void* stream);
/* unblock (arrays.py:181-190): blocks -> dense (cropped), stored as out_kind. */
int bz_unblock(const bz_layout* L, const double* blocks, void* out, int out_kind, void* stream);
/* forward / inverse transform of blocked f64 data (transforms.py:118-142). */
int bz_transform(const bz_layout* L, const double* in, double* out, int inverse,
                 void* workspace, size_t workspace_bytes, void* stream);
/* bin_coefficients (codec.py:253-278): coeffs[grid][block] -> maxima[grid],
 * full_indices[grid][block] (unpruned). */
int bz_bin(const bz_layout* L, const double* coeffs, void* maxima, void* full_indices,
           void* stream);
/* prune_and_flatten / unflatten (codec.py:281-318). */
int bz_prune(const bz_layout* L, const void* full_indices, void* flat, void* stream);
int bz_unflatten(const bz_layout* L, const void* flat, void* full_indices, void* stream);
/* specified_coefficients (codec.py:337-361): (F*N)/r as f64 blocks. */
int bz_specified(const bz_layout* L, const void* maxima, const void* flat, double* out,
                 void* stream);
/* Copy indices between index kinds (mixed-kind reductions). */
int bz_convert_indices(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                       void* stream);
/* Synthetic inputs (benchmark support): counter-based, partition
 * invariant: element at global flat index (offset + i) is identical for any
 * shard split.  dist 0 = N(0,1), 1 = U[0,1). */
int bz_fill_random(void* out, int kind, int64_t n, int64_t offset, uint64_t seed, int dist,
                   void* stream);

/* block_means (ops.py:355-359): per-block mean F0*N/r/sqrt(bsize) in the
 * reference's IEEE op order, row-major grid order, into out[nblocks] (f64). */
int bz_block_means(const bz_layout* L, const void* maxima, const void* indices, double* out,
                   void* stream);
/* block_means from the DC plane (indices[..., 0] stored contiguously, one
 * index per block -- the plane the compress / add kernels write): the same
 * values as bz_block_means, reading B*(idx+f) bytes instead of a K-strided
 * gather. */
int bz_block_means_dc(const bz_layout* L, const void* maxima, const void* dc, double* out,
                      void* stream);
/* approx_wasserstein (ops.py:362-384) entirely on the device: block means,
 * softmax where |sum - 1| > tol, radix sort, (mean |d|^order)^(1/order)
 * into result[0] (device f64).  ws: bz_wasserstein_workspace(La) bytes. */
size_t bz_wasserstein_workspace(const bz_layout* L);
int bz_approx_wasserstein(const bz_layout* La, const bz_layout* Lb, const void* a_max,
                          const void* a_idx, const void* b_max, const void* b_idx, double order,
                          double tol, double* result, void* ws, size_t ws_bytes, void* stream);
/* The same with the operands' DC planes (a_dc / b_dc; nullptr = gather the
 * first coefficients from a_idx / b_idx). */
int bz_approx_wasserstein_dc(const bz_layout* La, const bz_layout* Lb, const void* a_max,
                             const void* a_idx, const void* a_dc, const void* b_max,
                             const void* b_idx, const void* b_dc, double order, double tol,
                             double* result, void* ws, size_t ws_bytes, void* stream);
/* Fused time-series step (cli.py:240-243): the squared L2 norm of
 * subtract(a, b) = add(a, negate(b)) -- sum over blocks of N^2 * sum q^2 with
 * the rebinned q, N of the difference, bit-identical to materialising it --
 * written to out[0] (a device double, or pinned host memory under UVA: the
 * last CTA stores it) without writing the difference.  Returns
 * BZ_E_UNSUPPORTED for configurations without a fused kernel (other index
 * kinds, mixed float kinds, unaligned indices): compose bz_add + bz_moments.
 * ws: bz_subtract_l2_workspace() bytes, zeroed before first use. */
size_t bz_subtract_l2_workspace(void);
int bz_subtract_l2(const bz_layout* La, const bz_layout* Lb, const void* a_max, const void* a_idx,
                   const void* b_max, const void* b_idx, double* out, void* ws, size_t ws_bytes,
                   void* stream);

/* Error predictors (metrics.py:108-124), one value per block (f64):
 * bin_bound = N/(2r+1), loose_linf = max|C| * prod(i), l2_coeff =
 * sqrt(sum (Chat - C)^2) with Chat = (F*N)/r; coeffs = the true coefficient
 * blocks (nblocks x prod(i), row-major). */
int bz_error_bounds(const bz_layout* L, const void* maxima, const void* indices,
                    const double* coeffs, double* bin_bound, double* loose_linf, double* l2_coeff,
                    void* stream);
/* Round-trip errors (metrics.py:127-148): per block sum (x - y)^2 and
 * max |x - y| of two blocked f64 arrays. */
int bz_block_diff(int64_t nblocks, int bsize, const double* x, const double* y, double* l2sq,
                  double* maxabs, void* stream);

/* .bzc stream payload (format.py:108-127 serialize, 190-209 deserialize).
 * The payload -- maxima bytes then index bytes, little-endian -- occupies
 * stream bits [bit_offset, bit_offset + 8*(max_bytes+idx_bytes)); the host
 * owns the header.  pack writes 32-bit words bit_offset/32 .. out_words-1 of
 * `out` (4-byte aligned): the bits below bit_offset in the first word come
 * from head_word, bits past the payload are zero (padding).  unpack reads
 * `in_words` words of a stream (4-byte aligned) and fills both buffers. */
int bz_stream_pack(const void* maxima, int64_t max_bytes, const void* indices, int64_t idx_bytes,
                   int64_t bit_offset, uint32_t head_word, void* out, int64_t out_words,
                   void* stream);
int bz_stream_unpack(const void* in, int64_t in_words, int64_t bit_offset, void* maxima,
                     int64_t max_bytes, void* indices, int64_t idx_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BZC_B200_H */
