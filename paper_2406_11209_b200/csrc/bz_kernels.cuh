// bz_kernels.cuh -- launcher declarations shared by the translation units.
#pragma once
#include <algorithm>

#include "bz_common.cuh"

namespace bz {

// generic (bz_generic.cu)
int launch_round_to_kind(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                         int32_t* mismatch, cudaStream_t s);
int launch_convert_indices(const void* in, int in_kind, void* out, int out_kind, int64_t n,
                           cudaStream_t s);
int launch_gradient(int ndim, const int64_t* shape, int kind, void* out, cudaStream_t s);
int launch_fill_random(void* out, int kind, int64_t n, int64_t offset, uint64_t seed, int dist,
                       cudaStream_t s);
int launch_block(const Geo& g, const void* x, int x_kind, double* blocks, cudaStream_t s);
int launch_unblock(const Geo& g, const double* blocks, void* out, int out_kind, cudaStream_t s);
int launch_transform(const Geo& g, const double* in, double* out, int inverse, void* ws,
                     size_t ws_bytes, cudaStream_t s);
int launch_bin(const Geo& g, const double* coeffs, void* maxima, void* full, cudaStream_t s);
int launch_prune(const Geo& g, const void* full, void* flat, cudaStream_t s);
int launch_unflatten(const Geo& g, const void* flat, void* full, cudaStream_t s);
int launch_specified(const Geo& g, const void* maxima, const void* flat, double* out,
                     cudaStream_t s);
int launch_exact_compress(const Geo& g, const void* x, int x_kind, void* maxima, void* indices,
                          const int32_t* list, const int32_t* count, int64_t max_blocks,
                          void* ws, size_t ws_bytes, cudaStream_t s, void* dc = nullptr);
// DC plane (dc[b] = F[b][0], contiguous): gather from the indices
int launch_extract_dc(const Geo& g, const void* indices, void* dc, cudaStream_t s);
size_t exact_compress_workspace(const Geo& g, int64_t max_blocks);
int launch_exact_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                            int out_kind, void* ws, size_t ws_bytes, cudaStream_t s);

// fused fast paths (bz_fast_*.cu)
bool fast_supported(const Geo& g, int x_kind);
// dc (optional): the DC plane, written by every path but the 8^3 half-slice
// one (*dc_done reports which)
int launch_fast_compress(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s,
                         void* dc = nullptr, bool* dc_done = nullptr);
bool fast_decompress_supported(const Geo& g, int out_kind);
// 8x8x8 blocks, half slices (bz_half3.cu)
int launch_half3_compress(const Geo& g, const void* x, void* maxima, void* indices, cudaStream_t s);
int launch_half3_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                            int out_kind, cudaStream_t s);
int launch_fast_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                           int out_kind, cudaStream_t s);

// factored 8x8x8 DCT with exact fix-up (bz_dct8.cu)
bool dct8_supported(const Geo& g);
bool dct8_compress_supported(const Geo& g, int x_kind);
size_t dct8_compress_workspace(const Geo& g);
int launch_dct8_compress(const Geo& g, const void* x, void* maxima, void* indices, void* ws,
                         size_t ws_bytes, cudaStream_t s, void* dc = nullptr);
int launch_dct8_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                           int out_kind, cudaStream_t s);

// factored 4x4x4x4 DCT with exact fix-up (bz_dct4.cu)
bool dct4_supported(const Geo& g);
bool dct4_compress_supported(const Geo& g, int x_kind);
size_t dct4_compress_workspace(const Geo& g);
int launch_dct4_compress(const Geo& g, const void* x, void* maxima, void* indices, void* ws,
                         size_t ws_bytes, cudaStream_t s, void* dc = nullptr);
int launch_dct4_decompress(const Geo& g, const void* maxima, const void* indices, void* out,
                           int out_kind, cudaStream_t s);

// block means / approximate Wasserstein distance (bz_wasserstein.cu)
size_t wasserstein_workspace(int64_t nblocks);
// dc_plane: `indices` is the contiguous DC plane (one index per block)
int launch_block_means(const Geo& g, const void* maxima, const void* indices, double* out,
                       cudaStream_t s, bool dc_plane = false);
// a_dc / b_dc: the operands' DC planes, or nullptr (K-strided gather of a_idx / b_idx)
int launch_approx_wasserstein(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                              const void* b_max, const void* b_idx, double order, double tol,
                              double* result, void* ws, size_t ws_bytes, cudaStream_t s,
                              const void* a_dc = nullptr, const void* b_dc = nullptr);

// error predictors (bz_metrics.cu)
int launch_error_bounds(const Geo& g, const void* maxima, const void* indices,
                        const double* coeffs, double* bin_bound, double* loose_linf,
                        double* l2_coeff, cudaStream_t s);
int launch_block_diff(int64_t nblocks, int bsize, const double* x, const double* y, double* l2sq,
                      double* maxabs, cudaStream_t s);

// .bzc stream payload (bz_format.cu)
int launch_stream_pack(const void* maxima, int64_t max_bytes, const void* indices,
                       int64_t idx_bytes, int64_t bit_offset, uint32_t head_word, void* out,
                       int64_t out_words, cudaStream_t s);
int launch_stream_unpack(const void* in, int64_t in_words, int64_t bit_offset, void* maxima,
                         int64_t max_bytes, void* indices, int64_t idx_bytes, cudaStream_t s);

// compressed-domain ops (bz_ops.cu)
int launch_negate(int ik, const void* in, void* out, int64_t n, cudaStream_t s);
int launch_mul_scalar_indices(const Geo& g, const void* indices, double x, void* indices_out,
                              cudaStream_t s);
int launch_mul_scalar(const Geo& g, const void* maxima, const void* indices, double x,
                      void* maxima_out, void* indices_out, cudaStream_t s);
bool add8_supported(const Geo& ga, const Geo& gb, int mode, const void* a_idx, const void* b_idx,
                    const void* out_idx);
int launch_add8(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                const void* b_idx, int subtract, double shift, int mode, void* out_max,
                void* out_idx, cudaStream_t s, void* out_dc = nullptr);
// int8 / float32 blocks whose kept indices are not whole 16-byte vectors
// (K <= 128; bz_add_small.cu)
bool add_small_supported(const Geo& ga, const Geo& gb, int mode, const void* a_max,
                         const void* a_idx, const void* b_max, const void* b_idx,
                         const void* out_idx);
int launch_add_small(const Geo& ga, const void* a_max, const void* a_idx, const void* b_max,
                     const void* b_idx, int subtract, double shift, int mode, void* out_max,
                     void* out_idx, void* out_dc, cudaStream_t s);
int launch_subtract_l2_small(const Geo& ga, const void* a_max, const void* a_idx,
                             const void* b_max, const void* b_idx, double* red_ws, double* out,
                             cudaStream_t s);
int launch_subtract_l2_add8(const Geo& ga, const void* a_max, const void* a_idx,
                            const void* b_max, const void* b_idx, double* red_ws, double* out,
                            cudaStream_t s);
int launch_add(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
               const void* b_max, const void* b_idx, int subtract, double shift, int mode,
               void* out_max, void* out_idx, cudaStream_t s, void* out_dc = nullptr);
size_t subtract_l2_workspace();
int launch_subtract_l2(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                       const void* b_max, const void* b_idx, double* out, void* ws,
                       size_t ws_bytes, cudaStream_t s);
size_t moments_workspace(const Geo& g);
int launch_moments(const Geo& ga, const Geo& gb, const void* a_max, const void* a_idx,
                   const void* b_max, const void* b_idx, int pair, int dc_only, double* record,
                   void* ws, size_t ws_bytes, cudaStream_t s);
// mean record from the DC plane (contiguous first coefficients)
int launch_moments_plane(const Geo& g, const void* maxima, const void* dc, double* record,
                         void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace bz
