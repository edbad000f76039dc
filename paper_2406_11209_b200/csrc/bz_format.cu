// bz_format.cu -- the .bzc byte stream's payload on the GPU (format.py:11-33,
// 108-127, 190-209).
//
// The stream is LSB-first bits with little-endian multi-bit fields.  Every
// float / index kind is a whole number of bytes, so the payload -- raw
// maxima patterns (row-major grid order) followed by the kept indices (two's
// complement, blocks row-major) -- is exactly the concatenation of the two
// little-endian byte arrays, shifted to start at bit P = the header length
// (12 + 64*(2d+1) + block size bits, in general not a byte boundary).  Packing
// is therefore a funnel-shifted copy at 32-bit word granularity; the host
// writes the header words, and passes the header bits that share the first
// payload word.  Unpacking is the inverse shift.  Both are HBM-bound.
#include "bz_common.cuh"
#include "bz_kernels.cuh"

namespace bz {

// payload viewed as a virtual little-endian 32-bit word stream over the two
// buffers; word i covers payload bytes [4i, 4i+4), zero past the end
struct Payload {
  const unsigned char* a;  // maxima bytes
  const unsigned char* b;  // index bytes
  int64_t na, nb;          // byte counts
  bool aligned;            // na % 4 == 0 and both buffers 4-byte aligned
};

__device__ __forceinline__ uint32_t pay_byte(const Payload& p, int64_t j) {
  if (j < p.na) return p.a[j];
  j -= p.na;
  return j < p.nb ? p.b[j] : 0u;
}

__device__ __forceinline__ uint32_t pay_word(const Payload& p, int64_t i) {
  if (i < 0) return 0u;
  const int64_t j = i * 4;
  if (p.aligned) {
    if (j + 4 <= p.na) return __ldg(reinterpret_cast<const uint32_t*>(p.a + j));
    const int64_t k = j - p.na;
    if (k >= 0 && k + 4 <= p.nb) return __ldg(reinterpret_cast<const uint32_t*>(p.b + k));
  }
  return pay_byte(p, j) | (pay_byte(p, j + 1) << 8) | (pay_byte(p, j + 2) << 16) |
         (pay_byte(p, j + 3) << 24);
}

// out32[v] for v >= v0 = P / 32: stream bits [32v, 32v + 32)
__global__ void k_stream_pack(Payload p, int64_t P, uint32_t head_word, uint32_t* __restrict__ out,
                              int64_t v0, int64_t nwords) {
  const int sh = (int)(P & 31);
  for (int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nwords;
       v += (int64_t)gridDim.x * blockDim.x) {
    // payload bits [o, o + 32) with o = 32v - P
    const int64_t o = 32 * v - P;
    uint32_t word;
    if (o < 0) {  // first word: header bits below P, payload above
      const uint32_t low = sh ? (head_word & ((1u << sh) - 1u)) : 0u;
      word = low | (pay_word(p, 0) << sh);
    } else {
      const int64_t i = o >> 5;
      const uint32_t lo = pay_word(p, i), hi = pay_word(p, i + 1);
      word = __funnelshift_r(lo, hi, (int)(o & 31));
    }
    out[v] = word;
  }
}

// payload word i = stream bits [P + 32i, P + 32i + 32)
__global__ void k_stream_unpack(const uint32_t* __restrict__ in, int64_t in_words, int64_t P,
                                unsigned char* __restrict__ a, int64_t na, unsigned char* __restrict__ b,
                                int64_t nb, bool aligned) {
  const int64_t npay = (na + nb + 3) / 4;
  const int sh = (int)(P & 31);
  const int64_t w0 = P >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npay;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = w0 + i;
    const uint32_t lo = s < in_words ? __ldg(in + s) : 0u;
    const uint32_t hi = s + 1 < in_words ? __ldg(in + s + 1) : 0u;
    const uint32_t word = __funnelshift_r(lo, hi, sh);
    const int64_t j = i * 4;
    if (aligned && j + 4 <= na) {
      reinterpret_cast<uint32_t*>(a)[i] = word;
    } else if (aligned && j >= na && j - na + 4 <= nb) {
      reinterpret_cast<uint32_t*>(b + (j - na))[0] = word;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t jj = j + k;
        const unsigned char byte = (unsigned char)(word >> (8 * k));
        if (jj < na) a[jj] = byte;
        else if (jj - na < nb) b[jj - na] = byte;
      }
    }
  }
}

int launch_stream_pack(const void* maxima, int64_t max_bytes, const void* indices,
                       int64_t idx_bytes, int64_t bit_offset, uint32_t head_word, void* out,
                       int64_t out_words, cudaStream_t s) {
  if (((uintptr_t)out & 3) != 0) { set_error("stream_pack: output must be 4-byte aligned"); return BZ_E_INVALID; }
  if (bit_offset < 0 || out_words * 32 < bit_offset + 8 * (max_bytes + idx_bytes)) {
    set_error("stream_pack: output too small");
    return BZ_E_INVALID;
  }
  Payload p{reinterpret_cast<const unsigned char*>(maxima), reinterpret_cast<const unsigned char*>(indices),
            max_bytes, idx_bytes, false};
  p.aligned = (max_bytes % 4 == 0) && !(((uintptr_t)maxima | (uintptr_t)indices) & 3);
  const int64_t v0 = bit_offset >> 5;
  const int64_t n = out_words - v0;
  if (n <= 0) return BZ_OK;
  k_stream_pack<<<grid_for(n, 256, 16), 256, 0, s>>>(p, bit_offset, head_word,
                                                     reinterpret_cast<uint32_t*>(out), v0, out_words);
  return check_launch("stream_pack");
}

int launch_stream_unpack(const void* in, int64_t in_words, int64_t bit_offset, void* maxima,
                         int64_t max_bytes, void* indices, int64_t idx_bytes, cudaStream_t s) {
  if (((uintptr_t)in & 3) != 0) { set_error("stream_unpack: input must be 4-byte aligned"); return BZ_E_INVALID; }
  if (bit_offset < 0 || in_words * 32 < bit_offset + 8 * (max_bytes + idx_bytes)) {
    set_error("stream_unpack: stream truncated");
    return BZ_E_INVALID;
  }
  const bool aligned = (max_bytes % 4 == 0) && !(((uintptr_t)maxima | (uintptr_t)indices) & 3);
  const int64_t n = (max_bytes + idx_bytes + 3) / 4;
  if (n <= 0) return BZ_OK;
  k_stream_unpack<<<grid_for(n, 256, 16), 256, 0, s>>>(
      reinterpret_cast<const uint32_t*>(in), in_words, bit_offset,
      reinterpret_cast<unsigned char*>(maxima), max_bytes, reinterpret_cast<unsigned char*>(indices),
      idx_bytes, aligned);
  return check_launch("stream_unpack");
}

}  // namespace bz
