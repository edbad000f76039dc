// bz_ops.cu -- compressed-domain operators (ops.py:195-348).
//
//  negate / mul_scalar : elementwise over indices / maxima (ops.py:195-223)
//  add / subtract / add_scalar : bz_add.cu;  moments : bz_moments.cu
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

// sign(x) applied to indices (x <= 0 or NaN): -F or 0 (ops.py:222)
int launch_mul_scalar_indices(const Geo& g, const void* indices, double x, void* indices_out,
                              cudaStream_t s) {
  return launch_negate_mode(g.index_kind, indices, indices_out, g.nblocks * g.kept,
                            x < 0 ? -1 : 0, s);
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

}  // namespace bz
