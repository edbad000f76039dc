// bz_tma.cu -- host-side tensor-map encoding for the TMA box loads (bz_tma.cuh).
#include <cudaTypedefs.h>

#include <mutex>

#include "bz_tma.cuh"

namespace bz {
namespace tma {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_f32(CUtensorMap* map, const void* base, int rank, const int64_t* dims,
                const uint32_t* box, int swizzle_bytes) {
  return encode_tiled(map, base, 4, rank, dims, box, swizzle_bytes);
}

bool encode_tiled(CUtensorMap* map, const void* base, int elem_bytes, int rank,
                  const int64_t* dims, const uint32_t* box, int swizzle_bytes) {
  auto fn = encode_fn();
  if (!fn || rank < 1 || rank > 5 || ((uintptr_t)base & 15)) return false;
  if (elem_bytes != 4 && elem_bytes != 8) return false;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bdim[5], estride[5];
  uint64_t stride = (uint64_t)elem_bytes;  // bytes
  for (int i = 0; i < rank; ++i) {  // innermost first
    const int a = rank - 1 - i;
    if (dims[a] < 1 || dims[a] > (int64_t)0xffffffff) return false;
    gdim[i] = (cuuint64_t)dims[a];
    bdim[i] = box[a];
    estride[i] = 1;
    if (i > 0) {
      if (stride % 16) return false;
      gstride[i - 1] = stride;
    }
    stride *= (uint64_t)dims[a];
  }
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUresult r = fn(map, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank,
                        const_cast<void*>(base), gdim, gstride, bdim, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tma
}  // namespace bz
