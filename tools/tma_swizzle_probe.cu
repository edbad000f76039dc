// tma_swizzle_probe.cu -- where does a TMA box store with a swizzled map read
// each shared-memory byte from?  Fills a 4 KB shared box with its own 4-byte
// word offsets, stores it through a 2-D map (64 rows x R bytes, swizzle S),
// and prints, for the first rows, which shared word landed at each global
// word.  nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2406_11209_b200/csrc \
//      tools/tma_swizzle_probe.cu paper_2406_11209_b200/csrc/bz_tma.cu -o /tmp/tprobe -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include "bz_tma.cuh"

__global__ void k_store(const __grid_constant__ CUtensorMap map, int words) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (bz::tma::smem_u32(sm) & 1023u)) & 1023u);
  uint32_t* w = reinterpret_cast<uint32_t*>(base);
  for (int i = threadIdx.x; i < words; i += blockDim.x) w[i] = (uint32_t)i;
  bz::tma::fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
            reinterpret_cast<uint64_t>(&map)),
        "r"(bz::tma::smem_u32(base)), "r"(0), "r"(0)
        : "memory");
    bz::tma::bulk_commit();
    bz::tma::bulk_wait_all();
  }
}

int main(int argc, char** argv) {
  const int elem_arg = argc > 1 ? atoi(argv[1]) : 8, sw_arg = argc > 2 ? atoi(argv[2]) : 128;
  for (int elem : {elem_arg}) {
    for (int sw : {sw_arg}) {
      const int inner = 8, rows = 64;  // 8 elements per row
      const int64_t dims[2] = {rows, inner};
      const uint32_t box[2] = {(uint32_t)rows, (uint32_t)inner};
      void* d;
      const size_t bytes = (size_t)rows * inner * elem;
      cudaMalloc(&d, bytes);
      cudaMemset(d, 0xff, bytes);
      CUtensorMap map;
      if (!bz::tma::encode_tiled(&map, d, elem, 2, dims, box, sw)) { printf("encode failed elem %d sw %d\n", elem, sw); continue; }
      cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes + 1024));
      k_store<<<1, 128, bytes + 1024>>>(map, (int)(bytes / 4));
      printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
      cudaError_t e = cudaDeviceSynchronize();
      uint32_t h[2048];
      cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
      printf("elem %d B, row %d B, swizzle %d: %s\n", elem, inner * elem, sw, cudaGetErrorString(e));
      const int wpr = inner * elem / 4;
      for (int r = 0; r < 10; ++r) {
        printf("  global row %2d <- smem words:", r);
        for (int k = 0; k < wpr; ++k) printf(" %4u", h[r * wpr + k]);
        printf("\n");
      }
      cudaFree(d);
    }
  }
  return 0;
}
