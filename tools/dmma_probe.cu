// dmma_probe.cu -- B200 microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4
// f64) vs the FP64 FMA pipe.
//  1. bit-exactness: does D = A*B + C equal the sequential FMA chain
//     fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) (the reference's order)?
//  2. throughput of DMMA alone, DFMA alone, and both interleaved.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__global__ void k_exact(const double* A, const double* B, const double* C, double* D, int n) {
  // n independent 8x8x4 problems, one warp each
  int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (w >= n) return;
  const double* a = A + w * 32;  // 8x4 row-major
  const double* b = B + w * 32;  // 4x8 row-major (k, col)
  const double* c = C + w * 64;  // 8x8 row-major
  int g = lane >> 2, q = lane & 3;
  double av = a[g * 4 + q];
  double bv = b[q * 8 + g];
  double c0 = c[g * 8 + q * 2], c1 = c[g * 8 + q * 2 + 1];
  double d0, d1;
  dmma(d0, d1, av, bv, c0, c1);
  D[w * 64 + g * 8 + q * 2] = d0;
  D[w * 64 + g * 8 + q * 2 + 1] = d1;
}

__global__ void k_dmma_tput(double* out, int iters) {
  int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[2 * j], c[2 * j + 1], a, b, c[2 * j], c[2 * j + 1]);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma_tput(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = __fma_rn(a, c[j], b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// both in the same warp: 8 DMMA (=8*8*8*4 MACs) + 16 DFMA per iteration
__global__ void k_mixed_tput(double* out, int iters, int dfma_per) {
  int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[16], e[16];
  for (int i = 0; i < 16; ++i) { c[i] = i; e[i] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[2 * j], c[2 * j + 1], a, b, c[2 * j], c[2 * j + 1]);
#pragma unroll
    for (int j = 0; j < 16; ++j) e[j] = __fma_rn(a, e[j], b);
    if (dfma_per > 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) e[j] = __fma_rn(b, e[j], a);
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i] + e[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double drand(unsigned long long& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((double)(s >> 11) / 9007199254740992.0) * 4.0 - 2.0;
}

int main() {
  const int n = 4096;
  size_t na = n * 32, nc = n * 64;
  double *A, *B, *C, *D;
  cudaMallocManaged(&A, na * 8); cudaMallocManaged(&B, na * 8);
  cudaMallocManaged(&C, nc * 8); cudaMallocManaged(&D, nc * 8);
  unsigned long long s = 42;
  for (size_t i = 0; i < na; ++i) { A[i] = drand(s) * (1 << (i % 7)); B[i] = drand(s); }
  for (size_t i = 0; i < nc; ++i) C[i] = drand(s) * ((i % 3) ? 1e-3 : 1e3);
  k_exact<<<n / 4, 128>>>(A, B, C, D, n);
  cudaDeviceSynchronize();
  long seq_fwd = 0, seq_rev = 0, prod_first = 0, total = 0;
  for (int w = 0; w < n; ++w)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double c = C[w * 64 + i * 8 + j];
        double f = c;
        for (int k = 0; k < 4; ++k) f = __builtin_fma(A[w * 32 + i * 4 + k], B[w * 32 + k * 8 + j], f);
        double r = c;
        for (int k = 3; k >= 0; --k) r = __builtin_fma(A[w * 32 + i * 4 + k], B[w * 32 + k * 8 + j], r);
        double p = 0.0;
        for (int k = 0; k < 4; ++k) p = __builtin_fma(A[w * 32 + i * 4 + k], B[w * 32 + k * 8 + j], p);
        double pf = p + c;
        double d = D[w * 64 + i * 8 + j];
        seq_fwd += d == f;
        seq_rev += d == r;
        prod_first += d == pf;
        ++total;
      }
  printf("DMMA exactness over %ld outputs: seq_fma_k_ascending=%ld seq_fma_k_descending=%ld chain_then_add_c=%ld\n",
         total, seq_fwd, seq_rev, prod_first);

  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  float ms;
  int grid = 148 * 4, block = 256;
  k_dmma_tput<<<grid, block>>>(out, 10);
  cudaEventRecord(e0);
  k_dmma_tput<<<grid, block>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double dmma_macs = (double)grid * (block / 32) * iters * 8 * 256;
  printf("DMMA: %.3f ms, %.2f TFLOP/s (fp64 tensor)\n", ms, 2 * dmma_macs / ms / 1e9);
  k_dfma_tput<<<grid, block>>>(out, 10);
  cudaEventRecord(e0);
  k_dfma_tput<<<grid, block>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double dfma = (double)grid * block * iters * 16;
  printf("DFMA: %.3f ms, %.2f TFLOP/s (fp64 vector)\n", ms, 2 * dfma / ms / 1e9);
  for (int per : {16, 32}) {
    k_mixed_tput<<<grid, block>>>(out, 10, per);
    cudaEventRecord(e0);
    k_mixed_tput<<<grid, block>>>(out, iters, per);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2 * dmma_macs + 2.0 * grid * block * iters * per;
    printf("mixed (8 DMMA + %d DFMA per iter): %.3f ms, %.2f TFLOP/s combined (DMMA-only time share above)\n",
           per, ms, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("cuda: %s\n", cudaGetErrorString(err));
  return 0;
}
