// Throughput of the FP64-pipe instructions the codec kernels use (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096, CH = 8;

__global__ void k_dfma(double* out, double a) {
  double v[CH];
  for (int i = 0; i < CH; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = __fma_rn(v[i], a, 0.5);
  double s = 0; for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(double* out, double a) {
  double v[CH];
  for (int i = 0; i < CH; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = __dadd_rn(v[i], a);
  double s = 0; for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f2f64(double* out, float a) {   // F2F.F64.F32 (+ FADD to vary)
  float f[CH]; double s[CH];
  for (int i = 0; i < CH; ++i) { f[i] = threadIdx.x + i; s[i] = 0; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) { s[i] = __dadd_rn(s[i], (double)f[i]); f[i] = __fadd_rn(f[i], a); }
  double t = 0; for (int i = 0; i < CH; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_i2f64(double* out, int a) {     // I2F.F64.S32
  int f[CH]; double s[CH];
  for (int i = 0; i < CH; ++i) { f[i] = threadIdx.x + i; s[i] = 0; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) { s[i] = __dadd_rn(s[i], (double)f[i]); f[i] += a; }
  double t = 0; for (int i = 0; i < CH; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_f2f32(double* out, double a) {  // F2F.F32.F64
  double d[CH]; float s[CH];
  for (int i = 0; i < CH; ++i) { d[i] = threadIdx.x + i; s[i] = 0; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) { s[i] += __double2float_rn(d[i]); d[i] = d[i] * a; }
  double t = 0; for (int i = 0; i < CH; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_dsetp(double* out, double a) {  // fmax(|x|) = DSETP + 2 SEL
  double v[CH], m[CH];
  for (int i = 0; i < CH; ++i) { v[i] = threadIdx.x + i; m[i] = 0; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) { m[i] = fmax(m[i], fabs(v[i])); v[i] = -v[i]; }
  double s = 0; for (int i = 0; i < CH; ++i) s += m[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mix(double* out, float a) {  // 1 F2F.F64.F32 + 8 DFMA per step
  float f[CH]; double s[CH], u[CH];
  for (int i = 0; i < CH; ++i) { f[i] = threadIdx.x + i; s[i] = 0; u[i] = i; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      s[i] = __dadd_rn(s[i], (double)f[i]);
      f[i] = __fadd_rn(f[i], a);
#pragma unroll
      for (int k = 0; k < 7; ++k) u[i] = __fma_rn(u[i], 1.0000001, 0.5);
    }
  double t = 0; for (int i = 0; i < CH; ++i) t += s[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <typename K, typename A>
void run(const char* name, K k, A a, double ops_per_iter) {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  k<<<148 * 8, 256>>>(out, a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<148 * 8, 256>>>(out, a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 5.0 * 148 * 8 * 256 * (double)ITERS * CH * ops_per_iter;
  printf("%-12s %8.2f Gop/s  (%.1f per SM per clk @1.965GHz)\n", name, n / ms / 1e6,
         n / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}

int main() {
  run("DFMA", k_dfma, 1.0000001, 1);
  run("DADD", k_dadd, 1e-9, 1);
  run("F2F.F64.F32+DADD", k_f2f64, 1e-3f, 1);
  run("I2F.F64+DADD", k_i2f64, 3, 1);
  run("F2F.F32.F64+DMUL", k_f2f32, 1.0000001, 1);
  run("fmax|x|", k_dsetp, 1.0, 1);
  run("mix(per step: F2F+DADD+7DFMA)", k_mix, 1e-3f, 1);
  return 0;
}
