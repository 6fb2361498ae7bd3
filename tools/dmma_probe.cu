// Measures the fp64 peaks that bound the DMMA kernels (K5, K9) on this
// B200: mma.sync f64 shapes m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 and plain
// DFMA, issued back to back from registers (8 independent accumulators per
// warp), grid = 148 SMs x 4 CTAs x 8 warps. Prints TFLOP/s per variant as
// JSON. Not part of the library; built and run by tools/run_probe.sh.
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));         \
      return 1;                                                            \
    }                                                                      \
  } while (0)

constexpr int kIters = 4096;

__global__ void k_m16n8k4(double* out) {
  double acc[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1.0, b0 = a0 - 2.0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]), "+d"(acc[u][2]), "+d"(acc[u][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k8(double* out) {
  double acc[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1.0, a2 = a0 + 2.0, a3 = a0 + 3.0, b0 = a0 - 2.0, b1 = a0 - 1.0;
  for (int it = 0; it < kIters / 2; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+d"(acc[u][0]), "+d"(acc[u][1]), "+d"(acc[u][2]), "+d"(acc[u][3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k16(double* out) {
  double acc[8][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 1e-3 - i;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(acc[u][0]), "+d"(acc[u][1]), "+d"(acc[u][2]), "+d"(acc[u][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m8n8k4(double* out) {
  double acc[8][2] = {};
  double a0 = threadIdx.x * 1e-3, b0 = a0 - 2.0;
  for (int it = 0; it < kIters * 2; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[u][0]), "+d"(acc[u][1])
                   : "d"(a0), "d"(b0));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out) {
  double acc[8];
  for (int u = 0; u < 8; ++u) acc[u] = threadIdx.x + u;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < kIters * 8; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = fma(acc[u], a, b);
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double run(K kern, double flops_per_warp, double* out) {
  const int blocks = 148 * 4, threads = 256;
  kern<<<blocks, threads>>>(out);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double warps = blocks * (threads / 32.0) * 5;
  return flops_per_warp * warps / (ms * 1e-3) / 1e12;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * 148 * 4 * 256));
  // flops per warp: 2 * M * N * K per mma, 8 mmas per iteration
  const double f16x8x4 = 2.0 * 16 * 8 * 4 * 8 * kIters;
  const double f16x8x8 = 2.0 * 16 * 8 * 8 * 8 * (kIters / 2);
  const double f16x8x16 = 2.0 * 16 * 8 * 16 * 8 * (kIters / 4);
  const double f8x8x4 = 2.0 * 8 * 8 * 4 * 8 * (kIters * 2);
  const double fdfma = 2.0 * 32 * 8 * (kIters * 8);
  std::printf("{\"m16n8k4_tflops\": %.3f, \"m16n8k8_tflops\": %.3f, \"m16n8k16_tflops\": %.3f, "
              "\"m8n8k4_tflops\": %.3f, \"dfma_tflops\": %.3f}\n",
              run(k_m16n8k4, f16x8x4, out), run(k_m16n8k8, f16x8x8, out), run(k_m16n8k16, f16x8x16, out),
              run(k_m8n8k4, f8x8x4, out), run(k_dfma, fdfma, out));
  CK(cudaGetLastError());
  return 0;
}
