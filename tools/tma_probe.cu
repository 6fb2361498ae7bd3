// Streaming-read bandwidth probe for the near-field passes: how fast can one
// kernel pull a large fp64 array from HBM (a) with TMA bulk copies into a
// shared-memory ring (stage size S, NST stages, one producer warp, 8 consumer
// warps that touch every element), and (b) with plain 256-bit loads?
// Prints GB/s per configuration. Build: see run_tma_probe.sh.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// grid-stride over chunks of S doubles; every consumer thread sums its share
template <int NST>
__global__ void __launch_bounds__(288, 1) k_tma_stream(const double* __restrict__ a, long long nchunks, int S,
                                                       double* __restrict__ out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      int c = 0;
      for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++c) {
        const int slot = c % NST;
        if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
        mbar_expect_tx(&full[slot], S * 8u);
        bulk_g2s(sm + slot * S, a + ch * S, S * 8u, &full[slot]);
      }
    }
    return;
  }
  double acc = 0.0;
  int c = 0;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++c) {
    const int slot = c % NST;
    mbar_wait(&full[slot], (c / NST) & 1);
    const double* s = sm + slot * S;
    for (int e = tid; e < S; e += 256) acc += s[e];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg_stream(const double4* __restrict__ a, long long n4, double* out) {
  double acc = 0.0;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += 256ll * gridDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(a + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int NST>
int run_tma(const double* a, long long n, double* out, int S, int ctas_per_sm, int sms) {
  const size_t smem = static_cast<size_t>(NST) * S * 8;
  CK(cudaFuncSetAttribute(k_tma_stream<NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const long long nchunks = n / S;
  const int grid = sms * ctas_per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_tma_stream<NST><<<grid, 288, smem>>>(a, nchunks, S, out);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e0));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k_tma_stream<NST><<<grid, 288, smem>>>(a, nchunks, S, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma_stream<NST>, 288, smem));
  std::printf("tma  S=%6d B  NST=%d  grid=%4d (resident/SM %d)  %8.1f GB/s\n", S * 8, NST, grid, occ,
              nchunks * S * 8.0 * reps / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  const long long n = 1ll << 31;  // 16 GiB of doubles
  double *a, *out;
  if (cudaMalloc(&a, n * 8) != cudaSuccess) return 1;
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(a, 0, n * 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int per : {4, 8}) {
      k_ldg_stream<<<sms * per, 256>>>(reinterpret_cast<const double4*>(a), n / 4, out);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) k_ldg_stream<<<sms * per, 256>>>(reinterpret_cast<const double4*>(a), n / 4, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::printf("ldg256 grid=%d x 256   %8.1f GB/s\n", sms * per, n * 8.0 * 5 / (ms * 1e-3) / 1e9);
    }
  }
  for (int S : {1024, 2048, 4096, 5120, 8192}) {
    for (int cps : {1, 2}) {
      if (run_tma<2>(a, n, out, S, cps, sms)) return 1;
      if (run_tma<3>(a, n, out, S, cps, sms)) return 1;
      if (S <= 4096 && run_tma<4>(a, n, out, S, cps, sms)) return 1;
      if (S <= 2048 && run_tma<8>(a, n, out, S, cps, sms)) return 1;
    }
  }
  return 0;
}
