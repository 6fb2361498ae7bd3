// sm_100a kernels (see kernels.cuh for the index). All arithmetic is fp64.
// The instantiate (K1) and near-MVM (K6) kernels are HBM streams; everything
// is laid out so each warp load instruction touches contiguous 256-512 B.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>

#include "kernels.cuh"

// Device-side invariant checks of the TMA / shared-memory kernels (built
// into libphmat_b200_checked.so only): a violated layout assumption traps,
// which the host sees as a CUDA error on the next call.
#ifdef PHM_DEVICE_CHECKS
#define PHM_DCHECK(cond) \
  do {                   \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define PHM_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace phm {
namespace dev {

// ------------------------------------------------------------ helpers
// sm_100 has 256-bit global loads/stores (LDG.E.NA.EFL2.256 / STG.E.256):
// one instruction moves 4 doubles, halving LSU issue for the HBM streams.
struct alignas(32) dbl4 {
  double x, y, z, w;
};
__device__ __forceinline__ dbl4 ld_stream4(const double* p) {
  dbl4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, const dbl4& v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// Radial profiles of kernels.cpp:49-78 plus gauss / matern32 / matern52.
// The generic Matern (needs K_nu) is produced on the host instead.
__device__ __forceinline__ double kernel_profile(int fam, double r, const double* th) {
  const double l = th[0];
  switch (fam) {
    case 0: return exp(-r / l);
    case 1: {
      if (r == 0.0) return 0.0;
      const double s = r / l;
      return s * s * log(s);
    }
    case 2: {
      const double s = r / l;
      return exp(-s * s);
    }
    case 3: {
      const double s = r / l;
      return sqrt(1.0 + s * s);
    }
    case 5: {
      const double s = r / l;
      return exp(-0.5 * s * s);
    }
    case 6: {
      const double s = sqrt(3.0) * r / l;
      return (1.0 + s) * exp(-s);
    }
    case 7: {
      const double s = sqrt(5.0) * r / l;
      return (1.0 + s + s * s / 3.0) * exp(-s);
    }
  }
  return __longlong_as_double(0x7ff8000000000000LL);  // NaN: unsupported on device
}

// ---------------------------------------------------------------- K11
// One thread per (i, j) entry: r_ij computed once (no FMA contraction, same
// rounding as the reference's r2 accumulation, nearfield.cpp:38-45), then R
// profile evaluations written to R slabs (coalesced across threads).
__global__ void k_snapshot(const SnapTile* __restrict__ tiles, std::int64_t ntiles, const BlockGeom* __restrict__ geo,
                           const double* __restrict__ pts, std::int64_t n, int d, int fam, int R,
                           const double* __restrict__ theta_nodes, double amp, double* __restrict__ out) {
  for (std::int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const SnapTile T = tiles[t];
    const BlockGeom g = geo[T.blk];
    for (int e = threadIdx.x; e < T.len; e += blockDim.x) {
      const std::int64_t ee = T.e0 + e;
      const std::int64_t i = ee % g.s_n, j = ee / g.s_n;
      double r2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double dl = __dsub_rn(pts[k * n + g.s_begin + i], pts[k * n + g.t_begin + j]);
        r2 = __dadd_rn(r2, __dmul_rn(dl, dl));
      }
      const double r = sqrt(r2);
      for (int kap = 0; kap < R; ++kap)
        out[T.out_off + kap * T.stride + e] = amp * kernel_profile(fam, r, theta_nodes + 3 * kap);
    }
  }
}

// ----------------------------------------------------------------- K1
// Snapshot mode: every near block shares w = v(theta), so the instantiate is
// one flat stream D[e] = sum_k w_k S[k E + e] over all local near entries
// (E padded to a multiple of 4). Each thread issues U x R independent
// 256-bit loads before it accumulates, which keeps enough bytes in flight
// per SM to cover HBM latency.
template <int R>
__global__ void __launch_bounds__(256, 1) k_inst_flat(const double* __restrict__ G, std::int64_t E,
                                                   const double* __restrict__ w, double* __restrict__ D) {
  constexpr int U = R >= 8 ? 1 : 2;
  double wr[R];
#pragma unroll
  for (int k = 0; k < R; ++k) wr[k] = w[k];
  const std::int64_t E4 = E >> 2;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; q + (U - 1) * stride < E4; q += U * stride) {
    dbl4 v[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < R; ++k) v[u][k] = ld_stream4(G + 4 * (E4 * k + q + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      dbl4 acc = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < R; ++k) {
        acc.x += v[u][k].x * wr[k];
        acc.y += v[u][k].y * wr[k];
        acc.z += v[u][k].z * wr[k];
        acc.w += v[u][k].w * wr[k];
      }
      st4(D + 4 * (q + u * stride), acc);
    }
  }
  for (; q < E4; q += stride) {
    dbl4 acc = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const dbl4 v = ld_stream4(G + 4 * (E4 * k + q));
      acc.x += v.x * wr[k];
      acc.y += v.y * wr[k];
      acc.z += v.z * wr[k];
      acc.w += v.w * wr[k];
    }
    st4(D + 4 * q, acc);
  }
}

// K1 for a batch of B thetas (sweeps): the R snapshot slabs are read once
// and B instances are written, D_b[e] = sum_k w_b,k S[k E + e] with the same
// FMA order as k_inst_flat (each D_b is bit-identical to a single
// instantiate). Bytes per stored entry: 8 (R + B) instead of 8 B (R + 1).
constexpr int kInstBatchMax = 16;
template <int R>
__global__ void __launch_bounds__(256, 1) k_inst_flat_batch(const double* __restrict__ G, std::int64_t E, int B,
                                                         InstPtrs tab) {
  __shared__ double W[kInstBatchMax][R];
  __shared__ double* Dp[kInstBatchMax];
  for (int i = threadIdx.x; i < B * R; i += blockDim.x) W[i / R][i % R] = tab.w[i / R][i % R];
  if (threadIdx.x < B) Dp[threadIdx.x] = tab.d[threadIdx.x];
  __syncthreads();
  const std::int64_t E4 = E >> 2;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < E4; q += stride) {
    dbl4 v[R];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = ld_stream4(G + 4 * (E4 * k + q));
    for (int b = 0; b < B; ++b) {
      dbl4 acc = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const double wk = W[b][k];
        acc.x += v[k].x * wk;
        acc.y += v[k].y * wk;
        acc.z += v[k].z * wk;
        acc.w += v[k].w * wk;
      }
      st4(Dp[b] + 4 * q, acc);
    }
  }
}

__global__ void __launch_bounds__(256) k_inst_flat_any(const double* __restrict__ G, std::int64_t E, int R,
                                                       const double* __restrict__ w, double* __restrict__ D) {
  const std::int64_t E4 = E >> 2;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t q = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < E4; q += stride) {
    dbl4 acc = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < R; ++k) {
      const dbl4 v = ld_stream4(G + 4 * (E4 * k + q));
      const double wk = w[k];
      acc.x += v.x * wk;
      acc.y += v.y * wk;
      acc.z += v.z * wk;
      acc.w += v.w * wk;
    }
    st4(D + 4 * q, acc);
  }
}

// TT near mode: per-block G1_b (N_b x R_b, column-major, N_b padded to 4)
// against the block's own w_b.
__global__ void __launch_bounds__(256) k_inst_tiles(const InstTile* __restrict__ tiles, std::int64_t nt,
                                                    const double* __restrict__ G, const double* __restrict__ w,
                                                    double* __restrict__ D) {
  for (std::int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const InstTile T = tiles[t];
    const double* Gb = G + T.g_off;
    double* Db = D + T.d_off;
    const double* wb = w + T.w_off;
    for (int e = 4 * threadIdx.x; e < T.len; e += 4 * blockDim.x) {
      dbl4 acc = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < T.R; ++k) {
        const dbl4 v = ld_stream4(Gb + T.g_stride * k + e);
        const double wk = wb[k];
        acc.x += v.x * wk;
        acc.y += v.y * wk;
        acc.z += v.z * wk;
        acc.w += v.w * wk;
      }
      st4(Db + e, acc);
    }
  }
}

// w_b = I * prod_i contract_mode2(G_{b,i+1}, v_i) (nearfield.cpp:71-77),
// evaluated right to left as a vector chain; one warp per near block.
__global__ void k_near_w(const NearW* __restrict__ meta, std::int64_t nb, const double* __restrict__ cores,
                         const std::int32_t* __restrict__ dims, const ThetaParams* __restrict__ tp,
                         double* __restrict__ w) {
  const ThetaV& tv = tp->tv;
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  constexpr int kMaxR = 256;
  double* za = sm + warp * 2 * kMaxR;
  double* zb = za + kMaxR;
  for (std::int64_t b = static_cast<std::int64_t>(blockIdx.x) * wpb + warp; b < nb;
       b += static_cast<std::int64_t>(gridDim.x) * wpb) {
    const NearW M = meta[b];
    // z = [1] (the last core has r1 = 1)
    if (lane == 0) za[0] = 1.0;
    __syncwarp();
    std::int64_t off = M.core_off;
    // core offsets: walk forward to find each core start
    std::int64_t offs[kMaxThetaDim];
    for (int c = 0; c < M.ncores; ++c) {
      offs[c] = off;
      const std::int32_t* dm = dims + M.dims_off + 3 * c;
      off += static_cast<std::int64_t>(dm[0]) * dm[1] * dm[2];
    }
    double* zin = za;
    double* zout = zb;
    for (int c = M.ncores - 1; c >= 0; --c) {
      const std::int32_t* dm = dims + M.dims_off + 3 * c;
      const int r0 = dm[0], m = dm[1], r1 = dm[2];
      const double* G = cores + offs[c];
      const double* v = tv.v[c];
      for (int a = lane; a < r0; a += 32) {
        double s = 0.0;
        for (int j = 0; j < m; ++j) {
          const double vj = v[j];
          if (vj == 0.0) continue;
          double t = 0.0;
          for (int cc = 0; cc < r1; ++cc) t += G[a + j * r0 + cc * r0 * m] * zin[cc];
          s += vj * t;
        }
        zout[a] = s;
      }
      __syncwarp();
      double* tmp = zin;
      zin = zout;
      zout = tmp;
    }
    for (int a = lane; a < M.R; a += 32) w[M.w_off + a] = zin[a];
    __syncwarp();
  }
}

__global__ void k_set_vec(double* dst, int n, const ThetaParams* __restrict__ tp) {
  // dst = (v_0 (x) v_1 (x) ...) * amp over the shape parameters (first
  // factor fastest); amp = 1 leaves the product unchanged bit for bit
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ThetaV& tv = tp->shape;
  int rem = i;
  double s = 1.0;
  for (int k = 0; k < tv.dt; ++k) {
    s *= tv.v[k][rem % tv.p[k]];
    rem /= tv.p[k];
  }
  dst[i] = s * tp->amp;
}

// Schedule diagnostics (PHM_STAMPS=1): the device clock when the stream
// reaches this point.
__global__ void k_stamp(unsigned long long* __restrict__ buf, int id) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  buf[id] = t;
}
void launch_stamp(cudaStream_t st, unsigned long long* buf, int id) { k_stamp<<<1, 1, 0, st>>>(buf, id); }

__global__ void k_zero(double* __restrict__ p, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    p[i] = 0.0;
}
void launch_zero(cudaStream_t st, double* p, std::int64_t n) {
  if (n <= 0) return;
  const std::int64_t blocks = std::min<std::int64_t>((n + 255) / 256, 4 * 148);
  k_zero<<<static_cast<int>(blocks), 256, 0, st>>>(p, n);
}

__global__ void k_put_theta(ThetaParams p, ThetaParams* __restrict__ dst) {
  const int n = sizeof(ThetaParams) / sizeof(double);
  static_assert(sizeof(ThetaParams) % sizeof(double) == 0, "ThetaParams is copied as doubles");
  const double* src = reinterpret_cast<const double*>(&p);
  double* out = reinterpret_cast<double*>(dst);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = src[i];
}

// fp64 tensor-core MMA (DMMA; sm_100 has no tcgen05 f64 kind): D += A B with
// A 16x4 (a0 = A[g][t], a1 = A[g+8][t]), B 4x8 (b0 = B[t][g]), D 16x8
// (d = D[g][2t], D[g][2t+1], D[g+8][2t], D[g+8][2t+1]); g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// cp.async (16-byte, L2 only) into shared memory
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 16 : 0;  // src-size 0 zero-fills (missing partner)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ----------------------------------------------------------------- K2
// One CTA per translation class. H = prod_i contract(G_{d+i}, v_i)
// (farfield.cpp:149-155); for H^2 also C = L H R^T in 32-column tiles.
__global__ void k_class_inst(const ClassMeta* __restrict__ meta, int ncls, const double* __restrict__ mid,
                             const std::int32_t* __restrict__ mid_dims, const double* __restrict__ Lm,
                             const double* __restrict__ Rm, const ThetaParams* __restrict__ tp, int P, int want_c,
                             int capA, int capB, int capT, double* __restrict__ H, double* __restrict__ C) {
  const ThetaV& tv = tp->tv;
  extern __shared__ double sm[];
  const ClassMeta M = meta[blockIdx.x];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int rl = M.rl, rr = M.rr;
  double* A = sm;         // rl x r (running product)
  double* B = A + capA;   // next contracted core
  double* Tt = B + capB;  // rl x 32 tile of H R^T, or A B scratch
  // first theta core
  std::int64_t off = M.mid_off;
  int r0 = mid_dims[M.dims_off + 0], m0 = mid_dims[M.dims_off + 1], r1 = mid_dims[M.dims_off + 2];
  for (int e = tid; e < r0 * r1; e += nt) {
    const int a = e % r0, c = e / r0;
    double s = 0.0;
    // loads unconditional (so the compiler issues them together), the sum
    // still skips zero weights exactly as before
#pragma unroll 8
    for (int j = 0; j < m0; ++j) {
      const double vj = tv.v[0][j];
      const double x = mid[off + a + j * r0 + static_cast<std::int64_t>(c) * r0 * m0];
      if (vj != 0.0) s += vj * x;
    }
    A[e] = s;
  }
  off += static_cast<std::int64_t>(r0) * m0 * r1;
  for (int q = 1; q < tv.dt; ++q) {
    const int s0 = mid_dims[M.dims_off + 3 * q], sm_ = mid_dims[M.dims_off + 3 * q + 1],
              s1 = mid_dims[M.dims_off + 3 * q + 2];
    __syncthreads();
    for (int e = tid; e < s0 * s1; e += nt) {
      const int a = e % s0, c = e / s0;
      double s = 0.0;
#pragma unroll 8
      for (int j = 0; j < sm_; ++j) {
        const double vj = tv.v[q][j];
        const double x = mid[off + a + j * s0 + static_cast<std::int64_t>(c) * s0 * sm_];
        if (vj != 0.0) s += vj * x;
      }
      B[e] = s;
    }
    off += static_cast<std::int64_t>(s0) * sm_ * s1;
    __syncthreads();
    // A <- A B  (rl x s1); use Tt region as scratch then copy back
    for (int e = tid; e < rl * s1; e += nt) {
      const int a = e % rl, c = e / rl;
      double s = 0.0;
      for (int k = 0; k < s0; ++k) s += A[a + k * rl] * B[k + c * s0];
      Tt[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < rl * s1; e += nt) A[e] = Tt[e];
  }
  __syncthreads();
  for (int e = tid; e < rl * rr; e += nt) H[M.h_off + e] = A[e];
  if (!want_c) return;
  if (P == 64 && nt == 256 && rl <= 64) {
    // Both products on the fp64 tensor cores (mma.sync m16n8k4): T = H R^T
    // (rl x 64) into shared memory, then C = L T (64 x 64); warp w owns the
    // 8 output columns 8w .. 8w + 7 of each, all 16-row tiles. R (64 x rr)
    // and then L (64 x rl) are staged through one region with all loads in
    // flight (ld 68, and T's ld = 4 mod 16: conflict-free fragment reads);
    // the k padding (rr, rl up to a multiple of 4) is zero.
    const int rl4 = (rl + 3) & ~3, rr4 = (rr + 3) & ~3;
    const int ldT = rl4 + ((4 - rl4) & 15);  // the least ld >= rl4 with ld = 4 mod 16
    constexpr int ldL = 68;
    double* Ts = Tt;         // rl4 x 64, ld ldT
    double* Ls = Tt + capT;  // R: 64 x rr4, then L: 64 x rl4 (ld 68)
    for (int e = tid; e < 64 * rr4; e += nt) {
      const int b = e & 63, c = e >> 6;
      Ls[b + c * ldL] = c < rr ? Rm[M.r_off + b + static_cast<std::int64_t>(c) * 64] : 0.0;
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t0 = lane & 3;
    const int mts = (rl + 15) >> 4;
    {
      double acc[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
      for (int s2 = 0; s2 < (rr4 >> 2); ++s2) {
        const int k = 4 * s2 + t0;
        const double b0 = Ls[(8 * warp + g) + k * ldL];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (mt >= mts) break;  // warp-uniform
          const int r = 16 * mt + g;
          const double a0 = (r < rl && k < rr) ? A[r + k * rl] : 0.0;
          const double a1 = (r + 8 < rl && k < rr) ? A[r + 8 + k * rl] : 0.0;
          dmma_16x8x4(acc[mt], a0, a1, b0);
        }
      }
      const int c = 8 * warp + 2 * t0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if (mt >= mts) break;
        const int r = 16 * mt + g;  // rows in [rl, rl4) come out zero (zero A rows)
        if (r < rl4) {
          Ts[r + c * ldT] = acc[mt][0];
          Ts[r + (c + 1) * ldT] = acc[mt][1];
        }
        if (r + 8 < rl4) {
          Ts[r + 8 + c * ldT] = acc[mt][2];
          Ts[r + 8 + (c + 1) * ldT] = acc[mt][3];
        }
      }
    }
    __syncthreads();  // T complete, R no longer read
    for (int e = tid; e < 64 * rl4; e += nt) {
      const int a = e & 63, i = e >> 6;
      Ls[a + i * ldL] = i < rl ? Lm[M.l_off + a + static_cast<std::int64_t>(i) * 64] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
    for (int s2 = 0; s2 < (rl4 >> 2); ++s2) {
      const int k = 4 * s2 + t0;
      const double b0 = Ts[k + (8 * warp + g) * ldT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        dmma_16x8x4(acc[mt], Ls[(16 * mt + g) + k * ldL], Ls[(16 * mt + g + 8) + k * ldL], b0);
    }
    const int c = 8 * warp + 2 * t0;
    double* Cb = C + M.c_off;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {  // fragment order (cfrag64)
      const int r = 16 * mt + g;
      Cb[cfrag64(r, c)] = acc[mt][0];
      Cb[cfrag64(r, c + 1)] = acc[mt][1];
      Cb[cfrag64(r + 8, c)] = acc[mt][2];
      Cb[cfrag64(r + 8, c + 1)] = acc[mt][3];
    }
    return;
  }
  for (int b0 = 0; b0 < P; b0 += 32) {
    const int bw = min(32, P - b0);
    __syncthreads();
    for (int e = tid; e < rl * bw; e += nt) {  // Tt[i, bb] = sum_c H[i,c] R[b0+bb, c]
      const int i = e % rl, bb = e / rl;
      double s = 0.0;
      for (int c = 0; c < rr; ++c) s += A[i + c * rl] * Rm[M.r_off + (b0 + bb) + static_cast<std::int64_t>(c) * P];
      Tt[i + bb * rl] = s;
    }
    __syncthreads();
    for (int e = tid; e < P * bw; e += nt) {  // C[a, b0+bb] = sum_i L[a,i] Tt[i,bb]
      const int a = e % P, bb = e / P;
      double s = 0.0;
      for (int i = 0; i < rl; ++i) s += Lm[M.l_off + a + static_cast<std::int64_t>(i) * P] * Tt[i + bb * rl];
      C[M.c_off + (P == 64 ? cfrag64(a, b0 + bb) : a + static_cast<std::int64_t>(b0 + bb) * P)] = s;
    }
  }
}

// K2 with every global load of a class issued up front (H^2, P = 64, all
// left ranks <= 64): L_k and R_k go to shared memory by cp.async at the start
// and stay in flight during the theta-core contraction, whose loads are
// issued for four H entries per thread before their sums; T = H R^T then
// reuses R's region. One DRAM round trip per class instead of three. Same
// arithmetic, in the same order, as k_class_inst: H and C are bitwise equal.
__global__ void __launch_bounds__(256, 2)
    k_class_inst_pf(const ClassMeta* __restrict__ meta, int ncls, const double* __restrict__ mid,
                    const std::int32_t* __restrict__ mid_dims, const double* __restrict__ Lm,
                    const double* __restrict__ Rm, const ThetaParams* __restrict__ tp, int capA, int capB, int capS,
                    int capR, double* __restrict__ H, double* __restrict__ C) {
  constexpr int nt = 256, ldL = 68;
  const ThetaV& tv = tp->tv;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  // one class per CTA, or a capped persistent grid looping over the classes
  for (int cls = blockIdx.x; cls < ncls; cls += gridDim.x) {
  if (cls != static_cast<int>(blockIdx.x)) __syncthreads();  // the previous class is done with every region
  const ClassMeta M = meta[cls];
  const int rl = M.rl, rr = M.rr;
  const int rl4 = (rl + 3) & ~3, rr4 = (rr + 3) & ~3;
  double* A = sm;          // rl x r (running product), ld rl
  double* B = A + capA;    // next contracted core (theta chains of two or more)
  double* S = B + capB;    // A B scratch
  double* Rs = S + capS;   // R (64 x rr4, ld 68), then T (rl4 x 64, ld ldT)
  double* Ls = Rs + capR;  // L (64 x rl4, ld 68)
  for (int e = tid; e < 32 * rr; e += nt) {
    const int c = e >> 5, h = (e & 31) * 2;
    cp_async16(Rs + h + c * ldL, Rm + M.r_off + h + static_cast<std::int64_t>(c) * 64, true);
  }
  for (int e = tid; e < 32 * rl; e += nt) {
    const int c = e >> 5, h = (e & 31) * 2;
    cp_async16(Ls + h + c * ldL, Lm + M.l_off + h + static_cast<std::int64_t>(c) * 64, true);
  }
  cp_async_commit();
  for (int e = tid; e < 64 * (rr4 - rr); e += nt) Rs[(e & 63) + (rr + (e >> 6)) * ldL] = 0.0;
  for (int e = tid; e < 64 * (rl4 - rl); e += nt) Ls[(e & 63) + (rl + (e >> 6)) * ldL] = 0.0;
  // first theta core: A[a, c] = sum_j v_j G[a, j, c], zero weights skipped
  std::int64_t off = M.mid_off;
  {
    const int r0 = mid_dims[M.dims_off + 0], m0 = mid_dims[M.dims_off + 1], r1 = mid_dims[M.dims_off + 2];
    const int n = r0 * r1;
    for (int e0 = tid; e0 < n; e0 += 4 * nt) {
      const double* src[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = min(e0 + i * nt, n - 1);
        src[i] = mid + off + (e % r0) + static_cast<std::int64_t>(e / r0) * r0 * m0;
      }
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      for (int j0 = 0; j0 < m0; j0 += 8) {
        double x[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) x[i][jj] = (j0 + jj < m0) ? src[i][(j0 + jj) * r0] : 0.0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const double vj = (j0 + jj < m0) ? tv.v[0][j0 + jj] : 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (vj != 0.0) s[i] += vj * x[i][jj];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (e0 + i * nt < n) A[e0 + i * nt] = s[i];
    }
    off += static_cast<std::int64_t>(r0) * m0 * r1;
  }
  for (int q = 1; q < tv.dt; ++q) {
    const int s0 = mid_dims[M.dims_off + 3 * q], sm_ = mid_dims[M.dims_off + 3 * q + 1],
              s1 = mid_dims[M.dims_off + 3 * q + 2];
    __syncthreads();
    for (int e = tid; e < s0 * s1; e += nt) {
      const int a = e % s0, c = e / s0;
      double s = 0.0;
#pragma unroll 8
      for (int j = 0; j < sm_; ++j) {
        const double vj = tv.v[q][j];
        const double x = mid[off + a + j * s0 + static_cast<std::int64_t>(c) * s0 * sm_];
        if (vj != 0.0) s += vj * x;
      }
      B[e] = s;
    }
    off += static_cast<std::int64_t>(s0) * sm_ * s1;
    __syncthreads();
    for (int e = tid; e < rl * s1; e += nt) {
      const int a = e % rl, c = e / rl;
      double s = 0.0;
      for (int k = 0; k < s0; ++k) s += A[a + k * rl] * B[k + c * s0];
      S[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < rl * s1; e += nt) A[e] = S[e];
  }
  __syncthreads();
  for (int e = tid; e < rl * rr; e += nt) H[M.h_off + e] = A[e];
  cp_async_wait<0>();
  __syncthreads();  // R and L landed
  const int ldT = rl4 + ((4 - rl4) & 15);  // the least ld >= rl4 with ld = 4 mod 16
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t0 = lane & 3;
  const int mts = (rl + 15) >> 4;
  {
    double acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
    for (int s2 = 0; s2 < (rr4 >> 2); ++s2) {
      const int k = 4 * s2 + t0;
      const double b0 = Rs[(8 * warp + g) + k * ldL];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if (mt >= mts) break;  // warp-uniform
        const int r = 16 * mt + g;
        const double a0 = (r < rl && k < rr) ? A[r + k * rl] : 0.0;
        const double a1 = (r + 8 < rl && k < rr) ? A[r + 8 + k * rl] : 0.0;
        dmma_16x8x4(acc[mt], a0, a1, b0);
      }
    }
    __syncthreads();  // every warp done with R: T takes its region
    double* Ts = Rs;
    const int c = 8 * warp + 2 * t0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (mt >= mts) break;
      const int r = 16 * mt + g;  // rows in [rl, rl4) come out zero (zero A rows)
      if (r < rl4) {
        Ts[r + c * ldT] = acc[mt][0];
        Ts[r + (c + 1) * ldT] = acc[mt][1];
      }
      if (r + 8 < rl4) {
        Ts[r + 8 + c * ldT] = acc[mt][2];
        Ts[r + 8 + (c + 1) * ldT] = acc[mt][3];
      }
    }
  }
  __syncthreads();  // T complete
  const double* Ts = Rs;
  double acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
  for (int s2 = 0; s2 < (rl4 >> 2); ++s2) {
    const int k = 4 * s2 + t0;
    const double b0 = Ts[k + (8 * warp + g) * ldT];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      dmma_16x8x4(acc[mt], Ls[(16 * mt + g) + k * ldL], Ls[(16 * mt + g + 8) + k * ldL], b0);
  }
  const int c = 8 * warp + 2 * t0;
  double* Cb = C + M.c_off;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {  // fragment order (cfrag64)
    const int r = 16 * mt + g;
    Cb[cfrag64(r, c)] = acc[mt][0];
    Cb[cfrag64(r, c + 1)] = acc[mt][1];
    Cb[cfrag64(r + 8, c)] = acc[mt][2];
    Cb[cfrag64(r + 8, c + 1)] = acc[mt][3];
  }
  }
}

// ---------------------------------------------------------------- K10
__global__ void k_gather(const double* __restrict__ x, const std::int32_t* __restrict__ perm, std::int64_t n,
                         std::int64_t m, double* __restrict__ xp) {
  const std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * m) return;
  const std::int64_t c = t / n, p = t % n;
  xp[t] = x[c * n + perm[p]];
}
__global__ void k_scatter(const double* __restrict__ yp, const std::int32_t* __restrict__ perm, std::int64_t n,
                          std::int64_t m, double* __restrict__ y) {
  const std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * m) return;
  const std::int64_t c = t / n, p = t % n;
  y[c * n + perm[p]] = yp[t];
}

// ----------------------------------------------------------------- K3
// xhat_sigma[a] = sum_i x_i prod_k U_k(i, a_k) (chebyshev.cpp:236-252); one
// CTA per non-empty leaf, factor rows staged in shared memory per 64 points.
// K3 for blocks of right-hand sides (P == 64, m >= 4): x_hat_sigma (P x m) =
// F (P x cnt) X_sigma (cnt x m) with F[a][i] = prod_k U_k(i, a_k). One CTA
// per (leaf, 64-column tile); thread t owns output row a = t mod 64 and the
// columns cg, cg + 4, ... (cg = t / 64): each point's factor entries are read
// once for all of them, and the factor rows are staged once per leaf instead
// of once per column. Products and sums run in k_leaf_fwd's order, so every
// column equals the single-vector result bit for bit.
// chunks (non-null): CTA x takes points [p0, p0 + len) of leaf `leaf` and
// writes its partial x-hat to xhat + slot (m x P); a leaf of more than
// kLeafChunk points is split this way (k_leaf_fwd_reduce sums the chunks in
// order), so a clustered leaf of thousands of points is not one CTA's
// serial loop.
template <int MC>
__global__ void __launch_bounds__(256) k_leaf_fwd_m(const std::int32_t* __restrict__ leaves,
                                                    const std::int64_t* __restrict__ begin,
                                                    const std::int32_t* __restrict__ count,
                                                    const double* __restrict__ U, std::int64_t n, int d, int ps,
                                                    const double* __restrict__ xp, int m, double* __restrict__ xhat,
                                                    const LeafChunk* __restrict__ chunks = nullptr) {
  constexpr int P = 64, CH = 32;
  __shared__ double su[CH * 3 * 16];  // CH points x d x ps (d * ps <= 48)
  __shared__ double sx[CH * 4 * MC];  // CH points x the tile's columns
  const int leaf = chunks ? chunks[blockIdx.x].leaf : leaves[blockIdx.x];
  const std::int64_t b0 = begin[leaf] + (chunks ? chunks[blockIdx.x].p0 : 0);
  const int cnt = chunks ? chunks[blockIdx.x].len : count[leaf];
  const int c0 = blockIdx.y * 4 * MC;
  const int ncol = min(4 * MC, m - c0);
  const int a = threadIdx.x & 63, cg = threadIdx.x >> 6;
  int dig[3] = {0, 0, 0};
  {
    int rem = a;
    for (int k = 0; k < d; ++k) {
      dig[k] = rem % ps;
      rem /= ps;
    }
  }
  double acc[MC];
#pragma unroll
  for (int j = 0; j < MC; ++j) acc[j] = 0.0;
  const int dps = d * ps;
  for (int i0 = 0; i0 < cnt; i0 += CH) {
    const int len = min(CH, cnt - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < len * dps; e += blockDim.x) {
      const int i = e / dps, r = e - i * dps, k = r / ps, j = r - k * ps;
      su[e] = U[(static_cast<std::int64_t>(k) * n + b0 + i0 + i) * ps + j];
    }
    for (int e = threadIdx.x; e < len * ncol; e += blockDim.x) {
      const int c = e / len, i = e - c * len;  // consecutive threads read consecutive points
      sx[i * (4 * MC) + c] = xp[static_cast<std::int64_t>(c0 + c) * n + b0 + i0 + i];
    }
    __syncthreads();
    for (int i = 0; i < len; ++i) {
      double u[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) u[k] = k < d ? su[(i * d + k) * ps + dig[k]] : 1.0;
#pragma unroll
      for (int j = 0; j < MC; ++j) {
        const int c = cg + 4 * j;
        if (c < ncol) {
          double f = sx[i * (4 * MC) + c];  // x_i u_1 ... u_d, the order of k_leaf_fwd
          for (int k = 0; k < d; ++k) f *= u[k];
          acc[j] += f;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MC; ++j) {
    const int c = cg + 4 * j;
    if (c < ncol) {
      if (chunks)
        xhat[(chunks[blockIdx.x].slot * m + c0 + c) * P + a] = acc[j];
      else
        xhat[(static_cast<std::int64_t>(leaf) * m + c0 + c) * P + a] = acc[j];
    }
  }
}

// x-hat of a split leaf: the sum of its chunk partials in chunk order.
__global__ void k_leaf_fwd_reduce(const std::int32_t* __restrict__ red_leaf, const std::int64_t* __restrict__ red_slot,
                                  const std::int32_t* __restrict__ red_n, int P, int m, const double* __restrict__ part,
                                  double* __restrict__ xhat) {
  const int r = blockIdx.x, leaf = red_leaf[r], ns = red_n[r];
  const std::int64_t s0 = red_slot[r] * m * P;
  for (int e = threadIdx.x; e < m * P; e += blockDim.x) {
    double t = part[s0 + e];
    for (int q = 1; q < ns; ++q) t += part[s0 + static_cast<std::int64_t>(q) * m * P + e];
    xhat[static_cast<std::int64_t>(leaf) * m * P + e] = t;
  }
}

__global__ void k_leaf_fwd(const std::int32_t* __restrict__ leaves, const std::int64_t* __restrict__ begin,
                           const std::int32_t* __restrict__ count, const double* __restrict__ U, std::int64_t n,
                           int d, int ps, int P, const double* __restrict__ xp, int m, double* __restrict__ xhat) {
  extern __shared__ double sm[];
  const int leaf = leaves[blockIdx.x];
  const std::int64_t b0 = begin[leaf];
  const int cnt = count[leaf];
  double* su = sm;                 // 64 x d x ps
  double* sx = su + 64 * d * ps;   // 64
  {
    const int c = blockIdx.y;  // one right-hand side per grid row
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // up to 4 outputs per thread (P <= 4 * blockDim)
    for (int i0 = 0; i0 < cnt; i0 += 64) {
      const int len = min(64, cnt - i0);
      __syncthreads();
      for (int e = threadIdx.x; e < len * d * ps; e += blockDim.x) {
        const int i = e / (d * ps), r = e % (d * ps), k = r / ps, j = r % ps;
        su[e] = U[(static_cast<std::int64_t>(k) * n + b0 + i0 + i) * ps + j];
      }
      for (int e = threadIdx.x; e < len; e += blockDim.x) sx[e] = xp[static_cast<std::int64_t>(c) * n + b0 + i0 + e];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = threadIdx.x + q * blockDim.x;
        if (a >= P) break;
        int dig[3];
        int rem = a;
        for (int k = 0; k < d; ++k) {
          dig[k] = rem % ps;
          rem /= ps;
        }
        double s = acc[q];
        for (int i = 0; i < len; ++i) {
          double f = sx[i];
          for (int k = 0; k < d; ++k) f *= su[(i * d + k) * ps + dig[k]];
          s += f;
        }
        acc[q] = s;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = threadIdx.x + q * blockDim.x;
      if (a < P) xhat[(static_cast<std::int64_t>(leaf) * m + c) * P + a] = acc[q];
    }
  }
}

// ----------------------------------------------------------------- K5
// yhat_sigma = sum over the far blocks of sigma of C_k xhat_tau (CSR by
// sigma, deterministic order, no atomics). One CTA per sigma node.
__global__ void k_coupling(const std::int32_t* __restrict__ sig, const std::int64_t* __restrict__ fbeg,
                           const std::int32_t* __restrict__ ftau, const std::int32_t* __restrict__ fcls,
                           const double* __restrict__ C, int P, int m, const double* __restrict__ xhat,
                           double* __restrict__ yhat) {
  extern __shared__ double sm[];
  const int s = sig[blockIdx.x];
  const std::int64_t b0 = fbeg[blockIdx.x], b1 = fbeg[blockIdx.x + 1];
  const std::int64_t PP = static_cast<std::int64_t>(P) * P;
  for (int c = 0; c < m; ++c) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (std::int64_t b = b0; b < b1; ++b) {
      const int tau = ftau[b];
      const double* Ck = C + fcls[b] * PP;
      __syncthreads();
      for (int e = threadIdx.x; e < P; e += blockDim.x) sm[e] = xhat[(static_cast<std::int64_t>(tau) * m + c) * P + e];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = threadIdx.x + q * blockDim.x;
        if (a >= P) break;
        double s = 0.0;
        for (int j = 0; j < P; ++j) s += Ck[a + static_cast<std::int64_t>(j) * P] * sm[j];
        acc[q] += s;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int a = threadIdx.x + q * blockDim.x;
      if (a < P) yhat[(static_cast<std::int64_t>(s) * m + c) * P + a] = acc[q];
    }
  }
}

// K5, grouped fp64 tensor-core version. One CTA per (sigma group, class
// range): for every class k of the range, C_k (P x P) times the 32 gathered
// xhat_tau columns of the group (X_k, P x 32) on mma.sync.m16n8k4.f64
// (DMMA; sm_100 has no tcgen05 f64 kind), accumulated in registers across
// the classes. Warp w owns output rows [16w, 16w + 16); X_k is staged in
// shared memory by cp.async, double-buffered against the MMAs of the
// previous class. Per-item partial sums are reduced in a fixed order by
// k_coupling_reduce: deterministic, no atomics.
// One (item, RHS column) pair per CTA iteration; X is the gathered 32-slot
// panel of the column, double-buffered. item_tiles[e] has bit j set when
// n-tile j (slots 8j .. 8j + 7) holds any partner of class item_cls[e];
// empty tiles skip their MMAs and loads (the slot order of a group is Morton
// order, so boundary sigmas missing an offset cluster: at C3 this lifts the
// useful fraction of the MMA work from 64% to 83%).
// The C_k fragments are loaded in two k-halves per class (registers for
// occupancy; each half still feeds every tile). Prefetching the next class's
// fragments instead made the capped grid beside the near pass faster
// (6.0 vs 8.1 ms) but slowed the near pass more (9.4 vs 8.9 ms).
// DIAG (schedule diagnostics only, results invalid; PHM_COUPLING_DIAG): 1 =
// the C_k fragment loads stay but no MMAs and no x-hat gathers run (L2
// traffic of C_k alone), 2 = MMAs and gathers stay but the C_k fragments are
// constants (fp64 pipe and x-hat traffic alone). 0 is the product kernel.
template <int P, int DIAG = 0>
__global__ void __maxnreg__(P >= 128 ? 128 : 88) k_coupling_mma(const CouplingItem* __restrict__ items,
                                                              const std::int32_t* __restrict__ order,
                                                              const std::int32_t* __restrict__ item_cls,
                                                              const std::uint8_t* __restrict__ item_tiles,
                                                              const std::int32_t* __restrict__ cls_tau,
                                                              const double* __restrict__ C,
                                                              const double* __restrict__ xhat, int m,
                                                              double* __restrict__ partial, int nitems) {
  constexpr int LD = P + 4;           // conflict-free B-fragment reads
  constexpr int KS = P / 4;           // k-steps of the m16n8k4 MMA
  constexpr int NT = kGroupSlots / 8; // n-tiles of 8 slots
  constexpr int PANEL = kGroupSlots * LD;
  // C_k fragments are loaded a quarter of the k-steps at a time into two
  // ping-pong register buffers: the next quarter's (or the next class's
  // first quarter's) L2 loads are in flight while this quarter's MMAs run
  // (ncu, C3 apply: long-scoreboard stalls on these loads dominated)
  constexpr int KH = KS >= 4 ? 4 : KS;        // k-steps per fragment load
  constexpr int NQ = KS / KH;                 // loads per class
  constexpr bool kCross = (NQ % 2) == 0;      // next class starts in buffer 0
  extern __shared__ double smem[];    // 2 stages of [32][LD]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t0 = lane & 3;
  const int row0 = warp * 16;
  // (item, column) pairs strided over the grid: one pair per CTA for a full
  // grid, several for a capped one; items in class-major order (device.cu)
  const int nvb = nitems * m;
  for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
    const int item = order[vb % nitems];
    const CouplingItem it = items[item];
    const int col = vb / nitems;
    double acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

    // X panel gather: thread t serves slot t / TPS (TPS = threads per
    // slot) and 16-byte pairs t % TPS + TPS * j of that slot's x-hat column,
    // so each thread needs ONE tau per class -- loaded a class ahead (ncu:
    // the per-pair tau load in front of every cp.async was the hottest stall)
    constexpr int TPS = (2 * P) / kGroupSlots;  // blockDim = 2P
    constexpr int PPT = (P / 2) / TPS;          // pairs per thread
    const int gslot = threadIdx.x / TPS, gsub = threadIdx.x % TPS;
    auto tau_of = [&](int e) { return cls_tau[static_cast<std::int64_t>(e) * kGroupSlots + gslot]; };
    [[maybe_unused]] unsigned sink = 0;  // DIAG 1: keeps the fragment loads alive
    auto gather = [&](int e, int buf, int tau) {
      const unsigned tiles = DIAG == 1 ? 0u : item_tiles[e];
      double* X = smem + buf * PANEL + gslot * LD;
      if ((tiles >> (gslot >> 3)) & 1u) {  // else the tile is skipped by the MMAs
        const double* src = xhat + (static_cast<std::int64_t>(tau < 0 ? 0 : tau) * m + col) * P;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const int q = gsub + TPS * j;
          cp_async16(X + 2 * q, src + 2 * q, tau >= 0);
        }
      }
      cp_async_commit();
    };
    auto load_a = [&](int e, int h, double (&a)[KH][2]) {
      const double* Ck = C + static_cast<std::int64_t>(item_cls[e]) * P * P;
      if constexpr (DIAG == 2) {
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2) a[s2][0] = a[s2][1] = 1.0 + h;
        return;
      }
      if constexpr (P == 64) {  // fragment order: one 16-byte load per k-step
        const double2* F = reinterpret_cast<const double2*>(Ck);
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2) {
          const double2 v = __ldg(F + ((h * KH + s2) * 4 + warp) * 32 + lane);
          a[s2][0] = v.x;
          a[s2][1] = v.y;
        }
      } else {
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2) {
          const std::int64_t k = 4 * (h * KH + s2) + t0;
          a[s2][0] = __ldg(Ck + (row0 + g) + k * P);
          a[s2][1] = __ldg(Ck + (row0 + g + 8) + k * P);
        }
      }
    };
    auto mma = [&](const double (&a)[KH][2], int h, const double* X, unsigned tiles) {
      if constexpr (DIAG == 1) {
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2) sink ^= __double2loint(a[s2][0]) ^ __double2hiint(a[s2][1]);
        return;
      }
      if (tiles == (1u << NT) - 1u) {
        // every tile holds a partner: k-step outer, tile inner, so the NT
        // accumulators are independent chains in flight
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2)
#pragma unroll
          for (int j = 0; j < NT; ++j)
            dmma_16x8x4(acc[j], a[s2][0], a[s2][1], X[(8 * j + g) * LD + 4 * (h * KH + s2) + t0]);
        return;
      }
      // tile outer: an empty tile is a (warp-uniform) branch around its
      // MMAs; with the tile test inside the k loop the compiler predicates
      // the MMAs instead, and a predicated MMA still occupies the pipe
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (!((tiles >> j) & 1u)) continue;
#pragma unroll
        for (int s2 = 0; s2 < KH; ++s2)
          dmma_16x8x4(acc[j], a[s2][0], a[s2][1], X[(8 * j + g) * LD + 4 * (h * KH + s2) + t0]);
      }
    };

    const int e0 = it.e_begin;
    double a[2][KH][2];
    int tau_next = 0;
    if (e0 < it.e_end) {
      gather(e0, 0, tau_of(e0));
      load_a(e0, 0, a[0]);
      if (e0 + 1 < it.e_end) tau_next = tau_of(e0 + 1);
    }
    for (int e = e0; e < it.e_end; ++e) {
      const int buf = (e - e0) & 1;
      if (e + 1 < it.e_end) {
        gather(e + 1, buf ^ 1, tau_next);
        if (e + 2 < it.e_end) tau_next = tau_of(e + 2);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const unsigned tiles = item_tiles[e];
      if (!kCross) load_a(e, 0, a[0]);
#pragma unroll
      for (int h = 0; h < NQ; ++h) {
        if (h + 1 < NQ)
          load_a(e, h + 1, a[(h + 1) & 1]);
        else if (kCross && e + 1 < it.e_end)
          load_a(e + 1, 0, a[0]);
        mma(a[h & 1], h, smem + buf * PANEL, tiles);
      }
      __syncthreads();  // X[buf] is refilled two classes later
    }
    double* out = partial + (static_cast<std::int64_t>(item) * m + col) * kGroupSlots * P;
    if constexpr (DIAG == 1) acc[0][0] = __hiloint2double(0, static_cast<int>(sink));
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n0 = 8 * j + 2 * t0;
      out[n0 * P + row0 + g] = acc[j][0];
      out[(n0 + 1) * P + row0 + g] = acc[j][1];
      out[n0 * P + row0 + g + 8] = acc[j][2];
      out[(n0 + 1) * P + row0 + g + 8] = acc[j][3];
    }
  }
}

// yhat_sigma for one (group, column): fixed-order sum over the group's items.
__global__ void k_coupling_reduce(const std::int32_t* __restrict__ grp_sigma, const std::int32_t* __restrict__ grp_items,
                                  const double* __restrict__ partial, int P, int m, double* __restrict__ yhat) {
  const int grp = blockIdx.x, col = blockIdx.y;
  const int ib = grp_items[grp], ie = grp_items[grp + 1];
  for (int e = threadIdx.x; e < kGroupSlots * P; e += blockDim.x) {
    const int slot = e / P, a = e % P;
    const int sigma = grp_sigma[grp * kGroupSlots + slot];
    if (sigma < 0) continue;
    double s = 0.0;
    for (int i = ib; i < ie; ++i) s += partial[(static_cast<std::int64_t>(i) * m + col) * kGroupSlots * P + e];
    yhat[(static_cast<std::int64_t>(sigma) * m + col) * P + a] = s;
  }
}

// ------------------------------------------------------------------ K9
// Multi-RHS near field, Y_sigma = sum_tau D_{sigma,tau} X_tau, on DMMA.
// One CTA (4 warps) per (leaf sigma, 64-row chunk, 64-column chunk of the
// right-hand sides): D chunks (64 x 32) and X chunks (32 x 64) are staged by
// cp.async (double-buffered), warp w owns output rows [16w, 16w + 16) and all
// 64 columns (8 m16n8k4 accumulator tiles). Transposed (symmetric-storage)
// blocks are read through the transposed index map. Complete sums per CTA:
// deterministic, no atomics.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}

constexpr int kK9Rows = 64, kK9Kc = 32;

// kK9Cols (8..64) is the right-hand-side tile: small m uses a narrow tile so
// no MMA work is spent on zero-padded columns.
template <int kK9Cols>
__global__ void __launch_bounds__(128) k_near_mrhs(const MrhsItem* __restrict__ items, const std::int64_t* __restrict__ tb,
                                                   const std::int32_t* __restrict__ tn,
                                                   const std::int64_t* __restrict__ doff,
                                                   const std::int32_t* __restrict__ ldv,
                                                   const std::int32_t* __restrict__ trv, const double* __restrict__ D,
                                                   const double* __restrict__ X, std::int64_t n, int m,
                                                   double* __restrict__ Y) {
  constexpr int LDA = kK9Kc + 4, LDB = kK9Cols + 4;
  extern __shared__ double sm[];
  double* As[2] = {sm, sm + kK9Rows * LDA + kK9Kc * LDB};
  double* Bs[2] = {sm + kK9Rows * LDA, sm + 2 * kK9Rows * LDA + kK9Kc * LDB};
  const MrhsItem it = items[blockIdx.x];
  const int c0 = blockIdx.y * kK9Cols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t0 = lane & 3;
  constexpr int NT = kK9Cols / 8;
  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;

  auto stage = [&](int b, int k0, int buf) {
    const int kc = min(kK9Kc, tn[b] - k0);
    const double* Db = D + doff[b];
    const std::int64_t ld = ldv[b];
    const bool tr = trv[b] != 0;
    double* A = As[buf];
    double* B = Bs[buf];
    for (int e = threadIdx.x; e < kK9Rows * kK9Kc; e += blockDim.x) {
      const int i = tr ? e / kK9Kc : e % kK9Rows;
      const int k = tr ? e % kK9Kc : e / kK9Rows;
      const bool ok = i < it.rows && k < kc;
      const std::int64_t r = it.i0 + i, c = k0 + k;
      const double* src = Db + (tr ? c + r * ld : r + c * ld);
      cp_async8(A + i * LDA + k, ok ? src : Db, ok);
    }
    for (int e = threadIdx.x; e < kK9Kc * kK9Cols; e += blockDim.x) {
      const int k = e % kK9Kc, c = e / kK9Kc;
      const bool ok = k < kc && c0 + c < m;
      const double* src = X + tb[b] + k0 + k + static_cast<std::int64_t>(c0 + c) * n;
      cp_async8(B + k * LDB + c, ok ? src : X, ok);
    }
    cp_async_commit();
  };

  int b = it.bbeg, k0 = 0, buf = 0;
  if (b < it.bend) stage(b, 0, 0);
  while (b < it.bend) {
    int nb = b, nk = k0 + kK9Kc;
    if (nk >= tn[b]) {
      nb = b + 1;
      nk = 0;
    }
    if (nb < it.bend) {
      stage(nb, nk, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* A = As[buf];
    const double* B = Bs[buf];
    // only the k-steps this chunk holds, and only warps with rows: the
    // zero-padded remainder of a block (n_tau mod 32) and of a short row
    // slice costs no MMAs
    const int ksteps = (min(kK9Kc, tn[b] - k0) + 3) >> 2;
    if (16 * warp < it.rows) {
      for (int s = 0; s < ksteps; ++s) {
        const double a0 = A[(16 * warp + g) * LDA + 4 * s + t0];
        const double a1 = A[(16 * warp + g + 8) * LDA + 4 * s + t0];
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[j], a0, a1, B[(4 * s + t0) * LDB + 8 * j + g]);
      }
    }
    __syncthreads();
    b = nb;
    k0 = nk;
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        const int row = 16 * warp + g + 8 * r2;
        const int col = c0 + 8 * j + 2 * t0 + c2;
        if (row < it.rows && col < m) Y[it.row0 + row + static_cast<std::int64_t>(col) * n] = acc[j][2 * r2 + c2];
      }
}

// Copies the double pair src[0..1] into dst[0..1] (16 bytes when both are
// 16-byte aligned, else two 8-byte copies); n_valid < 2 zero-fills the rest
// (a zero-fill names the valid global address `safe` and reads nothing).
__device__ __forceinline__ void cp_pair(double* dst, const double* src, int n_valid, const double* safe) {
  if (n_valid == 2 && ((reinterpret_cast<std::uintptr_t>(src) | reinterpret_cast<std::uintptr_t>(dst)) & 15) == 0) {
    cp_async16(dst, src, true);
    return;
  }
  cp_async8(dst, n_valid > 0 ? src : safe, n_valid > 0);
  cp_async8(dst + 1, n_valid > 1 ? src + 1 : safe, n_valid > 1);
}

// K9, two-sided (symmetric storage; items are <= 128-row slices of a leaf): every stored block is
// read once and used twice on DMMA, Y_sigma += D X_tau (accumulated in
// registers over the item's blocks) and Z_tau = D^T X_sigma (per 32-column
// chunk, written to the block's column segment), so the near field of m
// right-hand sides costs one pass over the stored D instead of two. One CTA
// (8 warps) per (owner-leaf item, NC-column tile of the RHS). The D chunk is
// staged column-major with leading dimension 132 and the X panels with 36 /
// 132, which makes the four fragment reads (D, D^T, X_tau, X_sigma)
// conflict-free per half-warp. Outputs go to the partial buffer (column c at
// c * pstride) and k_near_gather sums them per leaf in a fixed order.
constexpr int kK9bKc = 32, kK9bLd = 132, kK9bLx = 36;
template <int NC>
__global__ void __launch_bounds__(256) k_near_mrhs2(const SymRowItem* __restrict__ items,
                                                    const SymBlock* __restrict__ blocks, const double* __restrict__ D,
                                                    const double* __restrict__ X, std::int64_t n, int m,
                                                    std::int64_t pstride, double* __restrict__ part) {
  constexpr int NTN = NC / 8;
  constexpr int STAGE = kK9bKc * kK9bLd + NC * kK9bLx;
  extern __shared__ __align__(128) double sm[];
  double* Xs = sm;                      // X_sigma: [c][r], ld 132
  double* St = sm + NC * kK9bLd;        // two stages: D chunk [k][r] then X_tau [c][k]
  const SymRowItem it = items[blockIdx.x];
  const int c0 = blockIdx.y * NC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t0 = lane & 3;
  const int R = it.rows;                // rows of this slice (<= 128)
  const std::int64_t ld = it.ld;        // stored column length (the leaf)
  const int R4 = (R + 3) & ~3;          // rows staged (zero beyond R)
  const int hp = R4 >> 1;               // pairs per staged column
  const int mtiles = (R + 15) >> 4;
  PHM_DCHECK(R >= 1 && R <= 128 && it.i0 + R <= it.ld);
  const int ypairs = mtiles * NTN;
  // X_sigma once per item: warp w stages columns w, w + 8, ..., lane l the
  // row pairs l, l + 32 (no index division on the staging path)
  for (int c = warp; c < NC; c += 8)
    for (int pr = lane; pr < hp; pr += 32) {
      const int r = 2 * pr;
      const int nv = c0 + c < m ? max(0, min(2, R - r)) : 0;
      cp_pair(Xs + c * kK9bLd + r, X + it.x_row0 + r + static_cast<std::int64_t>(c0 + c) * n, nv, X);
    }
  auto stage = [&](const SymBlock& blk, int j0, int buf) {
    double* Dc = St + buf * STAGE;
    double* Xt = Dc + kK9bKc * kK9bLd;
    const int kc = min(kK9bKc, blk.ncol - j0);
    const double* Db = D + blk.d_off + it.i0 + static_cast<std::int64_t>(j0) * ld;
#pragma unroll
    for (int kq = 0; kq < kK9bKc / 8; ++kq) {  // warp w: columns 4w .. 4w + 3
      const int k = 4 * warp + kq;
      for (int pr = lane; pr < hp; pr += 32) {
        const int r = 2 * pr;
        const int nv = k < kc ? max(0, min(2, R - r)) : 0;
        cp_pair(Dc + k * kK9bLd + r, Db + r + static_cast<std::int64_t>(k) * ld, nv, D);
      }
    }
    for (int q = tid; q < NC * (kK9bKc / 2); q += 256) {
      const int c = q >> 4, k = 2 * (q & 15);
      const int nv = c0 + c < m ? max(0, min(2, kc - k)) : 0;
      cp_pair(Xt + c * kK9bLx + k, X + blk.x_col0 + j0 + k + static_cast<std::int64_t>(c0 + c) * n, nv, X);
    }
    cp_async_commit();
  };
  double yacc[8][4];  // up to 8 (m-tile, n-tile) pairs of Y per warp
#pragma unroll
  for (int p = 0; p < 8; ++p) yacc[p][0] = yacc[p][1] = yacc[p][2] = yacc[p][3] = 0.0;

  int b = it.bbeg, j0 = 0, buf = 0;
  if (b < it.bend) stage(blocks[b], 0, 0);
  while (b < it.bend) {
    const SymBlock blk = blocks[b];
    int nb = b, nj = j0 + kK9bKc;
    if (nj >= blk.ncol) {
      nb = b + 1;
      nj = 0;
    }
    if (nb < it.bend) {
      stage(blocks[nb], nj, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* Dc = St + buf * STAGE;
    const double* Xt = Dc + kK9bKc * kK9bLd;
    const int kc = min(kK9bKc, blk.ncol - j0);
    const int ksy = (kc + 3) >> 2;
    // Y_sigma += D(:, chunk) X_tau(chunk, :)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int p = warp + 8 * q;
      if (p < ypairs) {
        const int mt = p / NTN, nt = p - mt * NTN;
        for (int s2 = 0; s2 < ksy; ++s2) {
          const int k = 4 * s2 + t0;
          dmma_16x8x4(yacc[q], Dc[k * kK9bLd + 16 * mt + g], Dc[k * kK9bLd + 16 * mt + g + 8],
                      Xt[(8 * nt + g) * kK9bLx + k]);
        }
      }
    }
    // Z_tau(chunk, :) = D(:, chunk)^T X_sigma (off-diagonal blocks)
    if (blk.p_col >= 0) {
      const int zpairs = ((kc + 15) >> 4) * NTN;
      for (int p = warp; p < zpairs; p += 8) {
        const int mt = p / NTN, nt = p - mt * NTN;
        double z[4] = {0.0, 0.0, 0.0, 0.0}, z1[4] = {0.0, 0.0, 0.0, 0.0};
        const int ksz = R4 >> 2;
        int s2 = 0;
        for (; s2 + 1 < ksz; s2 += 2) {  // two independent chains
          const int k = 4 * s2 + t0;
          dmma_16x8x4(z, Dc[(16 * mt + g) * kK9bLd + k], Dc[(16 * mt + g + 8) * kK9bLd + k],
                      Xs[(8 * nt + g) * kK9bLd + k]);
          dmma_16x8x4(z1, Dc[(16 * mt + g) * kK9bLd + k + 4], Dc[(16 * mt + g + 8) * kK9bLd + k + 4],
                      Xs[(8 * nt + g) * kK9bLd + k + 4]);
        }
        if (s2 < ksz) {
          const int k = 4 * s2 + t0;
          dmma_16x8x4(z, Dc[(16 * mt + g) * kK9bLd + k], Dc[(16 * mt + g + 8) * kK9bLd + k],
                      Xs[(8 * nt + g) * kK9bLd + k]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) z[e] += z1[e];
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int j = 16 * mt + g + 8 * r2, c = c0 + 8 * nt + 2 * t0 + cc;
            if (j < kc && c < m) part[static_cast<std::int64_t>(c) * pstride + blk.p_col + j0 + j] = z[2 * r2 + cc];
          }
      }
    }
    __syncthreads();
    b = nb;
    j0 = nj;
    buf ^= 1;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int p = warp + 8 * q;
    if (p < ypairs) {
      const int mt = p / NTN, nt = p - mt * NTN;
#pragma unroll
      for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int r = 16 * mt + g + 8 * r2, c = c0 + 8 * nt + 2 * t0 + cc;
          if (r < R && c < m) part[static_cast<std::int64_t>(c) * pstride + it.p_row + r] = yacc[q][2 * r2 + cc];
        }
    }
  }
}

// K6, symmetric storage: every stored block is streamed once and used twice
// (y_sigma += D x_tau and y_tau += D^T x_sigma), halving the near-field
// bytes of both instantiate and MVM for the (symmetric) radial kernels.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CSR-by-sigma version: a CTA streams every stored block owned by its leaf
// (ownership alternates by the parity of sigma + tau, which balances the
// lists), so each warp keeps loads in flight across blocks and the row sums
// stay in registers; per column the 8-warp split and a 5-shuffle reduction
// give the column sum D^T x_sigma.
__global__ void __launch_bounds__(256) k_near_mvm_symcsr(const SymRowItem* __restrict__ items,
                                                         const SymBlock* __restrict__ blocks,
                                                         const double* __restrict__ D, const double* __restrict__ xp,
                                                         double* __restrict__ part) {
  __shared__ double red[8][128];
  const SymRowItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double racc[4] = {0.0, 0.0, 0.0, 0.0};
  double xs[4];
  bool live[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    live[q] = lane + 32 * q < it.rows;
    xs[q] = live[q] ? xp[it.x_row0 + lane + 32 * q] : 0.0;
  }
  const std::int64_t ld = it.ld;
  for (int b = it.bbeg; b < it.bend; ++b) {
    const SymBlock blk = blocks[b];
    const double* Db = D + blk.d_off + it.i0 + lane;
    const double* xt = xp + blk.x_col0;
    const bool diag = blk.p_col < 0;
    int j = warp;
    for (; j + 8 < blk.ncol; j += 16) {
      const double x0 = xt[j], x1 = xt[j + 8];
      double v0[4], v1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v0[q] = live[q] ? ld_stream(Db + j * ld + 32 * q) : 0.0;
        v1[q] = live[q] ? ld_stream(Db + (j + 8) * ld + 32 * q) : 0.0;
      }
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        racc[q] += v0[q] * x0 + v1[q] * x1;
        c0 += v0[q] * xs[q];
        c1 += v1[q] * xs[q];
      }
      if (!diag) {
        c0 = warp_sum(c0);
        c1 = warp_sum(c1);
        if (lane == 0) {
          part[blk.p_col + j] = c0;
          part[blk.p_col + j + 8] = c1;
        }
      }
    }
    for (; j < blk.ncol; j += 8) {
      const double x0 = xt[j];
      double c0 = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double v = live[q] ? ld_stream(Db + j * ld + 32 * q) : 0.0;
        racc[q] += v * x0;
        c0 += v * xs[q];
      }
      if (!diag) {
        c0 = warp_sum(c0);
        if (lane == 0) part[blk.p_col + j] = c0;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) red[warp][lane + 32 * q] = racc[q];
  __syncthreads();
  if (threadIdx.x < it.rows) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    part[it.p_row + threadIdx.x] = s;
  }
}

// ------------------------------------------------------------ TMA near pass
// Near field through the Tensor Memory Accelerator: the CTA of an owner
// leaf walks its stored blocks in column chunks; for every chunk one thread
// issues R bulk copies (cp.async.bulk, one per snapshot slab, or one of D
// itself) into a shared-memory stage tracked by an mbarrier (expect_tx /
// complete_tx), double-buffered so the next chunk lands while this one is
// consumed. Consumers form d = sum_k w_k S_k (R = 1, w = 1 reads D as is),
// optionally store D (instantiate fused with apply), and accumulate the row
// product D x_tau (thread = row, conflict-free) and the column product
// D^T x_sigma (warp = column, shuffle reduction) straight from shared memory.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The same bulk copy with an L2 evict-first policy: a stream read once
// (apply's D) should not push out the L2-resident operands of kernels running
// beside it (the coupling's C_k, 83 MB at C3).
__device__ __forceinline__ std::uint64_t l2_evict_first_policy() {
  std::uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_ef(void* dst, const void* src, unsigned bytes, std::uint64_t* bar,
                                            std::uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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

// Warp-specialised pipeline: warp 8 (one elected lane) is the producer and
// keeps every free stage of an NST-deep ring filled with the next chunk
// (R bulk copies, one full[] mbarrier per stage); warps 0-7 consume. A
// consumer pass over a chunk forms d = sum_k w_k S_k into a double-buffered
// formed chunk (and stores it to D), meets the other consumers at a named
// barrier, releases the stage through its empty[] mbarrier, then runs the
// row and column products out of the formed chunk while the producer
// refills. Shared memory (doubles): NST R CH stages + 2 CH formed + 2 x 128
// x_tau panels.
constexpr int tma_smem_doubles(int R, int CH, int NST) { return NST * R * CH + 2 * CH + 256; }
constexpr int kTmaThreads = 288;    // 8 consumer warps + 1 producer warp

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int R, int CH, int NST>
__global__ void __launch_bounds__(kTmaThreads, 1) k_near_tma(const SymRowItem* __restrict__ items,
                                                          const SymBlock* __restrict__ blocks,
                                                          const double* __restrict__ G, std::int64_t E,
                                                          const double* __restrict__ w, double* __restrict__ D,
                                                          const double* __restrict__ xp, double* __restrict__ part) {
  static_assert(CH >= 256 && CH % 2 == 0, "a chunk holds at least two columns of a 128-row leaf");
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST];
  __shared__ double xs_sh[128];
  __shared__ SymBlock bl[kTmaMaxBlocks];
  const SymRowItem it = items[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ld = it.ld;  // == rows (the TMA path takes whole-height blocks)
  const int nb = it.bend - it.bbeg;
  const int jc = min(128, (CH / ld) & ~1);  // even column count per chunk
  PHM_DCHECK(ld >= 1 && ld <= 128 && it.rows == ld && it.i0 == 0 && nb <= kTmaMaxBlocks && jc >= 2);
  if (tid < it.rows) xs_sh[tid] = xp[it.x_row0 + tid];
  if (tid < nb) bl[tid] = blocks[it.bbeg + tid];
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {  // ---------------------------------------------- producer
    if (lane == 0) {
      int c = 0;
      for (int b = 0; b < nb; ++b) {
        const std::int64_t d_off = bl[b].d_off;
        const int ncol = bl[b].ncol;
        for (int j0 = 0; j0 < ncol; j0 += jc, ++c) {
          const int slot = c % NST;
          if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
          const int ncols = min(jc, ncol - j0);
          const unsigned bytes = static_cast<unsigned>(((static_cast<std::int64_t>(ncols) * ld * 8) + 15) & ~15LL);
          PHM_DCHECK(bytes <= CH * 8u && ((reinterpret_cast<std::uintptr_t>(G + d_off + static_cast<std::int64_t>(j0) * ld) & 15) == 0));
          mbar_expect_tx(&full[slot], bytes * R);
          const double* src = G + d_off + static_cast<std::int64_t>(j0) * ld;
#pragma unroll
          for (int k = 0; k < R; ++k) bulk_g2s(sm + (slot * R + k) * CH, src + k * E, bytes, &full[slot]);
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  double* dc0 = sm + NST * R * CH;  // formed chunk, two buffers
  double* xt0 = dc0 + 2 * CH;       // x_tau panel, two buffers of 128
  const int ng = 256 / ld, rg = tid / ld, rr = tid - rg * ld;  // row product: (row rr, column group rg)
  double wr[R];
#pragma unroll
  for (int k = 0; k < R; ++k) wr[k] = w[k];
  double racc = 0.0;
  // x_tau of the next chunk is loaded one chunk ahead (its latency would
  // otherwise sit between the stage landing and the row product)
  int b = 0, j0 = 0;
  double xnext = (nb > 0 && tid < min(jc, bl[0].ncol)) ? xp[bl[0].x_col0 + tid] : 0.0;
  for (int c = 0, buf = 0; b < nb; ++c, buf ^= 1) {
    const std::int64_t d_off = bl[b].d_off, p_col = bl[b].p_col;
    const int ncol = bl[b].ncol;
    const int slot = c % NST;
    const int ncols = min(jc, ncol - j0);
    double* dc = dc0 + buf * CH;
    double* xt = xt0 + buf * 128;
    if (tid < ncols) xt[tid] = xnext;
    int nb2 = b, nj2 = j0 + jc;  // cursor of the next chunk
    if (nj2 >= ncol) {
      ++nb2;
      nj2 = 0;
    }
    if (nb2 < nb && tid < min(jc, bl[nb2].ncol - nj2)) xnext = xp[bl[nb2].x_col0 + nj2 + tid];
    mbar_wait(&full[slot], (c / NST) & 1);
    const double* S = sm + slot * R * CH;
    const int nel = ncols * ld;
    double* Dg = D + d_off + static_cast<std::int64_t>(j0) * ld;
    // Coalesced 64-bit stores (a warp writes 256 contiguous bytes). A
    // 256-bit-store variant (each thread forming four consecutive elements)
    // read the stage with a stride of four doubles -- 4-way bank conflicts --
    // and cost the fused C3 step 23% (115 -> 87 theta/s, round 2).
    for (int e = tid; e < nel; e += 256) {
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) v += S[k * CH + e] * wr[k];
      dc[e] = v;
      Dg[e] = v;
    }
    consumers_sync();
    if (tid == 0) mbar_arrive(&empty[slot]);  // stage formed: the producer may refill it
    if (rg < ng) {
      double r = 0.0;
      for (int jj = rg; jj < ncols; jj += ng) r += dc[rr + jj * ld] * xt[jj];
      racc += r;
    }
    if (p_col >= 0) {
      for (int jj = warp; jj < ncols; jj += 8) {
        double cs = 0.0;
        for (int i = lane; i < ld; i += 32) cs += dc[i + jj * ld] * xs_sh[i];
        cs = warp_sum(cs);
        if (lane == 0) part[p_col + j0 + jj] = cs;
      }
    }
    b = nb2;
    j0 = nj2;
  }
  consumers_sync();
  double* red = dc0;  // reuse the formed-chunk buffers
  red[tid] = rg < ng ? racc : 0.0;
  consumers_sync();
  if (tid < it.rows) {
    double t = 0.0;
    for (int g = 0; g < ng; ++g) t += red[tid + g * ld];
    part[it.p_row + tid] = t;
  }
}

// K6 over TMA (apply alone, one RHS): the producer / consumer split of
// k_near_tma with D itself as the only slab, chunks of up to 64 columns of a
// block. Persistent: a fixed grid (one CTA per SM by default, so the far
// chain's kernels can sit beside it on every SM) takes items from a work
// counter; the producer warp fetches the next item's block list into a
// double-buffered slot while the consumers finish the current one, so the
// stage ring never drains at item boundaries.
// The consumers work register-tiled so that each D element costs a few
// instructions: thread t owns rows rt + 16 q (rt = t mod 16, q < 8) and the
// 4 columns 4 cg .. 4 cg + 3 of the chunk (cg = t / 16). Row partials
// (D x_tau) stay in registers across the item; column partials (D^T x_sigma)
// are reduced over the 16 lanes of a half-warp with a transpose-reduce (5
// shuffles for 4 columns). Each warp releases a stage on its own (empty[]
// counts 8 warp arrivals). 96 registers: 9 warps x 2 CTAs fit the per-SMSP
// register file.
template <int CH, int NST>
__global__ void __maxnreg__(96) k_near_tma_apply(const SymRowItem* __restrict__ items, int nitems,
                                                 const SymBlock* __restrict__ blocks, const double* __restrict__ D,
                                                 const double* __restrict__ xp, double* __restrict__ part,
                                                 int* __restrict__ counter) {
  static_assert(CH >= 128 * 16, "a chunk holds 16 columns of a 128-row leaf");
  // stage = D chunk (CH + 2 doubles, shifted by one when it starts on an odd
  // element) + the chunk's x_tau panel (64 + 2); then 8 x 128 row partials
  constexpr int kStage = CH + 2 + 66;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST], ifull[2], iempty[2];
  __shared__ SymBlock bl[2][kTmaMaxBlocks];
  __shared__ SymRowItem itm[2];
  __shared__ int iidx[2];
  __shared__ double xs_item[2][128];  // x_sigma of the item's rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&ifull[q], 1);
      mbar_init(&iempty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {  // ------------------------------------------------ producer
    int c = 0;
    for (int n = 0;; ++n) {
      const int ib = n & 1;
      if (n >= 2) mbar_wait(&iempty[ib], ((n >> 1) - 1) & 1);
      int idx = 0;
      if (lane == 0) idx = atomicAdd(counter, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx < nitems) {
        const SymRowItem it = items[idx];
        for (int t = lane; t < it.bend - it.bbeg; t += 32) bl[ib][t] = blocks[it.bbeg + t];
        for (int t = lane; t < 128; t += 32) xs_item[ib][t] = t < it.rows ? xp[it.x_row0 + t] : 0.0;
        if (lane == 0) itm[ib] = it;
      }
      if (lane == 0) iidx[ib] = idx;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ifull[ib]);
      if (idx >= nitems) break;
      if (lane == 0) {
        const SymRowItem& it = itm[ib];
        const int ld = it.ld, nb = it.bend - it.bbeg, jc = min(64, CH / ld);
        for (int b = 0; b < nb; ++b) {
          const std::int64_t d_off = bl[ib][b].d_off, x_col0 = bl[ib][b].x_col0;
          const int ncol = bl[ib][b].ncol;
          for (int j0 = 0; j0 < ncol; j0 += jc, ++c) {
            const int slot = c % NST;
            if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
            const int ncols = min(jc, ncol - j0);
            // the source may start 8 bytes past a 16-byte boundary (odd ld):
            // copy from the aligned address below and shift in shared memory
            const std::int64_t e0 = d_off + static_cast<std::int64_t>(j0) * ld;
            const std::int64_t ea = e0 & ~std::int64_t(1);
            const std::int64_t nbytes = (((e0 + static_cast<std::int64_t>(ncols) * ld - ea) + 1) & ~std::int64_t(1)) * 8;
            PHM_DCHECK(ld <= 128 && it.rows == ld && nbytes <= (CH + 2) * 8 && ncols <= 64);
            // x_tau panel: xp + column may sit on an odd element (odd n, RHS > 0)
            const double* xsrc = xp + x_col0 + j0;
            const int xsh = static_cast<int>((reinterpret_cast<std::uintptr_t>(xsrc) >> 3) & 1);
            const unsigned xbytes = static_cast<unsigned>(((ncols + xsh + 1) & ~1) * 8);
            PHM_DCHECK(xbytes <= 66 * 8);
            mbar_expect_tx(&full[slot], static_cast<unsigned>(nbytes) + xbytes);
            bulk_g2s(sm + slot * kStage, D + ea, static_cast<unsigned>(nbytes), &full[slot]);
            bulk_g2s(sm + slot * kStage + CH + 2, xsrc - xsh, xbytes, &full[slot]);
          }
        }
      }
      __syncwarp();
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  double* red = sm + NST * kStage;
  const int rt = tid & 15, cg = tid >> 4;  // row lane, column group
  const int l16 = lane & 15;
  int c = 0;
  for (int n = 0;; ++n) {
    const int ib = n & 1;
    mbar_wait(&ifull[ib], (n >> 1) & 1);
    if (iidx[ib] >= nitems) break;
    const SymRowItem it = itm[ib];
    const SymBlock* B = bl[ib];
    const int ld = it.ld, nb = it.bend - it.bbeg, jc = min(64, CH / ld);
    double xs[8], racc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      xs[q] = xs_item[ib][rt + 16 * q];
      racc[q] = 0.0;
    }
    for (int b = 0, j0 = 0; b < nb; ++c) {
      const std::int64_t p_col = B[b].p_col;
      const int ncol = B[b].ncol;
      const int slot = c % NST;
      const int ncols = min(jc, ncol - j0);
      int nb2 = b, nj2 = j0 + jc;
      if (nj2 >= ncol) {
        ++nb2;
        nj2 = 0;
      }
      mbar_wait(&full[slot], (c / NST) & 1);
      const double* Dc = sm + slot * kStage + ((B[b].d_off + static_cast<std::int64_t>(j0) * ld) & 1);
      const double* Xc = sm + slot * kStage + CH + 2 +
                         ((reinterpret_cast<std::uintptr_t>(xp + B[b].x_col0 + j0) >> 3) & 1);
      double xt[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) xt[k] = Xc[4 * cg + k];  // past ncols: finite, never used
      double cacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = 4 * cg + k;
        if (j < ncols) {
          const double* col = Dc + j * ld;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = rt + 16 * q;
            if (r < ld) {
              const double v = col[r];
              racc[q] += v * xt[k];
              cacc[k] += v * xs[q];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the stage
      if (p_col >= 0) {  // warp-uniform (one block per chunk)
        // transpose-reduce 4 column partials over the 16 lanes of the half-warp
        const bool b3 = l16 & 8, b2 = l16 & 4;
        double k0 = b3 ? cacc[2] : cacc[0], k1 = b3 ? cacc[3] : cacc[1];
        const double s0 = b3 ? cacc[0] : cacc[2], s1 = b3 ? cacc[1] : cacc[3];
        k0 += __shfl_xor_sync(0xffffffffu, s0, 8);
        k1 += __shfl_xor_sync(0xffffffffu, s1, 8);
        double kk = b2 ? k1 : k0;
        kk += __shfl_xor_sync(0xffffffffu, b2 ? k0 : k1, 4);
        kk += __shfl_xor_sync(0xffffffffu, kk, 2);
        kk += __shfl_xor_sync(0xffffffffu, kk, 1);
        const int j = 4 * cg + (l16 >> 2);
        if ((l16 & 3) == 0 && j < ncols) part[p_col + j0 + j] = kk;
      }
      b = nb2;
      j0 = nj2;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&iempty[ib]);  // block list no longer read
    // row sums over the 16 column groups: the two half-warps first, then the
    // 8 warps in warp order
#pragma unroll
    for (int q = 0; q < 8; ++q) racc[q] += __shfl_xor_sync(0xffffffffu, racc[q], 16);
    consumers_sync();
    if (lane < 16) {
#pragma unroll
      for (int q = 0; q < 8; ++q) red[warp * 128 + rt + 16 * q] = racc[q];
    }
    consumers_sync();
    if (tid < it.rows) {
      double t = 0.0;
      for (int g = 0; g < 8; ++g) t += red[g * 128 + tid];
      part[it.p_row + tid] = t;
    }
  }
}

// K6 lean (apply alone, one RHS; the default): the same TMA ring and item
// double-buffering as k_near_tma_apply with a quarter of its SM footprint, so
// that the H^2 coupling (DMMA pipe) runs on the same SMs at the same time as
// this HBM stream instead of time-sharing CTA slots with it. 4 consumer
// warps + 1 producer warp, one CTA per SM. Chunks are up to 64 columns of one
// block (a whole 64 x 64 block = 32 KB). Warp w owns columns 16w .. 16w + 15
// of a chunk, lane l rows l + 32q: per column two (or four) conflict-free
// 8-byte shared loads feed the row product (D x_tau, kept in registers across
// the item) and the column product (D^T x_sigma); the 16 column partials of a
// warp are reduced with one 16-step transpose-reduce (one shuffle per column
// and lane). Fixed summation order: deterministic.
template <int NCW>
__device__ __forceinline__ void lean_consumers_sync() { asm volatile("bar.sync 2, %0;" ::"n"(NCW * 32) : "memory"); }

template <int NQ, int NCW, int CH, int NST>
__device__ __forceinline__ void lean_item(const SymRowItem& it, const SymBlock* __restrict__ B,
                                          const double* __restrict__ xsi, const double* __restrict__ stages,
                                          std::uint64_t* full, std::uint64_t* empty, const double* __restrict__ xp,
                                          double* __restrict__ part, int& c, int warp, int lane,
                                          double (&racc)[2][4]) {
  constexpr int kStage = CH + 2 + 66;
  constexpr int CPW = 64 / NCW, NHB = CPW / 8;  // columns per warp, 8-column batches
  const int ld = it.ld, nb = it.bend - it.bbeg, jc = min(64, CH / ld);
  double xs[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) xs[q] = xsi[lane + 32 * q];  // zero past the item's rows
  for (int b = 0; b < nb; ++b) {
    const std::int64_t p_col = B[b].p_col, d_off = B[b].d_off, x_col0 = B[b].x_col0;
    const int ncol = B[b].ncol;
    for (int j0 = 0; j0 < ncol; j0 += jc, ++c) {
      const int slot = c % NST;
      const int ncols = min(jc, ncol - j0);
      mbar_wait(&full[slot], (c / NST) & 1);
      const double* st = stages + slot * kStage;
      const double* Dc = st + ((d_off + static_cast<std::int64_t>(j0) * ld) & 1);
      const double* Xc = st + CH + 2 + ((reinterpret_cast<std::uintptr_t>(xp + x_col0 + j0) >> 3) & 1);
      // two batches of 8 columns; every load of a batch is issued before its
      // FMAs (predicated, branch-free: one consumer warp per SMSP has only
      // instruction-level parallelism to hide shared-memory latency)
      double cp[NHB][8];
#pragma unroll
      for (int hb = 0; hb < NHB; ++hb) {
        // unpredicated loads: a column past the chunk reads the chunk's last
        // column with x_tau = 0, rows past ld read the next column's head
        // (finite: stages hold only D, x and the initial zeros) against
        // x_sigma = 0, and every read stays inside the stage
        double v[8][NQ], xt[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = CPW * warp + 8 * hb + jj;
          const bool jv = j < ncols;
          xt[jj] = jv ? Xc[j] : 0.0;
          const double* col = Dc + (jv ? j : ncols - 1) * ld + lane;
#pragma unroll
          for (int q = 0; q < NQ; ++q) v[jj][q] = col[32 * q];
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            racc[hb][q] = fma(v[jj][q], xt[jj], racc[hb][q]);
            s = fma(v[jj][q], xs[q], s);
          }
          cp[hb][jj] = s;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the stage
      if (p_col >= 0 && CPW * warp < ncols) {      // warp-uniform
        // transpose-reduce per batch: after the xor-16/8/4 steps lane l holds
        // the partial of column (l >> 2) & 7 over a quarter of the lanes;
        // xor 2 and 1 complete it
#pragma unroll
        for (int hb = 0; hb < NHB; ++hb) {
          double* c8 = cp[hb];
#pragma unroll
          for (int h = 4; h >= 1; h >>= 1) {
            const bool up = lane & (4 * h);
#pragma unroll
            for (int i = 0; i < h; ++i) {
              const double keep = up ? c8[i + h] : c8[i], send = up ? c8[i] : c8[i + h];
              c8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4 * h);
            }
          }
          c8[0] += __shfl_xor_sync(0xffffffffu, c8[0], 2);
          c8[0] += __shfl_xor_sync(0xffffffffu, c8[0], 1);
          const int j = CPW * warp + 8 * hb + ((lane >> 2) & 7);
          if (!(lane & 3) && j < ncols) part[p_col + j0 + j] = c8[0];
        }
      }
    }
  }
}

template <int NCW, int CH, int NST>
__global__ void __maxnreg__(96) k_near_gemv_lean(const SymRowItem* __restrict__ items, int nitems,
                                                                   const SymBlock* __restrict__ blocks,
                                                                   const double* __restrict__ D,
                                                                   const double* __restrict__ xp,
                                                                   double* __restrict__ part,
                                                                   int* __restrict__ counter, bool evict_first) {
  static_assert(CH >= 128 * 16, "a chunk holds 16 columns of a 128-row leaf");
  constexpr int kStage = CH + 2 + 66;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST], ifull[2], iempty[2];
  __shared__ SymBlock bl[2][kTmaMaxBlocks];
  __shared__ SymRowItem itm[2];
  __shared__ int iidx[2];
  __shared__ double xs_item[2][128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the consumers read whole stages unpredicated: start from finite zeros
  for (int e = tid; e < NST * kStage + NCW * 128; e += (NCW + 1) * 32) sm[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies overwrite them
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NCW);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&ifull[q], 1);
      mbar_init(&iempty[q], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {  // ------------------------------------------------ producer
    const std::uint64_t pol = l2_evict_first_policy();
    int c = 0;
    for (int n = 0;; ++n) {
      const int ib = n & 1;
      if (n >= 2) mbar_wait(&iempty[ib], ((n >> 1) - 1) & 1);
      int idx = 0;
      if (lane == 0) idx = atomicAdd(counter, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx < nitems) {
        const SymRowItem it = items[idx];
        for (int t = lane; t < it.bend - it.bbeg; t += 32) bl[ib][t] = blocks[it.bbeg + t];
        for (int t = lane; t < 128; t += 32) xs_item[ib][t] = t < it.rows ? xp[it.x_row0 + t] : 0.0;
        if (lane == 0) itm[ib] = it;
      }
      if (lane == 0) iidx[ib] = idx;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ifull[ib]);
      if (idx >= nitems) break;
      if (lane == 0) {
        const SymRowItem& it = itm[ib];
        const int ld = it.ld, nb = it.bend - it.bbeg, jc = min(64, CH / ld);
        for (int b = 0; b < nb; ++b) {
          const std::int64_t d_off = bl[ib][b].d_off, x_col0 = bl[ib][b].x_col0;
          const int ncol = bl[ib][b].ncol;
          for (int j0 = 0; j0 < ncol; j0 += jc, ++c) {
            const int slot = c % NST;
            if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
            const int ncols = min(jc, ncol - j0);
            const std::int64_t e0 = d_off + static_cast<std::int64_t>(j0) * ld;
            const std::int64_t ea = e0 & ~std::int64_t(1);
            const std::int64_t nbytes = (((e0 + static_cast<std::int64_t>(ncols) * ld - ea) + 1) & ~std::int64_t(1)) * 8;
            PHM_DCHECK(ld <= 128 && it.rows == ld && nbytes <= (CH + 2) * 8 && ncols <= 64);
            const double* xsrc = xp + x_col0 + j0;
            const int xsh = static_cast<int>((reinterpret_cast<std::uintptr_t>(xsrc) >> 3) & 1);
            const unsigned xbytes = static_cast<unsigned>(((ncols + xsh + 1) & ~1) * 8);
            PHM_DCHECK(xbytes <= 66 * 8);
            mbar_expect_tx(&full[slot], static_cast<unsigned>(nbytes) + xbytes);
            if (evict_first)
              bulk_g2s_ef(sm + slot * kStage, D + ea, static_cast<unsigned>(nbytes), &full[slot], pol);
            else
              bulk_g2s(sm + slot * kStage, D + ea, static_cast<unsigned>(nbytes), &full[slot]);
            bulk_g2s(sm + slot * kStage + CH + 2, xsrc - xsh, xbytes, &full[slot]);
          }
        }
      }
      __syncwarp();
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  double* red = sm + NST * kStage;  // NCW x 128 row partials
  int c = 0;
  for (int n = 0;; ++n) {
    const int ib = n & 1;
    mbar_wait(&ifull[ib], (n >> 1) & 1);
    if (iidx[ib] >= nitems) break;
    const SymRowItem it = itm[ib];
    double racc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    if (it.ld <= 64)
      lean_item<2, NCW, CH, NST>(it, bl[ib], xs_item[ib], sm, full, empty, xp, part, c, warp, lane, racc);
    else if (it.ld <= 96)
      lean_item<3, NCW, CH, NST>(it, bl[ib], xs_item[ib], sm, full, empty, xp, part, c, warp, lane, racc);
    else
      lean_item<4, NCW, CH, NST>(it, bl[ib], xs_item[ib], sm, full, empty, xp, part, c, warp, lane, racc);
    __syncwarp();
    if (lane == 0) mbar_arrive(&iempty[ib]);  // block list and x_sigma no longer read
    lean_consumers_sync<NCW>();                    // the previous item's reads of red are done
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp * 128 + lane + 32 * q] = racc[0][q] + racc[1][q];
    lean_consumers_sync<NCW>();
    if (tid < it.rows) {
      double t = red[tid];
#pragma unroll
      for (int w = 1; w < NCW; ++w) t += red[w * 128 + tid];
      part[it.p_row + tid] = t;
    }
  }
}

// K1 over TMA (instantiate alone, snapshot mode): the flat stream of
// k_inst_flat with the slabs moved by cp.async.bulk into an NST-deep ring
// (one producer lane, 8 consumer warps, full/empty mbarriers), persistent
// over chunks of CH doubles. Consumers form D_b[e] = sum_k w_b,k S_k[e] in
// k_inst_flat's FMA order (bit-identical D) for each of the B thetas of the
// call (B = 1: instantiate; B <= 16: the theta batch, whose weight and output
// tables are device arrays) and store with 256-bit stores. 96 registers:
// two CTAs per SM.
template <int R, int CH, int NST>
__global__ void __maxnreg__(96) k_inst_tma(const double* __restrict__ G, std::int64_t E, int B, InstPtrs tab) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST];
  __shared__ double W[kInstBatchMax][R];
  __shared__ double* Dp[kInstBatchMax];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::int64_t nchunks = (E + CH - 1) / CH;
  for (int i = tid; i < B * R; i += blockDim.x) W[i / R][i % R] = tab.w[i / R][i % R];
  if (tid < B) Dp[tid] = tab.d[tid];
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
      for (std::int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++c) {
        const int slot = c % NST;
        if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
        const std::int64_t e0 = ch * CH;
        const std::int64_t left = E - e0;
        const unsigned bytes = static_cast<unsigned>((left < CH ? left : CH) * 8);
        mbar_expect_tx(&full[slot], bytes * R);
#pragma unroll
        for (int k = 0; k < R; ++k) bulk_g2s(sm + (slot * R + k) * CH, G + k * E + e0, bytes, &full[slot]);
      }
    }
    return;
  }
  int c = 0;
  for (std::int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++c) {
    const int slot = c % NST;
    const std::int64_t e0 = ch * CH;
    const std::int64_t left = E - e0;
    const int len = static_cast<int>(left < CH ? left : CH);  // a multiple of 4
    PHM_DCHECK((len & 3) == 0 && B >= 1 && B <= kInstBatchMax);
    mbar_wait(&full[slot], (c / NST) & 1);
    const double* S = sm + slot * R * CH;
    for (int q = tid; q < (len >> 2); q += 256) {
      for (int b = 0; b < B; ++b) {
        dbl4 acc = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double* sk = S + k * CH + 4 * q;
          const double wk = W[b][k];
          acc.x += sk[0] * wk;
          acc.y += sk[1] * wk;
          acc.z += sk[2] * wk;
          acc.w += sk[3] * wk;
        }
        st4(Dp[b] + e0 + 4 * q, acc);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
}


// K9, two-sided over TMA (k_near_mrhs3): k_near_mrhs2's products with the
// staging moved to a producer warp. Per 32-column chunk its lanes issue one
// cp.async.bulk per D column (into the padded column-major chunk; a column
// that starts 8 bytes past a 16-byte boundary is copied from the aligned
// address below and read with a one-element shift) and one per RHS column of
// the X_tau panel; a 2-stage ring with full/empty mbarriers decouples them
// from the 8 consumer warps, which only run DMMA. Reads past the chunk (odd
// lengths, k beyond the chunk, rows beyond the slice) are masked to zero
// before they reach an MMA, so stale shared memory never contributes.
template <int NC, int NST>
__global__ void __maxnreg__(NC >= 64 ? 168 : 96) k_near_mrhs3(const SymRowItem* __restrict__ items,
                                              const SymBlock* __restrict__ blocks, const double* __restrict__ D,
                                              const double* __restrict__ X, std::int64_t n, int m,
                                              std::int64_t pstride, double* __restrict__ part, int dstage) {
  constexpr int NTN = NC / 8;
  constexpr int YQ = NC / 8;  // Y (m-tile, n-tile) pairs per consumer warp (<= 8 m-tiles x NTN / 8 warps)
  constexpr int LDX = kK9bKc + 4;
  // dstage: doubles of D per stage -- 32 x 132 when some item is a row
  // slice (column copies), else 32 x the tallest leaf (+2), which leaves
  // room for a deeper ring (NST) at two CTAs per SM
  const int STAGE = dstage + NC * LDX;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) std::uint64_t full[NST], empty[NST];
  double* Xs = sm;                      // X_sigma: [c][r], ld 132 (consumers stage it)
  double* St = sm + NC * kK9bLd;        // NST stages: D chunk [k][shift + r] then X_tau [c][shift + k]
  const SymRowItem it = items[blockIdx.x];
  const int c0 = blockIdx.y * NC;
  const int ncr = min(NC, m - c0);      // RHS columns of this tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t0 = lane & 3;
  const int R = it.rows;
  const std::int64_t ld = it.ld;
  const int R4 = (R + 3) & ~3;
  const int mtiles = (R + 15) >> 4;
  const int ypairs = mtiles * NTN;
  // whole-leaf item: a chunk of kc columns is contiguous in D, staged by one
  // bulk copy with column stride R (else one copy per column, stride 132)
  const bool dense = it.i0 == 0 && ld == R;
  const int cs = dense ? R : kK9bLd;
  PHM_DCHECK(R >= 1 && R <= 128 && it.i0 + R <= it.ld && (dense ? kK9bKc * R + 2 : kK9bKc * kK9bLd) <= dstage);
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {  // --------------------------------------------- producer
    int c = 0;
    for (int b = it.bbeg; b < it.bend; ++b) {
      const SymBlock blk = blocks[b];
      for (int j0 = 0; j0 < blk.ncol; j0 += kK9bKc, ++c) {
        const int slot = c % NST;
        if (c >= NST) mbar_wait(&empty[slot], ((c / NST) - 1) & 1);
        const int kc = min(kK9bKc, blk.ncol - j0);
        double* Dc = St + slot * STAGE;
        double* Xt = Dc + dstage;
        // lane k: column k of the chunk (whole-leaf items: lane 0 copies the
        // contiguous chunk at once); lane c (< ncr): RHS column c of X_tau
        unsigned bytes_d = 0, bytes_x = 0;
        const double* src_d = nullptr;
        const double* src_x = nullptr;
        if (dense) {
          if (lane == 0) {
            const double* ch = D + blk.d_off + static_cast<std::int64_t>(j0) * ld;
            const int sh = static_cast<int>((reinterpret_cast<std::uintptr_t>(ch) >> 3) & 1);
            src_d = ch - sh;
            bytes_d = static_cast<unsigned>(((kc * R + sh + 1) & ~1) * 8);
          }
        } else if (lane < kc) {
          const double* col = D + blk.d_off + it.i0 + static_cast<std::int64_t>(j0 + lane) * ld;
          const int sh = static_cast<int>((reinterpret_cast<std::uintptr_t>(col) >> 3) & 1);
          src_d = col - sh;
          bytes_d = static_cast<unsigned>(((R + sh + 1) & ~1) * 8);
        }
        // RHS columns lane, lane + 32 (NC = 64)
        constexpr int XC = NC > 32 ? NC / 32 : 1;
        const double* src_xs[XC];
        unsigned bytes_xs[XC];
#pragma unroll
        for (int u = 0; u < XC; ++u) {
          const int cc = lane + 32 * u;
          src_xs[u] = nullptr;
          bytes_xs[u] = 0;
          if (cc < ncr) {
            const double* xc = X + blk.x_col0 + j0 + static_cast<std::int64_t>(c0 + cc) * n;
            const int sh = static_cast<int>((reinterpret_cast<std::uintptr_t>(xc) >> 3) & 1);
            src_xs[u] = xc - sh;
            bytes_xs[u] = static_cast<unsigned>(((kc + sh + 1) & ~1) * 8);
            bytes_x += bytes_xs[u];
          }
        }
        (void)src_x;
        unsigned total = bytes_d + bytes_x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
        if (lane == 0) mbar_expect_tx(&full[slot], total);
        __syncwarp();
        if (bytes_d) bulk_g2s(Dc + lane * kK9bLd, src_d, bytes_d, &full[slot]);
#pragma unroll
        for (int u = 0; u < XC; ++u)
          if (bytes_xs[u]) bulk_g2s(Xt + (lane + 32 * u) * LDX, src_xs[u], bytes_xs[u], &full[slot]);
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  for (int q = tid; q < NC * R4; q += 256) {  // X_sigma, zero beyond the slice / the RHS count
    const int cc = q / R4, r = q - cc * R4;
    Xs[cc * kK9bLd + r] = (cc < ncr && r < R) ? X[it.x_row0 + r + static_cast<std::int64_t>(c0 + cc) * n] : 0.0;
  }
  consumers_sync();
  double yacc[YQ][4];
#pragma unroll
  for (int q = 0; q < YQ; ++q) yacc[q][0] = yacc[q][1] = yacc[q][2] = yacc[q][3] = 0.0;
  int c = 0;
  for (int b = it.bbeg; b < it.bend; ++b) {
    const SymBlock blk = blocks[b];
    const std::uintptr_t dbase = reinterpret_cast<std::uintptr_t>(D + blk.d_off + it.i0);
    for (int j0 = 0; j0 < blk.ncol; j0 += kK9bKc, ++c) {
      const int slot = c % NST;
      const int kc = min(kK9bKc, blk.ncol - j0);
      mbar_wait(&full[slot], (c / NST) & 1);
      const double* Dc = St + slot * STAGE;
      const double* Xt = Dc + dstage;
      // element (r, k) of the chunk sits at Dc[k * cs + sh(k) + r]
      const int sh_chunk = static_cast<int>(((dbase >> 3) + static_cast<std::uintptr_t>(j0 * ld)) & 1);
      auto dsh = [&](int k) {
        return dense ? sh_chunk : static_cast<int>(((dbase >> 3) + static_cast<std::uintptr_t>((j0 + k) * ld)) & 1);
      };
      const int ksy = (kc + 3) >> 2;
      // Y_sigma += D(:, chunk) X_tau(chunk, :)
      if (warp + 8 * (YQ - 1) < ypairs) {
        // every pair of this warp is live: k-step outer, pair inner, so the
        // YQ accumulators are independent DMMA chains (pair-outer made each
        // a serial chain of ksy dependent MMAs: ncu "wait" stalls); the
        // pairs share this lane's B column (nt = warp mod NTN)
        const int nt = warp % NTN;
        const int ncol_b = 8 * nt + g;
        const bool bin = ncol_b < ncr;
        const int xsh = bin ? static_cast<int>(((reinterpret_cast<std::uintptr_t>(
                                   X + blk.x_col0 + j0 + static_cast<std::int64_t>(c0 + ncol_b) * n)) >> 3) & 1)
                            : 0;
        for (int s2 = 0; s2 < ksy; ++s2) {
          const int k = 4 * s2 + t0;
          const bool kin = k < kc;
          const int sh = kin ? dsh(k) : 0;
          const double b0 = (kin && bin) ? Xt[ncol_b * LDX + xsh + k] : 0.0;
#pragma unroll
          for (int q = 0; q < YQ; ++q) {
            const int mt = (warp + 8 * q) / NTN;
            const double a0 = kin ? Dc[k * cs + sh + 16 * mt + g] : 0.0;
            const double a1 = kin ? Dc[k * cs + sh + 16 * mt + g + 8] : 0.0;
            dmma_16x8x4(yacc[q], a0, a1, b0);
          }
        }
      } else
#pragma unroll
      for (int q = 0; q < YQ; ++q) {
        const int p = warp + 8 * q;
        if (p < ypairs) {
          const int mt = p / NTN, nt = p - mt * NTN;
          const int ncol_b = 8 * nt + g;  // this lane's B column
          const int xsh = ncol_b < ncr ? static_cast<int>(((reinterpret_cast<std::uintptr_t>(
                                                               X + blk.x_col0 + j0 + static_cast<std::int64_t>(c0 + ncol_b) * n)) >> 3) & 1)
                                       : 0;
          for (int s2 = 0; s2 < ksy; ++s2) {
            const int k = 4 * s2 + t0;
            const bool kin = k < kc;
            const int sh = kin ? dsh(k) : 0;
            const double a0 = kin ? Dc[k * cs + sh + 16 * mt + g] : 0.0;
            const double a1 = kin ? Dc[k * cs + sh + 16 * mt + g + 8] : 0.0;
            const double b0 = (kin && ncol_b < ncr) ? Xt[ncol_b * LDX + xsh + k] : 0.0;
            dmma_16x8x4(yacc[q], a0, a1, b0);
          }
        }
      }
      // Z_tau(chunk, :) = D(:, chunk)^T X_sigma (off-diagonal blocks)
      if (blk.p_col >= 0) {
        const int zpairs = ((kc + 15) >> 4) * NTN;
        for (int p = warp; p < zpairs; p += 8) {
          const int mt = p / NTN, nt = p - mt * NTN;
          const int j_a0 = 16 * mt + g, j_a1 = j_a0 + 8;  // chunk columns of this lane's A rows
          const bool in0 = j_a0 < kc, in1 = j_a1 < kc;
          const int sh0 = in0 ? dsh(j_a0) : 0, sh1 = in1 ? dsh(j_a1) : 0;
          double z[4] = {0.0, 0.0, 0.0, 0.0}, z1[4] = {0.0, 0.0, 0.0, 0.0};
          const int ksz = R4 >> 2;
          int s2 = 0;
          for (; s2 + 1 < ksz; s2 += 2) {
            const int k = 4 * s2 + t0;
            dmma_16x8x4(z, (in0 && k < R) ? Dc[j_a0 * cs + sh0 + k] : 0.0,
                        (in1 && k < R) ? Dc[j_a1 * cs + sh1 + k] : 0.0, Xs[(8 * nt + g) * kK9bLd + k]);
            dmma_16x8x4(z1, (in0 && k + 4 < R) ? Dc[j_a0 * cs + sh0 + k + 4] : 0.0,
                        (in1 && k + 4 < R) ? Dc[j_a1 * cs + sh1 + k + 4] : 0.0, Xs[(8 * nt + g) * kK9bLd + k + 4]);
          }
          if (s2 < ksz) {
            const int k = 4 * s2 + t0;
            dmma_16x8x4(z, (in0 && k < R) ? Dc[j_a0 * cs + sh0 + k] : 0.0,
                        (in1 && k < R) ? Dc[j_a1 * cs + sh1 + k] : 0.0, Xs[(8 * nt + g) * kK9bLd + k]);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) z[e] += z1[e];
#pragma unroll
          for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const int j = 16 * mt + g + 8 * r2, col = c0 + 8 * nt + 2 * t0 + cc;
              if (j < kc && col < m) part[static_cast<std::int64_t>(col) * pstride + blk.p_col + j0 + j] = z[2 * r2 + cc];
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the stage
    }
  }
#pragma unroll
  for (int q = 0; q < YQ; ++q) {
    const int p = warp + 8 * q;
    if (p < ypairs) {
      const int mt = p / NTN, nt = p - mt * NTN;
#pragma unroll
      for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int r = 16 * mt + g + 8 * r2, col = c0 + 8 * nt + 2 * t0 + cc;
          if (r < R && col < m) part[static_cast<std::int64_t>(col) * pstride + it.p_row + r] = yacc[q][2 * r2 + cc];
        }
    }
  }
}

// y[rows of leaf] = sum of the leaf's partial segments, in list order. Small
// leaves: a thread per row walks the segments. Large leaves (clustered
// points): the rows are accumulated in shared memory (chunks of 4096 rows)
// while the segments are walked once in order, so the work is the total
// segment length (not rows x segments); every row sums in the same order
// either way.
// blockIdx.y is the right-hand-side column (part stride pstride, yp stride n).
__global__ void __launch_bounds__(128) k_near_gather(const std::int64_t* __restrict__ leaf_row0,
                                                     const std::int32_t* __restrict__ leaf_rows,
                                                     const std::int32_t* __restrict__ seg_beg,
                                                     const GatherSeg* __restrict__ segs, const double* __restrict__ part,
                                                     std::int64_t pstride, std::int64_t n, double* __restrict__ yp) {
  constexpr int kRows = 4096, kSegs = 64;
  __shared__ double acc[kRows];
  __shared__ GatherSeg sg[kSegs];
  const int l = blockIdx.x;
  const double* pc = part + blockIdx.y * pstride;
  double* yc = yp + blockIdx.y * n;
  const int sb = seg_beg[l], se = seg_beg[l + 1];
  const int rows = leaf_rows[l];
  if (rows <= 2 * static_cast<int>(blockDim.x)) {
    // small leaf: a thread per row walks the (few) segments itself. The
    // segment list is staged in shared memory first and the partial loads
    // of 16 segments are issued before their in-order sum, so a leaf costs
    // a few round trips instead of two per segment (C3: 65 -> 40 us).
    double s[2] = {0.0, 0.0};
    for (int k0 = sb; k0 < se; k0 += kSegs) {
      const int nk = min(kSegs, se - k0);
      __syncthreads();
      if (threadIdx.x < nk) sg[threadIdx.x] = segs[k0 + threadIdx.x];
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = threadIdx.x + h * blockDim.x;
        if (r >= rows) continue;
        for (int k = 0; k < nk; k += 16) {
          double v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            v[q] = 0.0;
            if (k + q < nk) {
              const GatherSeg g = sg[k + q];
              PHM_DCHECK(g.base >= 0 && g.len >= 0 && g.base + g.len <= rows);
              const int o = r - g.base;
              if (o >= 0 && o < g.len) v[q] = pc[g.poff + o];
            }
          }
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (k + q < nk) s[h] += v[q];
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = threadIdx.x + h * blockDim.x;
      if (r < rows) yc[leaf_row0[l] + r] = s[h];
    }
    return;
  }
  for (int r0 = 0; r0 < rows; r0 += kRows) {
    const int rn = min(kRows, rows - r0);
    for (int r = threadIdx.x; r < rn; r += blockDim.x) acc[r] = 0.0;
    __syncthreads();
    for (int k = sb; k < se; ++k) {
      const GatherSeg g = segs[k];
      const int lo = max(g.base, r0), hi = min(g.base + g.len, r0 + rn);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) acc[r - r0] += pc[g.poff + (r - g.base)];
      __syncthreads();  // next segment may overlap these rows
    }
    for (int r = threadIdx.x; r < rn; r += blockDim.x) yc[leaf_row0[l] + r0 + r] = acc[r];
    __syncthreads();
  }
}


// K8, H form: y_sigma += S_b (H_k (T_b^T x_tau)) per far block (one CTA per
// block: the T^T x reduction is split over the warps, H and S products over
// the threads), written to the block's partial segment; k_far_h_reduce then
// sums each sigma's segments in block order (deterministic, no atomics).
__global__ void __launch_bounds__(128) k_far_h_blocks(const FarHItem* __restrict__ items,
                                                      const std::int32_t* __restrict__ bitem,
                                                      const std::int64_t* __restrict__ tbeg,
                                                      const std::int32_t* __restrict__ tcnt,
                                                      const std::int32_t* __restrict__ cls,
                                                      const std::int64_t* __restrict__ s_off,
                                                      const std::int64_t* __restrict__ t_off,
                                                      const std::int64_t* __restrict__ p_off,
                                                      const ClassMeta* __restrict__ meta, const double* __restrict__ S,
                                                      const double* __restrict__ T, const double* __restrict__ H,
                                                      const double* __restrict__ xp, int b0,
                                                      double* __restrict__ part) {
  __shared__ double tv[128], uv[128];
  const int b = b0 + blockIdx.x;
  const FarHItem it = items[bitem[b]];
  const ClassMeta M = meta[cls[b]];
  const int rl = M.rl, rr = M.rr, nt = tcnt[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Tb = T + t_off[b];
  const double* Sb = S + s_off[b];
  const double* xb = xp + tbeg[b];
  for (int c = warp; c < rr; c += 4) {  // tv = T^T x_tau
    double s = 0.0;
    for (int j = lane; j < nt; j += 32) s += Tb[j + static_cast<std::int64_t>(c) * nt] * xb[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) tv[c] = s;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < rl; a += blockDim.x) {  // uv = H tv
    double s = 0.0;
    for (int c = 0; c < rr; ++c) s += H[M.h_off + a + static_cast<std::int64_t>(c) * rl] * tv[c];
    uv[a] = s;
  }
  __syncthreads();
  double* out = part + p_off[b];
  for (int i = threadIdx.x; i < it.rows; i += blockDim.x) {  // S uv
    double s = 0.0;
    for (int a = 0; a < rl; ++a) s += Sb[i + static_cast<std::int64_t>(a) * it.rows] * uv[a];
    out[i] = s;
  }
}

__global__ void k_far_h_reduce(const FarHItem* __restrict__ items, const std::int64_t* __restrict__ p_off,
                               const double* __restrict__ part, std::int64_t row_lo, std::int64_t row_hi,
                               double* __restrict__ yp) {
  const FarHItem it = items[blockIdx.x];
  for (int i = threadIdx.x; i < it.rows; i += blockDim.x) {
    double s = 0.0;
    for (int b = it.bbeg; b < it.bend; ++b) s += part[p_off[b] + i];
    const std::int64_t pos = it.row0 + i;
    if (pos >= row_lo && pos < row_hi) yp[pos] += s;
  }
}

// ---------------------------------------------- K4 / K7, mode-wise versions
// (A_d (x) ... (x) A_1)^(T) z as d sequential mode contractions in shared
// memory (the fast_kron of chebyshev.cpp:152-193): d * P * ps FMAs per child
// instead of P^2 * d.
__device__ __forceinline__ void mode_round(const double* __restrict__ zin, double* __restrict__ zout,
                                           const double* __restrict__ A, int ps, int P, int stride, bool transposed,
                                           bool accumulate) {
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int bk = (q / stride) % ps;
    const int base = q - bk * stride;
    double s = 0.0;
    for (int a = 0; a < ps; ++a) {
      const double f = transposed ? A[a * ps + bk] : A[bk * ps + a];
      s += f * zin[base + a * stride];
    }
    zout[q] = accumulate ? zout[q] + s : s;
  }
}

// xhat_p = sum over non-empty children c of (E_{c,d} (x) ... (x) E_{c,1})^T xhat_c.
__global__ void k_up2(const std::int32_t* __restrict__ nodes, const std::int32_t* __restrict__ first_child,
                      const std::int32_t* __restrict__ count, const double* __restrict__ E, int d, int ps, int P,
                      int nc, int m, double* __restrict__ xhat) {
  extern __shared__ double sm[];
  const int p = nodes[blockIdx.x];
  const int fc = first_child[p];
  const int fsz = d * ps * ps;
  double* se = sm;               // d x ps x ps factors of the current child
  double* za = se + fsz;         // ping
  double* zb = za + P;           // pong
  double* acc = zb + P;          // P
  {
    const int c = blockIdx.y;  // one right-hand side per grid row
    for (int e = threadIdx.x; e < P; e += blockDim.x) acc[e] = 0.0;
    for (int ch = 0; ch < nc; ++ch) {
      if (count[fc + ch] == 0) continue;
      __syncthreads();
      for (int e = threadIdx.x; e < fsz; e += blockDim.x) se[e] = E[static_cast<std::int64_t>(fc + ch) * fsz + e];
      for (int e = threadIdx.x; e < P; e += blockDim.x)
        za[e] = xhat[(static_cast<std::int64_t>(fc + ch) * m + c) * P + e];
      __syncthreads();
      double* in = za;
      double* out = zb;
      int stride = 1;
      for (int k = 0; k < d; ++k) {
        if (k == d - 1) {
          mode_round(in, acc, se + k * ps * ps, ps, P, stride, true, true);
        } else {
          mode_round(in, out, se + k * ps * ps, ps, P, stride, true, false);
          __syncthreads();
          double* t = in;
          in = out;
          out = t;
        }
        stride *= ps;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < P; e += blockDim.x) xhat[(static_cast<std::int64_t>(p) * m + c) * P + e] = acc[e];
    __syncthreads();
  }
}

// yhat_child += (E_d (x) ... (x) E_1) yhat_parent.
__global__ void k_down2(const std::int32_t* __restrict__ nodes, const std::int32_t* __restrict__ parent,
                        const double* __restrict__ E, int d, int ps, int P, int m, double* __restrict__ yhat) {
  extern __shared__ double sm[];
  const int ch = nodes[blockIdx.x];
  const int p = parent[ch];
  const int fsz = d * ps * ps;
  double* se = sm;
  double* za = se + fsz;
  double* zb = za + P;
  double* yc = zb + P;
  for (int e = threadIdx.x; e < fsz; e += blockDim.x) se[e] = E[static_cast<std::int64_t>(ch) * fsz + e];
  {
    const int c = blockIdx.y;  // one right-hand side per grid row
    __syncthreads();
    for (int e = threadIdx.x; e < P; e += blockDim.x) {
      za[e] = yhat[(static_cast<std::int64_t>(p) * m + c) * P + e];
      yc[e] = yhat[(static_cast<std::int64_t>(ch) * m + c) * P + e];
    }
    __syncthreads();
    double* in = za;
    double* out = zb;
    int stride = 1;
    for (int k = 0; k < d; ++k) {
      if (k == d - 1) {
        mode_round(in, yc, se + k * ps * ps, ps, P, stride, false, true);
      } else {
        mode_round(in, out, se + k * ps * ps, ps, P, stride, false, false);
        __syncthreads();
        double* t = in;
        in = out;
        out = t;
      }
      stride *= ps;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < P; e += blockDim.x) yhat[(static_cast<std::int64_t>(ch) * m + c) * P + e] = yc[e];
  }
}

// y_i += <kron row of point i, yhat> folded one dimension at a time, last
// dimension first (chebyshev.cpp:270-282); one CTA per leaf, the partial
// folds of all points of a 32-point chunk live in shared memory.
constexpr int kLeafBwdChunk = 32;  // points per pass of k_leaf_bwd2 (64: no faster)
__global__ void k_leaf_bwd2(const std::int32_t* __restrict__ leaves, const std::int64_t* __restrict__ begin,
                            const std::int32_t* __restrict__ count, const double* __restrict__ U, std::int64_t n,
                            int d, int ps, int P, const double* __restrict__ yhat, int m, std::int64_t row_lo,
                            std::int64_t row_hi, double* __restrict__ yp) {
  extern __shared__ double sm[];
  constexpr int kChunk = kLeafBwdChunk;
  const int leaf = leaves[blockIdx.x];
  const std::int64_t b0 = begin[leaf];
  const int cnt = count[leaf];
  double* yh = sm;                 // P
  double* ta = yh + P;             // kChunk x P/ps
  double* tb = ta + kChunk * (P / ps);
  {
    const int c = blockIdx.y;  // one right-hand side per grid row
    __syncthreads();
    for (int e = threadIdx.x; e < P; e += blockDim.x) yh[e] = yhat[(static_cast<std::int64_t>(leaf) * m + c) * P + e];
    __syncthreads();
    for (int i0 = 0; i0 < cnt; i0 += kChunk) {
      const int len = min(kChunk, cnt - i0);
      const double* in = yh;
      int inlen = P;   // per-point length (shared yh has no point stride)
      bool shared_in = true;
      double* out = ta;
      for (int k = d - 1; k >= 1; --k) {
        const int olen = inlen / ps;
        for (int e = threadIdx.x; e < len * olen; e += blockDim.x) {
          const int i = e / olen, q = e % olen;
          const std::int64_t pos = b0 + i0 + i;
          const double* u = U + (static_cast<std::int64_t>(k) * n + pos) * ps;
          const double* z = shared_in ? in : in + i * inlen;
          double s = 0.0;
          for (int a = 0; a < ps; ++a) s += z[q + a * olen] * u[a];
          out[i * olen + q] = s;
        }
        __syncthreads();
        in = out;
        out = (out == ta) ? tb : ta;
        inlen = olen;
        shared_in = false;
      }
      for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const std::int64_t pos = b0 + i0 + i;
        const double* u = U + pos * ps;  // dimension 0
        const double* z = shared_in ? in : in + i * inlen;
        double s = 0.0;
        for (int a = 0; a < ps; ++a) s += u[a] * z[a];
        if (pos >= row_lo && pos < row_hi) yp[static_cast<std::int64_t>(c) * n + pos] += s;
      }
      __syncthreads();
    }
  }
}

// estimate_error (harness.cpp:183-236): exact rows (K x)_J for the probe
// rows J by direct kernel evaluation, one CTA per probe row, fixed-order
// block reduction.
__global__ void __launch_bounds__(256) k_exact_rows(const std::int64_t* __restrict__ rows, const double* __restrict__ pts,
                                                    std::int64_t n, int d, int fam, const double* __restrict__ theta,
                                                    double amp, const double* __restrict__ xp,
                                                    double* __restrict__ out) {
  __shared__ double red[256];
  const std::int64_t r = rows[blockIdx.x];
  double pr[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < d; ++k) pr[k] = pts[k * n + r];
  double th[3] = {theta[0], theta[1], theta[2]};
  double s = 0.0;
  for (std::int64_t l = threadIdx.x; l < n; l += blockDim.x) {
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double dl = __dsub_rn(pr[k], pts[k * n + l]);
      r2 = __dadd_rn(r2, __dmul_rn(dl, dl));
    }
    s += amp * kernel_profile(fam, sqrt(r2), th) * xp[l];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// ------------------------------------------------------------ launchers
namespace {
// cudaFuncSetAttribute once per (kernel, device, size): the attributes live
// in each device's context, and launches may come from several host threads.
void smem_attr(const void* fn, int bytes, bool max_carveout) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert(std::make_tuple(fn, dev, bytes)).second) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (max_carveout)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}
}  // namespace

void launch_exact_rows(cudaStream_t st, const std::int64_t* rows, int nrows, const double* pts, std::int64_t n, int d,
                       int fam, const double* theta, double amp, const double* xp, double* out) {
  if (nrows == 0) return;
  k_exact_rows<<<nrows, 256, 0, st>>>(rows, pts, n, d, fam, theta, amp, xp, out);
}
void launch_snapshot(cudaStream_t st, const SnapTile* tiles, std::int64_t ntiles, const BlockGeom* geo,
                     const double* pts, std::int64_t n, int d, int fam, int R, const double* theta_nodes, double amp,
                     double* out) {
  const int grid = static_cast<int>(std::min<std::int64_t>(ntiles, 148 * 16));
  if (grid > 0) k_snapshot<<<grid, 256, 0, st>>>(tiles, ntiles, geo, pts, n, d, fam, R, theta_nodes, amp, out);
}

bool launch_inst_flat_batch(cudaStream_t st, const double* G, std::int64_t E, int R, int B, const InstPtrs& tab) {
  if (B < 1 || B > kInstBatchMax) return false;
  static const int per_sm = [] {
    const char* e = std::getenv("PHM_K1_CTAS");
    const int k = e ? std::atoi(e) : 4;
    return k >= 1 && k <= 8 ? k : 4;
  }();
  const std::int64_t E4 = E >> 2;
  const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((E4 + 255) / 256, 148 * per_sm)));
  switch (R) {
    case 1: k_inst_flat_batch<1><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 2: k_inst_flat_batch<2><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 3: k_inst_flat_batch<3><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 4: k_inst_flat_batch<4><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 5: k_inst_flat_batch<5><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 6: k_inst_flat_batch<6><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 8: k_inst_flat_batch<8><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 10: k_inst_flat_batch<10><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 12: k_inst_flat_batch<12><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    case 16: k_inst_flat_batch<16><<<grid, 256, 0, st>>>(G, E, B, tab); return true;
    default: return false;
  }
}
bool launch_inst_tma(cudaStream_t st, const double* G, std::int64_t E, int R, int B, const InstPtrs& tab, int per_sm) {
  if (E == 0) return true;
  if (B < 1 || B > kInstBatchMax) return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const int k1_env = [] {  // A/B override of the caller's choice
    const char* e = std::getenv("PHM_K1_TMA_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  const int k1_per_sm = k1_env == 1 || k1_env == 2 ? k1_env : (per_sm == 1 ? 1 : 2);
#define PHM_K1T(RR)                                                                                           \
  case RR: {                                                                                                  \
    constexpr int CH = ((5120 / RR) & ~63) < 256 ? 256 : (((5120 / RR) & ~63) > 1024 ? 1024 : ((5120 / RR) & ~63)); \
    constexpr int NST = 2;                                                                                    \
    const size_t smem = static_cast<size_t>(NST * RR * CH) * sizeof(double);                                 \
    smem_attr(reinterpret_cast<const void*>(k_inst_tma<RR, CH, NST>), static_cast<int>(smem), true);          \
    const int grid = static_cast<int>(std::min<std::int64_t>((E + CH - 1) / CH, k1_per_sm * sms));           \
    k_inst_tma<RR, CH, NST><<<grid, kTmaThreads, smem, st>>>(G, E, B, tab);                                   \
    return true;                                                                                              \
  }
  switch (R) {
    PHM_K1T(1)
    PHM_K1T(2)
    PHM_K1T(4)
    PHM_K1T(6)
    PHM_K1T(8)
    PHM_K1T(10)
    PHM_K1T(12)
    PHM_K1T(16)
    default: return false;
  }
#undef PHM_K1T
}

void launch_inst_flat(cudaStream_t st, const double* G, std::int64_t E, int R, const double* w, double* D) {
  const std::int64_t E4 = E / 4;
  if (E4 == 0) return;
  // Grid of 148 x k resident CTAs (grid-stride). k = 4 leaves half of each
  // SM's warp slots to the compute-bound far-field chain that runs on the
  // side stream during the fused instantiate+apply; PHM_K1_CTAS overrides.
  static const int per_sm = [] {
    const char* e = std::getenv("PHM_K1_CTAS");
    const int k = e ? std::atoi(e) : 4;
    return k >= 1 && k <= 8 ? k : 4;
  }();
  const int grid = static_cast<int>(std::min<std::int64_t>((E4 + 255) / 256, 148 * per_sm));
  switch (R) {
    case 1: k_inst_flat<1><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 2: k_inst_flat<2><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 4: k_inst_flat<4><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 6: k_inst_flat<6><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 8: k_inst_flat<8><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 10: k_inst_flat<10><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 12: k_inst_flat<12><<<grid, 256, 0, st>>>(G, E, w, D); break;
    case 16: k_inst_flat<16><<<grid, 256, 0, st>>>(G, E, w, D); break;
    default: k_inst_flat_any<<<grid, 256, 0, st>>>(G, E, R, w, D); break;
  }
}

void launch_inst_tiles(cudaStream_t st, const InstTile* tiles, std::int64_t nt, const double* G, const double* w,
                       double* D) {
  const int grid = static_cast<int>(std::min<std::int64_t>(nt, 148 * 8));
  if (grid > 0) k_inst_tiles<<<grid, 256, 0, st>>>(tiles, nt, G, w, D);
}


void launch_near_w(cudaStream_t st, const NearW* meta, std::int64_t nb, const double* cores, const std::int32_t* dims,
                   const ThetaParams* tp, double* w) {
  if (nb == 0) return;
  const int wpb = 8;
  const int grid = static_cast<int>(std::min<std::int64_t>((nb + wpb - 1) / wpb, 148 * 16));
  k_near_w<<<grid, 32 * wpb, wpb * 2 * 256 * sizeof(double), st>>>(meta, nb, cores, dims, tp, w);
}

void launch_set_vec(cudaStream_t st, double* dst, int n, const ThetaParams* tp) {
  k_set_vec<<<(n + 127) / 128, 128, 0, st>>>(dst, n, tp);
}
void launch_put_theta(cudaStream_t st, const ThetaParams& p, ThetaParams* dst) {
  k_put_theta<<<1, 128, 0, st>>>(p, dst);
}


void launch_class_inst(cudaStream_t st, const ClassMeta* meta, int ncls, const double* mid, const std::int32_t* dims,
                       const double* L, const double* R, const ThetaParams* tp, int P, bool want_c, int capA,
                       int capB, int capT, int capL, int capR, int ctas, double* H, double* C) {
  if (ncls == 0) return;
  if (capR > 0) {  // k_class_inst_pf: capT is its theta-chain scratch, capR the R / T region
    const size_t smem = static_cast<size_t>(capA + capB + capT + capR + capL) * sizeof(double);
    smem_attr(reinterpret_cast<const void*>(k_class_inst_pf), 227 * 1024, false);
    const int grid = ctas > 0 ? std::min(ctas, ncls) : ncls;
    k_class_inst_pf<<<grid, 256, smem, st>>>(meta, ncls, mid, dims, L, R, tp, capA, capB, capT, capR, H, C);
    return;
  }
  const size_t smem = static_cast<size_t>(capA + capB + capT + capL) * sizeof(double);
  smem_attr(reinterpret_cast<const void*>(k_class_inst), 227 * 1024, false);
  k_class_inst<<<ncls, 256, smem, st>>>(meta, ncls, mid, dims, L, R, tp, P, want_c ? 1 : 0, capA, capB, capT, H, C);
}

void launch_gather(cudaStream_t st, const double* x, const std::int32_t* perm, std::int64_t n, std::int64_t m,
                   double* xp) {
  const std::int64_t t = n * m;
  k_gather<<<static_cast<unsigned>((t + 255) / 256), 256, 0, st>>>(x, perm, n, m, xp);
}
void launch_scatter(cudaStream_t st, const double* yp, const std::int32_t* perm, std::int64_t n, std::int64_t m,
                    double* y) {
  const std::int64_t t = n * m;
  k_scatter<<<static_cast<unsigned>((t + 255) / 256), 256, 0, st>>>(yp, perm, n, m, y);
}

static int threads_for(int P) { return P <= 64 ? 64 : (P <= 128 ? 128 : 256); }

void launch_leaf_fwd(cudaStream_t st, const std::int32_t* leaves, int nleaves, const std::int64_t* begin,
                     const std::int32_t* count, const double* U, std::int64_t n, int d, int ps, int P, const double* xp,
                     int m, double* xhat) {
  if (nleaves == 0) return;
  if (P == 64 && m >= 4 && d * ps <= 48) {
    if (m <= 16) {
      k_leaf_fwd_m<4><<<dim3(nleaves, (m + 15) / 16), 256, 0, st>>>(leaves, begin, count, U, n, d, ps, xp, m, xhat);
    } else {
      k_leaf_fwd_m<16><<<dim3(nleaves, (m + 63) / 64), 256, 0, st>>>(leaves, begin, count, U, n, d, ps, xp, m, xhat);
    }
    return;
  }
  const size_t smem = (64 * d * ps + 64) * sizeof(double);
  if (smem > 48 * 1024) smem_attr(reinterpret_cast<const void*>(k_leaf_fwd), static_cast<int>(smem), false);
  k_leaf_fwd<<<dim3(nleaves, m), threads_for(P), smem, st>>>(leaves, begin, count, U, n, d, ps, P, xp, m, xhat);
}
// The big leaves of a list (more than kLeafChunk points, m >= 4, P = 64):
// chunk partials, then the ordered sum per leaf.
void launch_leaf_fwd_chunks(cudaStream_t st, const LeafChunk* chunks, int nchunks, const std::int32_t* red_leaf,
                            const std::int64_t* red_slot, const std::int32_t* red_n, int nred,
                            const std::int64_t* begin, const std::int32_t* count, const double* U, std::int64_t n,
                            int d, int ps, const double* xp, int m, double* part, double* xhat) {
  if (nchunks == 0) return;
  if (m <= 16)
    k_leaf_fwd_m<4><<<dim3(nchunks, (m + 15) / 16), 256, 0, st>>>(nullptr, begin, count, U, n, d, ps, xp, m, part,
                                                                   chunks);
  else
    k_leaf_fwd_m<16><<<dim3(nchunks, (m + 63) / 64), 256, 0, st>>>(nullptr, begin, count, U, n, d, ps, xp, m, part,
                                                                    chunks);
  k_leaf_fwd_reduce<<<nred, 256, 0, st>>>(red_leaf, red_slot, red_n, 64, m, part, xhat);
}
void launch_up(cudaStream_t st, const std::int32_t* nodes, int cnt, const std::int32_t* first_child,
               const std::int32_t* count, const double* E, int d, int ps, int P, int m, double* xhat) {
  if (cnt == 0) return;
  const int nc = 1 << d;
  const size_t smem = (d * ps * ps + 3 * P) * sizeof(double);
  if (smem > 48 * 1024) smem_attr(reinterpret_cast<const void*>(k_up2), static_cast<int>(smem), false);
  k_up2<<<dim3(cnt, m), threads_for(P), smem, st>>>(nodes, first_child, count, E, d, ps, P, nc, m, xhat);
}
void launch_coupling(cudaStream_t st, const std::int32_t* sig, int nsig, const std::int64_t* fbeg,
                     const std::int32_t* ftau, const std::int32_t* fcls, const double* C, int P, int m,
                     const double* xhat, double* yhat) {
  if (nsig == 0) return;
  k_coupling<<<nsig, threads_for(P), P * sizeof(double), st>>>(sig, fbeg, ftau, fcls, C, P, m, xhat, yhat);
}
void launch_near_tma_apply(cudaStream_t st, const SymRowItem* items, int nitems, const SymBlock* blocks,
                           const double* D, const double* xp, double* part, int* counter) {
  if (nitems == 0) return;
  // 3 stages of 24 KB (48 columns of a 64-row leaf): two CTAs per SM
  constexpr int CH = 3072, NST = 3;
  const size_t smem = static_cast<size_t>(NST * (CH + 2 + 66) + 8 * 128) * sizeof(double);
  smem_attr(reinterpret_cast<const void*>(k_near_tma_apply<CH, NST>), static_cast<int>(smem), true);
  static const int per_sm = [] {
    const char* e = std::getenv("PHM_NEAR_CTAS_PER_SM");
    const int k = e ? std::atoi(e) : 2;
    return k >= 1 && k <= 2 ? k : 2;
  }();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  static const int lean = [] {  // PHM_NEAR_GEMV=0: the 8-consumer-warp kernel at two CTAs per SM
    const char* e = std::getenv("PHM_NEAR_GEMV");
    return e ? std::atoi(e) : 1;
  }();
  if (lean) {
    // one CTA per SM (a quarter of the SM's registers): the coupling's CTAs
    // fill the rest of every SM while this stream runs
    static const int lnst = [] {  // ring depth (two stages: room for the coupling's CTAs)
      const char* e = std::getenv("PHM_NEAR_LEAN_NST");
      const int k = e ? std::atoi(e) : 2;
      return k == 3 || k == 4 ? k : 2;
    }();
    static const int lch = [] {  // chunk doubles: 4096 = a whole 64 x 64 block
      const char* e = std::getenv("PHM_NEAR_LEAN_CH");
      const int k = e ? std::atoi(e) : 4096;
      return k == 3072 ? 3072 : 4096;
    }();
    static const int lwarps = [] {  // consumer warps per CTA
      const char* e = std::getenv("PHM_NEAR_LEAN_WARPS");
      const int k = e ? std::atoi(e) : 4;
      return k == 8 ? 8 : 4;
    }();
    static const int lean_per_sm = [] {
      const char* e = std::getenv("PHM_NEAR_LEAN_PER_SM");
      const int k = e ? std::atoi(e) : 2;
      return k >= 1 && k <= 2 ? k : 1;
    }();
    const int grid = std::min(nitems, sms * lean_per_sm);
    static const bool lef = [] {  // D by evict-first bulk copies (C_k stays in L2 for the coupling beside)
      const char* e = std::getenv("PHM_GEMV_EVICT_FIRST");
      return !(e && std::atoi(e) == 0);
    }();
#define PHM_LEAN(WW, LCH, NN)                                                                               \
  if (lnst == NN && lwarps == WW && lch == LCH) {                                                           \
    const size_t lsmem = static_cast<size_t>(NN * (LCH + 2 + 66) + WW * 128) * sizeof(double);             \
    smem_attr(reinterpret_cast<const void*>(k_near_gemv_lean<WW, LCH, NN>), static_cast<int>(lsmem), true); \
    k_near_gemv_lean<WW, LCH, NN><<<grid, (WW + 1) * 32, lsmem, st>>>(items, nitems, blocks, D, xp, part, counter, lef); \
    return;                                                                                                 \
  }
    PHM_LEAN(4, 4096, 2) PHM_LEAN(4, 3072, 2) PHM_LEAN(4, 4096, 3) PHM_LEAN(4, 3072, 3) PHM_LEAN(4, 4096, 4)
    PHM_LEAN(8, 4096, 2) PHM_LEAN(8, 4096, 3) PHM_LEAN(8, 4096, 4)
#undef PHM_LEAN
    {  // any other PHM_NEAR_LEAN_* combination: the default kernel
      const size_t lsmem = static_cast<size_t>(2 * (4096 + 2 + 66) + 4 * 128) * sizeof(double);
      smem_attr(reinterpret_cast<const void*>(k_near_gemv_lean<4, 4096, 2>), static_cast<int>(lsmem), true);
      k_near_gemv_lean<4, 4096, 2><<<grid, 5 * 32, lsmem, st>>>(items, nitems, blocks, D, xp, part, counter, lef);
    }
    return;
  }
  const int grid = std::min(nitems, sms * per_sm);
  k_near_tma_apply<CH, NST><<<grid, kTmaThreads, smem, st>>>(items, nitems, blocks, D, xp, part, counter);
}
void launch_near_mvm_symcsr(cudaStream_t st, const SymRowItem* items, int nitems, const SymBlock* blocks,
                            const double* D, const double* xp, double* part) {
  if (nitems == 0) return;
  k_near_mvm_symcsr<<<nitems, 256, 0, st>>>(items, blocks, D, xp, part);
}
// Chunk length (doubles per slab) of k_near_tma for rank R: about 40 KB per
// stage, 256 <= CH <= 1024, a multiple of 64.
constexpr int near_tma_ch(int R) {
  return ((5120 / R) & ~63) < 256 ? 256 : (((5120 / R) & ~63) > 1024 ? 1024 : ((5120 / R) & ~63));
}

namespace {
// CTAs of kernel b that fit on one SM beside na CTAs of kernel a (registers,
// shared memory, threads; per-warp register allocation in units of 256).
int fit_beside(const void* fa, size_t dyn_a, int thr_a, int na, const void* fb, size_t dyn_b, int thr_b) {
  int dev = 0;
  cudaGetDevice(&dev);
  struct {
    int regsPerMultiprocessor, sharedMemPerMultiprocessor, reservedSharedMemPerBlock, maxThreadsPerMultiProcessor;
  } pr{};
  cudaFuncAttributes a, b;
  if (cudaDeviceGetAttribute(&pr.regsPerMultiprocessor, cudaDevAttrMaxRegistersPerMultiprocessor, dev) ||
      cudaDeviceGetAttribute(&pr.sharedMemPerMultiprocessor, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) ||
      cudaDeviceGetAttribute(&pr.reservedSharedMemPerBlock, cudaDevAttrReservedSharedMemoryPerBlock, dev) ||
      cudaDeviceGetAttribute(&pr.maxThreadsPerMultiProcessor, cudaDevAttrMaxThreadsPerMultiProcessor, dev) ||
      cudaFuncGetAttributes(&a, fa) != cudaSuccess || cudaFuncGetAttributes(&b, fb) != cudaSuccess)
    return 0;
  auto regs = [](const cudaFuncAttributes& f, int thr) {
    return ((thr + 31) / 32) * ((f.numRegs * 32 + 255) / 256 * 256);
  };
  auto smem = [&](const cudaFuncAttributes& f, size_t dyn) {
    return static_cast<long>(f.sharedSizeBytes + dyn + pr.reservedSharedMemPerBlock);
  };
  long r = pr.regsPerMultiprocessor - static_cast<long>(na) * regs(a, thr_a);
  long sm = static_cast<long>(pr.sharedMemPerMultiprocessor) - na * smem(a, dyn_a);
  long th = pr.maxThreadsPerMultiProcessor - static_cast<long>(na) * thr_a;
  int k = 0;
  while (r >= regs(b, thr_b) && sm >= smem(b, dyn_b) && th >= thr_b && k < 8) {
    r -= regs(b, thr_b);
    sm -= smem(b, dyn_b);
    th -= thr_b;
    ++k;
  }
  return k;
}
}  // namespace

int coupling_fit(int R, int P);
// Coupling CTAs (k_coupling_mma<P>) that fit on one SM beside the two CTAs
// per SM of the fused near pass (k_near_tma for rank R); 0 when none does.
// Memoised: it runs on every (ungraphed) step.
int coupling_beside_near(int R, int P) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, int> memo;  // (device, R, P) -> CTAs
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, R, P);
  const auto hit = memo.find(key);
  if (hit != memo.end()) return hit->second;
  return memo[key] = coupling_fit(R, P);
}
int coupling_fit(int R, int P) {
  const size_t cpl = 2 * kGroupSlots * (P + 4) * sizeof(double);
  const void* fb = nullptr;
  switch (P) {
    case 16: fb = reinterpret_cast<const void*>(k_coupling_mma<16>); break;
    case 32: fb = reinterpret_cast<const void*>(k_coupling_mma<32>); break;
    case 64: fb = reinterpret_cast<const void*>(k_coupling_mma<64>); break;
    case 128: fb = reinterpret_cast<const void*>(k_coupling_mma<128>); break;
    default: return 0;
  }
  switch (R) {
#define PHM_FIT(RR)                                                                                             \
  case RR:                                                                                                      \
    return fit_beside(reinterpret_cast<const void*>(k_near_tma<RR, near_tma_ch(RR), 2>),                        \
                      static_cast<size_t>(tma_smem_doubles(RR, near_tma_ch(RR), 2)) * sizeof(double), kTmaThreads, 2, \
                      fb, cpl, P / 16 * 32);
    PHM_FIT(1) PHM_FIT(2) PHM_FIT(3) PHM_FIT(4) PHM_FIT(5) PHM_FIT(6) PHM_FIT(7) PHM_FIT(8)
    PHM_FIT(9) PHM_FIT(10) PHM_FIT(11) PHM_FIT(12) PHM_FIT(13) PHM_FIT(14) PHM_FIT(15) PHM_FIT(16)
#undef PHM_FIT
    default: return 0;
  }
}

// Snapshot-mode instantiate fused with apply (K1 + K6 in one pass over the
// snapshots). Returns false for a rank without an instantiation (R > 16).
bool launch_near_inst_tma(cudaStream_t st, const SymRowItem* items, int nitems, const SymBlock* blocks,
                          const double* G, std::int64_t E, int R, const double* w, double* D, const double* xp,
                          double* part) {
  if (nitems == 0) return true;
#define PHM_TMA(RR, NST) PHM_TMA_CH(RR, near_tma_ch(RR), NST)
#define PHM_TMA_CH(RR, CHv, NST)                                                                              \
  {                                                                                                           \
    constexpr int CHc = CHv;                                                                                  \
    const size_t smem = static_cast<size_t>(tma_smem_doubles(RR, CHc, NST)) * sizeof(double);                \
    smem_attr(reinterpret_cast<const void*>(k_near_tma<RR, CHc, NST>), static_cast<int>(smem), true);       \
    k_near_tma<RR, CHc, NST><<<nitems, kTmaThreads, smem, st>>>(items, blocks, G, E, w, D, xp, part);                 \
    return true;                                                                                              \
  }
  // two stages of about 40 KB (R slabs x CH doubles, 256 <= CH <= 1024): two
  // CTAs per SM. Measured at C3 (R = 8): 8.9 ms for CH 640 x 2 stages and
  // CH 512 x 3, 9.4 ms for 512 x 2, 10.3 ms for 768 x 2 (one CTA per SM),
  // 18.5 ms for 256 x 6 (the per-chunk cost dominates small chunks).
  switch (R) {
    case 1: PHM_TMA(1, 2)
    case 2: PHM_TMA(2, 2)
    case 3: PHM_TMA(3, 2)
    case 4: PHM_TMA(4, 2)
    case 5: PHM_TMA(5, 2)
    case 6: PHM_TMA(6, 2)
    case 7: PHM_TMA(7, 2)
    case 8: PHM_TMA(8, 2)
    case 9: PHM_TMA(9, 2)
    case 10: PHM_TMA(10, 2)
    case 11: PHM_TMA(11, 2)
    case 12: PHM_TMA(12, 2)
    case 13: PHM_TMA(13, 2)
    case 14: PHM_TMA(14, 2)
    case 15: PHM_TMA(15, 2)
    case 16: PHM_TMA(16, 2)
    default: break;
  }
#undef PHM_TMA
#undef PHM_TMA_CH
  return false;
}

void launch_near_gather(cudaStream_t st, int nleaves, const std::int64_t* leaf_row0, const std::int32_t* leaf_rows,
                        const std::int32_t* seg_beg, const GatherSeg* segs, const double* part, std::int64_t pstride,
                        std::int64_t n, int m, double* yp) {
  if (nleaves == 0 || m == 0) return;
  k_near_gather<<<dim3(nleaves, m), 128, 0, st>>>(leaf_row0, leaf_rows, seg_beg, segs, part, pstride, n, yp);
}

void launch_near_mrhs3(cudaStream_t st, const SymRowItem* items, int nitems, const SymBlock* blocks, const double* D,
                       const double* X, std::int64_t n, int m, std::int64_t pstride, double* part, int dense_rows) {
  if (nitems == 0) return;
  // D per stage: 32 columns of the tallest leaf when every item is a whole
  // leaf (one bulk copy per chunk), else 32 padded columns of 132
  const int dstage = dense_rows > 0 ? ((kK9bKc * dense_rows + 2 + 1) & ~1) : kK9bKc * kK9bLd;
  static const int nst_env = [] {  // tuning: ring depth
    const char* e = std::getenv("PHM_K9_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  auto bytes = [&](int nc, int nst) {
    return static_cast<size_t>(nc * kK9bLd + nst * (dstage + nc * (kK9bKc + 4))) * sizeof(double);
  };
  // more than 32 RHS: one 64-column tile, so D is read once (one CTA per SM)
  const int nc = m <= 8 ? 8 : (m <= 16 ? 16 : (m <= 32 ? 32 : 64));
  // the deepest ring (<= 4) that keeps two CTAs per SM (one for 64 columns)
  const size_t budget = nc == 64 ? 226 * 1024 : 113 * 1024;
  int nst = 2;
  for (int q = 4; q > 2; --q)
    if (bytes(nc, q) + 2048 <= budget) {
      nst = q;
      break;
    }
  if (nst_env >= 2 && nst_env <= 4) nst = nst_env;
#define PHM_K9C(NC, NST)                                                                                    \
  if (nc == NC && nst == NST) {                                                                             \
    const size_t smem = bytes(NC, NST);                                                                     \
    smem_attr(reinterpret_cast<const void*>(k_near_mrhs3<NC, NST>), static_cast<int>(smem), true);         \
    const dim3 grid(static_cast<unsigned>(nitems), static_cast<unsigned>((m + NC - 1) / NC));               \
    k_near_mrhs3<NC, NST><<<grid, kTmaThreads, smem, st>>>(items, blocks, D, X, n, m, pstride, part, dstage); \
    return;                                                                                                 \
  }
  PHM_K9C(8, 2) PHM_K9C(8, 3) PHM_K9C(8, 4)
  PHM_K9C(16, 2) PHM_K9C(16, 3) PHM_K9C(16, 4)
  PHM_K9C(32, 2) PHM_K9C(32, 3) PHM_K9C(32, 4)
  PHM_K9C(64, 2) PHM_K9C(64, 3) PHM_K9C(64, 4)
#undef PHM_K9C
}

void launch_near_mrhs2(cudaStream_t st, const SymRowItem* items, int nitems, const SymBlock* blocks, const double* D,
                       const double* X, std::int64_t n, int m, std::int64_t pstride, double* part) {
  if (nitems == 0) return;
#define PHM_K9B(NC)                                                                                         \
  {                                                                                                         \
    const size_t smem = (NC * kK9bLd + 2 * (kK9bKc * kK9bLd + NC * kK9bLx)) * sizeof(double);             \
    smem_attr(reinterpret_cast<const void*>(k_near_mrhs2<NC>), static_cast<int>(smem), true);              \
    const dim3 grid(static_cast<unsigned>(nitems), static_cast<unsigned>((m + NC - 1) / NC));               \
    k_near_mrhs2<NC><<<grid, 256, smem, st>>>(items, blocks, D, X, n, m, pstride, part);                    \
    return;                                                                                                 \
  }
  if (m <= 8) PHM_K9B(8)
  if (m <= 16) PHM_K9B(16)
  if (m <= 32) PHM_K9B(32)
  PHM_K9B(64)
#undef PHM_K9B
}

void launch_near_mrhs(cudaStream_t st, const MrhsItem* items, int nitems, const std::int64_t* tb, const std::int32_t* tn,
                      const std::int64_t* doff, const std::int32_t* ld, const std::int32_t* tr, const double* D,
                      const double* X, std::int64_t n, int m, double* Y) {
  if (nitems == 0) return;
#define PHM_K9(NC)                                                                                          \
  {                                                                                                         \
    const size_t smem = 2 * (kK9Rows * (kK9Kc + 4) + kK9Kc * (NC + 4)) * sizeof(double);                   \
    smem_attr(reinterpret_cast<const void*>(k_near_mrhs<NC>), 96 * 1024, false);                           \
    const dim3 grid(static_cast<unsigned>(nitems), static_cast<unsigned>((m + NC - 1) / NC));               \
    k_near_mrhs<NC><<<grid, 128, smem, st>>>(items, tb, tn, doff, ld, tr, D, X, n, m, Y);                   \
    return;                                                                                                 \
  }
  if (m <= 8) PHM_K9(8)
  if (m <= 16) PHM_K9(16)
  if (m <= 32) PHM_K9(32)
  PHM_K9(64)
#undef PHM_K9
}

bool coupling_mma_supported(int P) { return P == 16 || P == 32 || P == 64 || P == 128; }

void launch_coupling_mma(cudaStream_t st, const CouplingItem* items, const std::int32_t* order, int nitems,
                         const std::int32_t* item_cls, const std::uint8_t* item_tiles, const std::int32_t* cls_tau,
                         const double* C, int P, const double* xhat, int m, double* partial, int max_ctas) {
  if (nitems == 0) return;
  // one RHS column per CTA iteration: at C3 it beat two columns sharing each
  // C_k fragment load at every m measured (4: 3.3 vs 3.5 ms, 10: 7.9 vs 8.4,
  // 64: 49.4 vs 52.2) -- occupancy over reuse
  const size_t smem = 2 * kGroupSlots * (P + 4) * sizeof(double);
  const std::int64_t nvb = static_cast<std::int64_t>(nitems) * m;
  const int grid = static_cast<int>(max_ctas > 0 && max_ctas < nvb ? max_ctas : nvb);
  static const int diag = [] {  // schedule diagnostics (results invalid), P = 64 only
    const char* e = std::getenv("PHM_COUPLING_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  if (P == 64 && (diag == 1 || diag == 2)) {
    if (diag == 1) {
      smem_attr(reinterpret_cast<const void*>(k_coupling_mma<64, 1>), 200 * 1024, false);
      k_coupling_mma<64, 1><<<grid, 128, smem, st>>>(items, order, item_cls, item_tiles, cls_tau, C, xhat, m, partial,
                                                     nitems);
    } else {
      smem_attr(reinterpret_cast<const void*>(k_coupling_mma<64, 2>), 200 * 1024, false);
      k_coupling_mma<64, 2><<<grid, 128, smem, st>>>(items, order, item_cls, item_tiles, cls_tau, C, xhat, m, partial,
                                                     nitems);
    }
    return;
  }
#define PHM_CASE(PP)                                                                                        \
  if (P == PP) {                                                                                            \
    smem_attr(reinterpret_cast<const void*>(k_coupling_mma<PP>), 200 * 1024, false);                       \
    k_coupling_mma<PP><<<grid, PP / 16 * 32, smem, st>>>(items, order, item_cls, item_tiles, cls_tau, C, xhat, m, \
                                                         partial, nitems);                                      \
    return;                                                                                                 \
  }
  PHM_CASE(16)
  PHM_CASE(32)
  PHM_CASE(64)
  PHM_CASE(128)
#undef PHM_CASE
}

void launch_coupling_reduce(cudaStream_t st, const std::int32_t* grp_sigma, const std::int32_t* grp_items, int ngroups,
                            const double* partial, int P, int m, double* yhat) {
  if (ngroups == 0) return;
  k_coupling_reduce<<<dim3(static_cast<unsigned>(ngroups), static_cast<unsigned>(m)), 256, 0, st>>>(
      grp_sigma, grp_items, partial, P, m, yhat);
}

void launch_down(cudaStream_t st, const std::int32_t* nodes, int cnt, const std::int32_t* parent, const double* E,
                 int d, int ps, int P, int m, double* yhat) {
  if (cnt == 0) return;
  const size_t smem = (d * ps * ps + 3 * P) * sizeof(double);
  if (smem > 48 * 1024) smem_attr(reinterpret_cast<const void*>(k_down2), static_cast<int>(smem), false);
  k_down2<<<dim3(cnt, m), threads_for(P), smem, st>>>(nodes, parent, E, d, ps, P, m, yhat);
}
void launch_leaf_bwd(cudaStream_t st, const std::int32_t* leaves, int nleaves, const std::int64_t* begin,
                     const std::int32_t* count, const double* U, std::int64_t n, int d, int ps, int P,
                     const double* yhat, int m, std::int64_t row_lo, std::int64_t row_hi, double* yp) {
  if (nleaves == 0) return;
  const size_t smem = (P + 2 * kLeafBwdChunk * (P / ps)) * sizeof(double);
  if (smem > 48 * 1024) smem_attr(reinterpret_cast<const void*>(k_leaf_bwd2), static_cast<int>(smem), false);
  k_leaf_bwd2<<<dim3(nleaves, m), 128, smem, st>>>(leaves, begin, count, U, n, d, ps, P, yhat, m, row_lo, row_hi, yp);
}
void launch_far_h(cudaStream_t st, const FarHItem* items, int item0, int nitems, const std::int32_t* bitem, int b0,
                  int nblocks, const std::int64_t* tbeg, const std::int32_t* tcnt, const std::int32_t* cls,
                  const std::int64_t* s_off, const std::int64_t* t_off, const std::int64_t* p_off,
                  const ClassMeta* meta, const double* S, const double* T, const double* H, const double* xp,
                  double* part, std::int64_t row_lo, std::int64_t row_hi, double* yp) {
  if (nitems == 0 || nblocks == 0) return;
  k_far_h_blocks<<<nblocks, 128, 0, st>>>(items, bitem, tbeg, tcnt, cls, s_off, t_off, p_off, meta, S, T, H, xp, b0,
                                          part);
  k_far_h_reduce<<<nitems, 128, 0, st>>>(items + item0, p_off, part, row_lo, row_hi, yp);
}

}  // namespace dev
}  // namespace phm
