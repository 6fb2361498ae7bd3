// sm_100a kernels of the online stage (instantiate + MVM) and the offline
// snapshot generator. Numbering follows SURVEY.md §2.1:
//   K11   k_snapshot          near-field kernel snapshots at theta nodes (offline)
//   K1+K6 k_near_tma          snapshot instantiate fused with the near GEMV (TMA ring)
//   K1    k_inst_flat         D = sum_k w_k S_k  (snapshot mode, flat HBM stream)
//   K1    k_inst_flat_batch   the same for B thetas per snapshot pass (sweeps)
//   K1    k_inst_tiles        D_b = G1_b w_b     (TT near mode, per-block tiles)
//   --    k_near_w            w_b = prod_i contract(G_{b,i+1}, v_i) (TT mode)
//   K2    k_class_inst        H_k(theta) and C_k = L_k H_k R_k^T per class
//   K10   k_gather/k_scatter  tree-order permutation of x / y
//   K3    k_leaf_fwd          xhat_sigma = U_sigma^T x_sigma
//   K4    k_up2               xhat_parent += E^T xhat_child (one launch per level)
//   K5    k_coupling_mma      yhat_sigma += C_k xhat_tau (grouped fp64 DMMA) + reduce
//   K6    k_near_tma_apply    two-sided near GEMV over TMA (apply alone)
//   K6    k_near_mvm_symcsr   the same with plain loads (leaves > 128 rows)
//   --    k_near_gather       fixed-order sum of the near partial segments
//   K7    k_down2/k_leaf_bwd2 yhat_child += E yhat_parent; y += U yhat
//   K8    k_far_h             y_sigma += S_b H_k T_b^T x_tau (H form, per level)
//   K9    k_near_mrhs         Y_sigma += D_b X_tau on fp64 DMMA (m >= 4 RHS)
//   --    k_exact_rows        exact probe rows for estimate_error
#pragma once

#include <cstdint>

namespace phm {
namespace dev {

constexpr int kMaxThetaDim = 3;
constexpr int kMaxThetaNodes = 32;

struct ThetaV {  // parametric vectors v_k(theta_k) (farfield.cpp:16-29), by value
  double v[kMaxThetaDim][kMaxThetaNodes];
  int p[kMaxThetaDim];
  int dt;
};

struct BlockGeom {  // one near block in tree order
  std::int64_t s_begin, t_begin;
  std::int32_t s_n, t_n;
};

struct SnapTile {  // K11 tile: entries [e0, e0+len) of block blk
  std::int64_t out_off;  // output offset of entry e0 in slab 0
  std::int64_t stride;   // slab stride
  std::int32_t e0, len, blk, pad;
};

struct InstTile {  // K1 (TT mode) tile, len even, offsets even
  std::int64_t d_off, g_off, g_stride, w_off;
  std::int32_t len, R;
};

struct NearW {  // theta-core chain of one TT near block
  std::int64_t core_off;  // into near_cores
  std::int64_t w_off;     // into w
  std::int32_t dims_off;  // into near_core_dims (3 ints per core)
  std::int32_t ncores;    // number of theta cores (= d_theta)
  std::int32_t R;
  std::int32_t pad;
};

// The theta-dependent inputs of an instantiate, in device memory so the
// launch sequence is the same for every theta (CUDA graphs): the parametric
// vectors, the snapshot-shape subset of them and the amplitude factor.
struct ThetaParams {
  ThetaV tv;
  ThetaV shape;
  double amp;
};

// K1 output table, passed by value (no host staging): per theta of the call,
// its snapshot weights w (R doubles, device) and its D (device).
struct InstPtrs {
  const double* w[16];
  double* d[16];
};

struct ClassMeta {
  std::int64_t mid_off, l_off, r_off, h_off, c_off;
  std::int32_t rl, rr, dims_off, pad;  // dims_off into class_mid_dims (3 per theta core)
};

// K5 (grouped DMMA): a group is up to 32 sigma nodes of one level with the
// same child parity (so their far partners share translation classes); an
// item is a contiguous range of that group's classes. cls_tau[e*32 + slot] is
// the tau node of (sigma slot, class item_cls[e]) or -1.
// Chunk of a leaf for the split leaf forward pass (K3): points [p0, p0 + len)
// of `leaf`, partial x-hat at chunk ordinal `slot` (m x P doubles each).
constexpr int kLeafChunk = 256;
struct LeafChunk {
  std::int32_t leaf, p0, len, pad;
  std::int64_t slot;
};

// C_k with P = 64 is stored in DMMA fragment order: element (i, j) (row i of
// sigma's basis, column j of tau's) at cfrag64(i, j), so that the coupling's
// m16n8k4 A fragment of (k-step s, m-tile mt) is 32 lanes x 16 contiguous
// bytes -- one coalesced 16-byte load per lane, and a contiguous 8 KB per
// quarter of k-steps.
__host__ __device__ inline int cfrag64(int i, int j) {
  const int mt = i >> 4, r = i & 15, s = j >> 2, t0 = j & 3;
  return (((s * 4 + mt) * 32 + ((r & 7) << 2) + t0) << 1) + (r >> 3);
}

constexpr int kGroupSlots = 32;
struct CouplingItem {
  std::int32_t group, e_begin, e_end, pad;
};

// CSR form of the symmetric near GEMV: one item per (leaf sigma, 128-row
// chunk) streaming all stored blocks owned by sigma; row sums accumulate
// across those blocks, column sums are written per block.
struct SymRowItem {
  std::int64_t x_row0, p_row;
  std::int32_t rows, ld, i0, bbeg, bend, pad;
};
// Owned blocks per near item at most (the TMA passes cache an item's block
// list in shared memory; device.cu splits longer runs). Small, so that a
// coupling CTA fits beside two near CTAs on one SM.
constexpr int kTmaMaxBlocks = 32;
struct SymBlock {
  std::int64_t d_off, x_col0, p_col;  // p_col < 0: diagonal block
  std::int32_t ncol, pad;
};
struct GatherSeg {  // contribution to rows [base, base + len) of one leaf
  std::int64_t poff;
  std::int32_t base, len;
};

// K9 (multi-RHS near field on DMMA): one item per (leaf sigma, 64-row
// chunk); its near blocks are nb_* entries [bbeg, bend) (tau begin, n_tau,
// stored offset, stored leading dimension, transposed flag).
struct MrhsItem {
  std::int64_t row0;
  std::int32_t rows, i0, bbeg, bend;
};

struct FarHItem {  // K8 work item: one sigma node at one level
  std::int64_t row0;
  std::int32_t rows, bbeg, bend, pad;
};

}  // namespace dev
}  // namespace phm
