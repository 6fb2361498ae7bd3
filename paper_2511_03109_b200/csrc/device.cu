// Device layer: flattens a HostMatrix into HBM-resident arrays once
// (upload), generates near-field snapshots on the GPU (K11), and runs the
// online stage (instantiate, apply) as a sequence of sm_100a kernels on one
// stream. No CPU fallback: every online computation is a kernel launch.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "comm.hpp"
#include "engine.hpp"
#include "kernels.cuh"

#define CK(x)                                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess)                                                                            \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
  } while (0)

namespace phm {
namespace dev {
void launch_snapshot(cudaStream_t, const SnapTile*, std::int64_t, const BlockGeom*, const double*, std::int64_t, int,
                     int, int, const double*, double, double*);
void launch_inst_flat(cudaStream_t, const double*, std::int64_t, int, const double*, double*);
bool launch_inst_flat_batch(cudaStream_t, const double*, std::int64_t, int, int, const InstPtrs&);
bool launch_inst_tma(cudaStream_t, const double*, std::int64_t, int, int, const InstPtrs&, int per_sm = 2);
void launch_inst_tiles(cudaStream_t, const InstTile*, std::int64_t, const double*, const double*, double*);
void launch_near_w(cudaStream_t, const NearW*, std::int64_t, const double*, const std::int32_t*, const ThetaParams*,
                   double*);
void launch_set_vec(cudaStream_t, double*, int, const ThetaParams*);
void launch_put_theta(cudaStream_t, const ThetaParams&, ThetaParams*);
void launch_stamp(cudaStream_t, unsigned long long*, int);
void launch_zero(cudaStream_t, double*, std::int64_t);
void launch_class_inst(cudaStream_t, const ClassMeta*, int, const double*, const std::int32_t*, const double*,
                       const double*, const ThetaParams*, int, bool, int, int, int, int, int, int, double*, double*);
void launch_gather(cudaStream_t, const double*, const std::int32_t*, std::int64_t, std::int64_t, double*);
void launch_scatter(cudaStream_t, const double*, const std::int32_t*, std::int64_t, std::int64_t, double*);
void launch_leaf_fwd_chunks(cudaStream_t, const LeafChunk*, int, const std::int32_t*, const std::int64_t*,
                            const std::int32_t*, int, const std::int64_t*, const std::int32_t*, const double*,
                            std::int64_t, int, int, const double*, int, double*, double*);
void launch_leaf_fwd(cudaStream_t, const std::int32_t*, int, const std::int64_t*, const std::int32_t*, const double*,
                     std::int64_t, int, int, int, const double*, int, double*);
void launch_up(cudaStream_t, const std::int32_t*, int, const std::int32_t*, const std::int32_t*, const double*, int,
               int, int, int, double*);
void launch_coupling(cudaStream_t, const std::int32_t*, int, const std::int64_t*, const std::int32_t*,
                     const std::int32_t*, const double*, int, int, const double*, double*);
bool coupling_mma_supported(int P);
int coupling_beside_near(int R, int P);
void launch_coupling_mma(cudaStream_t, const CouplingItem*, const std::int32_t*, int, const std::int32_t*,
                         const std::uint8_t*,
                         const std::int32_t*, const double*, int, const double*, int, double*, int);
void launch_coupling_reduce(cudaStream_t, const std::int32_t*, const std::int32_t*, int, const double*, int, int,
                            double*);
void launch_near_tma_apply(cudaStream_t, const SymRowItem*, int, const SymBlock*, const double*, const double*,
                           double*, int*);
void launch_near_mrhs2(cudaStream_t, const SymRowItem*, int, const SymBlock*, const double*, const double*,
                       std::int64_t, int, std::int64_t, double*);
void launch_near_mrhs3(cudaStream_t, const SymRowItem*, int, const SymBlock*, const double*, const double*,
                       std::int64_t, int, std::int64_t, double*, int);
void launch_near_mvm_symcsr(cudaStream_t, const SymRowItem*, int, const SymBlock*, const double*, const double*,
                            double*);
bool launch_near_inst_tma(cudaStream_t, const SymRowItem*, int, const SymBlock*, const double*, std::int64_t, int,
                          const double*, double*, const double*, double*);
void launch_exact_rows(cudaStream_t, const std::int64_t*, int, const double*, std::int64_t, int, int, const double*,
                       double, const double*, double*);
void launch_near_mrhs(cudaStream_t, const MrhsItem*, int, const std::int64_t*, const std::int32_t*,
                      const std::int64_t*, const std::int32_t*, const std::int32_t*, const double*, const double*,
                      std::int64_t, int, double*);
void launch_near_gather(cudaStream_t, int, const std::int64_t*, const std::int32_t*, const std::int32_t*,
                        const GatherSeg*, const double*, std::int64_t, std::int64_t, int, double*);
void launch_down(cudaStream_t, const std::int32_t*, int, const std::int32_t*, const double*, int, int, int, int,
                 double*);
void launch_leaf_bwd(cudaStream_t, const std::int32_t*, int, const std::int64_t*, const std::int32_t*, const double*,
                     std::int64_t, int, int, int, const double*, int, std::int64_t, std::int64_t, double*);
void launch_far_h(cudaStream_t, const FarHItem*, int, int, const std::int32_t*, int, int, const std::int64_t*,
                  const std::int32_t*, const std::int32_t*, const std::int64_t*, const std::int64_t*,
                  const std::int64_t*, const ClassMeta*, const double*, const double*, const double*, const double*,
                  double*, std::int64_t, std::int64_t, double*);
}  // namespace dev

// ---------------------------------------------------------------- buffers
namespace {

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b) {
    release();
    if (b == 0) return;
    CK(cudaMalloc(&p, b));
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <typename T>
void upload(DBuf& buf, const std::vector<T>& v, cudaStream_t st) {
  buf.alloc(v.size() * sizeof(T));
  if (!v.empty()) {
    CK(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // host vector may die after return
  }
}

}  // namespace

// ---------------------------------------------------------------- context
// NVTX range for the lifetime of the object (header-only NVTX 3; a no-op
// unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Context {
  int device = 0;
  std::recursive_mutex exec_mu;  // see DevMatrix::exec_mu()
  int sms = 148;  // multiprocessors of the device
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  bool timing = false;
  std::int64_t launches = 0;
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<double, std::int64_t>> totals;
  ~Context() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (aux_ev) cudaEventDestroy(aux_ev);
    if (leaf_ev) cudaEventDestroy(leaf_ev);
    if (up_ev) cudaEventDestroy(up_ev);
    if (stamps) cudaFree(stamps);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (own) cudaStreamDestroy(own);
  }
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // Brackets one kernel launch with events on the launching stream.
  template <typename F>
  void run(const char* name, F&& f) {
    run_on(stream, name, std::forward<F>(f));
  }
  template <typename F>
  void run_on(cudaStream_t s, const char* name, F&& f) {
    ++launches;
    NvtxRange nvtx(name);  // host-side launch range (nsys / ncu --nvtx)
    if (!timing) {
      f();
      CK(cudaGetLastError());
      keep_priority(s);
      return;
    }
    Rec r{name, ev(), ev()};
    CK(cudaEventRecord(r.a, s));
    f();
    CK(cudaGetLastError());
    CK(cudaEventRecord(r.b, s));
    recs.push_back(r);
  }
  // Under stream capture, give the kernel node just captured on s the
  // priority of s: graph nodes otherwise carry no priority, and the far
  // chain would queue behind the near pass's CTAs instead of taking SM
  // slots beside it (graphs are instantiated with UseNodePriority).
  static void keep_priority(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd));
    if (cs != cudaStreamCaptureStatusActive) return;
    int prio = 0;
    CK(cudaStreamGetPriority(s, &prio));
    for (size_t i = 0; i < nd; ++i) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(deps[i], &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeAttrValue v{};
      v.priority = prio;
      CK(cudaGraphKernelNodeSetAttribute(deps[i], cudaKernelNodeAttributePriority, &v));
    }
  }
  // PHM_STAMPS=1: device-clock stamps at fixed points of the fused step,
  // printed to stderr after each step (schedule diagnostics only)
  unsigned long long* stamps = nullptr;
  static bool stamps_on() {
    static const bool on = [] {
      const char* e = std::getenv("PHM_STAMPS");
      return e && std::atoi(e) == 1;
    }();
    return on;
  }
  void stamp(cudaStream_t s, int id) {
    if (!stamps_on()) return;
    if (!stamps) CK(cudaMallocManaged(&stamps, 16 * sizeof(unsigned long long)));
    dev::launch_stamp(s, stamps, id);
    keep_priority(s);
  }
  void print_stamps() {
    if (!stamps_on() || !stamps) return;
    CK(cudaDeviceSynchronize());
    std::fprintf(stderr, "stamps(us):");
    for (int i = 1; i < 16; ++i)
      if (stamps[i] >= stamps[0]) std::fprintf(stderr, " %d:%.1f", i, (stamps[i] - stamps[0]) * 1e-3);
    std::fprintf(stderr, "\n");
  }
  // Second stream for the H^2 far-field chain, which overlaps the near-field
  // GEMV (compute-bound DMMA next to an HBM stream); fork/join by events.
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, aux_ev = nullptr;
  // Third stream (same priority as side): in apply, the transfer pass and the
  // upper-level coupling run here while the leaf-level coupling, which needs
  // only the leaf x-hat, already runs on side (far_chain).
  cudaStream_t side2 = nullptr;
  cudaEvent_t leaf_ev = nullptr, up_ev = nullptr;
  void fork() {
    CK(cudaEventRecord(fork_ev, stream));
    CK(cudaStreamWaitEvent(side, fork_ev, 0));
  }
  void join() {
    CK(cudaEventRecord(join_ev, side));
    CK(cudaStreamWaitEvent(stream, join_ev, 0));
  }
  void flush_timers() {
    if (recs.empty()) return;
    CK(cudaStreamSynchronize(stream));
    for (auto& r : recs) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      auto& t = totals[r.name];
      t.first += ms;
      t.second += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    recs.clear();
  }
};

std::shared_ptr<Context> context_create(int device) {
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) throw std::runtime_error("no such CUDA device");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) throw std::runtime_error("phmat_b200 is built for sm_100a (B200); found sm_" +
                                                 std::to_string(prop.major) + std::to_string(prop.minor));
  auto ctx = std::make_shared<Context>();
  ctx->device = device;
  ctx->sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
  {
    // the side stream carries the compute-bound far chain that runs beside
    // the HBM-bound near pass; with the higher priority its CTAs take SM
    // slots as soon as near-pass CTAs retire
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* e = std::getenv("PHM_SIDE_PRIORITY");
    const bool prio = !(e && std::atoi(e) == 0);
    CK(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, prio ? hi : lo));
    CK(cudaStreamCreateWithPriority(&ctx->side2, cudaStreamNonBlocking, prio ? hi : lo));
  }
  CK(cudaEventCreateWithFlags(&ctx->leaf_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->up_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->aux_ev, cudaEventDisableTiming));
  ctx->stream = ctx->own;
  return ctx;
}
void context_set_stream(Context& ctx, void* s) {
  std::lock_guard<std::recursive_mutex> lk(ctx.exec_mu);
  ctx.stream = s ? static_cast<cudaStream_t>(s) : ctx.own;
}
void* context_stream(Context& ctx) { return ctx.stream; }
void context_sync(Context& ctx) { CK(cudaStreamSynchronize(ctx.stream)); }
void context_enable_timing(Context& ctx, bool on) {
  std::lock_guard<std::recursive_mutex> lk(ctx.exec_mu);
  ctx.timing = on;
}
void context_timer(Context& ctx, const std::string& name, double* ms, std::int64_t* count) {
  std::lock_guard<std::recursive_mutex> lk(ctx.exec_mu);
  ctx.flush_timers();
  auto it = ctx.totals.find(name);
  *ms = it == ctx.totals.end() ? 0.0 : it->second.first;
  *count = it == ctx.totals.end() ? 0 : it->second.second;
}
void context_reset_timers(Context& ctx) {
  std::lock_guard<std::recursive_mutex> lk(ctx.exec_mu);
  ctx.flush_timers();
  ctx.totals.clear();
}
std::int64_t context_launches(Context& ctx) { return ctx.launches; }
int context_device(const Context& ctx) { return ctx.device; }

// ----------------------------------------------------------------- matrix
struct DevMatrix {
  std::shared_ptr<Context> ctx;
  std::unique_ptr<HostMatrix> hm;
  int d = 0, ps = 0, P = 0, dt = 0, nnodes = 0;
  Index n = 0;
  bool h2 = true;
  NearMode mode = NearMode::TT;

  // structure
  DBuf perm, pts, node_begin, node_count, node_first_child, node_parent;
  // near field
  std::vector<std::int64_t> near_doff;  // per global near block, -1 if not local
  std::vector<std::int64_t> near_goff;  // start of G1 / snapshot slab 0
  std::vector<std::int64_t> near_gstride;
  std::vector<int> near_R;
  std::int64_t E = 0;    // padded local near entries (D length)
  std::int64_t E_raw = 0, E_rank = 0;
  int R_snap = 0;        // snapshot mode: shared rank
  double snap_amp_nodes_unused = 0;
  DBuf G;                // near payload
  DBuf snap_tiles, geo;  // K11 (snapshot / direct)
  std::int64_t n_snap_tiles = 0;
  DBuf inst_tiles, near_w_meta, near_cores, near_core_dims;
  std::int64_t n_inst_tiles = 0, n_near_local = 0, w_len = 0;
  // symmetric near storage (sigma <= tau blocks only)
  bool sym = false;
  bool sharded = false;          // a row shard (rows [row_begin, row_end) of y)
  std::vector<char> near_trans;  // block stored as the transpose of its partner
  std::int64_t E_logical = 0;    // sum of n_sigma n_tau over local near blocks
  DBuf sym_items, sym_blocks, g_row0, g_rows, g_sbeg, g_segs, sym_part;
  std::int64_t sym_pstride = 0;  // partial segments per right-hand side
  DBuf sym_part_m;               // two-sided K9: sym_pstride x m partials
  int n_sym_items = 0, n_gather_leaves = 0;
  int k9_dense_rows = 0;  // tallest whole-leaf item, 0 if some item is a row slice (K9 stage size)
  bool near_tma = false;  // every item spans its whole leaf: TMA near pass
  DBuf theta_dev;         // dev::ThetaParams of the instantiate in flight
  DBuf work_ctr;          // persistent near kernels' item counter
  // K9 multi-RHS near field (DMMA), CSR by sigma over stored blocks
  DBuf k9_items, k9_tb, k9_tn, k9_doff, k9_ld, k9_tr;
  int n_k9_items = 0;
  // far field
  int ncls = 0;
  // classes the class stage instantiates: all of them, or on a row shard
  // only those some local far block uses (the rest are never read)
  DBuf cmeta_run;
  int ncls_run = 0;
  std::vector<char> cls_run;  // per class: instantiated by this matrix's class stage
  std::vector<dev::ClassMeta> cmeta_h;
  DBuf cmeta, class_mid, class_mid_dims, class_L, class_R;
  bool baseline = false;  // fixed far field (H-ACA / H^2-HCA at one theta)
  DBuf fixed_H, fixed_C;
  std::int64_t H_len = 0, C_len = 0;
  int capA = 0, capB = 0, capT = 0, capL = 0, capR = 0;  // capR > 0: k_class_inst_pf
  // H^2 coupling CSR by sigma node
  DBuf cp_sig, cp_beg, cp_tau, cp_cls;
  int n_cp_sig = 0;
  // H^2 coupling, grouped DMMA path (P in {16, 32, 64, 128})
  bool cp_mma = false;
  DBuf cg_items, cg_order, cg_cls, cg_tiles, cg_tau, cg_grp_sigma, cg_grp_items, cg_partial;
  int n_cg_items = 0, n_cg_groups = 0;
  // cg_order lists the items of levels above the leaf level first: the first
  // cg_n_upper entries need the transfer pass, the rest only the leaf x-hat
  // (-1: order not by level)
  int cg_n_upper = -1;
  // lowest level (nearest the root) holding far blocks, over ALL ranks' blocks
  // (class keys): x-hat / y-hat of the levels above it are never used
  int far_min_level = 0;
  // H form far CSR by level
  DBuf fh_items, fh_tb, fh_tn, fh_cls, fh_soff, fh_toff, fh_S, fh_T, fh_bitem, fh_poff, fh_part;
  std::vector<dev::FarHItem> fh_items_h;
  std::vector<std::pair<int, int>> fh_level_range;  // [item begin, item end) per level
  // basis
  DBuf U, Etr;
  DBuf leaves_all, leaves_local;
  int n_leaves_all = 0, n_leaves_local = 0;
  // split leaf forward pass (K3, m >= 4): per list (0 all, 1 local) the leaves
  // of at most kLeafChunk points, the chunks of the bigger ones and their
  // ordered reduction
  struct LeafPlan {
    DBuf small, chunks, red_leaf, red_slot, red_n;
    int n_small = 0, n_chunks = 0, n_red = 0;
  } lf[2];
  DBuf lf_part;
  std::vector<std::pair<int, int>> up_range, down_range;  // per level into level_nodes arrays
  DBuf up_nodes, down_nodes;
  // sharded forward pass with an x-hat exchange: upward lists restricted to
  // nodes that hold local rows (their x-hat is this rank's partial sum)
  std::vector<std::pair<int, int>> upl_range;
  DBuf upl_nodes;
  // apply workspace
  DBuf xp, yp, xhat, yhat, xdev, ydev;
  Index ws_m = 0;
  std::int64_t ws_gen = 0;  // bumped whenever the workspace is reallocated
  // pooled instance buffers
  std::vector<DBuf> pool_D;
  std::mutex mu;
  // Serialises the public entry points: a matrix's workspace (xp, yp,
  // x-hat, ...) is its own, but its stream, side stream, fork / join events,
  // launch counter and timer records live on the Context that every matrix
  // built on it shares, so the lock is the Context's (own_mu for host-only
  // matrices, which have none).
  std::recursive_mutex own_mu;
  std::recursive_mutex& exec_mu() { return ctx ? ctx->exec_mu : own_mu; }
  std::int64_t device_bytes = 0;

  cudaStream_t st() const { return ctx->stream; }
};

struct DevInstance {
  std::shared_ptr<DevMatrix> M;
  std::vector<double> theta;
  DBuf D, H, C, w;
  // apply_tree_order captured as a CUDA graph per RHS count (the launch
  // sequence is fixed for an instance: the buffers never move); tagged with
  // the matrix's workspace generation, which changes when the workspace is
  // reallocated.
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    std::int64_t ws_gen = -1;
    std::int64_t launches = 0;  // kernels in the graph (for the launch count)
    bool seen = false;          // the first call runs directly (lazy buffers)
    std::uint64_t last_use = 0;
  };
  // LRU bound: the fused step's graphs are keyed by the caller's x pointer,
  // which an HPO loop over a caching allocator may vary without end
  static constexpr std::size_t kMaxGraphs = 16;
  std::uint64_t graph_tick = 0;
  // key: (launch sequence, input pointer it reads, RHS count)
  std::map<std::tuple<int, const void*, Index>, Graph> graphs;
  ~DevInstance() {
    for (auto& g : graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    if (M && D.p) {
      std::lock_guard<std::mutex> lk(M->mu);
      M->pool_D.push_back(std::move(D));
    }
  }
};

namespace {

dev::ThetaV make_theta_v(const std::vector<std::vector<double>>& v) {
  dev::ThetaV tv{};
  tv.dt = static_cast<int>(v.size());
  PHM_CHECK(tv.dt <= dev::kMaxThetaDim, "too many theta dimensions");
  for (int k = 0; k < tv.dt; ++k) {
    PHM_CHECK(static_cast<int>(v[k].size()) <= dev::kMaxThetaNodes, "p_theta above 32 unsupported on device");
    tv.p[k] = static_cast<int>(v[k].size());
    for (size_t j = 0; j < v[k].size(); ++j) tv.v[k][j] = v[k][j];
  }
  return tv;
}

std::int64_t pad4(std::int64_t x) { return (x + 3) & ~std::int64_t(3); }

// Right-hand-side count from which the near field switches from the HBM GEMV
// (K6, one pass per vector) to the DMMA block kernel (K9, one pass for all).
constexpr Index kMrhsMin = 4;

void ensure_workspace(DevMatrix& M, Index m) {
  if (M.ws_m >= m) return;
  // +4: the TMA panel copies of K9 may read one double past a column
  M.xp.alloc(sizeof(double) * (M.n * m + 4));
  M.yp.alloc(sizeof(double) * M.n * m);
  M.xdev.alloc(sizeof(double) * M.n * m);
  M.ydev.alloc(sizeof(double) * M.n * m);
  if (M.h2) {
    M.xhat.alloc(sizeof(double) * M.nnodes * M.P * m);
    M.yhat.alloc(sizeof(double) * M.nnodes * M.P * m);
  }
  M.ws_m = m;
  ++M.ws_gen;
}

}  // namespace

const HostMatrix& matrix_host(const DevMatrix& m) { return *m.hm; }
bool matrix_on_device(const DevMatrix& m) { return m.ctx != nullptr; }

std::shared_ptr<DevMatrix> matrix_build_host_only(const double* points, Index n, int d, const Config& cfg) {
  auto M = std::make_shared<DevMatrix>();
  M->hm = build_host(points, n, d, cfg);
  M->n = n;
  M->d = d;
  return M;
}
std::int64_t matrix_device_bytes(const DevMatrix& m) { return m.device_bytes; }
std::int64_t matrix_near_rank(const DevMatrix& m, Index b) {
  if (!m.ctx) throw std::logic_error("host-only matrix has no device near payload");
  if (b < 0 || b >= static_cast<Index>(m.near_R.size())) throw std::out_of_range("near block index");
  return m.near_R[b];
}
std::int64_t matrix_near_elems(const DevMatrix& m, int kind) {
  return kind == 0 ? m.E_logical : (kind == 1 ? m.E_raw : m.E_rank);
}

void matrix_near_column(const DevMatrix& m, Index b, Index kap, double* out) {
  if (!m.ctx) throw std::logic_error("host-only matrix has no device near payload");
  if (b < 0 || b >= static_cast<Index>(m.near_doff.size()) || m.near_doff[b] < 0)
    throw std::out_of_range("near block not resident");
  if (kap < 0 || kap >= m.near_R[b]) throw std::out_of_range("near column index");
  const HostMatrix& H = *m.hm;
  const Block blk = H.blocks.near[b];
  const Index ns = H.tree->nodes[blk.sigma].count, nt = H.tree->nodes[blk.tau].count;
  CK(cudaSetDevice(m.ctx->device));
  std::vector<double> tmp(static_cast<size_t>(ns * nt));
  CK(cudaMemcpyAsync(tmp.data(), m.G.as<double>() + m.near_goff[b] + kap * m.near_gstride[b], ns * nt * sizeof(double),
                     cudaMemcpyDeviceToHost, m.st()));
  CK(cudaStreamSynchronize(m.st()));
  for (Index j = 0; j < nt; ++j)
    for (Index i = 0; i < ns; ++i) out[i + j * ns] = m.near_trans[b] ? tmp[j + i * nt] : tmp[i + j * ns];
}

std::shared_ptr<DevMatrix> matrix_upload(std::shared_ptr<Context> ctx, std::unique_ptr<HostMatrix> hm);

std::shared_ptr<DevMatrix> matrix_build(std::shared_ptr<Context> ctx, const double* points, Index n, int d,
                                        const Config& cfg) {
  CK(cudaSetDevice(ctx->device));
  if (cfg.spec.family == kMatern && cfg.near_mode == NearMode::Direct)
    throw std::invalid_argument("direct near mode needs a closed-form kernel family on the GPU");
  return matrix_upload(ctx, build_host(points, n, d, cfg));
}

void matrix_save(const DevMatrix& M, const std::string& path) {
  const HostMatrix& H = *M.hm;
  const Tree& T = *H.tree;
  write_artifact(H, path, [&](Index b) {
    if (H.cfg.near_mode == NearMode::TT) return H.near_tt[b];
    // Snapshot mode: the full-rank NearBlockTT (G1 = the R snapshot columns,
    // identity theta cores), SURVEY.md §8(a).
    const Block blk = H.blocks.near[b];
    const Index N = T.nodes[blk.sigma].count * T.nodes[blk.tau].count;
    const Index R = matrix_near_rank(M, b);
    TTTensor tt;
    TTCore g1 = TTCore::zeros(1, N, R);
    for (Index k = 0; k < R; ++k) matrix_near_column(M, b, k, g1.data.data() + k * N);
    tt.cores.push_back(std::move(g1));
    Index rin = R;
    for (const Grid1D& g : H.grids.grids) {
      const Index p = g.p;
      TTCore c = TTCore::zeros(rin, p, rin / p);
      for (Index rest = 0; rest < rin / p; ++rest)
        for (Index j = 0; j < p; ++j) c.data[(j + p * rest) + j * c.r0 + rest * c.r0 * c.m] = 1.0;
      tt.cores.push_back(std::move(c));
      rin /= p;
    }
    return tt;
  });
}

std::shared_ptr<DevMatrix> matrix_load_host_only(const std::string& path, int threads) {
  auto M = std::make_shared<DevMatrix>();
  M->hm = read_artifact(path, threads);
  M->n = M->hm->n();
  M->d = M->hm->d();
  return M;
}

std::shared_ptr<DevMatrix> matrix_load(std::shared_ptr<Context> ctx, const std::string& path, int threads) {
  CK(cudaSetDevice(ctx->device));
  return matrix_upload(ctx, read_artifact(path, threads));
}

std::shared_ptr<DevMatrix> matrix_upload(std::shared_ptr<Context> ctx, std::unique_ptr<HostMatrix> hm) {
  CK(cudaSetDevice(ctx->device));
  auto Mp = std::make_shared<DevMatrix>();
  DevMatrix& M = *Mp;
  M.ctx = ctx;
  M.hm = std::move(hm);
  const Config& cfg = M.hm->cfg;
  const Index n = M.hm->n();
  const int d = M.hm->d();
  if (cfg.spec.family == kMatern && cfg.near_mode == NearMode::Direct)
    throw std::invalid_argument("direct near mode needs a closed-form kernel family on the GPU");
  const auto t_up = std::chrono::steady_clock::now();
  HostMatrix& H = *M.hm;
  const Tree& T = *H.tree;
  cudaStream_t st = ctx->stream;
  M.d = d;
  M.n = n;
  M.ps = cfg.p_s;
  M.P = static_cast<int>(H.P());
  M.dt = H.grids.d_theta();
  M.nnodes = static_cast<int>(T.nodes.size());
  M.h2 = cfg.format == Format::H2;
  M.mode = cfg.near_mode;
  if (M.h2) PHM_CHECK(M.ps <= 16 && M.P <= 1024, "H2 on device needs p_s <= 16 and p_s^d <= 1024");

  // --- structure
  {
    upload(M.perm, T.perm, st);
    std::vector<double> soa(static_cast<size_t>(d * n));
    for (int k = 0; k < d; ++k)
      for (Index p = 0; p < n; ++p) soa[k * n + p] = T.coord(T.perm[p], k);
    upload(M.pts, soa, st);
    std::vector<std::int64_t> nb(M.nnodes);
    std::vector<std::int32_t> nc(M.nnodes), fc(M.nnodes), par(M.nnodes);
    for (int i = 0; i < M.nnodes; ++i) {
      nb[i] = T.nodes[i].begin;
      nc[i] = static_cast<std::int32_t>(T.nodes[i].count);
      fc[i] = T.nodes[i].first_child;
      par[i] = T.nodes[i].parent;
    }
    upload(M.node_begin, nb, st);
    upload(M.node_count, nc, st);
    upload(M.node_first_child, fc, st);
    upload(M.node_parent, par, st);
  }

  // --- near field layout
  const Index nnear = static_cast<Index>(H.blocks.near.size());
  M.near_doff.assign(nnear, -1);
  M.near_goff.assign(nnear, -1);
  M.near_gstride.assign(nnear, 0);
  M.near_R.assign(nnear, 0);
  int Rshape = 1;  // snapshot rank: product of non-amplitude theta grids
  for (int k = 0; k < cfg.spec.shape_params(); ++k) Rshape *= H.grids.grids[k].p;
  // Symmetric near storage: the near relation is symmetric and every kernel
  // family is radial, so with snapshots (or direct evaluation) D_{tau,sigma}
  // equals D_{sigma,tau}^T bit for bit (the squared distance accumulates the
  // same rounded squares). Only blocks with sigma <= tau are stored.
  // On a row shard the rank stores the pairs whose owner leaf it holds; the
  // transposed products land on rows of other ranks, so a sharded apply
  // yields a full-length partial y that the ranks sum (all-reduce).
  M.sym = M.mode == NearMode::Snapshot && cfg.symmetric_near;
  M.sharded = H.row_begin != 0 || H.row_end != n;
  M.near_trans.assign(nnear, 0);
  std::vector<Index> canon(nnear);
  for (Index b = 0; b < nnear; ++b) canon[b] = b;
  if (M.sym) {
    std::unordered_map<std::uint64_t, Index> where;
    auto key = [](int s, int t) { return (static_cast<std::uint64_t>(s) << 32) | static_cast<std::uint32_t>(t); };
    for (Index b = 0; b < nnear; ++b) where[key(H.blocks.near[b].sigma, H.blocks.near[b].tau)] = b;
    // Owner of the pair {a, b}, a < b: a when a + b is even, b otherwise.
    // Alternating by parity gives every leaf about half of its partners
    // (a plain sigma < tau rule would give the first leaves all of them).
    for (Index b = 0; b < nnear; ++b) {
      const Block blk = H.blocks.near[b];
      if (blk.sigma == blk.tau) continue;
      const bool owner = (blk.sigma < blk.tau) == (((blk.sigma + blk.tau) & 1) == 0);
      if (!owner) {
        canon[b] = where.at(key(blk.tau, blk.sigma));
        M.near_trans[b] = 1;
      }
    }
  }
  {
    std::int64_t off = 0;
    for (Index b = 0; b < nnear; ++b) {
      if (!H.near_local[b]) continue;
      const Block blk = H.blocks.near[b];
      const std::int64_t N = T.nodes[blk.sigma].count * T.nodes[blk.tau].count;
      M.E_logical += N;
      ++M.n_near_local;
      if (M.near_trans[b]) continue;
      M.near_doff[b] = off;
      off += pad4(N);
      M.E_raw += N;
    }
    for (Index b = 0; b < nnear; ++b)
      if (M.near_trans[b]) M.near_doff[b] = M.near_doff[canon[b]];
    M.E = off;
  }
  std::vector<dev::BlockGeom> geo(nnear);
  for (Index b = 0; b < nnear; ++b) {
    const Block blk = H.blocks.near[b];
    geo[b] = {T.nodes[blk.sigma].begin, T.nodes[blk.tau].begin, static_cast<std::int32_t>(T.nodes[blk.sigma].count),
              static_cast<std::int32_t>(T.nodes[blk.tau].count)};
  }
  if (M.mode == NearMode::Snapshot || M.mode == NearMode::Direct) {
    upload(M.geo, geo, st);
    std::vector<dev::SnapTile> tiles;
    const int kTile = 4096;
    for (Index b = 0; b < nnear; ++b) {
      if (M.near_doff[b] < 0 || M.near_trans[b]) continue;
      const std::int64_t N = static_cast<std::int64_t>(geo[b].s_n) * geo[b].t_n;
      for (std::int64_t e0 = 0; e0 < N; e0 += kTile)
        tiles.push_back({M.near_doff[b] + e0, M.E, static_cast<std::int32_t>(e0),
                         static_cast<std::int32_t>(std::min<std::int64_t>(kTile, N - e0)), static_cast<std::int32_t>(b),
                         0});
    }
    M.n_snap_tiles = static_cast<std::int64_t>(tiles.size());
    upload(M.snap_tiles, tiles, st);
  }
  if (M.mode == NearMode::Snapshot) {
    M.R_snap = Rshape;
    M.E_rank = M.E_raw * (Rshape + 1);
    for (Index b = 0; b < nnear; ++b)
      if (M.near_doff[b] >= 0) {
        M.near_goff[b] = M.near_doff[b];
        M.near_gstride[b] = M.E;
        M.near_R[b] = Rshape;
      }
    M.G.alloc(sizeof(double) * M.E * Rshape);
    CK(cudaMemsetAsync(M.G.p, 0, M.G.bytes, st));
    // theta-node table (kappa -> shape parameters, first grid fastest)
    std::vector<double> tn(3 * Rshape, 1.0);
    for (int kap = 0; kap < Rshape; ++kap) {
      int rem = kap;
      for (int k = 0; k < cfg.spec.shape_params(); ++k) {
        tn[3 * kap + k] = H.grids.grids[k].nodes[rem % H.grids.grids[k].p];
        rem /= H.grids.grids[k].p;
      }
    }
    if (cfg.spec.family == kMatern) {
      // K_nu has no device implementation: evaluate the snapshots on host
      // threads (offline data production, not the online path) and upload.
      KernelSpec shape = cfg.spec;
      shape.amplitude = false;
      std::vector<double> host(static_cast<size_t>(M.E * Rshape), 0.0);
      parallel_for(
          nnear,
          [&](Index b) {
            if (M.near_doff[b] < 0 || M.near_trans[b]) return;
            const auto& g = geo[b];
            for (std::int64_t j = 0; j < g.t_n; ++j)
              for (std::int64_t i = 0; i < g.s_n; ++i) {
                const Index oi = T.perm[g.s_begin + i], oj = T.perm[g.t_begin + j];
                double r2 = 0.0;
                for (int k = 0; k < d; ++k) {
                  const double dl = T.coord(oi, k) - T.coord(oj, k);
                  r2 += dl * dl;
                }
                const double r = std::sqrt(r2);
                for (int kap = 0; kap < Rshape; ++kap)
                  host[kap * M.E + M.near_doff[b] + i + j * g.s_n] = kernel_value(shape, r, &tn[3 * kap]);
              }
          },
          cfg.threads);
      CK(cudaMemcpyAsync(M.G.p, host.data(), M.G.bytes, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    } else {
      DBuf dtn;
      upload(dtn, tn, st);
      ctx->run("snapshot", [&] {
        dev::launch_snapshot(st, M.snap_tiles.as<dev::SnapTile>(), M.n_snap_tiles, M.geo.as<dev::BlockGeom>(),
                             M.pts.as<double>(), n, d, cfg.spec.family, Rshape, dtn.as<double>(), 1.0,
                             M.G.as<double>());
      });
      CK(cudaStreamSynchronize(st));
    }
    H.counters.offline.add(static_cast<std::uint64_t>(M.E_raw) * Rshape);
    H.stats.nf_evals += static_cast<std::uint64_t>(M.E_raw) * Rshape;
  } else if (M.mode == NearMode::TT) {
    // G1_b per block (N_b padded even, column-major), theta cores, w chain
    std::int64_t goff = 0, woff = 0, coff = 0;
    std::vector<dev::InstTile> tiles;
    std::vector<dev::NearW> wm;
    std::vector<std::int32_t> cdims;
    std::vector<double> cores;
    for (Index b = 0; b < nnear; ++b) {
      if (M.near_doff[b] < 0) continue;
      const TTTensor& tt = H.near_tt[b];
      const std::int64_t N = tt.cores[0].m, Np = pad4(N), R = tt.cores[0].r1;
      PHM_CHECK(R <= 256, "near TT rank above 256 unsupported on device");
      M.near_goff[b] = goff;
      M.near_gstride[b] = Np;
      M.near_R[b] = static_cast<int>(R);
      M.E_rank += N * (R + 1);
      const int kTile = 2048;
      for (std::int64_t e0 = 0; e0 < Np; e0 += kTile)
        tiles.push_back({M.near_doff[b] + e0, goff + e0, Np, woff,
                         static_cast<std::int32_t>(std::min<std::int64_t>(kTile, Np - e0)),
                         static_cast<std::int32_t>(R)});
      dev::NearW nw{};
      nw.core_off = coff;
      nw.w_off = woff;
      nw.dims_off = static_cast<std::int32_t>(cdims.size());
      nw.ncores = tt.order() - 1;
      nw.R = static_cast<std::int32_t>(R);
      for (int c = 1; c < tt.order(); ++c) {
        cdims.push_back(static_cast<std::int32_t>(tt.cores[c].r0));
        cdims.push_back(static_cast<std::int32_t>(tt.cores[c].m));
        cdims.push_back(static_cast<std::int32_t>(tt.cores[c].r1));
        cores.insert(cores.end(), tt.cores[c].data.begin(), tt.cores[c].data.end());
        coff += tt.cores[c].size();
      }
      wm.push_back(nw);
      goff += Np * R;
      woff += R;
    }
    M.G.alloc(sizeof(double) * goff);
    {
      std::vector<double> host(static_cast<size_t>(goff), 0.0);
      for (Index b = 0; b < nnear; ++b) {
        if (M.near_doff[b] < 0) continue;
        const TTCore& g1 = H.near_tt[b].cores[0];
        for (Index k = 0; k < g1.r1; ++k)
          std::memcpy(&host[M.near_goff[b] + k * M.near_gstride[b]], &g1.data[k * g1.m], g1.m * sizeof(double));
      }
      if (goff) CK(cudaMemcpyAsync(M.G.p, host.data(), M.G.bytes, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    M.n_inst_tiles = static_cast<std::int64_t>(tiles.size());
    upload(M.inst_tiles, tiles, st);
    upload(M.near_w_meta, wm, st);
    upload(M.near_cores, cores, st);
    upload(M.near_core_dims, cdims, st);
    M.w_len = woff;
  } else {  // Direct
    M.E_rank = M.E_raw;
  }

  {
    // K6, CSR by owner leaf: one item per (leaf, 128-row chunk) over the
    // stored blocks the leaf owns (all of its blocks with full storage);
    // with symmetric storage each stored block also yields the column
    // product for its partner leaf. Partial segments are gathered per leaf
    // in a fixed order.
    std::vector<std::vector<Index>> owned(M.nnodes);
    for (Index b = 0; b < nnear; ++b)
      if (M.near_doff[b] >= 0 && !M.near_trans[b]) owned[H.blocks.near[b].sigma].push_back(b);
    std::vector<dev::SymRowItem> items;
    std::vector<dev::SymBlock> blocks;
    std::vector<std::vector<dev::GatherSeg>> segs_of(M.nnodes);
    std::int64_t poff = 0;
    // Enough items for ~8 waves of two CTAs per SM: a row shard (few leaves)
    // splits each leaf's blocks over several items, so the near pass does
    // not end on a partial wave of long CTAs; the unsharded C3 keeps one
    // item per leaf.
    std::size_t kItemBlocks = dev::kTmaMaxBlocks;
    {
      std::size_t total = 0;
      for (const auto& o : owned) total += o.size();
      const std::size_t target = 8 * 2 * 148;
      static const std::size_t floor_blocks = [] {  // tuning: smallest item run
        const char* e = std::getenv("PHM_ITEM_MIN_BLOCKS");
        const int k = e ? std::atoi(e) : 8;
        return static_cast<std::size_t>(k >= 1 && k <= dev::kTmaMaxBlocks ? k : 8);
      }();
      kItemBlocks = std::min<std::size_t>(dev::kTmaMaxBlocks,
                                          std::max<std::size_t>(floor_blocks, (total + target - 1) / target));
    }
    for (int s = 0; s < M.nnodes; ++s) {
      if (owned[s].empty()) continue;
      const int ns = static_cast<int>(T.nodes[s].count);
      // items: 128-row slices of the leaf x runs of at most kItemBlocks owned
      // blocks (the TMA pass caches an item's block list in shared memory)
      for (int i0 = 0; i0 < ns; i0 += 128)
      for (std::size_t q0 = 0; q0 < owned[s].size(); q0 += kItemBlocks) {
        dev::SymRowItem it{};
        it.x_row0 = T.nodes[s].begin + i0;
        it.rows = std::min(128, ns - i0);
        it.ld = ns;
        it.i0 = i0;
        it.bbeg = static_cast<std::int32_t>(blocks.size());
        for (std::size_t q = q0; q < std::min(owned[s].size(), q0 + kItemBlocks); ++q) {
          const Index b = owned[s][q];
          const int tau = H.blocks.near[b].tau;
          const int nt = static_cast<int>(T.nodes[tau].count);
          dev::SymBlock sb{};
          sb.d_off = M.near_doff[b];
          sb.x_col0 = T.nodes[tau].begin;
          sb.ncol = nt;
          sb.p_col = -1;
          if (M.sym && tau != s) {
            sb.p_col = poff;
            segs_of[tau].push_back({poff, 0, nt});
            poff += nt;
          }
          blocks.push_back(sb);
        }
        it.bend = static_cast<std::int32_t>(blocks.size());
        it.p_row = poff;
        segs_of[s].push_back({poff, i0, it.rows});
        poff += it.rows;
        items.push_back(it);
      }
    }
    // Longest items first (stable): the near passes take items in index
    // order (one CTA per item, or a work counter), so the last wave is made
    // of the shortest items instead of whichever leaves come last in tree
    // order. Each item writes fixed partial segments: the order changes no
    // result.
    static const bool lpt = [] {
      const char* e = std::getenv("PHM_ITEM_ORDER");
      return !(e && std::atoi(e) == 0);
    }();
    if (lpt) {
      auto work = [&](const dev::SymRowItem& it) {
        std::int64_t w = 0;
        for (int b = it.bbeg; b < it.bend; ++b) w += blocks[b].ncol;
        return w * it.rows;
      };
      std::stable_sort(items.begin(), items.end(),
                       [&](const dev::SymRowItem& a, const dev::SymRowItem& b) { return work(a) > work(b); });
    }
    upload(M.sym_blocks, blocks, st);
    std::vector<std::int64_t> lrow0;
    std::vector<std::int32_t> lrows, sbeg{0};
    std::vector<dev::GatherSeg> segs;
    for (int id = 0; id < M.nnodes; ++id) {
      if (segs_of[id].empty()) continue;
      lrow0.push_back(T.nodes[id].begin);
      lrows.push_back(static_cast<std::int32_t>(T.nodes[id].count));
      segs.insert(segs.end(), segs_of[id].begin(), segs_of[id].end());
      sbeg.push_back(static_cast<std::int32_t>(segs.size()));
    }
    M.n_sym_items = static_cast<int>(items.size());
    M.k9_dense_rows = 1;
    for (const auto& it : items)
      M.k9_dense_rows = (it.i0 == 0 && it.rows == it.ld && M.k9_dense_rows > 0) ? std::max(M.k9_dense_rows, it.rows) : 0;
    M.n_gather_leaves = static_cast<int>(lrow0.size());
    M.near_tma = !items.empty();
    M.work_ctr.alloc(sizeof(int));
    M.theta_dev.alloc(sizeof(dev::ThetaParams));
    for (const auto& it : items)  // whole-leaf items (k_near_tma)
      M.near_tma = M.near_tma && it.i0 == 0 && it.rows == it.ld;
    upload(M.sym_items, items, st);
    upload(M.g_row0, lrow0, st);
    upload(M.g_rows, lrows, st);
    upload(M.g_sbeg, sbeg, st);
    upload(M.g_segs, segs, st);
    M.sym_part.alloc(sizeof(double) * std::max<std::int64_t>(poff, 1));
    M.sym_pstride = std::max<std::int64_t>(poff, 1);
  }
  {
    // K9 work (multi-RHS): CSR by sigma over every local near block; blocks
    // kept as transposes read their partner through the transposed map.
    std::vector<std::vector<Index>> by_sigma(M.nnodes);
    for (Index b = 0; b < nnear; ++b)
      if (M.near_doff[b] >= 0) by_sigma[H.blocks.near[b].sigma].push_back(b);
    std::vector<dev::MrhsItem> items;
    std::vector<std::int64_t> tb, dof;
    std::vector<std::int32_t> tn, ld, tr;
    for (int s = 0; s < M.nnodes; ++s) {
      if (by_sigma[s].empty()) continue;
      const int bbeg = static_cast<int>(tb.size());
      for (Index b : by_sigma[s]) {
        const Block blk = H.blocks.near[b];
        tb.push_back(T.nodes[blk.tau].begin);
        tn.push_back(static_cast<std::int32_t>(T.nodes[blk.tau].count));
        dof.push_back(M.near_doff[b]);
        ld.push_back(static_cast<std::int32_t>(M.near_trans[b] ? T.nodes[blk.tau].count : T.nodes[blk.sigma].count));
        tr.push_back(M.near_trans[b] ? 1 : 0);
      }
      const int bend = static_cast<int>(tb.size());
      const int ns = static_cast<int>(T.nodes[s].count);
      for (int i0 = 0; i0 < ns; i0 += 64)
        items.push_back({T.nodes[s].begin + i0, std::min(64, ns - i0), i0, bbeg, bend});
    }
    M.n_k9_items = static_cast<int>(items.size());
    upload(M.k9_items, items, st);
    upload(M.k9_tb, tb, st);
    upload(M.k9_tn, tn, st);
    upload(M.k9_doff, dof, st);
    upload(M.k9_ld, ld, st);
    upload(M.k9_tr, tr, st);
  }
  // --- far field: classes
  if (H.baseline.method != Baseline::None) {
    // fixed far field (baselines): per class H = I_t and, for H^2, C_k; the
    // instance copies them (no theta-core contraction)
    const BaselineData& B = H.baseline;
    M.baseline = true;
    M.ncls = static_cast<int>(B.rank.size());
    for (int k = 0; k < M.ncls; ++k) {
      dev::ClassMeta cm{};
      cm.rl = cm.rr = B.rank[k];
      PHM_CHECK(cm.rl <= 128, "baseline far rank above 128 unsupported on device");
      cm.h_off = B.h_off[k];
      if (M.h2) cm.c_off = static_cast<std::int64_t>(k) * M.P * M.P;
      M.cmeta_h.push_back(cm);
    }
    M.H_len = static_cast<std::int64_t>(B.fixed_h.size());
    M.C_len = M.h2 ? static_cast<std::int64_t>(M.ncls) * M.P * M.P : 0;
    upload(M.cmeta, M.cmeta_h, st);
    upload(M.fixed_H, B.fixed_h, st);
    if (M.h2) {
      if (M.P == 64) {  // C_k in DMMA fragment order (kernels.cuh cfrag64)
        std::vector<double> fc(B.fixed_c.size());
        for (std::size_t k = 0; k * 4096 < fc.size(); ++k)
          for (int j = 0; j < 64; ++j)
            for (int i = 0; i < 64; ++i) fc[k * 4096 + dev::cfrag64(i, j)] = B.fixed_c[k * 4096 + i + j * 64];
        upload(M.fixed_C, fc, st);
      } else {
        upload(M.fixed_C, B.fixed_c, st);
      }
    }
  } else {
    M.ncls = static_cast<int>(H.couplings.size());
    std::vector<double> mid, L, R;
    std::vector<std::int32_t> mdims;
    std::int64_t hoff = 0;
    int maxrl = 1, maxrr = 1, maxA = 1, maxB = 1, maxs1 = 1, maxdt = 0;
    for (int k = 0; k < M.ncls; ++k) {
      const Coupling& c = H.couplings[k];
      dev::ClassMeta cm{};
      cm.rl = static_cast<std::int32_t>(c.rank_left());
      cm.rr = static_cast<std::int32_t>(c.rank_right());
      PHM_CHECK(cm.rl <= 128 && cm.rr <= 128, "coupling rank above 128 unsupported on device");
      cm.mid_off = static_cast<std::int64_t>(mid.size());
      cm.dims_off = static_cast<std::int32_t>(mdims.size());
      int cur = 1;
      maxdt = std::max(maxdt, c.d_theta);
      for (int q = 0; q < c.d_theta; ++q) {
        const TTCore& g = c.tt.cores[c.d + q];
        mdims.push_back(static_cast<std::int32_t>(g.r0));
        mdims.push_back(static_cast<std::int32_t>(g.m));
        mdims.push_back(static_cast<std::int32_t>(g.r1));
        mid.insert(mid.end(), g.data.begin(), g.data.end());
        if (q == 0) maxA = std::max<int>(maxA, static_cast<int>(g.r0 * g.r1));
        else {
          maxB = std::max<int>(maxB, static_cast<int>(g.r0 * g.r1));
          maxs1 = std::max<int>(maxs1, static_cast<int>(g.r1));
        }
        cur = static_cast<int>(g.r1);
      }
      (void)cur;
      maxA = std::max(maxA, cm.rl * cm.rr);
      maxrl = std::max(maxrl, cm.rl);
      maxrr = std::max(maxrr, cm.rr);
      cm.h_off = hoff;
      hoff += static_cast<std::int64_t>(cm.rl) * cm.rr;
      if (M.h2) {
        cm.l_off = static_cast<std::int64_t>(L.size());
        cm.r_off = static_cast<std::int64_t>(R.size());
        L.insert(L.end(), H.class_l[k].a.begin(), H.class_l[k].a.end());
        R.insert(R.end(), H.class_r[k].a.begin(), H.class_r[k].a.end());
        cm.c_off = static_cast<std::int64_t>(k) * M.P * M.P;
      }
      M.cmeta_h.push_back(cm);
    }
    // A needs rl x (running r) for every step of the chain
    M.capA = std::max(maxA, maxrl * maxs1);
    M.capB = maxB;
    M.capT = std::max(maxrl * 32, maxrl * maxs1);
    if (M.h2 && M.P == 64) {  // C = L (H R^T) on DMMA: T (rl4 x 64, ld ldT), then R / L (ld 68) staged
      // only classes with rl <= 64 take the DMMA path in k_class_inst; the
      // others use the plain path sized by maxrl above
      int mrl = 0, mrr = 0, ldT = 0;  // ldT: the least ld >= rl4 with ld = 4 mod 16
      for (const auto& cm : M.cmeta_h) {
        if (cm.rl > 64) continue;
        mrl = std::max(mrl, cm.rl);
        mrr = std::max(mrr, cm.rr);
        const int r4 = (cm.rl + 3) & ~3;
        ldT = std::max(ldT, r4 + ((4 - r4) & 15));
      }
      const int rl4 = (mrl + 3) & ~3, rr4 = (mrr + 3) & ~3;
      M.capT = std::max(M.capT, ldT * 64);
      M.capL = 68 * std::max(rl4, rr4);  // L, and R before it
      // every class on the DMMA path: k_class_inst_pf (all loads of a class
      // in flight at once; its own region sizes, each a multiple of two
      // doubles for the 16-byte cp.async destinations)
      static const bool pf_env = [] {
        const char* e = std::getenv("PHM_CLASS_PF");
        return !(e && std::atoi(e) == 0);
      }();
      bool all_dmma = true;
      for (const auto& cm : M.cmeta_h) all_dmma = all_dmma && cm.rl <= 64;
      // one theta core (the chain of two or more measured slower with it:
      // C4 proxy 0.43 -> 0.60 ms)
      if (pf_env && all_dmma && maxdt == 1) {
        auto even = [](int v) { return (v + 1) & ~1; };
        M.capA = even(std::max(maxA, maxrl * maxs1));
        M.capB = even(maxB);
        M.capT = even(maxrl * maxs1);               // theta-chain scratch
        M.capR = even(std::max(68 * rr4, ldT * 64));  // R, then T
        M.capL = 68 * rl4;                          // L
      }
    }
    PHM_CHECK((M.capA + M.capB + M.capT + M.capR + M.capL) * 8 <= 227 * 1024,
              "class instantiate shared memory over 227 KB");
    M.H_len = hoff;
    M.C_len = M.h2 ? static_cast<std::int64_t>(M.ncls) * M.P * M.P : 0;
    upload(M.cmeta, M.cmeta_h, st);
    {
      const char* e = std::getenv("PHM_CLASS_SUBSET");
      const bool subset = H.cfg.shard_count > 1 && !(e && std::atoi(e) == 0);
      std::vector<char> need(M.ncls, subset ? 0 : 1);
      for (Index i = 0; i < static_cast<Index>(H.blocks.far.size()); ++i)
        if (H.far_local[i]) need[H.far_key[i]] = 1;
      std::vector<dev::ClassMeta> run;
      for (int k = 0; k < M.ncls; ++k)
        if (need[k]) run.push_back(M.cmeta_h[k]);
      M.ncls_run = static_cast<int>(run.size());
      M.cls_run = need;
      if (M.ncls_run == M.ncls)
        M.ncls_run = -1;  // all classes: use cmeta itself
      else if (M.ncls_run > 0)
        upload(M.cmeta_run, run, st);
    }
    upload(M.class_mid, mid, st);
    upload(M.class_mid_dims, mdims, st);
    upload(M.class_L, L, st);
    upload(M.class_R, R, st);
  }
  if (M.h2) {
    // coupling CSR by sigma node (local far blocks, list order inside sigma)
    std::vector<std::vector<Index>> by_sigma(M.nnodes);
    for (Index i = 0; i < static_cast<Index>(H.blocks.far.size()); ++i)
      if (H.far_local[i]) by_sigma[H.blocks.far[i].sigma].push_back(i);
    std::vector<std::int32_t> sig, tau, cls;
    std::vector<std::int64_t> beg{0};
    for (int s = 0; s < M.nnodes; ++s) {
      if (by_sigma[s].empty()) continue;
      sig.push_back(s);
      for (Index i : by_sigma[s]) {
        tau.push_back(H.blocks.far[i].tau);
        cls.push_back(H.far_key[i]);
      }
      beg.push_back(static_cast<std::int64_t>(tau.size()));
    }
    M.n_cp_sig = static_cast<int>(sig.size());
    upload(M.cp_sig, sig, st);
    upload(M.cp_beg, beg, st);
    upload(M.cp_tau, tau, st);
    upload(M.cp_cls, cls, st);
    M.cp_mma = dev::coupling_mma_supported(M.P);
    if (M.cp_mma) {
      // Groups: sigma nodes of one level with the same child parity, in node
      // id (Morton) order, 32 per group; classes of a group split into items.
      constexpr int kSlots = dev::kGroupSlots;
      std::map<std::pair<int, int>, std::vector<int>> by_lp;  // (level, parity) -> sigmas
      for (int s = 0; s < M.nnodes; ++s) {
        if (by_sigma[s].empty()) continue;
        int parity = 0;
        for (int k = 0; k < d; ++k) parity |= static_cast<int>(T.nodes[s].coords[k] & 1) << k;
        by_lp[{T.nodes[s].level, parity}].push_back(s);
      }
      std::vector<std::int32_t> grp_sigma, grp_items{0}, item_cls, cls_tau;
      std::vector<std::uint8_t> item_tiles;
      std::vector<dev::CouplingItem> items;
      std::vector<std::array<int, 3>> granges;  // (group, first class entry, end)
      for (auto& kv : by_lp) {
        const auto& sigs = kv.second;
        for (size_t g0 = 0; g0 < sigs.size(); g0 += kSlots) {
          const int grp = static_cast<int>(grp_items.size()) - 1;
          std::map<int, std::array<std::int32_t, kSlots>> table;
          for (int slot = 0; slot < kSlots; ++slot) {
            const size_t si = g0 + slot;
            grp_sigma.push_back(si < sigs.size() ? sigs[si] : -1);
            if (si >= sigs.size()) continue;
            for (Index i : by_sigma[sigs[si]]) {
              auto it = table.find(H.far_key[i]);
              if (it == table.end()) {
                std::array<std::int32_t, kSlots> row;
                row.fill(-1);
                it = table.emplace(H.far_key[i], row).first;
              }
              it->second[slot] = H.blocks.far[i].tau;
            }
          }
          int e = static_cast<int>(item_cls.size());
          for (auto& cr : table) {
            item_cls.push_back(cr.first);
            cls_tau.insert(cls_tau.end(), cr.second.begin(), cr.second.end());
            std::uint8_t tiles = 0;  // n-tiles of 8 slots holding a partner
            for (int slot = 0; slot < kSlots; ++slot)
              if (cr.second[slot] >= 0) tiles |= static_cast<std::uint8_t>(1u << (slot >> 3));
            item_tiles.push_back(tiles);
          }
          granges.push_back({grp, e, static_cast<int>(item_cls.size())});
          grp_items.push_back(0);  // filled below
        }
      }
      // Items of up to kItemClasses classes, sized so the launch has at least
      // ~4 items per SM: a small matrix (C2: ~40 groups) would otherwise run
      // ~40 CTAs that each walk ~60 classes one after another.
      const int kItemClasses = static_cast<int>(std::min<std::size_t>(
          64, std::max<std::size_t>(4, (item_cls.size() + 4 * 148 - 1) / (4 * 148))));
      for (const auto& gr : granges) {
        for (int e = gr[1]; e < gr[2]; e += kItemClasses)
          items.push_back({gr[0], e, std::min(e + kItemClasses, gr[2]), 0});
        grp_items[gr[0] + 1] = static_cast<std::int32_t>(items.size());
      }
      M.n_cg_items = static_cast<int>(items.size());
      M.n_cg_groups = static_cast<int>(grp_items.size()) - 1;
      // Traversal order: by (level, first class, group), so that the CTAs
      // running at one time stream the same C_k (L2 hits instead of HBM
      // re-reads while the near pass floods L2); partial sums stay indexed by
      // item, so the reduction order does not change.
      {
        std::vector<int> grp_level(M.n_cg_groups);
        for (int g = 0; g < M.n_cg_groups; ++g) grp_level[g] = T.nodes[grp_sigma[g * kSlots]].level;
        std::vector<std::int32_t> order(items.size());
        for (size_t i = 0; i < items.size(); ++i) order[i] = static_cast<std::int32_t>(i);
        std::stable_sort(order.begin(), order.end(), [&](std::int32_t a, std::int32_t b) {
          const auto& ia = items[a];
          const auto& ib = items[b];
          const auto ka = std::make_tuple(grp_level[ia.group], item_cls[ia.e_begin], ia.group);
          const auto kb = std::make_tuple(grp_level[ib.group], item_cls[ib.e_begin], ib.group);
          return ka < kb;
        });
        static const bool ordered = [] {
          const char* e = std::getenv("PHM_COUPLING_ORDER");
          return !(e && std::atoi(e) == 0);
        }();
        if (!ordered)
          for (size_t i = 0; i < items.size(); ++i) order[i] = static_cast<std::int32_t>(i);
        M.cg_n_upper = -1;
        if (ordered) {
          M.cg_n_upper = 0;
          for (std::int32_t i : order)
            if (grp_level[items[i].group] < T.l_max) ++M.cg_n_upper;
        }
        upload(M.cg_order, order, st);
      }
      upload(M.cg_items, items, st);
      upload(M.cg_cls, item_cls, st);
      upload(M.cg_tiles, item_tiles, st);
      upload(M.cg_tau, cls_tau, st);
      upload(M.cg_grp_sigma, grp_sigma, st);
      upload(M.cg_grp_items, grp_items, st);
      M.cg_partial.alloc(sizeof(double) * std::max(1, M.n_cg_items) * kSlots * M.P);
    }
    // basis: leaf factors [k][pos][j] for all points, transfers per node
    std::vector<double> u(static_cast<size_t>(d) * n * M.ps, 0.0);
    std::vector<std::int32_t> lall, lloc;
    for (int id = 0; id < M.nnodes; ++id) {
      const TreeNode& nd = T.nodes[id];
      if (!nd.leaf() || nd.count == 0) continue;
      lall.push_back(id);
      if (H.node_local[id]) lloc.push_back(id);
      std::vector<double> row(M.ps);
      for (int k = 0; k < d; ++k) {
        const Grid1D g = cheb_grid(nd.box.lo[k], nd.box.hi[k], M.ps);
        for (Index i = 0; i < nd.count; ++i) {
          lagrange_all(g, T.coord(T.perm[nd.begin + i], k), row.data());
          for (int j = 0; j < M.ps; ++j) u[(static_cast<size_t>(k) * n + nd.begin + i) * M.ps + j] = row[j];
        }
      }
    }
    std::vector<double> e(static_cast<size_t>(M.nnodes) * d * M.ps * M.ps, 0.0);
    for (int id = 1; id < M.nnodes; ++id) {
      const TreeNode& ch = T.nodes[id];
      const TreeNode& pa = T.nodes[ch.parent];
      std::vector<double> row(M.ps);
      for (int k = 0; k < d; ++k) {
        const Grid1D pg = cheb_grid(pa.box.lo[k], pa.box.hi[k], M.ps);
        const Grid1D cg = cheb_grid(ch.box.lo[k], ch.box.hi[k], M.ps);
        for (int i = 0; i < M.ps; ++i) {  // E_k(i, j): parent cardinal j at child node i
          lagrange_all(pg, cg.nodes[i], row.data());
          for (int j = 0; j < M.ps; ++j) e[((static_cast<size_t>(id) * d + k) * M.ps + i) * M.ps + j] = row[j];
        }
      }
    }
    upload(M.U, u, st);
    upload(M.Etr, e, st);
    M.n_leaves_all = static_cast<int>(lall.size());
    M.n_leaves_local = static_cast<int>(lloc.size());
    upload(M.leaves_all, lall, st);
    upload(M.leaves_local, lloc, st);
    for (int li = 0; li < 2; ++li) {
      const auto& lst = li == 0 ? lall : lloc;
      std::vector<std::int32_t> small, rleaf, rn;
      std::vector<dev::LeafChunk> ch;
      std::vector<std::int64_t> rslot;
      for (std::int32_t leaf : lst) {
        const int cnt = static_cast<int>(T.nodes[leaf].count);
        if (cnt <= dev::kLeafChunk) {
          small.push_back(leaf);
          continue;
        }
        rleaf.push_back(leaf);
        rslot.push_back(static_cast<std::int64_t>(ch.size()));
        int k = 0;
        for (int p0 = 0; p0 < cnt; p0 += dev::kLeafChunk, ++k)
          ch.push_back({leaf, p0, std::min(dev::kLeafChunk, cnt - p0), 0, static_cast<std::int64_t>(ch.size())});
        rn.push_back(k);
      }
      auto& L = M.lf[li];
      L.n_small = static_cast<int>(small.size());
      L.n_chunks = static_cast<int>(ch.size());
      L.n_red = static_cast<int>(rleaf.size());
      upload(L.small, small, st);
      upload(L.chunks, ch, st);
      upload(L.red_leaf, rleaf, st);
      upload(L.red_slot, rslot, st);
      upload(L.red_n, rn, st);
    }
    // level lists: upward = internal non-empty nodes per level (all);
    // downward = non-empty local non-root nodes per level
    std::vector<std::int32_t> upn, dnn, upl;
    M.up_range.assign(T.l_max + 1, {0, 0});
    M.down_range.assign(T.l_max + 1, {0, 0});
    M.upl_range.assign(T.l_max + 1, {0, 0});
    for (int l = 0; l <= T.l_max; ++l) {
      M.up_range[l].first = static_cast<int>(upn.size());
      M.down_range[l].first = static_cast<int>(dnn.size());
      M.upl_range[l].first = static_cast<int>(upl.size());
      for (int id = 0; id < M.nnodes; ++id) {
        const TreeNode& nd = T.nodes[id];
        if (nd.level != l || nd.count == 0) continue;
        if (!nd.leaf()) upn.push_back(id);
        if (!nd.leaf() && H.node_local[id]) upl.push_back(id);
        if (nd.parent >= 0 && H.node_local[id]) dnn.push_back(id);
      }
      M.up_range[l].second = static_cast<int>(upn.size());
      M.down_range[l].second = static_cast<int>(dnn.size());
      M.upl_range[l].second = static_cast<int>(upl.size());
    }
    upload(M.up_nodes, upn, st);
    upload(M.down_nodes, dnn, st);
    upload(M.upl_nodes, upl, st);
    // Levels above the first one with far blocks take no part in the product
    // (chebyshev.cpp:223-298 runs them; their x-hat / y-hat are never read).
    // Class keys cover every rank's far blocks, so shards agree on the level.
    M.far_min_level = T.l_max;
    for (const auto& key : H.class_keys) M.far_min_level = std::min<int>(M.far_min_level, static_cast<int>(key[0]));
    if (H.class_keys.empty()) M.far_min_level = 0;
    {
      const char* e = std::getenv("PHM_SKIP_TOP_LEVELS");
      if (e && std::atoi(e) == 0) M.far_min_level = 0;
    }
  } else {
    // H form: far blocks grouped per level, CSR by sigma, S/T payloads
    std::vector<dev::FarHItem> items;
    std::vector<std::int64_t> tb, soff, toff, poff;
    std::vector<std::int32_t> tn, cls, bitem;
    std::vector<double> S, Tm;
    std::int64_t pnext = 0;  // per-block partial segments (n_sigma each)
    M.fh_level_range.assign(T.l_max + 1, {0, 0});
    for (int l = 0; l <= T.l_max; ++l) {
      std::map<int, std::vector<Index>> by_sigma;
      for (Index i = 0; i < static_cast<Index>(H.blocks.far.size()); ++i)
        if (H.far_local[i] && T.nodes[H.blocks.far[i].sigma].level == l) by_sigma[H.blocks.far[i].sigma].push_back(i);
      M.fh_level_range[l].first = static_cast<int>(items.size());
      for (auto& kv : by_sigma) {
        const TreeNode& s = T.nodes[kv.first];
        dev::FarHItem it{};
        it.row0 = s.begin;
        it.rows = static_cast<std::int32_t>(s.count);
        it.bbeg = static_cast<std::int32_t>(tb.size());
        for (Index i : kv.second) {
          const TreeNode& u = T.nodes[H.blocks.far[i].tau];
          tb.push_back(u.begin);
          tn.push_back(static_cast<std::int32_t>(u.count));
          cls.push_back(H.far_key[i]);
          soff.push_back(static_cast<std::int64_t>(S.size()));
          toff.push_back(static_cast<std::int64_t>(Tm.size()));
          S.insert(S.end(), H.far_s[i].a.begin(), H.far_s[i].a.end());
          Tm.insert(Tm.end(), H.far_t[i].a.begin(), H.far_t[i].a.end());
        }
        it.bend = static_cast<std::int32_t>(tb.size());
        for (int q = it.bbeg; q < it.bend; ++q) {
          bitem.push_back(static_cast<std::int32_t>(items.size()));
          poff.push_back(pnext);
          pnext += it.rows;
        }
        items.push_back(it);
      }
      M.fh_level_range[l].second = static_cast<int>(items.size());
    }
    upload(M.fh_bitem, bitem, st);
    upload(M.fh_poff, poff, st);
    M.fh_part.alloc(sizeof(double) * std::max<std::int64_t>(pnext, 1));
    upload(M.fh_items, items, st);
    M.fh_items_h = items;
    upload(M.fh_tb, tb, st);
    upload(M.fh_tn, tn, st);
    upload(M.fh_cls, cls, st);
    upload(M.fh_soff, soff, st);
    upload(M.fh_toff, toff, st);
    upload(M.fh_S, S, st);
    upload(M.fh_T, Tm, st);
  }
  CK(cudaStreamSynchronize(st));
  {
    std::int64_t bytes = 0;
    for (const DBuf* b : {&M.perm, &M.pts, &M.G, &M.class_mid, &M.class_L, &M.class_R, &M.U, &M.Etr, &M.fh_S, &M.fh_T,
                          &M.near_cores, &M.snap_tiles, &M.inst_tiles})
      bytes += static_cast<std::int64_t>(b->bytes);
    M.device_bytes = bytes;
  }
  H.stats.upload_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_up).count();
  return Mp;
}

// ----------------------------------------------------------- instantiate
namespace {

// Class stage of instantiate: H_k(theta) and C_k = L_k H_k R_k^T (K2).
// Writes the theta-dependent inputs (parametric vectors, snapshot weights'
// shape part, amplitude) to M.theta_dev on stream s: the kernels of the
// class stage and of the near weights read them there, so their launch
// parameters do not depend on theta.
void put_theta(DevMatrix& M, const std::vector<std::vector<double>>& v, const dev::ThetaV& tv, cudaStream_t s) {
  const KernelSpec& spec = M.hm->cfg.spec;
  dev::ThetaParams p{};
  p.tv = tv;
  p.shape = tv;
  p.shape.dt = spec.shape_params();
  p.amp = 1.0;
  if (spec.amplitude && M.mode == NearMode::Snapshot) {
    const auto& g = M.hm->grids.grids[spec.shape_params()];
    p.amp = 0.0;
    for (int j = 0; j < g.p; ++j) p.amp += v[spec.shape_params()][j] * g.nodes[j];
  }
  M.ctx->run_on(s, "put_theta", [&] { dev::launch_put_theta(s, p, M.theta_dev.as<dev::ThetaParams>()); });
}

// ctas > 0 caps the grid of k_class_inst_pf (a persistent loop over the
// classes): beside the fused near pass, one class CTA per SM leaves room for
// a near CTA from the start instead of holding every slot until its last wave.
void inst_classes(DevInstance& I, cudaStream_t s, int ctas = 0) {
  DevMatrix& M = *I.M;
  const bool all = M.ncls_run < 0 || M.baseline;
  if (!all && M.ncls_run == 0) return;  // a shard without far blocks
  M.ctx->run_on(s, "class_inst", [&] {
    dev::launch_class_inst(s, all ? M.cmeta.as<dev::ClassMeta>() : M.cmeta_run.as<dev::ClassMeta>(),
                           all ? M.ncls : M.ncls_run, M.class_mid.as<double>(),
                           M.class_mid_dims.as<std::int32_t>(), M.class_L.as<double>(), M.class_R.as<double>(),
                           M.theta_dev.as<dev::ThetaParams>(), M.P, M.h2, M.capA, M.capB, M.capT, M.capL, M.capR, ctas,
                           I.H.as<double>(), I.C.as<double>());
  });
}

// Snapshot weights w = v_shape (x) ... times the amplitude interpolant
// sum_j v_j s_j (the full-rank NearBlockTT theta-core chain).
void inst_snapshot_w(DevInstance& I, cudaStream_t s) {
  DevMatrix& M = *I.M;
  M.ctx->run_on(s, "near_w", [&] {
    dev::launch_set_vec(s, I.w.as<double>(), M.R_snap, M.theta_dev.as<dev::ThetaParams>());
  });
}

// K1 moves the snapshot slabs by TMA (k_inst_tma) unless PHM_K1_TMA=0
// (k_inst_flat: 256-bit loads): 8.5 vs 9.3 ms at C3.
bool k1_tma() {
  static const bool on = [] {
    const char* e = std::getenv("PHM_K1_TMA");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// Near stage of instantiate: every stored D_b(theta) (K1).
// k1_per_sm: CTAs per SM of the TMA K1 stream -- 1 when the far chain runs
// beside it on the side stream (instantiate + block apply), so the class
// stage, the leaf forward pass and the coupling get SM room during K1
// instead of queueing behind its persistent grid (C4 rank 0 of 8: 71.3 vs
// 74.2 ms per step)
void inst_near(DevInstance& I, const double* theta, cudaStream_t s, StageCounters* counters, int k1_per_sm = 2) {
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  Context& ctx = *M.ctx;
  if (M.mode == NearMode::Snapshot) {
    inst_snapshot_w(I, s);
    ctx.run_on(s, "near_inst", [&] {
      dev::InstPtrs tab{};
      tab.w[0] = I.w.as<double>();
      tab.d[0] = I.D.as<double>();
      // the TMA ring pays off on large snapshot sets; small ones (C1: 160 MB)
      // run faster as the plain 256-bit stream
      const bool big = static_cast<double>(M.E) * M.R_snap * 8.0 > 1e9;
      if (!big || !k1_tma() || !dev::launch_inst_tma(s, M.G.as<double>(), M.E, M.R_snap, 1, tab, k1_per_sm))
        dev::launch_inst_flat(s, M.G.as<double>(), M.E, M.R_snap, I.w.as<double>(), I.D.as<double>());
    });
  } else if (M.mode == NearMode::TT) {
    ctx.run_on(s, "near_w", [&] {
      dev::launch_near_w(s, M.near_w_meta.as<dev::NearW>(), M.n_near_local, M.near_cores.as<double>(),
                         M.near_core_dims.as<std::int32_t>(), M.theta_dev.as<dev::ThetaParams>(),
                         I.w.as<double>());
    });
    ctx.run_on(s, "near_inst", [&] {
      dev::launch_inst_tiles(s, M.inst_tiles.as<dev::InstTile>(), M.n_inst_tiles, M.G.as<double>(),
                             I.w.as<double>(), I.D.as<double>());
    });
  } else {
    // Direct: evaluate the kernel at theta for every near entry (counted)
    std::vector<double> th(3, 1.0);
    for (int k = 0; k < H.cfg.spec.shape_params(); ++k) th[k] = theta[k];
    double amp = H.cfg.spec.amplitude ? theta[H.cfg.spec.shape_params()] : 1.0;
    if (!I.w.p) I.w.alloc(3 * sizeof(double));
    CK(cudaMemcpyAsync(I.w.p, th.data(), 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    ctx.run_on(s, "near_direct", [&] {
      dev::launch_snapshot(s, M.snap_tiles.as<dev::SnapTile>(), M.n_snap_tiles, M.geo.as<dev::BlockGeom>(),
                           M.pts.as<double>(), M.n, M.d, H.cfg.spec.family, 1, I.w.as<double>(), amp, I.D.as<double>());
    });
    CK(cudaStreamSynchronize(s));  // th lives on this stack frame
    if (counters) counters->online.add(static_cast<std::uint64_t>(M.E_raw));
  }
}

void run_instantiate(DevInstance& I, const double* theta, int n_theta, StageCounters* counters) {
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  CK(cudaSetDevice(M.ctx->device));
  if (M.baseline) {
    // baselines: the far field was factorised at the build theta; the dense
    // near blocks are evaluated now (charged to the build's near_evals)
    const BaselineData& B = H.baseline;
    cudaStream_t st = M.ctx->stream;
    I.theta = B.theta;
    if (M.H_len) CK(cudaMemcpyAsync(I.H.p, M.fixed_H.p, sizeof(double) * M.H_len, cudaMemcpyDeviceToDevice, st));
    if (M.C_len) CK(cudaMemcpyAsync(I.C.p, M.fixed_C.p, sizeof(double) * M.C_len, cudaMemcpyDeviceToDevice, st));
    inst_near(I, B.theta.data(), st, nullptr);
    return;
  }
  // theta box check before any launch (farfield.cpp:23-24)
  const auto v = parametric_vectors(H.grids, theta, n_theta);
  I.theta.assign(theta, theta + n_theta);
  const dev::ThetaV tv = make_theta_v(v);
  // (Overlapping the class stage with K1 on the side stream measured
  // slower: its CTAs displaced K1's and K1 lost 1.8 ms.)
  put_theta(M, v, tv, M.ctx->stream);
  inst_classes(I, M.ctx->stream);
  inst_near(I, theta, M.ctx->stream, counters);
}

}  // namespace

namespace {
std::shared_ptr<DevInstance> alloc_instance(const std::shared_ptr<DevMatrix>& m) {
  auto I = std::make_shared<DevInstance>();
  I->M = m;
  {
    std::lock_guard<std::mutex> lk(m->mu);
    if (!m->pool_D.empty()) {
      I->D = std::move(m->pool_D.back());
      m->pool_D.pop_back();
    }
  }
  if (I->D.bytes < static_cast<size_t>(m->E) * sizeof(double)) {
    I->D.alloc(static_cast<size_t>(m->E) * sizeof(double));
    CK(cudaMemsetAsync(I->D.p, 0, I->D.bytes, m->st()));  // block pads stay zero
  }
  I->H.alloc(static_cast<size_t>(std::max<std::int64_t>(m->H_len, 1)) * sizeof(double));
  if (m->C_len) I->C.alloc(static_cast<size_t>(m->C_len) * sizeof(double));
  const std::int64_t wl = m->mode == NearMode::Snapshot ? m->R_snap : m->w_len;
  if (wl) I->w.alloc(static_cast<size_t>(wl) * sizeof(double));
  return I;
}

// instantiate for B thetas at once: the class stage per theta, then (snapshot
// mode) one K1 pass that reads the snapshots once and writes all B D's.
void run_instantiate_batch(const std::vector<DevInstance*>& insts, const double* thetas, int n_theta,
                           StageCounters* counters) {
  DevMatrix& M = *insts[0]->M;
  const HostMatrix& H = *M.hm;
  CK(cudaSetDevice(M.ctx->device));
  const int B = static_cast<int>(insts.size());
  std::vector<std::vector<std::vector<double>>> vs(B);
  for (int b = 0; b < B; ++b) vs[b] = parametric_vectors(H.grids, thetas + b * n_theta, n_theta);  // all checked first
  cudaStream_t st = M.ctx->stream;
  // per theta, in stream order: its parameters, class stage and near
  // weights (non-snapshot modes: its whole near stage)
  for (int b = 0; b < B; ++b) {
    insts[b]->theta.assign(thetas + b * n_theta, thetas + (b + 1) * n_theta);
    put_theta(M, vs[b], make_theta_v(vs[b]), st);
    inst_classes(*insts[b], st);
    if (M.mode == NearMode::Snapshot)
      inst_snapshot_w(*insts[b], st);
    else
      inst_near(*insts[b], thetas + b * n_theta, st, counters);
  }
  if (M.mode != NearMode::Snapshot) return;
  constexpr int kMax = 16;  // dev::kInstBatchMax
  for (int b0 = 0; b0 < B; b0 += kMax) {
    const int nb = std::min(kMax, B - b0);
    dev::InstPtrs tab{};  // by value: no host staging buffer to race with
    for (int b = 0; b < nb; ++b) {
      tab.w[b] = insts[b0 + b]->w.as<double>();
      tab.d[b] = insts[b0 + b]->D.as<double>();
    }
    bool ok = false;
    M.ctx->run_on(st, "near_inst", [&] {
      // larger batches are bound by the formation work, where the plain
      // 256-bit stream is as fast (8 thetas: 16.7 vs 17.0 ms at C3)
      ok = (nb <= 2 && k1_tma() && dev::launch_inst_tma(st, M.G.as<double>(), M.E, M.R_snap, nb, tab)) ||
           dev::launch_inst_flat_batch(st, M.G.as<double>(), M.E, M.R_snap, nb, tab);
    });
    if (!ok)
      for (int b = 0; b < nb; ++b)
        M.ctx->run_on(st, "near_inst", [&] {
          dev::launch_inst_flat(st, M.G.as<double>(), M.E, M.R_snap, insts[b0 + b]->w.as<double>(),
                                insts[b0 + b]->D.as<double>());
        });
  }
}
}  // namespace

std::shared_ptr<DevInstance> baseline_instance(std::shared_ptr<DevMatrix> m) {
  std::lock_guard<std::recursive_mutex> exec_lock(m->exec_mu());
  PHM_CHECK(m->baseline, "baseline_instance: not a baseline matrix");
  CK(cudaSetDevice(m->ctx->device));
  auto I = alloc_instance(m);
  run_instantiate(*I, nullptr, 0, nullptr);
  return I;
}

std::shared_ptr<DevMatrix> baseline_build(std::shared_ptr<Context> ctx, const double* points, Index n, int d,
                                          const Config& cfg, Baseline method, const double* theta, int n_theta,
                                          double eps, Index r_max) {
  return matrix_upload(ctx, build_baseline_host(points, n, d, cfg, method, theta, n_theta, eps, r_max));
}

std::shared_ptr<DevInstance> instantiate(std::shared_ptr<DevMatrix> m, const double* theta, int n_theta,
                                         StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(m->exec_mu());
  if (!m->ctx) throw std::logic_error("instantiate: host-only matrix (built without a device)");
  if (m->baseline) throw std::logic_error("instantiate: a baseline matrix is built at a fixed theta");
  CK(cudaSetDevice(m->ctx->device));
  // validate theta first so nothing is allocated for a bad call
  (void)parametric_vectors(m->hm->grids, theta, n_theta);
  auto I = alloc_instance(m);
  run_instantiate(*I, theta, n_theta, counters);
  return I;
}

std::vector<std::shared_ptr<DevInstance>> instantiate_batch(std::shared_ptr<DevMatrix> m, const double* thetas,
                                                            int n_theta, int count, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(m->exec_mu());
  if (!m->ctx) throw std::logic_error("instantiate: host-only matrix (built without a device)");
  if (m->baseline) throw std::logic_error("instantiate: a baseline matrix is built at a fixed theta");
  PHM_CHECK(count >= 1, "instantiate_batch: count must be >= 1");
  CK(cudaSetDevice(m->ctx->device));
  for (int b = 0; b < count; ++b) (void)parametric_vectors(m->hm->grids, thetas + b * n_theta, n_theta);
  std::vector<std::shared_ptr<DevInstance>> out;
  std::vector<DevInstance*> raw;
  for (int b = 0; b < count; ++b) {
    out.push_back(alloc_instance(m));
    raw.push_back(out.back().get());
  }
  run_instantiate_batch(raw, thetas, n_theta, counters);
  return out;
}

void reinstantiate_batch(const std::vector<DevInstance*>& insts, const double* thetas, int n_theta,
                         StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(insts.at(0)->M->exec_mu());
  PHM_CHECK(!insts.empty(), "reinstantiate_batch: no instances");
  if (insts[0]->M->baseline) throw std::logic_error("reinstantiate: a baseline matrix is built at a fixed theta");
  for (DevInstance* I : insts) PHM_CHECK(I->M == insts[0]->M, "reinstantiate_batch: instances of different matrices");
  run_instantiate_batch(insts, thetas, n_theta, counters);
}

void reinstantiate(DevInstance& inst, const double* theta, int n_theta, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(inst.M->exec_mu());
  NvtxRange nvtx("phm::instantiate");
  if (inst.M->baseline) throw std::logic_error("reinstantiate: a baseline matrix is built at a fixed theta");
  run_instantiate(inst, theta, n_theta, counters);
}
const std::vector<double>& instance_theta(const DevInstance& inst) { return inst.theta; }
void instance_sync(DevInstance& inst) { CK(cudaStreamSynchronize(inst.M->st())); }

void instance_far_h(DevInstance& I, Index far_index, std::vector<double>& out, Index& rows, Index& cols) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  const DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  if (far_index < 0 || far_index >= static_cast<Index>(H.blocks.far.size())) throw std::out_of_range("far index");
  if (!M.cls_run.empty() && !M.cls_run[H.far_key[far_index]])
    throw std::logic_error("far_h: the block's class is not instantiated on this row shard (no local far block uses it)");
  const dev::ClassMeta& cm = M.cmeta_h[H.far_key[far_index]];
  rows = cm.rl;
  cols = cm.rr;
  out.resize(static_cast<size_t>(rows * cols));
  CK(cudaMemcpyAsync(out.data(), I.H.as<double>() + cm.h_off, out.size() * sizeof(double), cudaMemcpyDeviceToHost,
                     M.st()));
  CK(cudaStreamSynchronize(M.st()));
}

void instance_near_d(DevInstance& I, Index b, std::vector<double>& out) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  const DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  if (b < 0 || b >= static_cast<Index>(H.blocks.near.size())) throw std::out_of_range("near index");
  if (M.near_doff[b] < 0) throw std::out_of_range("near block not resident on this shard");
  const Block blk = H.blocks.near[b];
  const Index ns = H.tree->nodes[blk.sigma].count, nt = H.tree->nodes[blk.tau].count;
  out.resize(static_cast<size_t>(ns * nt));
  CK(cudaMemcpyAsync(out.data(), I.D.as<double>() + M.near_doff[b], ns * nt * sizeof(double), cudaMemcpyDeviceToHost,
                     M.st()));
  CK(cudaStreamSynchronize(M.st()));
  if (M.near_trans[b]) {  // stored as the (nt x ns) partner block
    std::vector<double> t(out.size());
    for (Index j = 0; j < nt; ++j)
      for (Index i = 0; i < ns; ++i) t[i + j * ns] = out[j + i * nt];
    out.swap(t);
  }
}

void instance_class_c(DevInstance& I, Index k, std::vector<double>& out) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  const DevMatrix& M = *I.M;
  if (!M.h2) throw std::invalid_argument("explicit C_k exists only for the H2 format");
  if (k < 0 || k >= M.ncls) throw std::out_of_range("class index");
  if (!M.cls_run.empty() && !M.cls_run[k])
    throw std::logic_error("class_c: the class is not instantiated on this row shard (no local far block uses it)");
  out.resize(static_cast<size_t>(M.P) * M.P);
  CK(cudaMemcpyAsync(out.data(), I.C.as<double>() + k * static_cast<std::int64_t>(M.P) * M.P,
                     out.size() * sizeof(double), cudaMemcpyDeviceToHost, M.st()));
  CK(cudaStreamSynchronize(M.st()));
  if (M.P == 64) {  // stored in DMMA fragment order (kernels.cuh cfrag64)
    std::vector<double> cm(out.size());
    for (int j = 0; j < 64; ++j)
      for (int i = 0; i < 64; ++i) cm[i + j * 64] = out[dev::cfrag64(i, j)];
    out.swap(cm);
  }
}

// ------------------------------------------------------------------ apply
namespace {

// H^2 far-field chain on stream fs: forward (K3, K4), coupling (K5),
// downward (K7 internal). Reads xp and C_k; writes yhat.
void far_chain(DevInstance& I, Index m, cudaStream_t fs, int coupling_ctas, Comm* ex = nullptr,
               bool leaf_level_first = false) {
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  Context& ctx = *M.ctx;
  const int P = M.P;
  const int mm = static_cast<int>(m);
  // On a row shard with an exchange, the forward pass covers only the local
  // leaves and the nodes above them (x-hat of a node spanning ranks is this
  // rank's partial sum; every other entry is zero), and one all-reduce of
  // x-hat completes it: the transfer pass is linear, so the ranks' partial
  // sums add up to the unsharded x-hat (to rounding). Replaces the forward
  // pass every rank otherwise repeats in full.
  static const bool split_env = [] {
    const char* e = std::getenv("PHM_SPLIT_FORWARD");
    return !(e && std::atoi(e) == 0);
  }();
  const bool split = ex != nullptr && M.sharded && split_env;
  if (split)
    ctx.run_on(fs, "zero", [&] { dev::launch_zero(fs, M.xhat.as<double>(), static_cast<std::int64_t>(M.nnodes) * P * m); });
  const auto& LP = M.lf[split ? 1 : 0];
  if (LP.n_chunks > 0 && P == 64 && m >= 4 && M.d * M.ps <= 48) {
    // big (clustered) leaves split into chunks of kLeafChunk points
    const size_t need = sizeof(double) * LP.n_chunks * m * P;
    if (M.lf_part.bytes < need) {
      M.lf_part.alloc(need);
      ++M.ws_gen;  // captured graphs hold the old pointer
    }
    ctx.run_on(fs, "leaf_fwd", [&] {
      dev::launch_leaf_fwd_chunks(fs, LP.chunks.as<dev::LeafChunk>(), LP.n_chunks, LP.red_leaf.as<std::int32_t>(),
                                  LP.red_slot.as<std::int64_t>(), LP.red_n.as<std::int32_t>(), LP.n_red,
                                  M.node_begin.as<std::int64_t>(), M.node_count.as<std::int32_t>(), M.U.as<double>(),
                                  M.n, M.d, M.ps, M.xp.as<double>(), mm, M.lf_part.as<double>(), M.xhat.as<double>());
      dev::launch_leaf_fwd(fs, LP.small.as<std::int32_t>(), LP.n_small, M.node_begin.as<std::int64_t>(),
                           M.node_count.as<std::int32_t>(), M.U.as<double>(), M.n, M.d, M.ps, P, M.xp.as<double>(),
                           mm, M.xhat.as<double>());
    });
  } else {
    ctx.run_on(fs, "leaf_fwd", [&] {
      dev::launch_leaf_fwd(fs, (split ? M.leaves_local : M.leaves_all).as<std::int32_t>(),
                           split ? M.n_leaves_local : M.n_leaves_all, M.node_begin.as<std::int64_t>(),
                           M.node_count.as<std::int32_t>(), M.U.as<double>(), M.n, M.d, M.ps, P, M.xp.as<double>(),
                           mm, M.xhat.as<double>());
    });
  }
  // PHM_LEAF_LEVEL_FIRST=1 (diagnostic, off by default): leaf-level blocks
  // (2.02M of 2.16M at C3) read only the leaf x-hat, so in apply their
  // coupling launch can start right after K3 while the transfer pass and the
  // upper levels' coupling run on a second side stream. Items write disjoint
  // partial slots and the reduction order is per item, so y is bitwise the
  // same. Measured at C3: no gain (1.691 vs 1.677 ms) -- the MVM is bound by
  // the SM time the GEMV and the coupling share, not by the K3 -> K4 -> K5
  // dependency chain; the earlier coupling just overlaps more of the GEMV
  // and both slow down (profiles/r02d_apply_level_split_sweep.txt).
  static const bool llf_env = [] {
    const char* e = std::getenv("PHM_LEAF_LEVEL_FIRST");
    return e && std::atoi(e) == 1;
  }();
  const bool llf = leaf_level_first && llf_env && !split && M.cp_mma && coupling_ctas == 0 && M.cg_n_upper > 0 &&
                   M.cg_n_upper < M.n_cg_items;
  cudaStream_t us = llf ? ctx.side2 : fs;  // transfer pass (and upper-level coupling)
  if (M.cp_mma) {
    const size_t need = sizeof(double) * std::max(1, M.n_cg_items) * m * dev::kGroupSlots * P;
    if (M.cg_partial.bytes < need) {
      M.cg_partial.alloc(need);
      ++M.ws_gen;  // captured graphs hold the old pointer
    }
  }
  auto coupling_launch = [&](cudaStream_t s, int first, int count) {
    ctx.run_on(s, "coupling", [&] {
      dev::launch_coupling_mma(s, M.cg_items.as<dev::CouplingItem>(), M.cg_order.as<std::int32_t>() + first, count,
                               M.cg_cls.as<std::int32_t>(), M.cg_tiles.as<std::uint8_t>(),
                               M.cg_tau.as<std::int32_t>(), I.C.as<double>(), P, M.xhat.as<double>(), mm,
                               M.cg_partial.as<double>(), coupling_ctas);
    });
  };
  // a kernel, not a memset: a memset node of a graph carries no priority and
  // would wait behind the near pass's CTAs
  ctx.run_on(fs, "zero", [&] { dev::launch_zero(fs, M.yhat.as<double>(), static_cast<std::int64_t>(M.nnodes) * P * m); });
  if (llf) {
    CK(cudaEventRecord(ctx.leaf_ev, fs));
    CK(cudaStreamWaitEvent(us, ctx.leaf_ev, 0));
    coupling_launch(fs, M.cg_n_upper, M.n_cg_items - M.cg_n_upper);
  }
  for (int l = H.tree->l_max - 1; l >= M.far_min_level; --l) {
    const auto r = split ? M.upl_range[l] : M.up_range[l];
    if (r.second == r.first) continue;
    ctx.run_on(us, "up", [&] {
      dev::launch_up(us, (split ? M.upl_nodes : M.up_nodes).as<std::int32_t>() + r.first, r.second - r.first,
                     M.node_first_child.as<std::int32_t>(), M.node_count.as<std::int32_t>(), M.Etr.as<double>(), M.d,
                     M.ps, P, mm, M.xhat.as<double>());
    });
  }
  if (llf) {
    coupling_launch(us, 0, M.cg_n_upper);
    CK(cudaEventRecord(ctx.up_ev, us));
    CK(cudaStreamWaitEvent(fs, ctx.up_ev, 0));
  }
  if (split) ex->allreduce(M.xhat.as<double>(), static_cast<std::int64_t>(M.nnodes) * P * m, fs);
  if (M.cp_mma) {
    ctx.stamp(fs, 5);
    if (!llf) coupling_launch(fs, 0, M.n_cg_items);
    ctx.stamp(fs, 6);
    ctx.run_on(fs, "coupling_reduce", [&] {
      dev::launch_coupling_reduce(fs, M.cg_grp_sigma.as<std::int32_t>(), M.cg_grp_items.as<std::int32_t>(),
                                  M.n_cg_groups, M.cg_partial.as<double>(), P, mm, M.yhat.as<double>());
    });
  } else {
    ctx.run_on(fs, "coupling", [&] {
      dev::launch_coupling(fs, M.cp_sig.as<std::int32_t>(), M.n_cp_sig, M.cp_beg.as<std::int64_t>(),
                           M.cp_tau.as<std::int32_t>(), M.cp_cls.as<std::int32_t>(), I.C.as<double>(), P, mm,
                           M.xhat.as<double>(), M.yhat.as<double>());
    });
  }
  for (int l = std::max(1, M.far_min_level + 1); l <= H.tree->l_max; ++l) {
    const auto r = M.down_range[l];
    if (r.second == r.first) continue;
    ctx.run_on(fs, "down", [&] {
      dev::launch_down(fs, M.down_nodes.as<std::int32_t>() + r.first, r.second - r.first,
                       M.node_parent.as<std::int32_t>(), M.Etr.as<double>(), M.d, M.ps, P, mm, M.yhat.as<double>());
    });
  }
}

// Near-field product on stream st: writes this shard's rows of yp.
// Fixed-order per-leaf sum of the near partials into column c of yp.
void near_gather(DevInstance& I, Index c, cudaStream_t st) {
  DevMatrix& M = *I.M;
  M.ctx->run_on(st, "near_gather", [&] {
    dev::launch_near_gather(st, M.n_gather_leaves, M.g_row0.as<std::int64_t>(), M.g_rows.as<std::int32_t>(),
                            M.g_sbeg.as<std::int32_t>(), M.g_segs.as<dev::GatherSeg>(), M.sym_part.as<double>(), 0,
                            M.n, 1, M.yp.as<double>() + c * M.n);
  });
}

// Column c of the near product by the two-sided HBM GEMV (K6) and its
// ordered per-leaf sum.
void near_gemv_column(DevInstance& I, Index c, cudaStream_t st) {
  DevMatrix& M = *I.M;
  M.ctx->run_on(st, "near_mvm", [&] {
    static const bool tma = [] {
      const char* e = std::getenv("PHM_NEAR_TMA");
      return !(e && std::atoi(e) == 0);
    }();
    if (M.near_tma && tma)
      dev::launch_near_tma_apply(st, M.sym_items.as<dev::SymRowItem>(), M.n_sym_items,
                                 M.sym_blocks.as<dev::SymBlock>(), I.D.as<double>(), M.xp.as<double>() + c * M.n,
                                 M.sym_part.as<double>(), M.work_ctr.as<int>());
    else
      dev::launch_near_mvm_symcsr(st, M.sym_items.as<dev::SymRowItem>(), M.n_sym_items,
                                  M.sym_blocks.as<dev::SymBlock>(), I.D.as<double>(), M.xp.as<double>() + c * M.n,
                                  M.sym_part.as<double>());
  });
  near_gather(I, c, st);
}

void near_product(DevInstance& I, Index m, cudaStream_t st) {
  DevMatrix& M = *I.M;
  Context& ctx = *M.ctx;
  const int mm = static_cast<int>(m);
  // A shard's gather touches only the leaves its blocks reach: clear the rest.
  if (M.n_gather_leaves == 0 || M.n_k9_items == 0 || M.sharded)
    CK(cudaMemsetAsync(M.yp.p, 0, sizeof(double) * M.n * m, st));
  // Block right-hand sides: the near product is a dense contraction, so it
  // runs on fp64 tensor cores (K9); single vectors stay on the HBM GEMV.
  // K9 computes rows sigma only, so a symmetric shard (whose transposed
  // products belong to other ranks' rows) keeps the two-sided GEMV.
  static const int two_sided_env = [] {  // 0: never, 2: also above 32 RHS unsharded (diagnostics)
    const char* e = std::getenv("PHM_K9_TWO_SIDED");
    return e ? std::atoi(e) : 1;
  }();
  const bool two_sided = two_sided_env != 0;
  // up to 32 RHS: each stored block read once, both products on DMMA
  // (k_near_mrhs3, TMA-staged: C3 at 10 RHS 3.5 ms against 6.4 for the
  // one-sided K9). At 64 RHS the one-sided K9 is faster (13.8 vs 16.8 ms +
  // 3.3 ms of gather), except on a symmetric shard, which needs both sides.
  if (m >= kMrhsMin && M.n_sym_items > 0 && two_sided && (m <= 32 || (M.sym && M.sharded) || two_sided_env == 2)) {
    const size_t need = sizeof(double) * M.sym_pstride * m;
    if (M.sym_part_m.bytes < need) {
      M.sym_part_m.alloc(need);
      ++M.ws_gen;  // captured graphs hold the old pointer
    }
    static const int k9v = [] {
      const char* e = std::getenv("PHM_K9_TMA");
      return e ? std::atoi(e) : 1;
    }();
    // Measured and dropped (profiles/r02d_k9_tail_gemv_sweep.txt): K9 on the
    // first 8k columns and the HBM GEMV for a tail of one or two (m = 10:
    // apply 10.4 -> 11.7 ms). Beside the coupling K9 is not paced by its own
    // MMA padding: the high-priority coupling grid takes the SM slots and K9
    // finishes after it, so the schedule is the sum of the kernels' own times
    // and the GEMV passes only add to it.
    ctx.run_on(st, "near_mrhs", [&] {
      if (k9v == 1)
        dev::launch_near_mrhs3(st, M.sym_items.as<dev::SymRowItem>(), M.n_sym_items, M.sym_blocks.as<dev::SymBlock>(),
                               I.D.as<double>(), M.xp.as<double>(), M.n, mm, M.sym_pstride, M.sym_part_m.as<double>(),
                               M.k9_dense_rows);
      else
        dev::launch_near_mrhs2(st, M.sym_items.as<dev::SymRowItem>(), M.n_sym_items, M.sym_blocks.as<dev::SymBlock>(),
                               I.D.as<double>(), M.xp.as<double>(), M.n, mm, M.sym_pstride, M.sym_part_m.as<double>());
    });
    ctx.run_on(st, "near_gather", [&] {
      dev::launch_near_gather(st, M.n_gather_leaves, M.g_row0.as<std::int64_t>(), M.g_rows.as<std::int32_t>(),
                              M.g_sbeg.as<std::int32_t>(), M.g_segs.as<dev::GatherSeg>(), M.sym_part_m.as<double>(),
                              M.sym_pstride, M.n, mm, M.yp.as<double>());
    });
    return;
  }
  const bool block_rhs = m >= kMrhsMin && !(M.sym && M.sharded);
  if (block_rhs)
    ctx.run_on(st, "near_mrhs", [&] {
      dev::launch_near_mrhs(st, M.k9_items.as<dev::MrhsItem>(), M.n_k9_items, M.k9_tb.as<std::int64_t>(),
                            M.k9_tn.as<std::int32_t>(), M.k9_doff.as<std::int64_t>(), M.k9_ld.as<std::int32_t>(),
                            M.k9_tr.as<std::int32_t>(), I.D.as<double>(), M.xp.as<double>(), M.n, mm,
                            M.yp.as<double>());
    });
  for (Index c = 0; c < (block_rhs ? 0 : m); ++c) near_gemv_column(I, c, st);
}

// Far-field contribution added into yp on stream st: the leaf step of the
// downward pass (H^2, after far_chain) or the S H T^T products (H form).
void far_finish(DevInstance& I, Index m, cudaStream_t st) {
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  Context& ctx = *M.ctx;
  const int mm = static_cast<int>(m);
  if (M.h2) {
    ctx.run_on(st, "leaf_bwd", [&] {
      dev::launch_leaf_bwd(st, M.leaves_local.as<std::int32_t>(), M.n_leaves_local, M.node_begin.as<std::int64_t>(),
                           M.node_count.as<std::int32_t>(), M.U.as<double>(), M.n, M.d, M.ps, M.P,
                           M.yhat.as<double>(), mm, H.row_begin, H.row_end, M.yp.as<double>());
    });
    return;
  }
  for (int l = 0; l <= H.tree->l_max; ++l) {
    const auto r = M.fh_level_range[l];
    if (r.second == r.first) continue;
    const int b0 = M.fh_items_h[r.first].bbeg, b1 = M.fh_items_h[r.second - 1].bend;
    for (Index c = 0; c < m; ++c)
      ctx.run_on(st, "far_h", [&] {
        dev::launch_far_h(st, M.fh_items.as<dev::FarHItem>(), r.first, r.second - r.first,
                          M.fh_bitem.as<std::int32_t>(), b0, b1 - b0, M.fh_tb.as<std::int64_t>(),
                          M.fh_tn.as<std::int32_t>(), M.fh_cls.as<std::int32_t>(), M.fh_soff.as<std::int64_t>(),
                          M.fh_toff.as<std::int64_t>(), M.fh_poff.as<std::int64_t>(), M.cmeta.as<dev::ClassMeta>(),
                          M.fh_S.as<double>(), M.fh_T.as<double>(), I.H.as<double>(), M.xp.as<double>() + c * M.n,
                          M.fh_part.as<double>(), H.row_begin, H.row_end, M.yp.as<double>() + c * M.n);
      });
  }
}

// Computes this shard's rows of y in tree order into M.yp (n x m layout;
// only rows [row_begin, row_end) are defined) from xp (tree order). The H^2
// far chain runs on the side stream, concurrent with the near GEMV.
void apply_tree_order(DevInstance& I, Index m, Comm* ex = nullptr) {
  DevMatrix& M = *I.M;
  Context& ctx = *M.ctx;
  static const int overlap = [] {
    const char* e = std::getenv("PHM_APPLY_OVERLAP");
    return e ? std::atoi(e) : 1;
  }();
  if (M.h2 && overlap == 0) {  // serial: far chain, then the near GEMV
    far_chain(I, m, ctx.stream, 0, ex);
    near_product(I, m, ctx.stream);
    far_finish(I, m, ctx.stream);
    return;
  }
  if (M.h2 && overlap == 2) {  // serial: near GEMV first
    near_product(I, m, ctx.stream);
    far_chain(I, m, ctx.stream, 0, ex);
    far_finish(I, m, ctx.stream);
    return;
  }
  static const int apply_cp_per_sm = [] {  // diagnostics: coupling CTAs per SM in apply (0: full grid)
    const char* e = std::getenv("PHM_APPLY_COUPLING_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  if (M.h2) {
    ctx.fork();
    far_chain(I, m, ctx.side, apply_cp_per_sm * ctx.sms, ex, /*leaf_level_first=*/true);
  }
  near_product(I, m, ctx.stream);
  if (M.h2) ctx.join();
  far_finish(I, m, ctx.stream);
}

}  // namespace

// Runs body (a theta-independent launch sequence on the context's streams)
// through the instance's CUDA graph for key: the first call per key runs it
// directly (lazy allocations happen there), the second captures it, later
// calls replay it as one graph launch; a workspace move re-captures.
// Per-kernel timing (ctx.timing) and PHM_GRAPHS=0 take the direct path.
// Measured effect is within noise on the benchmarked configurations (C1-C3):
// their steps are dominated by kernel time, not by launch gaps.
template <typename F>
void run_graphed(DevInstance& I, int seq, const void* input, Index m, F&& body) {
  DevMatrix& M = *I.M;
  Context& ctx = *M.ctx;
  static const bool use = [] {
    const char* e = std::getenv("PHM_GRAPHS");
    return !(e && std::atoi(e) == 0);
  }();
  if (!use || ctx.timing) {
    body();
    return;
  }
  const auto key = std::make_tuple(seq, input, m);
  if (I.graphs.find(key) == I.graphs.end() && I.graphs.size() >= DevInstance::kMaxGraphs) {
    auto lru = I.graphs.begin();
    for (auto it = I.graphs.begin(); it != I.graphs.end(); ++it)
      if (it->second.last_use < lru->second.last_use) lru = it;
    if (lru->second.exec) CK(cudaGraphExecDestroy(lru->second.exec));
    I.graphs.erase(lru);
  }
  DevInstance::Graph& g = I.graphs[key];
  g.last_use = ++I.graph_tick;
  if (!g.seen || g.ws_gen != M.ws_gen) {
    if (g.exec) CK(cudaGraphExecDestroy(g.exec));
    g.exec = nullptr;
    g.seen = true;
    g.ws_gen = M.ws_gen;
    body();
    return;
  }
  if (!g.exec) {
    cudaGraph_t graph = nullptr;
    const std::int64_t l0 = ctx.launches;
    CK(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(ctx.stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    CK(cudaStreamEndCapture(ctx.stream, &graph));
    if (Context::stamps_on()) {
      size_t nn = 0;
      CK(cudaGraphGetNodes(graph, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
      int nk = 0, np = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        ++nk;
        cudaKernelNodeAttrValue v{};
        CK(cudaGraphKernelNodeGetAttribute(nd, cudaKernelNodeAttributePriority, &v));
        if (v.priority != 0) ++np;
      }
      std::fprintf(stderr, "graph: %zu nodes, %d kernels, %d with priority\n", nn, nk, np);
    }
    // keep the side stream's priority per node (a graph otherwise runs every
    // node at the priority of the stream it is launched into)
    CK(cudaGraphInstantiate(&g.exec, graph, cudaGraphInstantiateFlagUseNodePriority));
    CK(cudaGraphDestroy(graph));
    g.launches = ctx.launches - l0;
    ctx.launches = l0;  // counted when the graph runs
  }
  CK(cudaGraphLaunch(g.exec, ctx.stream));
  ctx.launches += g.launches;
}

void apply_device(DevInstance& I, const double* x_dev, double* y_dev, Index m) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  NvtxRange nvtx("phm::apply");
  DevMatrix& M = *I.M;
  PHM_CHECK(m >= 1, "apply: m must be >= 1");
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  M.ctx->run("gather", [&] { dev::launch_gather(st, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
  run_graphed(I, 0, nullptr, m, [&] { apply_tree_order(I, m); });
  M.ctx->run("scatter", [&] { dev::launch_scatter(st, M.yp.as<double>(), M.perm.as<std::int32_t>(), M.n, m, y_dev); });
}

void apply_host(DevInstance& I, const double* x, double* y, Index m) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  if (H.row_begin != 0 || H.row_end != M.n)
    throw std::logic_error("apply on a row shard: use the sharded apply and gather y across ranks");
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  CK(cudaMemcpyAsync(M.xdev.p, x, sizeof(double) * M.n * m, cudaMemcpyHostToDevice, st));
  apply_device(I, M.xdev.as<double>(), M.ydev.as<double>(), m);
  CK(cudaMemcpyAsync(y, M.ydev.p, sizeof(double) * M.n * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}
// The launch sequence of instantiate(theta) + apply(x) after put_theta (H^2,
// snapshot or TT near mode): the class stage and the whole H^2 far chain on
// the side stream, the near stage (fused with the GEMV for one vector in
// snapshot mode) on the main stream. It depends on theta only through
// M.theta_dev, so it is graph-captured per (instance, x, m).
void instantiate_apply_sequence(DevInstance& I, const double* x_dev, Index m, StageCounters* counters,
                                Comm* ex = nullptr) {
  DevMatrix& M = *I.M;
  Context& ctx = *M.ctx;
  cudaStream_t st = ctx.stream, fs = ctx.side;
  ctx.stamp(st, 0);
  ctx.fork();  // side stream sees x (and everything before) as ready
  ctx.stamp(fs, 1);
  ctx.run_on(fs, "gather", [&] { dev::launch_gather(fs, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
  ctx.stamp(fs, 9);
  CK(cudaEventRecord(ctx.aux_ev, fs));
  // PHM_CLASS_PER_SM=k: k class CTAs per SM beside the fused near pass
  // (k_class_inst_pf as a persistent loop) instead of one CTA per class.
  // Measured on row shard 8 of 8 at C3 and not the default: with k = 1 the
  // near pass starts at once but runs a CTA short per SM while the class
  // stage takes 2x longer (1.277 -> 1.314 ms per step); k = 2 equals the
  // full grid (1.274).
  static const int class_per_sm = [] {
    const char* e = std::getenv("PHM_CLASS_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  const bool fuse_near = M.near_tma && M.mode == NearMode::Snapshot && m == 1;
  inst_classes(I, fs, fuse_near && class_per_sm > 0 ? class_per_sm * ctx.sms : 0);
  ctx.stamp(fs, 2);
  // The coupling as a capped grid that stays resident beside the fused near
  // pass (one CTA per SM where it fits next to the pass's two) instead of
  // taking the pass's SM slots as its CTAs retire: C3 9.6 -> 9.2 ms per step
  // (DESIGN.md). PHM_COUPLING_RESIDENT=0 restores the full grid.
  static const int resident_env = [] {
    const char* e = std::getenv("PHM_COUPLING_RESIDENT");
    return e ? std::atoi(e) : -1;
  }();
  static const bool use_fused = [] {
    const char* e = std::getenv("PHM_FUSED_NEAR");
    return !(e && std::atoi(e) == 0);
  }();
  const bool fuse = use_fused && M.near_tma && M.mode == NearMode::Snapshot && m == 1;
  // Only for a long near pass (>= 16 GB streamed, ~2.5 ms): the capped grid
  // needs about 8x the full grid's time, which a short pass does not cover
  // (row shard 8 of C3: 1.48 vs 1.44 ms per step; shard 4 of 4: equal).
  const bool long_pass = 8.0 * static_cast<double>(M.E_rank) >= 16e9;
  int coupling_ctas = 0;
  if (fuse && M.cp_mma && resident_env != 0 && (long_pass || resident_env > 0)) {
    const int fit = dev::coupling_beside_near(M.R_snap, M.P);
    const int per_sm = resident_env > 0 ? resident_env : std::min(fit, 1);
    coupling_ctas = per_sm * ctx.sms;
  }
  far_chain(I, m, fs, coupling_ctas, ex);
  bool fused = false;
  // Snapshot mode, one vector: K1 and K6 fused into one TMA pass over the
  // snapshots (k_near_tma) -- 10.8 ms at C3 against 9.8 + 1.6 ms for the
  // separate kernels. D is bit-identical to K1's; y agrees with the separate
  // path to rounding (row sums are accumulated in a different order).
  // PHM_FUSED_NEAR=0 selects the separate kernels.
  if (fuse) {
    // one pass over the snapshots: D is formed, stored and multiplied at once
    inst_snapshot_w(I, st);
    ctx.stamp(st, 10);
    CK(cudaStreamWaitEvent(st, ctx.aux_ev, 0));  // xp gathered
    ctx.stamp(st, 3);
    ctx.run_on(st, "near_inst_mvm", [&] {
      fused = dev::launch_near_inst_tma(st, M.sym_items.as<dev::SymRowItem>(), M.n_sym_items,
                                        M.sym_blocks.as<dev::SymBlock>(), M.G.as<double>(), M.E, M.R_snap,
                                        I.w.as<double>(), I.D.as<double>(), M.xp.as<double>(),
                                        M.sym_part.as<double>());
    });
    ctx.stamp(st, 4);
    if (fused) {
      if (M.n_gather_leaves == 0 || M.sharded) CK(cudaMemsetAsync(M.yp.p, 0, sizeof(double) * M.n * m, st));
      near_gather(I, 0, st);
    }
  }
  if (!fused) {
    inst_near(I, nullptr, st, counters, M.h2 ? 1 : 2);
    CK(cudaStreamWaitEvent(st, ctx.aux_ev, 0));  // xp gathered
    near_product(I, m, st);
  }
  ctx.stamp(fs, 7);
  ctx.join();
  far_finish(I, m, st);
  ctx.stamp(st, 8);
}

namespace {
// instantiate(theta) + apply(x) leaving y (this shard's part) in tree order
// in M.yp: put_theta, then instantiate_apply_sequence (replayed as a CUDA
// graph). H form and direct mode run instantiate and apply one after the
// other. y equals reinstantiate() + apply_device() to rounding (D bitwise).
void instantiate_apply_tree(DevInstance& I, const double* theta, int n_theta, const double* x_dev, Index m,
                            StageCounters* counters, Comm* ex = nullptr) {
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  PHM_CHECK(m >= 1, "apply: m must be >= 1");
  if (M.baseline) throw std::logic_error("instantiate: a baseline matrix is built at a fixed theta");
  CK(cudaSetDevice(M.ctx->device));
  const auto v = parametric_vectors(H.grids, theta, n_theta);
  const dev::ThetaV tv = make_theta_v(v);
  ensure_workspace(M, m);
  if (!M.h2 || M.mode == NearMode::Direct) {
    run_instantiate(I, theta, n_theta, counters);
    cudaStream_t st = M.st();
    M.ctx->run("gather", [&] { dev::launch_gather(st, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
    apply_tree_order(I, m, ex);
    return;
  }
  I.theta.assign(theta, theta + n_theta);
  Context& ctx = *M.ctx;
  put_theta(M, v, tv, ctx.stream);  // the only theta-dependent launch
  if (ex == nullptr)
    run_graphed(I, 1, x_dev, m, [&] { instantiate_apply_sequence(I, x_dev, m, counters); });
  else if (ex->capturable())
    run_graphed(I, 2, x_dev, m, [&] { instantiate_apply_sequence(I, x_dev, m, counters, ex); });
  else
    instantiate_apply_sequence(I, x_dev, m, counters, ex);
}
}  // namespace

void instantiate_apply_device(DevInstance& I, const double* theta, int n_theta, const double* x_dev, double* y_dev,
                              Index m, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  NvtxRange nvtx("phm::instantiate_apply");
  DevMatrix& M = *I.M;
  if (M.sharded)
    throw std::logic_error("fused instantiate+apply on a row shard: use the partial apply and sum across ranks");
  instantiate_apply_tree(I, theta, n_theta, x_dev, m, counters);
  M.ctx->run("scatter", [&] {
    dev::launch_scatter(M.st(), M.yp.as<double>(), M.perm.as<std::int32_t>(), M.n, m, y_dev);
  });
  M.ctx->print_stamps();
}

// The sharded HPO step as one library call: this rank's
// instantiate + partial apply (its near blocks -- with symmetric storage also
// the transposed products that land on other ranks' rows -- its far blocks,
// its share of the forward pass), the x-hat all-reduce between the forward
// pass and the coupling, the y all-reduce of the tree-order partials on the
// context stream, and the un-permute into y (original point order, every
// rank). With an NCCL comm the whole sequence is captured as one CUDA graph.
void instantiate_apply_sharded(DevInstance& I, Comm& ex, const double* theta, int n_theta, const double* x_dev,
                               double* y_dev, Index m, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  NvtxRange nvtx("phm::instantiate_apply_sharded");
  DevMatrix& M = *I.M;
  PHM_CHECK(ex.world == M.hm->cfg.shard_count && ex.rank == M.hm->cfg.shard_rank,
            "sharded step: communicator rank / world differ from the matrix's shard");
  instantiate_apply_tree(I, theta, n_theta, x_dev, m, counters, &ex);
  // world 1 still runs the (local) all-reduce: the same path as at N > 1
  ex.allreduce(M.yp.as<double>(), M.n * m, M.st());
  M.ctx->run("scatter", [&] {
    dev::launch_scatter(M.st(), M.yp.as<double>(), M.perm.as<std::int32_t>(), M.n, m, y_dev);
  });
  M.ctx->print_stamps();
}

void instantiate_apply_sharded_host(DevInstance& I, Comm& ex, const double* theta, int n_theta, const double* x,
                                    double* y, Index m, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  CK(cudaMemcpyAsync(M.xdev.p, x, sizeof(double) * M.n * m, cudaMemcpyHostToDevice, st));
  instantiate_apply_sharded(I, ex, theta, n_theta, M.xdev.as<double>(), M.ydev.as<double>(), m, counters);
  CK(cudaMemcpyAsync(y, M.ydev.p, sizeof(double) * M.n * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void apply_sharded(DevInstance& I, Comm& ex, const double* x_dev, double* y_dev, Index m) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  NvtxRange nvtx("phm::apply_sharded");
  DevMatrix& M = *I.M;
  PHM_CHECK(ex.world == M.hm->cfg.shard_count && ex.rank == M.hm->cfg.shard_rank,
            "sharded apply: communicator rank / world differ from the matrix's shard");
  PHM_CHECK(m >= 1, "apply: m must be >= 1");
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  M.ctx->run("gather", [&] { dev::launch_gather(st, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
  if (ex.capturable())
    run_graphed(I, 3, nullptr, m, [&] { apply_tree_order(I, m, &ex); });
  else
    apply_tree_order(I, m, &ex);
  ex.allreduce(M.yp.as<double>(), M.n * m, st);
  M.ctx->run("scatter", [&] { dev::launch_scatter(st, M.yp.as<double>(), M.perm.as<std::int32_t>(), M.n, m, y_dev); });
}

void instantiate_apply_partial_device(DevInstance& I, const double* theta, int n_theta, const double* x_dev,
                                      double* ypart_dev, Index m, StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  instantiate_apply_tree(I, theta, n_theta, x_dev, m, counters);
  CK(cudaMemcpyAsync(ypart_dev, M.yp.p, sizeof(double) * M.n * m, cudaMemcpyDeviceToDevice, M.st()));
}

// estimate_error (harness.cpp:183-236) for this instance: probe rows J
// sampled without replacement and x ~ U[0,1) from Rng(mix_seed(seed,
// "erro")), exact rows (K x)_J evaluated directly on the GPU (charged to the
// audit counter), approximate rows from the GPU MVM; returns
// ||exact - approx||_J / ||exact||_J.
double estimate_error(DevInstance& I, Index probe_rows, std::uint64_t seed, StageCounters* counters,
                      std::vector<Index>* rows_out, std::vector<double>* exact_out, std::vector<double>* approx_out,
                      std::vector<double>* x_out) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  const Tree& T = *H.tree;
  const KernelSpec& spec = H.cfg.spec;
  if (spec.family == kMatern) throw std::invalid_argument("estimate_error on the GPU needs a closed-form kernel");
  PHM_CHECK(probe_rows >= 1, "estimate_error: probe_rows must be >= 1");
  const Index n = M.n;
  Rng rng(mix_seed(seed, 0x6572726fULL));
  std::vector<Index> all(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) all[i] = i;
  const Index m = std::min<Index>(probe_rows, n);
  for (Index i = 0; i < m; ++i) std::swap(all[i], all[i + static_cast<Index>(rng.integer(n - i))]);
  all.resize(static_cast<size_t>(m));
  std::vector<double> x(static_cast<size_t>(n)), y(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) x[i] = rng.uniform();
  apply_host(I, x.data(), y.data(), 1);  // leaves x in tree order in M.xp
  std::vector<Index> inv(static_cast<size_t>(n));
  for (Index p = 0; p < n; ++p) inv[T.perm[p]] = p;
  std::vector<std::int64_t> pos(static_cast<size_t>(m));
  for (Index j = 0; j < m; ++j) pos[j] = inv[all[j]];
  std::vector<double> th(3, 1.0);
  for (int k = 0; k < spec.shape_params(); ++k) th[k] = I.theta[k];
  const double amp = spec.amplitude ? I.theta[spec.shape_params()] : 1.0;
  DBuf dpos, dth, dout;
  cudaStream_t st = M.st();
  upload(dpos, pos, st);
  upload(dth, th, st);
  dout.alloc(sizeof(double) * m);
  M.ctx->run("exact_rows", [&] {
    dev::launch_exact_rows(st, dpos.as<std::int64_t>(), static_cast<int>(m), M.pts.as<double>(), n, M.d, spec.family,
                           dth.as<double>(), amp, M.xp.as<double>(), dout.as<double>());
  });
  std::vector<double> exact(static_cast<size_t>(m));
  CK(cudaMemcpyAsync(exact.data(), dout.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (counters) counters->audit.add(static_cast<std::uint64_t>(m * n));
  double num = 0.0, den = 0.0;
  std::vector<double> approx(static_cast<size_t>(m));
  for (Index j = 0; j < m; ++j) {
    approx[j] = y[all[j]];
    const double diff = exact[j] - approx[j];
    num += diff * diff;
    den += exact[j] * exact[j];
  }
  if (rows_out) *rows_out = all;
  if (exact_out) *exact_out = exact;
  if (approx_out) *approx_out = approx;
  if (x_out) *x_out = x;
  return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

void instantiate_apply_host(DevInstance& I, const double* theta, int n_theta, const double* x, double* y, Index m,
                            StageCounters* counters) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  CK(cudaMemcpyAsync(M.xdev.p, x, sizeof(double) * M.n * m, cudaMemcpyHostToDevice, st));
  instantiate_apply_device(I, theta, n_theta, M.xdev.as<double>(), M.ydev.as<double>(), m, counters);
  CK(cudaMemcpyAsync(y, M.ydev.p, sizeof(double) * M.n * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void apply_device_partial(DevInstance& I, const double* x_dev, double* ypart_dev, Index m) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  PHM_CHECK(m >= 1, "apply: m must be >= 1");
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  M.ctx->run("gather", [&] { dev::launch_gather(st, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
  apply_tree_order(I, m);
  CK(cudaMemcpyAsync(ypart_dev, M.yp.p, sizeof(double) * M.n * m, cudaMemcpyDeviceToDevice, st));
}

void apply_device_rows(DevInstance& I, const double* x_dev, double* yrows_dev, Index m) {
  std::lock_guard<std::recursive_mutex> exec_lock(I.M->exec_mu());
  DevMatrix& M = *I.M;
  const HostMatrix& H = *M.hm;
  if (M.sym && M.sharded)
    throw std::logic_error(
        "symmetric near storage on a row shard: rows of y get contributions from other ranks; use the partial "
        "apply and sum across ranks (or build with symmetric_near = 0)");
  CK(cudaSetDevice(M.ctx->device));
  ensure_workspace(M, m);
  cudaStream_t st = M.st();
  M.ctx->run("gather", [&] { dev::launch_gather(st, x_dev, M.perm.as<std::int32_t>(), M.n, m, M.xp.as<double>()); });
  apply_tree_order(I, m);
  const Index rows = H.row_end - H.row_begin;
  if (rows > 0)
    CK(cudaMemcpy2DAsync(yrows_dev, rows * sizeof(double), M.yp.as<double>() + H.row_begin, M.n * sizeof(double),
                         rows * sizeof(double), m, cudaMemcpyDeviceToDevice, st));
}

void unpermute_device(DevMatrix& M, const double* yperm_dev, double* y_dev, Index mcols) {
  CK(cudaSetDevice(M.ctx->device));
  M.ctx->run("scatter", [&] {
    dev::launch_scatter(M.st(), yperm_dev, M.perm.as<std::int32_t>(), M.n, mcols, y_dev);
  });
}

}  // namespace phm
