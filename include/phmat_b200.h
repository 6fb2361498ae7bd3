/*
 * phmat_b200 — C ABI of the B200-native online stage of parametric H / H^2
 * matrices (arXiv 2511.03109).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (/root/reference/proj) is a C++ library with no FFI of its own (its
 * python module is an empty pybind11 stub, proj/python/phmat_module.cpp:1-2),
 * so the entry points below mirror its public C++ API, one C function per
 * reference entry point, with plain pointers and sizes:
 *
 *   phm_matrix_build       <- phmat::offline_h / offline_h2
 *                             (proj/include/phmat/phmatrix.hpp:82-91)
 *   phm_instantiate        <- phmat::instantiate(pm, theta, counter)
 *                             (proj/include/phmat/phmatrix.hpp:133-138,
 *                              proj/src/phmatrix.cpp:168-225)
 *   phm_apply              <- LinearOperator::apply / Instantiated{H,H2}Matrix::apply
 *                             (proj/include/phmat/phmatrix.hpp:95-128,
 *                              proj/src/phmatrix.cpp:227-269), plus m > 1
 *   phm_instance_far_h     <- InstantiatedXMatrix::far_h[i]   (phmatrix.hpp:105,119)
 *   phm_instance_near_d    <- InstantiatedXMatrix::near_d[i]  (phmatrix.hpp:106,120)
 *   phm_to_dense           <- InstantiatedXMatrix::to_dense   (phmatrix.hpp:110,124)
 *   phm_matrix_metrics     <- phmat::metrics                  (phmatrix.hpp:141-153)
 *   phm_matrix_perm/nodes/blocks/class_keys
 *                          <- ClusterTree / BlockClusterTree / far_key views
 *                             (geometry.hpp:49-92, phmatrix.hpp:56-57)
 *   phm_parametric_vectors <- phmat::parametric_vectors       (farfield.hpp:31-34)
 *   phm_generate_points    <- phmat::generate_points          (harness.hpp:77)
 *
 * Conventions: every function returns PHM_OK (0) or an error code; no C++
 * exception crosses the ABI. The code maps back to the reference's exception
 * types (domain_error, invalid_argument, logic_error, runtime_error) and
 * phm_last_error() returns the message (thread-local). Matrices are
 * column-major doubles; point sets are n x d row-major (the reference's
 * Eigen row access order). Vectors are in the ORIGINAL point order, as in the
 * reference; the tree-order permutation is internal.
 */
#ifndef PHMAT_B200_H_
#define PHMAT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum phm_status {
  PHM_OK = 0,
  PHM_ERR_RUNTIME = 1,   /* std::runtime_error (size guards, artifact problems) */
  PHM_ERR_DOMAIN = 2,    /* std::domain_error  (theta outside the box) */
  PHM_ERR_INVALID = 3,   /* std::invalid_argument (length mismatch, bad spec) */
  PHM_ERR_LOGIC = 4,     /* std::logic_error   (PHMAT_CHECK failures) */
  PHM_ERR_CUDA = 5,      /* CUDA runtime failure / no sm_100 device */
  PHM_ERR_RANGE = 6      /* index out of range */
};

/* Kernel families: reference ids e, tps, se, mc, mn (kernels.hpp:14-23) plus
 * the single-parameter Gaussian and Matern-3/2, -5/2 families. */
enum phm_family {
  PHM_KERNEL_E = 0,
  PHM_KERNEL_TPS = 1,
  PHM_KERNEL_SE = 2,
  PHM_KERNEL_MC = 3,
  PHM_KERNEL_MN = 4,
  PHM_KERNEL_GAUSS = 5,
  PHM_KERNEL_MATERN32 = 6,
  PHM_KERNEL_MATERN52 = 7
};

enum phm_format { PHM_FORMAT_H = 0, PHM_FORMAT_H2 = 1 };
/* Near-field modes: the reference's TT and Direct (phmatrix.hpp:18) plus
 * Snapshot (full-rank NearBlockTT generated on the GPU). */
enum phm_near_mode { PHM_NEAR_TT = 0, PHM_NEAR_DIRECT = 1, PHM_NEAR_SNAPSHOT = 2 };

/* PHConfig (phmatrix.hpp:20-35) + KernelSpec (kernels.hpp:31-38) + the
 * extensions of SURVEY.md Appendix A (amplitude parameter, per-dimension
 * p_theta) + row sharding for multi-GPU. */
typedef struct phm_config {
  int32_t family;
  int32_t amplitude;   /* 1: trailing theta component sigma^2 multiplies the kernel */
  int32_t d_theta;
  int32_t p_theta[3];
  double theta_lo[3];
  double theta_hi[3];
  int32_t format;
  int32_t l_max;
  int32_t p_s;
  int32_t near_mode;
  double eps;
  double eta;          /* <= 0 selects sqrt(d) */
  int64_t r_max_far;
  int64_t r_max_near;
  uint64_t seed;
  int32_t translation_cache;
  int32_t threads;     /* 0: PHMAT_THREADS / hardware */
  int32_t shard_rank;
  int32_t shard_count;
  int32_t symmetric_near; /* snapshot mode: store sigma <= tau blocks only (D_ts = D_st^T) */
  int32_t reserved;
} phm_config;

/* StructureMetrics (phmatrix.hpp:141-153) + build statistics. */
typedef struct phm_info {
  int64_t n, d, nodes, n_near, n_far, n_classes, c_sp, constructed;
  int64_t P;                 /* p_s^d */
  int64_t row_begin, row_end;/* tree-order rows owned by this shard */
  int64_t near_entries;      /* sum over local near blocks of n_sigma n_tau */
  int64_t near_stored;       /* near entries actually stored (symmetric storage halves them) */
  int64_t near_stream_elems; /* sum of n_sigma n_tau (R_b + 1): K1's algorithmic elements */
  int64_t device_bytes;
  int64_t storage_entries;
  double storage_gb, nf_ratio, ff_ratio, coupling_ratio, rank;
  double tree_s, ff_s, nf_s, upload_s;
  uint64_t evals_offline, evals_online, evals_audit;
  int32_t any_rank_capped;
  int32_t pad;
} phm_info;

typedef struct phm_context_s* phm_context;
typedef struct phm_matrix_s* phm_matrix;
typedef struct phm_instance_s* phm_instance;

const char* phm_last_error(void);
int phm_version(void);
void phm_config_default(phm_config* cfg);

/* Context: one CUDA device and one stream (own, or a caller's stream). */
int phm_context_create(int device, phm_context* out);
int phm_context_destroy(phm_context ctx);
int phm_context_set_stream(phm_context ctx, void* cuda_stream);
int phm_context_get_stream(phm_context ctx, void** cuda_stream);
int phm_context_sync(phm_context ctx);
/* CUDA-event timing of every kernel launch, aggregated by kernel name. */
int phm_context_enable_timing(phm_context ctx, int on);
int phm_context_timer(phm_context ctx, const char* name, double* total_ms, int64_t* launches);
int phm_context_reset_timers(phm_context ctx);
int phm_context_launches(phm_context ctx, int64_t* launches);

/* Offline build (host structure + TT-cross, upload, GPU snapshots). */
int phm_matrix_build(phm_context ctx, const double* points, int64_t n, int d, const phm_config* cfg,
                     phm_matrix* out);
/* Host-only build (no device): structure + offline TT data for inspection;
 * instantiate / apply on such a handle fail with PHM_ERR_LOGIC. */
int phm_matrix_build_host(const double* points, int64_t n, int d, const phm_config* cfg, phm_matrix* out);
/* HMAT v1 artifacts, byte-compatible with the reference's save_parametric /
 * load_parametric_{h,h2} / artifact_is_h2 (serialize.cpp:108-294): load
 * rebuilds and validates the tree and block lists, then uploads the stored
 * TT data (threads = host threads for the L/R assembly, 0 = all). */
int phm_matrix_load(phm_context ctx, const char* path, int threads, phm_matrix* out);
int phm_matrix_load_host(const char* path, int threads, phm_matrix* out); /* no device (inspection) */
int phm_matrix_save(phm_matrix m, const char* path);
int phm_artifact_is_h2(const char* path, int* is_h2);
/* The matrix's configuration (e.g. after phm_matrix_load). */
int phm_matrix_config(phm_matrix m, phm_config* out);
int phm_matrix_destroy(phm_matrix m);
int phm_matrix_info(phm_matrix m, phm_info* info);
/* Structure views (bit-exact with the reference's tree and block lists). */
int phm_matrix_perm(phm_matrix m, int32_t* perm /* n */);
int phm_matrix_nodes(phm_matrix m, int32_t* ints /* 7 per node: level,parent,first_child,count,coords[3] */,
                     double* boxes /* 6 per node: lo[3], hi[3] */);
int phm_matrix_blocks(phm_matrix m, int32_t* near_pairs /* 2 per near block */,
                      int32_t* far_pairs /* 2 per far block */, int32_t* far_key /* per far block */);
int phm_matrix_class_keys(phm_matrix m, int64_t* keys /* 4 per class: level, offset[3] */);
int phm_matrix_theta_grid(phm_matrix m, int k, double* nodes /* p_theta[k] */);
/* Offline payload views, two-call pattern: pass data == NULL to get sizes.
 * dims: 3 per core (r0, m, r1); *ncores <= 10. */
int phm_matrix_coupling(phm_matrix m, int64_t cls, int32_t* ncores, int64_t* dims, double* data, int64_t* len);
int phm_matrix_near_tt(phm_matrix m, int64_t near_block, int32_t* ncores, int64_t* dims, double* data, int64_t* len);
int phm_matrix_near_rank(phm_matrix m, int64_t near_block, int64_t* rank);
int phm_matrix_near_column(phm_matrix m, int64_t near_block, int64_t kap, double* out /* n_sigma n_tau */);
int phm_matrix_far_st(phm_matrix m, int64_t far_index, double* S, double* T, int64_t* dims /* 4 */);
int phm_matrix_class_lr(phm_matrix m, int64_t cls, double* L, double* R, int64_t* dims /* 4 */);
int phm_parametric_vectors(phm_matrix m, const double* theta, int n_theta, double* out /* sum p_theta */);

/* Online stage. */
int phm_instantiate(phm_matrix m, const double* theta, int n_theta, phm_instance* out);
int phm_reinstantiate(phm_instance inst, const double* theta, int n_theta);
/* Non-parametric baselines at one fixed theta (proj/include/phmat/baselines.hpp):
 * PHM_BASELINE_H_ACA = HAcaMatrix (baselines.hpp:27-50: ACA far blocks,
 * dense near blocks), PHM_BASELINE_H2_HCA = H2HcaMatrix (:52-82: ACA of the
 * Chebyshev node-interaction matrices per translation class, nested basis
 * shared with the parametric build). Factorisation on the host (the
 * reference's aca_engine, aca_impl.hpp:34-173), near blocks evaluated on the
 * GPU; the returned instance applies through phm_apply / phm_to_dense like a
 * parametric one (LinearOperator, harness.cpp:314-336). The config supplies
 * the kernel, tree depth, eta and p_s (H^2-HCA); eps and r_max are the ACA's.
 * phm_instantiate / phm_reinstantiate reject baseline instances. */
enum { PHM_BASELINE_H_ACA = 1, PHM_BASELINE_H2_HCA = 2 };
typedef struct phm_baseline_info {
  int32_t method;
  int32_t any_capped;      /* some ACA hit r_max */
  double mean_far_rank;    /* HAcaMatrix::mean_far_rank / H2HcaMatrix::mean_far_rank */
  double coupling_ratio;   /* H2HcaMatrix::coupling_ratio, (2/n^2) sum_b p_s^d t_b; 0 for H-ACA */
  double far_build_s;      /* host ACA time (far_build_seconds) */
  double near_build_s;     /* device near evaluation time (near_build_seconds) */
  uint64_t far_evals;      /* kernel evaluations of the ACAs */
  uint64_t near_evals;     /* dense near entries evaluated */
  int64_t n_far, n_near, n_classes;
} phm_baseline_info;
int phm_baseline_build(phm_context ctx, const double* points, int64_t n, int d, const phm_config* cfg, int method,
                       const double* theta, int n_theta, double eps, int64_t r_max, phm_instance* out);
int phm_baseline_info_get(phm_instance inst, phm_baseline_info* out);
/* aca_partial (baselines.hpp:22-24) on a dense m x n column-major matrix:
 * A ~ V Y^T, V m x rank, Y n x rank (buffers of min(m, n, r_max) columns). */
int phm_aca_partial_dense(const double* a, int64_t m, int64_t n, double eps, int64_t r_max, uint64_t seed,
                          int64_t* rank, int32_t* capped, double* v, double* y);

/* theta-batched instantiate for sweeps: count thetas
 * (count x n_theta, row-major) -> count instances in out[]. Snapshot mode
 * reads the snapshots once for the whole batch (K1 batch kernel); every D is
 * bit-identical to phm_instantiate's. Each instance is destroyed with
 * phm_instance_destroy. Replaces a loop of instantiate(pm, theta) calls
 * (harness.cpp:293-312 per theta). */
int phm_instantiate_batch(phm_matrix m, const double* thetas, int n_theta, int count, phm_instance* out);
/* In place: instances of one matrix re-instantiated at count thetas. */
int phm_reinstantiate_batch(phm_instance* insts, int count, const double* thetas, int n_theta);
int phm_instance_destroy(phm_instance inst);
int phm_instance_sync(phm_instance inst);
int phm_instance_far_h(phm_instance inst, int64_t far_index, double* out, int64_t* rows, int64_t* cols);
int phm_instance_near_d(phm_instance inst, int64_t near_block, double* out);
int phm_instance_class_c(phm_instance inst, int64_t cls, double* out /* P x P, column-major (the device keeps P = 64 in DMMA fragment order and converts here) */);
/* y = K(theta) x, host buffers, n_rows must equal n (length check before
 * any launch, phmatrix.cpp:228); m right-hand sides, column-major. */
int phm_apply(phm_instance inst, const double* x, int64_t n_rows, double* y, int64_t m);
/* reinstantiate(theta) followed by apply(x) in one call (the HPO step): the
 * class stage and the H^2 far chain overlap the near-field instantiate
 * stream; results equal phm_reinstantiate + phm_apply. */
int phm_instantiate_apply(phm_instance inst, const double* theta, int n_theta, const double* x, int64_t n_rows,
                          double* y, int64_t m);
int phm_instantiate_apply_device(phm_instance inst, const double* theta, int n_theta, const double* x_dev,
                                 double* y_dev, int64_t m);
/* Device buffers, asynchronous on the context stream. */
int phm_apply_device(phm_instance inst, const double* x_dev, double* y_dev, int64_t m);
/* Row-sharded apply: this shard's rows [row_begin, row_end) of y in tree
 * order (rows x m, column-major); gather across ranks, then unpermute. */
int phm_apply_rows_device(phm_instance inst, const double* x_dev, double* yrows_dev, int64_t m);
/* Row-sharded apply with symmetric near storage (each rank stores the near
 * pairs its owner leaves hold, so its transposed products reach other
 * ranks' rows): this shard's full-length partial y in tree order (n x m);
 * sum the partials across ranks (all-reduce), then unpermute. Also valid on
 * an unsharded matrix (the partial is then y itself, in tree order). */
int phm_apply_partial_device(phm_instance inst, const double* x_dev, double* ypart_dev, int64_t m);
/* phm_reinstantiate(theta) + phm_apply_partial_device in one schedule (the
 * sharded HPO step). */
int phm_instantiate_apply_partial_device(phm_instance inst, const double* theta, int n_theta, const double* x_dev,
                                         double* ypart_dev, int64_t m);
int phm_unpermute_device(phm_matrix m, const double* yperm_dev, double* y_dev, int64_t mcols);

/* Multi-GPU inside the library: one process per GPU, each
 * holding the row shard cfg.shard_rank of cfg.shard_count. A communicator
 * carries the two exchanges of the sharded step, both in-place sum
 * all-reduces on the context stream: x-hat (nodes x P per RHS) between each
 * rank's share of the forward pass and the coupling, and the tree-order
 * partial y at the end. It replaces the caller-side loop of
 * run_experiment (proj/src/harness.cpp:287-352) over one shared matrix.
 *   NCCL: rank 0 calls phm_comm_unique_id and broadcasts the 128 bytes; every
 *   rank calls phm_comm_create_nccl (libnccl.so.2 is loaded at run time).
 *   Callback: fn(buf_dev, count, cuda_stream, user) must leave buf summed
 *   over the ranks, ordered on cuda_stream (used to test the sharded step
 *   with any transport, e.g. gloo). */
typedef struct phm_comm_s* phm_comm;
typedef int (*phm_allreduce_fn)(double* buf_dev, int64_t count, void* cuda_stream, void* user);
int phm_comm_unique_id(uint8_t* id /* 128 bytes */);
int phm_comm_create_nccl(phm_context ctx, const uint8_t* id /* 128 bytes */, int rank, int world, phm_comm* out);
int phm_comm_create_callback(phm_allreduce_fn fn, void* user, int rank, int world, phm_comm* out);
/* Single-GPU timing probe of one rank's sharded step: both exchanges are
 * no-ops (the partials stay partial; y is NOT the product). Diagnostics only. */
int phm_comm_create_probe(int rank, int world, phm_comm* out);
int phm_comm_destroy(phm_comm comm);
int phm_comm_info(phm_comm comm, int* rank, int* world, int* is_nccl);
/* reinstantiate(theta) + apply(x) on this rank's shard, exchanges included;
 * y (original point order, n x m) is complete on every rank. Device buffers
 * (asynchronous on the context stream; NCCL: one CUDA graph per step) or
 * host buffers (synchronous, like phm_instantiate_apply). */
int phm_instantiate_apply_sharded(phm_instance inst, phm_comm comm, const double* theta, int n_theta,
                                  const double* x_dev, double* y_dev, int64_t m);
int phm_instantiate_apply_sharded_host(phm_instance inst, phm_comm comm, const double* theta, int n_theta,
                                       const double* x, int64_t n_rows, double* y, int64_t m);
int phm_apply_sharded(phm_instance inst, phm_comm comm, const double* x_dev, double* y_dev, int64_t m);
/* estimate_error of the reference harness (harness.cpp:183-236): probe rows
 * sampled without replacement and x ~ U[0,1) from the reference's Rng
 * stream, exact rows (K x)_J by direct kernel evaluation on the GPU (audit
 * counted), ||exact - approx|| / ||exact|| over J. Outputs other than err are
 * optional (min(probe_rows, n) entries; x_out has n). */
int phm_estimate_error(phm_instance inst, int64_t probe_rows, uint64_t seed, double* err, int64_t* rows_out,
                       double* exact_out, double* approx_out, double* x_out);
/* Induced dense matrix (n x n column-major), refuses n > guard. */
int phm_to_dense(phm_instance inst, double* out, int64_t guard);

/* Seeded generators (harness.cpp:174-181; mixture and normal are new). */
int phm_generate_points(int64_t n, int d, uint64_t seed, double* out);
int phm_generate_mixture_points(int64_t n, int d, int clusters, double sigma, uint64_t seed, double* out);
int phm_generate_normal(int64_t n, uint64_t seed, double* out);
/* Offline TT tooling on a dense tensor (first index fastest): TT-cross with
 * the reference's options (tt.hpp:107-130, tt.cpp:269-480) and TT-rounding
 * (tt.cpp:159-224; abs_budget < 0 selects the relative form with eps).
 * Cores are written when cap >= *len; flags = {rank_capped, converged}. */
int phm_tt_cross_dense(const double* tensor, const int64_t* dims, int ndims, double eps, int64_t r_max,
                       uint64_t seed, int round_after, int32_t* ncores, int64_t* core_dims, double* core_data,
                       int64_t cap, int64_t* len, uint64_t* evals, int32_t* flags, double* est);
int phm_tt_round(int ncores_in, const int64_t* dims_in, const double* data_in, double eps, double abs_budget,
                 int32_t* ncores, int64_t* dims, double* data, int64_t cap, int64_t* len);
/* theta draws of run_experiment (harness.cpp:254-260), one parameter. */
int phm_theta_draws(double lo, double hi, int64_t count, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PHMAT_B200_H_ */
