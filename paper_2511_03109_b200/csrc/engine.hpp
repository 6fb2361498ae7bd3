// Engine interface between the C ABI (capi.cpp) and the CUDA layer
// (device.cu). Plain C++: no CUDA types cross this header.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "host/phm.hpp"

namespace phm {

struct Context;     // device, stream, timers
struct DevMatrix;   // parametric matrix resident on the GPU
struct DevInstance; // matrix instantiated at one theta
class Comm;         // rank-to-rank all-reduce (comm.hpp)

std::shared_ptr<Context> context_create(int device);
void context_set_stream(Context& ctx, void* stream);  // nullptr = own stream
void* context_stream(Context& ctx);
void context_sync(Context& ctx);
void context_enable_timing(Context& ctx, bool on);
// Sum of CUDA-event durations (ms) and launch count of the named kernel
// recorded since the last reset (synchronises the stream).
void context_timer(Context& ctx, const std::string& name, double* ms, std::int64_t* count);
void context_reset_timers(Context& ctx);
std::int64_t context_launches(Context& ctx);  // kernels launched so far
int context_device(const Context& ctx);

// Offline build: host structure + TT-cross (host), upload, and for
// NearMode::Snapshot the GPU snapshot generator (K11).
std::shared_ptr<DevMatrix> matrix_build(std::shared_ptr<Context> ctx, const double* points, Index n, int d,
                                        const Config& cfg);
// HMAT v1 artifact (proj/src/serialize.cpp format): load = rebuild +
// validate the structure, take the stored TT data, upload; save writes the
// reference-readable file (snapshot near data as full-rank TTs).
std::shared_ptr<DevMatrix> matrix_load(std::shared_ptr<Context> ctx, const std::string& path, int threads);
void matrix_save(const DevMatrix& m, const std::string& path);
std::shared_ptr<DevMatrix> matrix_load_host_only(const std::string& path, int threads);
// Host-only build: structure and offline TT data, no device (CPU tests).
std::shared_ptr<DevMatrix> matrix_build_host_only(const double* points, Index n, int d, const Config& cfg);
bool matrix_on_device(const DevMatrix& m);
const HostMatrix& matrix_host(const DevMatrix& m);
// Near payload actually resident on the device (bytes), and per-near-block
// rank R_b (0 for non-local blocks).
std::int64_t matrix_device_bytes(const DevMatrix& m);
std::int64_t matrix_near_rank(const DevMatrix& m, Index near_block);
// Device -> host copy of one snapshot / G1 column kap of a near block.
void matrix_near_column(const DevMatrix& m, Index near_block, Index kap, double* out);
// kind 0: sum over local near blocks of n_sigma n_tau (the logical near
// field); 1: entries actually stored (symmetric storage keeps sigma <= tau);
// 2: stored entries times (R_b + 1), the instantiate stream's elements.
std::int64_t matrix_near_elems(const DevMatrix& m, int kind);

std::shared_ptr<DevInstance> instantiate(std::shared_ptr<DevMatrix> m, const double* theta, int n_theta,
                                         StageCounters* counters);
// Baselines (baselines.hpp): H-ACA / H^2-HCA built at one theta; the
// instance holds the dense near blocks (evaluated on the device) and the
// fixed far field, and applies through the same kernels.
std::shared_ptr<DevMatrix> baseline_build(std::shared_ptr<Context> ctx, const double* points, Index n, int d,
                                          const Config& cfg, Baseline method, const double* theta, int n_theta,
                                          double eps, Index r_max);
std::shared_ptr<DevInstance> baseline_instance(std::shared_ptr<DevMatrix> m);
// Re-instantiate in place at a new theta (reuses the device buffers).
void reinstantiate(DevInstance& inst, const double* theta, int n_theta, StageCounters* counters);
// theta-batched instantiate (sweeps): count thetas (count x n_theta,
// row-major); in snapshot mode one K1 pass reads the snapshots once and
// writes every instance's D (bit-identical to single instantiates).
std::vector<std::shared_ptr<DevInstance>> instantiate_batch(std::shared_ptr<DevMatrix> m, const double* thetas,
                                                            int n_theta, int count, StageCounters* counters);
void reinstantiate_batch(const std::vector<DevInstance*>& insts, const double* thetas, int n_theta,
                         StageCounters* counters);
const std::vector<double>& instance_theta(const DevInstance& inst);
void instance_sync(DevInstance& inst);

// H_b(theta) of far block i (rows x cols, column-major), D_b of near block b
// (n_sigma x n_tau column-major), explicit C_k of class k (P x P).
void instance_far_h(DevInstance& inst, Index far_index, std::vector<double>& out, Index& rows, Index& cols);
void instance_near_d(DevInstance& inst, Index near_index, std::vector<double>& out);
void instance_class_c(DevInstance& inst, Index cls, std::vector<double>& out);

// y = K(theta) x for m right-hand sides (column-major n x m), original point
// order. Host variants copy in/out and synchronise; device variants are
// asynchronous on the context stream.
void apply_host(DevInstance& inst, const double* x, double* y, Index m);
// instantiate(theta) then apply(x) as one schedule: the class stage and the
// H^2 far chain overlap the near-field instantiate stream.
void instantiate_apply_device(DevInstance& inst, const double* theta, int n_theta, const double* x_dev, double* y_dev,
                              Index m, StageCounters* counters);
void instantiate_apply_host(DevInstance& inst, const double* theta, int n_theta, const double* x, double* y, Index m,
                            StageCounters* counters);
// estimate_error of harness.cpp:183-236 on the GPU (exact probe rows by
// direct kernel evaluation; audit-counted).
double estimate_error(DevInstance& inst, Index probe_rows, std::uint64_t seed, StageCounters* counters,
                      std::vector<Index>* rows_out, std::vector<double>* exact_out, std::vector<double>* approx_out,
                      std::vector<double>* x_out);
void apply_device(DevInstance& inst, const double* x_dev, double* y_dev, Index m);
// Sharded pieces: rows [row_begin, row_end) of y in tree order (full near
// storage only), the shard's full-length partial y in tree order (sum the
// partials of all ranks), and the final un-permute of a tree-order vector.
void apply_device_rows(DevInstance& inst, const double* x_dev, double* yrows_dev, Index m);
void apply_device_partial(DevInstance& inst, const double* x_dev, double* ypart_dev, Index m);
void instantiate_apply_partial_device(DevInstance& inst, const double* theta, int n_theta, const double* x_dev,
                                      double* ypart_dev, Index m, StageCounters* counters);
void unpermute_device(DevMatrix& m, const double* yperm_dev, double* y_dev, Index mcols);
// The row-sharded step as one call per rank: this rank's
// partial instantiate + apply, the x-hat and y all-reduces over `comm`
// (NCCL, or a callback), and the un-permute; y (original point order) is
// complete on every rank. The matrix must be shard comm.rank of comm.world.
void instantiate_apply_sharded(DevInstance& inst, Comm& comm, const double* theta, int n_theta, const double* x_dev,
                               double* y_dev, Index m, StageCounters* counters);
void instantiate_apply_sharded_host(DevInstance& inst, Comm& comm, const double* theta, int n_theta, const double* x,
                                    double* y, Index m, StageCounters* counters);
void apply_sharded(DevInstance& inst, Comm& comm, const double* x_dev, double* y_dev, Index m);

}  // namespace phm
