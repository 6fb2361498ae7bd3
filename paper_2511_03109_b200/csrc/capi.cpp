// C ABI over the engine (include/phmat_b200.h). Exceptions never cross the
// boundary; they become status codes that map back to the reference's
// exception types, with the message in phm_last_error().
#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/phmat_b200.h"
#include "comm.hpp"
#include "engine.hpp"

struct phm_context_s {
  std::shared_ptr<phm::Context> ctx;
};
struct phm_matrix_s {
  std::shared_ptr<phm::Context> ctx;
  std::shared_ptr<phm::DevMatrix> m;
};
struct phm_instance_s {
  std::shared_ptr<phm::DevMatrix> m;
  std::shared_ptr<phm::DevInstance> inst;
};
struct phm_comm_s {
  std::shared_ptr<phm::Comm> c;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PHM_OK;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return PHM_ERR_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PHM_ERR_INVALID;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return PHM_ERR_RANGE;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return PHM_ERR_LOGIC;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return std::strncmp(e.what(), "CUDA", 4) == 0 || std::strstr(e.what(), "sm_100") ? PHM_ERR_CUDA : PHM_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PHM_ERR_RUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return PHM_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null ") + what);
}

phm::Config to_config(const phm_config& c) {
  phm::Config cfg;
  cfg.spec.family = c.family;
  cfg.spec.amplitude = c.amplitude != 0;
  if (c.d_theta < 1 || c.d_theta > 3) throw std::invalid_argument("d_theta must be 1..3");
  for (int k = 0; k < c.d_theta; ++k) cfg.spec.box.push_back({c.theta_lo[k], c.theta_hi[k]});
  cfg.p_theta.assign(c.p_theta, c.p_theta + c.d_theta);
  for (int p : cfg.p_theta)
    if (p < 1) throw std::invalid_argument("p_theta must be >= 1");
  cfg.format = c.format == PHM_FORMAT_H ? phm::Format::H : phm::Format::H2;
  cfg.l_max = c.l_max;
  cfg.p_s = c.p_s;
  if (c.p_s < 1) throw std::invalid_argument("p_s must be >= 1");
  cfg.eps = c.eps;
  cfg.eta = c.eta;
  cfg.r_max_far = c.r_max_far;
  cfg.r_max_near = c.r_max_near;
  cfg.seed = c.seed;
  cfg.near_mode = c.near_mode == PHM_NEAR_DIRECT     ? phm::NearMode::Direct
                  : c.near_mode == PHM_NEAR_SNAPSHOT ? phm::NearMode::Snapshot
                                                     : phm::NearMode::TT;
  cfg.translation_cache = c.translation_cache != 0;
  cfg.threads = c.threads;
  cfg.shard_rank = c.shard_rank;
  cfg.shard_count = c.shard_count < 1 ? 1 : c.shard_count;
  cfg.symmetric_near = c.symmetric_near != 0;
  return cfg;
}

void export_cores(const std::vector<phm::TTCore>& cores, int32_t* ncores, int64_t* dims, double* data, int64_t* len) {
  if (cores.size() > 10) throw std::logic_error("more than 10 cores");
  int64_t total = 0;
  for (size_t i = 0; i < cores.size(); ++i) {
    if (dims) {
      dims[3 * i] = cores[i].r0;
      dims[3 * i + 1] = cores[i].m;
      dims[3 * i + 2] = cores[i].r1;
    }
    if (data) std::memcpy(data + total, cores[i].data.data(), cores[i].data.size() * sizeof(double));
    total += cores[i].size();
  }
  if (ncores) *ncores = static_cast<int32_t>(cores.size());
  if (len) *len = total;
}

// StructureMetrics, phmatrix.cpp:319-422.
void fill_metrics(const phm::DevMatrix& dm, phm_info* info) {
  const phm::HostMatrix& H = phm::matrix_host(dm);
  const phm::Tree& T = *H.tree;
  const double n2 = static_cast<double>(T.n) * static_cast<double>(T.n);
  int64_t near_dense = 0;
  for (const auto& b : H.blocks.near) near_dense += T.nodes[b.sigma].count * T.nodes[b.tau].count;
  info->nf_ratio = near_dense / n2;
  const int d = T.d;
  const int64_t ps = H.cfg.p_s;
  int64_t basis = 0;
  if (H.cfg.format == phm::Format::H2) {
    for (const auto& nd : T.nodes) {
      if (nd.leaf() && nd.count > 0) basis += d * nd.count * ps;
      if (nd.parent >= 0) basis += d * ps * ps;
    }
  }
  auto coupling_online = [&](const phm::Coupling& c) {
    const int delta = c.tt.order();
    int64_t pl = 0, pr = 0;
    for (int i = 1; i <= c.d; ++i) pl += c.tt.rank(i - 1) * c.tt.rank(i);
    for (int i = c.d + c.d_theta + 1; i <= delta - 1; ++i) pr += c.tt.rank(i) * c.tt.rank(i + 1);
    return ps * (pl + pr) + c.rank_left() * c.rank_right();
  };
  double rank_sum = 0.0, coupling_sum = 0.0;
  int64_t ff_online = 0;
  for (size_t i = 0; i < H.blocks.far.size(); ++i) {
    const phm::Coupling& c = H.couplings[H.far_key[i]];
    rank_sum += static_cast<double>(std::max(c.rank_left(), c.rank_right()));
    if (H.cfg.format == phm::Format::H) {
      ff_online += T.nodes[H.blocks.far[i].sigma].count * c.rank_left() + c.rank_left() * c.rank_right() +
                   T.nodes[H.blocks.far[i].tau].count * c.rank_right();
    } else {
      const int64_t e = coupling_online(c);
      ff_online += e;
      coupling_sum += static_cast<double>(e);
    }
  }
  info->rank = H.blocks.far.empty() ? 0.0 : rank_sum / static_cast<double>(H.blocks.far.size());
  int64_t storage = 0;
  for (size_t b = 0; b < H.blocks.near.size(); ++b) {
    if (H.cfg.near_mode == phm::NearMode::TT && b < H.near_tt.size()) storage += H.near_tt[b].storage();
    if (H.cfg.near_mode == phm::NearMode::Snapshot && phm::matrix_on_device(dm)) {
      const auto& blk = H.blocks.near[b];
      storage += T.nodes[blk.sigma].count * T.nodes[blk.tau].count * phm::matrix_near_rank(dm, static_cast<int64_t>(b));
    }
  }
  if (H.cfg.format == phm::Format::H) {
    for (size_t i = 0; i < H.far_s.size(); ++i) storage += static_cast<int64_t>(H.far_s[i].a.size() + H.far_t[i].a.size());
    for (const auto& c : H.couplings)
      for (int q = c.d; q < c.d + c.d_theta; ++q) storage += c.tt.cores[q].size();
  } else {
    for (const auto& c : H.couplings) storage += c.tt.storage();
    storage += basis;
    ff_online += basis;
    info->coupling_ratio = coupling_sum / n2;
  }
  info->ff_ratio = static_cast<double>(ff_online) / n2;
  info->storage_entries = storage;
  info->storage_gb = static_cast<double>(storage) * 8.0 / 1e9;
}

}  // namespace

extern "C" {

const char* phm_last_error(void) { return g_last_error.c_str(); }
int phm_version(void) { return 1; }

void phm_config_default(phm_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->family = PHM_KERNEL_SE;  // reference defaults: phmatrix.hpp:20-35, kernels.cpp:41-47
  c->d_theta = 1;
  c->p_theta[0] = c->p_theta[1] = c->p_theta[2] = 27;
  c->theta_lo[0] = 0.25;
  c->theta_hi[0] = 1.0;
  c->format = PHM_FORMAT_H2;
  c->l_max = 2;
  c->p_s = 15;
  c->near_mode = PHM_NEAR_TT;
  c->eps = 1e-5;
  c->eta = 0.0;
  c->r_max_far = 120;
  c->r_max_near = 150;
  c->seed = 0;
  c->translation_cache = 1;
  c->threads = 0;
  c->shard_rank = 0;
  c->shard_count = 1;
  c->symmetric_near = 1;
}

int phm_context_create(int device, phm_context* out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<phm_context_s>();
    c->ctx = phm::context_create(device);
    *out = c.release();
  });
}
int phm_context_destroy(phm_context ctx) {
  return guarded([&] { delete ctx; });
}
int phm_context_set_stream(phm_context ctx, void* s) {
  return guarded([&] {
    need(ctx, "context");
    phm::context_set_stream(*ctx->ctx, s);
  });
}
int phm_context_get_stream(phm_context ctx, void** s) {
  return guarded([&] {
    need(ctx, "context");
    need(s, "out");
    *s = phm::context_stream(*ctx->ctx);
  });
}
int phm_context_sync(phm_context ctx) {
  return guarded([&] {
    need(ctx, "context");
    phm::context_sync(*ctx->ctx);
  });
}
int phm_context_enable_timing(phm_context ctx, int on) {
  return guarded([&] {
    need(ctx, "context");
    phm::context_enable_timing(*ctx->ctx, on != 0);
  });
}
int phm_context_timer(phm_context ctx, const char* name, double* ms, int64_t* launches) {
  return guarded([&] {
    need(ctx, "context");
    need(name, "name");
    double t = 0;
    int64_t c = 0;
    phm::context_timer(*ctx->ctx, name, &t, &c);
    if (ms) *ms = t;
    if (launches) *launches = c;
  });
}
int phm_context_reset_timers(phm_context ctx) {
  return guarded([&] {
    need(ctx, "context");
    phm::context_reset_timers(*ctx->ctx);
  });
}
int phm_context_launches(phm_context ctx, int64_t* launches) {
  return guarded([&] {
    need(ctx, "context");
    need(launches, "out");
    *launches = phm::context_launches(*ctx->ctx);
  });
}

int phm_matrix_build(phm_context ctx, const double* points, int64_t n, int d, const phm_config* cfg, phm_matrix* out) {
  return guarded([&] {
    need(ctx, "context");
    need(points, "points");
    need(cfg, "config");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("n must be >= 1");
    if (d < 1 || d > 3) throw std::invalid_argument("d must be 1..3");
    auto m = std::make_unique<phm_matrix_s>();
    m->ctx = ctx->ctx;
    m->m = phm::matrix_build(ctx->ctx, points, n, d, to_config(*cfg));
    *out = m.release();
  });
}
int phm_baseline_build(phm_context ctx, const double* points, int64_t n, int d, const phm_config* cfg, int method,
                       const double* theta, int n_theta, double eps, int64_t r_max, phm_instance* out) {
  return guarded([&] {
    need(ctx, "context");
    need(points, "points");
    need(cfg, "config");
    need(theta, "theta");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("n must be >= 1");
    if (d < 1 || d > 3) throw std::invalid_argument("d must be 1..3");
    if (method != PHM_BASELINE_H_ACA && method != PHM_BASELINE_H2_HCA) throw std::invalid_argument("unknown baseline");
    if (r_max < 1) throw std::invalid_argument("r_max must be >= 1");
    auto m = phm::baseline_build(ctx->ctx, points, n, d, to_config(*cfg),
                                 method == PHM_BASELINE_H_ACA ? phm::Baseline::HAca : phm::Baseline::H2Hca, theta,
                                 n_theta, eps, r_max);
    const auto t0 = std::chrono::steady_clock::now();
    auto inst = phm::baseline_instance(m);
    phm::instance_sync(*inst);
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*m));
    H.stats.nf_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    auto I = std::make_unique<phm_instance_s>();
    I->m = m;
    I->inst = inst;
    *out = I.release();
  });
}
int phm_baseline_info_get(phm_instance inst, phm_baseline_info* out) {
  return guarded([&] {
    need(inst, "instance");
    need(out, "out");
    const auto& H = phm::matrix_host(*inst->m);
    const phm::BaselineData& B = H.baseline;
    if (B.method == phm::Baseline::None) throw std::logic_error("not a baseline instance");
    *out = phm_baseline_info{};
    out->method = B.method == phm::Baseline::HAca ? PHM_BASELINE_H_ACA : PHM_BASELINE_H2_HCA;
    out->mean_far_rank = B.mean_far_rank;
    out->coupling_ratio = B.coupling_ratio;
    out->far_build_s = B.far_s;
    out->near_build_s = H.stats.nf_s;
    out->far_evals = B.far_evals;
    out->near_evals = B.near_evals;
    out->any_capped = B.any_capped ? 1 : 0;
    out->n_far = static_cast<int64_t>(H.blocks.far.size());
    out->n_near = static_cast<int64_t>(H.blocks.near.size());
    out->n_classes = static_cast<int64_t>(B.rank.size());
  });
}
int phm_aca_partial_dense(const double* a, int64_t m, int64_t n, double eps, int64_t r_max, uint64_t seed,
                          int64_t* rank, int32_t* capped, double* v, double* y) {
  return guarded([&] {
    need(a, "a");
    need(rank, "rank");
    if (m < 1 || n < 1) throw std::invalid_argument("aca_partial: empty matrix");
    auto f = phm::aca_partial([&](phm::Index i, phm::Index j) { return a[i + j * m]; }, m, n, eps, r_max, seed);
    *rank = f.rank();
    if (capped) *capped = f.capped ? 1 : 0;
    if (v) std::memcpy(v, f.v.a.data(), f.v.a.size() * sizeof(double));
    if (y) std::memcpy(y, f.y.a.data(), f.y.a.size() * sizeof(double));
  });
}
int phm_matrix_build_host(const double* points, int64_t n, int d, const phm_config* cfg, phm_matrix* out) {
  return guarded([&] {
    need(points, "points");
    need(cfg, "config");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("n must be >= 1");
    if (d < 1 || d > 3) throw std::invalid_argument("d must be 1..3");
    auto m = std::make_unique<phm_matrix_s>();
    m->m = phm::matrix_build_host_only(points, n, d, to_config(*cfg));
    *out = m.release();
  });
}
int phm_matrix_load(phm_context ctx, const char* path, int threads, phm_matrix* out) {
  return guarded([&] {
    need(ctx, "context");
    need(path, "path");
    need(out, "out");
    auto m = std::make_unique<phm_matrix_s>();
    m->ctx = ctx->ctx;
    m->m = phm::matrix_load(ctx->ctx, path, threads);
    *out = m.release();
  });
}
int phm_matrix_load_host(const char* path, int threads, phm_matrix* out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    auto m = std::make_unique<phm_matrix_s>();
    m->m = phm::matrix_load_host_only(path, threads);
    *out = m.release();
  });
}
int phm_matrix_save(phm_matrix m, const char* path) {
  return guarded([&] {
    need(m, "matrix");
    need(path, "path");
    if (!phm::matrix_on_device(*m->m) && phm::matrix_host(*m->m).cfg.near_mode == phm::NearMode::Snapshot)
      throw std::logic_error("snapshot near data lives on the device; save from a device matrix");
    phm::matrix_save(*m->m, path);
  });
}
int phm_matrix_config(phm_matrix m, phm_config* out) {
  return guarded([&] {
    need(m, "matrix");
    need(out, "out");
    const phm::Config& c = phm::matrix_host(*m->m).cfg;
    phm_config_default(out);
    out->family = c.spec.family;
    out->amplitude = c.spec.amplitude ? 1 : 0;
    out->d_theta = c.spec.d_theta();
    for (int k = 0; k < c.spec.d_theta(); ++k) {
      out->theta_lo[k] = c.spec.box[k].lo;
      out->theta_hi[k] = c.spec.box[k].hi;
      out->p_theta[k] = c.p_theta.size() == 1 ? c.p_theta[0] : c.p_theta[k];
    }
    out->format = c.format == phm::Format::H2 ? PHM_FORMAT_H2 : PHM_FORMAT_H;
    out->l_max = c.l_max;
    out->p_s = c.p_s;
    out->near_mode = c.near_mode == phm::NearMode::Direct     ? PHM_NEAR_DIRECT
                     : c.near_mode == phm::NearMode::Snapshot ? PHM_NEAR_SNAPSHOT
                                                              : PHM_NEAR_TT;
    out->eps = c.eps;
    out->eta = c.eta;
    out->r_max_far = c.r_max_far;
    out->r_max_near = c.r_max_near;
    out->seed = c.seed;
    out->translation_cache = c.translation_cache ? 1 : 0;
    out->threads = c.threads;
    out->shard_rank = c.shard_rank;
    out->shard_count = c.shard_count;
    out->symmetric_near = c.symmetric_near ? 1 : 0;
  });
}
int phm_artifact_is_h2(const char* path, int* is_h2) {
  return guarded([&] {
    need(path, "path");
    need(is_h2, "out");
    *is_h2 = phm::artifact_is_h2(path) ? 1 : 0;
  });
}
int phm_matrix_destroy(phm_matrix m) {
  return guarded([&] { delete m; });
}

int phm_matrix_info(phm_matrix m, phm_info* info) {
  return guarded([&] {
    need(m, "matrix");
    need(info, "info");
    std::memset(info, 0, sizeof(*info));
    const phm::HostMatrix& H = phm::matrix_host(*m->m);
    const phm::Tree& T = *H.tree;
    info->n = T.n;
    info->d = T.d;
    info->nodes = static_cast<int64_t>(T.nodes.size());
    info->n_near = static_cast<int64_t>(H.blocks.near.size());
    info->n_far = static_cast<int64_t>(H.blocks.far.size());
    std::map<int, int> distinct;
    for (int k : H.far_key) distinct[k] = 1;
    info->n_classes = static_cast<int64_t>(H.couplings.size());
    info->c_sp = H.blocks.c_sp;
    info->constructed = H.blocks.constructed;
    info->P = H.P();
    info->row_begin = H.row_begin;
    info->row_end = H.row_end;
    if (phm::matrix_on_device(*m->m)) {
      info->near_entries = phm::matrix_near_elems(*m->m, 0);
      info->near_stored = phm::matrix_near_elems(*m->m, 1);
      info->near_stream_elems = phm::matrix_near_elems(*m->m, 2);
      info->device_bytes = phm::matrix_device_bytes(*m->m);
    }
    info->tree_s = H.stats.tree_s;
    info->ff_s = H.stats.ff_s;
    info->nf_s = H.stats.nf_s;
    info->upload_s = H.stats.upload_s;
    info->evals_offline = H.counters.offline.value();
    info->evals_online = H.counters.online.value();
    info->evals_audit = H.counters.audit.value();
    info->any_rank_capped = H.stats.any_rank_capped ? 1 : 0;
    fill_metrics(*m->m, info);
  });
}

int phm_matrix_perm(phm_matrix m, int32_t* perm) {
  return guarded([&] {
    need(m, "matrix");
    need(perm, "perm");
    const auto& T = *phm::matrix_host(*m->m).tree;
    std::memcpy(perm, T.perm.data(), T.perm.size() * sizeof(int32_t));
  });
}

int phm_matrix_nodes(phm_matrix m, int32_t* ints, double* boxes) {
  return guarded([&] {
    need(m, "matrix");
    const auto& T = *phm::matrix_host(*m->m).tree;
    for (size_t i = 0; i < T.nodes.size(); ++i) {
      const auto& nd = T.nodes[i];
      if (ints) {
        ints[7 * i] = nd.level;
        ints[7 * i + 1] = nd.parent;
        ints[7 * i + 2] = nd.first_child;
        ints[7 * i + 3] = static_cast<int32_t>(nd.count);
        for (int k = 0; k < 3; ++k) ints[7 * i + 4 + k] = static_cast<int32_t>(nd.coords[k]);
      }
      if (boxes)
        for (int k = 0; k < 3; ++k) {
          boxes[6 * i + k] = k < T.d ? nd.box.lo[k] : 0.0;
          boxes[6 * i + 3 + k] = k < T.d ? nd.box.hi[k] : 0.0;
        }
    }
  });
}

int phm_matrix_blocks(phm_matrix m, int32_t* near_pairs, int32_t* far_pairs, int32_t* far_key) {
  return guarded([&] {
    need(m, "matrix");
    const auto& H = phm::matrix_host(*m->m);
    for (size_t i = 0; i < H.blocks.near.size(); ++i)
      if (near_pairs) {
        near_pairs[2 * i] = H.blocks.near[i].sigma;
        near_pairs[2 * i + 1] = H.blocks.near[i].tau;
      }
    for (size_t i = 0; i < H.blocks.far.size(); ++i) {
      if (far_pairs) {
        far_pairs[2 * i] = H.blocks.far[i].sigma;
        far_pairs[2 * i + 1] = H.blocks.far[i].tau;
      }
      if (far_key) far_key[i] = H.far_key[i];
    }
  });
}

int phm_matrix_class_keys(phm_matrix m, int64_t* keys) {
  return guarded([&] {
    need(m, "matrix");
    need(keys, "keys");
    const auto& H = phm::matrix_host(*m->m);
    for (size_t k = 0; k < H.class_keys.size(); ++k)
      for (int q = 0; q < 4; ++q) keys[4 * k + q] = H.class_keys[k][q];
  });
}

int phm_matrix_theta_grid(phm_matrix m, int k, double* nodes) {
  return guarded([&] {
    need(m, "matrix");
    need(nodes, "nodes");
    const auto& H = phm::matrix_host(*m->m);
    const auto& g = H.grids.grids.at(k);
    std::memcpy(nodes, g.nodes.data(), g.nodes.size() * sizeof(double));
  });
}

int phm_matrix_coupling(phm_matrix m, int64_t cls, int32_t* ncores, int64_t* dims, double* data, int64_t* len) {
  return guarded([&] {
    need(m, "matrix");
    const auto& H = phm::matrix_host(*m->m);
    if (cls < 0 || cls >= static_cast<int64_t>(H.couplings.size())) throw std::out_of_range("class index");
    export_cores(H.couplings[cls].tt.cores, ncores, dims, data, len);
  });
}

int phm_matrix_near_tt(phm_matrix m, int64_t b, int32_t* ncores, int64_t* dims, double* data, int64_t* len) {
  return guarded([&] {
    need(m, "matrix");
    const auto& H = phm::matrix_host(*m->m);
    if (H.cfg.near_mode != phm::NearMode::TT) throw std::invalid_argument("near blocks are not in TT mode");
    if (b < 0 || b >= static_cast<int64_t>(H.near_tt.size())) throw std::out_of_range("near block index");
    if (H.near_tt[b].cores.empty()) throw std::out_of_range("near block not built on this shard");
    export_cores(H.near_tt[b].cores, ncores, dims, data, len);
  });
}

int phm_matrix_near_rank(phm_matrix m, int64_t b, int64_t* rank) {
  return guarded([&] {
    need(m, "matrix");
    need(rank, "out");
    *rank = phm::matrix_near_rank(*m->m, b);
  });
}

int phm_matrix_near_column(phm_matrix m, int64_t b, int64_t kap, double* out) {
  return guarded([&] {
    need(m, "matrix");
    need(out, "out");
    phm::matrix_near_column(*m->m, b, kap, out);
  });
}

int phm_matrix_far_st(phm_matrix m, int64_t i, double* S, double* T, int64_t* dims) {
  return guarded([&] {
    need(m, "matrix");
    const auto& H = phm::matrix_host(*m->m);
    if (H.cfg.format != phm::Format::H) throw std::invalid_argument("S/T factors exist only for the H format");
    if (i < 0 || i >= static_cast<int64_t>(H.far_s.size())) throw std::out_of_range("far index");
    const auto& s = H.far_s[i];
    const auto& t = H.far_t[i];
    if (dims) {
      dims[0] = s.rows;
      dims[1] = s.cols;
      dims[2] = t.rows;
      dims[3] = t.cols;
    }
    if (S) std::memcpy(S, s.a.data(), s.a.size() * sizeof(double));
    if (T) std::memcpy(T, t.a.data(), t.a.size() * sizeof(double));
  });
}

int phm_matrix_class_lr(phm_matrix m, int64_t k, double* L, double* R, int64_t* dims) {
  return guarded([&] {
    need(m, "matrix");
    const auto& H = phm::matrix_host(*m->m);
    if (H.cfg.format != phm::Format::H2) throw std::invalid_argument("L/R exist only for the H2 format");
    if (k < 0 || k >= static_cast<int64_t>(H.class_l.size())) throw std::out_of_range("class index");
    if (dims) {
      dims[0] = H.class_l[k].rows;
      dims[1] = H.class_l[k].cols;
      dims[2] = H.class_r[k].rows;
      dims[3] = H.class_r[k].cols;
    }
    if (L) std::memcpy(L, H.class_l[k].a.data(), H.class_l[k].a.size() * sizeof(double));
    if (R) std::memcpy(R, H.class_r[k].a.data(), H.class_r[k].a.size() * sizeof(double));
  });
}

int phm_parametric_vectors(phm_matrix m, const double* theta, int n_theta, double* out) {
  return guarded([&] {
    need(m, "matrix");
    need(theta, "theta");
    need(out, "out");
    const auto v = phm::parametric_vectors(phm::matrix_host(*m->m).grids, theta, n_theta);
    size_t o = 0;
    for (const auto& vk : v)
      for (double x : vk) out[o++] = x;
  });
}

int phm_instantiate(phm_matrix m, const double* theta, int n_theta, phm_instance* out) {
  return guarded([&] {
    need(m, "matrix");
    need(theta, "theta");
    need(out, "out");
    auto I = std::make_unique<phm_instance_s>();
    I->m = m->m;
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*m->m));
    I->inst = phm::instantiate(m->m, theta, n_theta, &H.counters);
    *out = I.release();
  });
}
int phm_instantiate_batch(phm_matrix m, const double* thetas, int n_theta, int count, phm_instance* out) {
  return guarded([&] {
    need(m, "matrix");
    need(thetas, "thetas");
    need(out, "out");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*m->m));
    auto insts = phm::instantiate_batch(m->m, thetas, n_theta, count, &H.counters);
    for (int b = 0; b < count; ++b) {
      auto I = std::make_unique<phm_instance_s>();
      I->m = m->m;
      I->inst = insts[b];
      out[b] = I.release();
    }
  });
}
int phm_reinstantiate_batch(phm_instance* insts, int count, const double* thetas, int n_theta) {
  return guarded([&] {
    need(insts, "instances");
    need(thetas, "thetas");
    PHM_CHECK(count >= 1, "reinstantiate_batch: count must be >= 1");
    std::vector<phm::DevInstance*> raw;
    for (int b = 0; b < count; ++b) {
      need(insts[b], "instance");
      PHM_CHECK(insts[b]->m == insts[0]->m, "reinstantiate_batch: instances of different matrices");
      raw.push_back(insts[b]->inst.get());
    }
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*insts[0]->m));
    phm::reinstantiate_batch(raw, thetas, n_theta, &H.counters);
  });
}
int phm_reinstantiate(phm_instance inst, const double* theta, int n_theta) {
  return guarded([&] {
    need(inst, "instance");
    need(theta, "theta");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    phm::reinstantiate(*inst->inst, theta, n_theta, &H.counters);
  });
}
int phm_instance_destroy(phm_instance inst) {
  return guarded([&] { delete inst; });
}
int phm_instance_sync(phm_instance inst) {
  return guarded([&] {
    need(inst, "instance");
    phm::instance_sync(*inst->inst);
  });
}
int phm_instance_far_h(phm_instance inst, int64_t i, double* out, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    need(inst, "instance");
    std::vector<double> h;
    phm::Index r = 0, c = 0;
    phm::instance_far_h(*inst->inst, i, h, r, c);
    if (rows) *rows = r;
    if (cols) *cols = c;
    if (out) std::memcpy(out, h.data(), h.size() * sizeof(double));
  });
}
int phm_instance_near_d(phm_instance inst, int64_t b, double* out) {
  return guarded([&] {
    need(inst, "instance");
    need(out, "out");
    std::vector<double> v;
    phm::instance_near_d(*inst->inst, b, v);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}
int phm_instance_class_c(phm_instance inst, int64_t k, double* out) {
  return guarded([&] {
    need(inst, "instance");
    need(out, "out");
    std::vector<double> v;
    phm::instance_class_c(*inst->inst, k, v);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}
int phm_apply(phm_instance inst, const double* x, int64_t n_rows, double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(x, "x");
    need(y, "y");
    if (n_rows != phm::matrix_host(*inst->m).n()) throw std::invalid_argument("mvm: length mismatch");
    if (m < 1) throw std::invalid_argument("mvm: m must be >= 1");
    phm::apply_host(*inst->inst, x, y, m);
  });
}
int phm_instantiate_apply(phm_instance inst, const double* theta, int n_theta, const double* x, int64_t n_rows,
                          double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(theta, "theta");
    need(x, "x");
    need(y, "y");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    (void)phm::parametric_vectors(H.grids, theta, n_theta);  // domain check first
    if (n_rows != H.n()) throw std::invalid_argument("mvm: length mismatch");
    if (m < 1) throw std::invalid_argument("mvm: m must be >= 1");
    phm::instantiate_apply_host(*inst->inst, theta, n_theta, x, y, m, &H.counters);
  });
}
int phm_instantiate_apply_device(phm_instance inst, const double* theta, int n_theta, const double* x, double* y,
                                 int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(theta, "theta");
    need(x, "x");
    need(y, "y");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    phm::instantiate_apply_device(*inst->inst, theta, n_theta, x, y, m, &H.counters);
  });
}
int phm_comm_unique_id(uint8_t* id) {
  return guarded([&] {
    need(id, "id");
    phm::nccl_unique_id(id);
  });
}
int phm_comm_create_nccl(phm_context ctx, const uint8_t* id, int rank, int world, phm_comm* out) {
  return guarded([&] {
    need(ctx, "context");
    need(id, "id");
    need(out, "out");
    auto c = std::make_unique<phm_comm_s>();
    c->c = phm::comm_nccl(phm::context_device(*ctx->ctx), id, rank, world);
    *out = c.release();
  });
}
int phm_comm_create_callback(phm_allreduce_fn fn, void* user, int rank, int world, phm_comm* out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<phm_comm_s>();
    c->c = phm::comm_callback(fn, user, rank, world);
    *out = c.release();
  });
}
int phm_comm_create_probe(int rank, int world, phm_comm* out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<phm_comm_s>();
    c->c = phm::comm_probe(rank, world);
    *out = c.release();
  });
}
int phm_comm_destroy(phm_comm c) {
  return guarded([&] { delete c; });
}
int phm_comm_info(phm_comm c, int* rank, int* world, int* is_nccl) {
  return guarded([&] {
    need(c, "comm");
    if (rank) *rank = c->c->rank;
    if (world) *world = c->c->world;
    if (is_nccl) *is_nccl = c->c->capturable() ? 1 : 0;
  });
}
int phm_instantiate_apply_sharded(phm_instance inst, phm_comm comm, const double* theta, int n_theta,
                                  const double* x, double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(comm, "comm");
    need(theta, "theta");
    need(x, "x");
    need(y, "y");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    (void)phm::parametric_vectors(H.grids, theta, n_theta);  // domain check before any launch
    if (m < 1) throw std::invalid_argument("mvm: m must be >= 1");
    phm::instantiate_apply_sharded(*inst->inst, *comm->c, theta, n_theta, x, y, m, &H.counters);
  });
}
int phm_instantiate_apply_sharded_host(phm_instance inst, phm_comm comm, const double* theta, int n_theta,
                                       const double* x, int64_t n_rows, double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(comm, "comm");
    need(theta, "theta");
    need(x, "x");
    need(y, "y");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    (void)phm::parametric_vectors(H.grids, theta, n_theta);
    if (n_rows != H.n()) throw std::invalid_argument("mvm: length mismatch");
    if (m < 1) throw std::invalid_argument("mvm: m must be >= 1");
    phm::instantiate_apply_sharded_host(*inst->inst, *comm->c, theta, n_theta, x, y, m, &H.counters);
  });
}
int phm_apply_sharded(phm_instance inst, phm_comm comm, const double* x, double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(comm, "comm");
    need(x, "x");
    need(y, "y");
    phm::apply_sharded(*inst->inst, *comm->c, x, y, m);
  });
}
int phm_estimate_error(phm_instance inst, int64_t probe_rows, uint64_t seed, double* err, int64_t* rows_out,
                       double* exact_out, double* approx_out, double* x_out) {
  return guarded([&] {
    need(inst, "instance");
    need(err, "err");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    std::vector<phm::Index> rows;
    std::vector<double> ex, ap, xs;
    *err = phm::estimate_error(*inst->inst, probe_rows, seed, &H.counters, &rows, &ex, &ap, &xs);
    if (rows_out) std::memcpy(rows_out, rows.data(), rows.size() * sizeof(int64_t));
    if (exact_out) std::memcpy(exact_out, ex.data(), ex.size() * sizeof(double));
    if (approx_out) std::memcpy(approx_out, ap.data(), ap.size() * sizeof(double));
    if (x_out) std::memcpy(x_out, xs.data(), xs.size() * sizeof(double));
  });
}
int phm_apply_device(phm_instance inst, const double* x, double* y, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(x, "x");
    need(y, "y");
    const auto& H = phm::matrix_host(*inst->m);
    if (H.row_begin != 0 || H.row_end != H.n())
      throw std::logic_error("apply on a row shard: use phm_apply_partial_device (or phm_apply_rows_device) across ranks");
    phm::apply_device(*inst->inst, x, y, m);
  });
}
int phm_apply_rows_device(phm_instance inst, const double* x, double* yrows, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(x, "x");
    need(yrows, "y");
    phm::apply_device_rows(*inst->inst, x, yrows, m);
  });
}
int phm_apply_partial_device(phm_instance inst, const double* x, double* ypart, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(x, "x");
    need(ypart, "y");
    phm::apply_device_partial(*inst->inst, x, ypart, m);
  });
}
int phm_instantiate_apply_partial_device(phm_instance inst, const double* theta, int n_theta, const double* x,
                                         double* ypart, int64_t m) {
  return guarded([&] {
    need(inst, "instance");
    need(theta, "theta");
    need(x, "x");
    need(ypart, "y");
    auto& H = const_cast<phm::HostMatrix&>(phm::matrix_host(*inst->m));
    phm::instantiate_apply_partial_device(*inst->inst, theta, n_theta, x, ypart, m, &H.counters);
  });
}
int phm_unpermute_device(phm_matrix m, const double* yperm, double* y, int64_t mcols) {
  return guarded([&] {
    need(m, "matrix");
    need(yperm, "yperm");
    need(y, "y");
    phm::unpermute_device(*m->m, yperm, y, mcols);
  });
}
int phm_to_dense(phm_instance inst, double* out, int64_t guard) {
  return guarded([&] {
    need(inst, "instance");
    need(out, "out");
    const int64_t n = phm::matrix_host(*inst->m).n();
    if (n > guard) throw std::runtime_error("to_dense: matrix exceeds the size guard");
    // Columns K e_j through the GPU MVM in batches of 256 right-hand sides.
    const int64_t batch = std::min<int64_t>(n, 256);
    std::vector<double> eye(static_cast<size_t>(n * batch));
    for (int64_t j0 = 0; j0 < n; j0 += batch) {
      const int64_t bw = std::min(batch, n - j0);
      std::fill(eye.begin(), eye.end(), 0.0);
      for (int64_t c = 0; c < bw; ++c) eye[c * n + j0 + c] = 1.0;
      phm::apply_host(*inst->inst, eye.data(), out + j0 * n, bw);
    }
  });
}

int phm_generate_points(int64_t n, int d, uint64_t seed, double* out) {
  return guarded([&] {
    need(out, "out");
    phm::generate_points(n, d, seed, out);
  });
}
int phm_generate_mixture_points(int64_t n, int d, int clusters, double sigma, uint64_t seed, double* out) {
  return guarded([&] {
    need(out, "out");
    if (clusters < 1) throw std::invalid_argument("clusters must be >= 1");
    phm::generate_mixture_points(n, d, clusters, sigma, seed, out);
  });
}
namespace {
void export_tt(const phm::TTTensor& tt, int32_t* ncores, int64_t* dims, double* data, int64_t cap, int64_t* len) {
  int64_t total = 0;
  for (const auto& c : tt.cores) total += c.size();
  if (len) *len = total;
  if (ncores) *ncores = tt.order();
  if (dims)
    for (int i = 0; i < tt.order(); ++i) {
      dims[3 * i] = tt.cores[i].r0;
      dims[3 * i + 1] = tt.cores[i].m;
      dims[3 * i + 2] = tt.cores[i].r1;
    }
  if (data && cap >= total) {
    int64_t off = 0;
    for (const auto& c : tt.cores) {
      std::memcpy(data + off, c.data.data(), c.data.size() * sizeof(double));
      off += c.size();
    }
  }
}
}  // namespace

int phm_tt_cross_dense(const double* tensor, const int64_t* dims, int ndims, double eps, int64_t r_max,
                       uint64_t seed, int round_after, int32_t* ncores, int64_t* core_dims, double* core_data,
                       int64_t cap, int64_t* len, uint64_t* evals, int32_t* flags, double* est) {
  return guarded([&] {
    need(tensor, "tensor");
    need(dims, "dims");
    if (ndims < 1 || ndims > 16) throw std::invalid_argument("ndims must be 1..16");
    phm::EntryFn f;
    f.dims.assign(dims, dims + ndims);
    std::vector<int64_t> strides(ndims, 1);
    for (int k = 1; k < ndims; ++k) strides[k] = strides[k - 1] * dims[k - 1];
    f.fn = [tensor, strides, ndims](const phm::Index* idx) {
      int64_t o = 0;
      for (int k = 0; k < ndims; ++k) o += idx[k] * strides[k];
      return tensor[o];
    };
    phm::CrossOptions co;
    co.eps = eps;
    co.r_max = r_max;
    co.seed = seed;
    co.round_after = round_after != 0;
    const phm::CrossResult r = phm::tt_cross(f, co);
    export_tt(r.tt, ncores, core_dims, core_data, cap, len);
    if (evals) *evals = r.evals;
    if (flags) {
      flags[0] = r.rank_capped ? 1 : 0;
      flags[1] = r.converged ? 1 : 0;
    }
    if (est) *est = r.est_rel_error;
  });
}

int phm_tt_round(int ncores_in, const int64_t* dims_in, const double* data_in, double eps, double abs_budget,
                 int32_t* ncores, int64_t* dims, double* data, int64_t cap, int64_t* len) {
  return guarded([&] {
    need(dims_in, "dims");
    need(data_in, "data");
    phm::TTTensor tt;
    int64_t off = 0;
    for (int i = 0; i < ncores_in; ++i) {
      phm::TTCore c = phm::TTCore::zeros(dims_in[3 * i], dims_in[3 * i + 1], dims_in[3 * i + 2]);
      std::memcpy(c.data.data(), data_in + off, c.data.size() * sizeof(double));
      off += c.size();
      tt.cores.push_back(std::move(c));
    }
    export_tt(phm::tt_round(tt, eps, abs_budget), ncores, dims, data, cap, len);
  });
}

int phm_theta_draws(double lo, double hi, int64_t count, uint64_t seed, double* out) {
  return guarded([&] {
    need(out, "out");
    phm::Rng rng(phm::mix_seed(seed, 0x74686574ULL));  // harness.cpp:254-260
    for (int64_t i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
  });
}
int phm_generate_normal(int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    need(out, "out");
    phm::generate_normal(n, seed, out);
  });
}

}  // extern "C"
