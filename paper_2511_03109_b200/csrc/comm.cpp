// NCCL and callback implementations of phm::Comm (comm.hpp).
#include "comm.hpp"

#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>

namespace phm {

namespace {

// The few NCCL entry points the sharded step needs, resolved from the
// process's libnccl.so.2 (torch's if it is loaded, the system one otherwise).
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL not available: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.init_rank || !api.destroy || !api.all_reduce || !api.error_string)
      err = "NCCL library lacks a required symbol";
  });
  if (!err.empty()) throw std::runtime_error(err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(int device, const void* id128, int rank_, int world_) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("comm: cudaSetDevice failed");
    nccl_check(nccl().init_rank(&comm_, world_, id, rank_), "ncclCommInitRank");
    rank = rank_;
    world = world_;
  }
  ~NcclComm() override {
    if (comm_) nccl().destroy(comm_);
  }
  void allreduce(double* buf, std::int64_t count, void* stream) override {
    nccl_check(nccl().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, comm_,
                                 static_cast<cudaStream_t>(stream)),
               "ncclAllReduce");
  }
  bool capturable() const override { return true; }
  const char* kind() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
};

class CallbackComm final : public Comm {
 public:
  CallbackComm(AllreduceFn fn, void* user, int rank_, int world_) : fn_(fn), user_(user) {
    if (!fn_) throw std::invalid_argument("comm: null all-reduce callback");
    rank = rank_;
    world = world_;
  }
  void allreduce(double* buf, std::int64_t count, void* stream) override {
    if (fn_(buf, count, stream, user_) != 0) throw std::runtime_error("comm: all-reduce callback failed");
  }
  bool capturable() const override { return false; }
  const char* kind() const override { return "callback"; }

 private:
  AllreduceFn fn_;
  void* user_;
};

class ProbeComm final : public Comm {
 public:
  ProbeComm(int rank_, int world_) {
    rank = rank_;
    world = world_;
  }
  void allreduce(double*, std::int64_t, void*) override {}
  bool capturable() const override { return true; }
  const char* kind() const override { return "probe"; }
};

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::shared_ptr<Comm> comm_nccl(int device, const void* id128, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm: bad rank / world");
  return std::make_shared<NcclComm>(device, id128, rank, world);
}

std::shared_ptr<Comm> comm_probe(int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm: bad rank / world");
  return std::make_shared<ProbeComm>(rank, world);
}

std::shared_ptr<Comm> comm_callback(AllreduceFn fn, void* user, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm: bad rank / world");
  return std::make_shared<CallbackComm>(fn, user, rank, world);
}

}  // namespace phm
