// Rank-to-rank exchange of the row-sharded step: an
// in-place sum all-reduce of doubles, enqueued on a CUDA stream.
//
// Two implementations behind one interface:
//   * NCCL (production): libnccl.so.2 is dlopen'd on first use, so the
//     library has no link-time NCCL dependency and shares whichever NCCL the
//     process already loaded (torch's, when torch.distributed is in use).
//     NVLink / NVSwitch (NVLS) transport is NCCL's choice. Capturable in a
//     CUDA graph.
//   * a caller callback (the C ABI's phm_allreduce_fn): lets a test drive
//     the library's sharded step with any exchange (two processes on one
//     GPU over gloo); not capturable.
#pragma once

#include <cstdint>
#include <memory>
#include <string>

namespace phm {

using AllreduceFn = int (*)(double* buf_dev, std::int64_t count, void* stream, void* user);

class Comm {
 public:
  virtual ~Comm() = default;
  // buf (device, count doubles) <- sum over ranks, ordered on `stream`
  virtual void allreduce(double* buf, std::int64_t count, void* stream) = 0;
  virtual bool capturable() const = 0;
  virtual const char* kind() const = 0;
  int rank = 0, world = 1;
};

// 128-byte ncclUniqueId of rank 0, to be broadcast to the other ranks.
void nccl_unique_id(void* out128);
std::shared_ptr<Comm> comm_nccl(int device, const void* id128, int rank, int world);
std::shared_ptr<Comm> comm_callback(AllreduceFn fn, void* user, int rank, int world);
// Timing probe of one rank on one GPU: the exchanges are no-ops (the rank's
// partials stay partial), capturable, so the rank's step replays as a graph.
std::shared_ptr<Comm> comm_probe(int rank, int world);

}  // namespace phm
