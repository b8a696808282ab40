// SPMD plumbing: NCCL communicator (barrier, byte all-gather) and the peer
// block directory built on CUDA IPC.
//
// Replaces the reference's in-process TransportHub
// (gridgemm/transport.hpp:99-213) for the one thing the GEMM path needs from
// it: every worker can read the blocks it needs from their owner.  Instead of
// copying messages, each rank exports its owned blocks as CUDA IPC handles
// once per matrix; peers map them and the split kernel reads them directly
// over NVLink (no staging copy, no NCCL kernel on the data path).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "layout.hpp"
#include "session.hpp"

namespace dm {

class Comm {
 public:
  Comm(int world, int rank, const void* nccl_id, int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  // Stream-ordered all-reduce of one int followed by a host wait: returns
  // once every rank has reached the same point.
  void barrier();
  // Same collective enqueued on `s` without a host wait: work issued on `s`
  // afterwards starts only once every rank's `s` reached this point.
  // `channel` selects a dedicated communicator (0: copy-in stream, 1: pulls).
  void barrier_on(cudaStream_t s, int channel);
  // Fixed-size all-gather of host bytes; result is world * bytes.
  std::vector<std::uint8_t> allgather(const void* data, std::size_t bytes);

  // Export this rank's owned blocks of `id` and map every peer's.
  void publish(MatrixId id, const LayoutSpec& layout, const std::map<BlockKey, StoredBlock>& owned);
  // Same for raw allocations (this rank's blocks of `id` -> base pointers).
  void publish_raw(MatrixId id, const LayoutSpec& layout, const std::map<BlockKey, void*>& mine);
  void unpublish(MatrixId id);
  const float* remote_ptr(MatrixId id, BlockCoord c) const;

 private:
  void* comm_ = nullptr;  // ncclComm_t
  std::array<void*, 2> channels_{};
  int world_ = 1, rank_ = 0, device_ = 0;
  cudaStream_t stream_ = nullptr;
  void* dev_buf_ = nullptr;
  void* bar_buf_ = nullptr;
  std::size_t dev_buf_bytes_ = 0;
  struct Mapping {
    void* ptr = nullptr;
    int refs = 0;
  };
  std::map<std::string, Mapping> opened_;           // handle bytes -> mapping
  std::map<BlockKey, std::pair<std::string, const float*>> dir_;
};

}  // namespace dm
