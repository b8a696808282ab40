#include "comm.hpp"

#include <nccl.h>

#include <cstring>

namespace dm {

namespace {
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

Comm::Comm(int world, int rank, const void* nccl_id, int device)
    : world_(world), rank_(rank), device_(device) {
  if (nccl_id == nullptr) throw UsageError("SPMD session requires an NCCL unique id");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t c = nullptr;
  nccl_check(ncclCommInitRank(&c, world_, id, rank_), "ncclCommInitRank");
  comm_ = c;
  // one extra communicator per device-barrier channel: NCCL orders the
  // collectives of one communicator, so barriers on the copy and pull streams
  // must not share one (that would chain the streams together)
  for (auto& ch : channels_) {
    ncclComm_t d = nullptr;
    nccl_check(ncclCommSplit(c, 0, rank_, &d, nullptr), "ncclCommSplit");
    ch = d;
  }
  dev_buf_bytes_ = 1 << 20;
  cuda_check(cudaMalloc(&dev_buf_, dev_buf_bytes_), "cudaMalloc(comm)");
  cuda_check(cudaMalloc(&bar_buf_, 256), "cudaMalloc(barrier)");  // never reallocated
}

Comm::~Comm() {
  cudaSetDevice(device_);
  for (auto& [h, m] : opened_)
    if (m.ptr) cudaIpcCloseMemHandle(m.ptr);
  opened_.clear();
  for (void* ch : channels_)
    if (ch) ncclCommDestroy(static_cast<ncclComm_t>(ch));
  if (comm_) ncclCommDestroy(static_cast<ncclComm_t>(comm_));
  if (dev_buf_) cudaFree(dev_buf_);
  if (bar_buf_) cudaFree(bar_buf_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Comm::barrier() {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  int* buf = static_cast<int*>(bar_buf_);
  nccl_check(ncclAllReduce(buf, buf + 1, 1, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm_),
                           stream_),
             "ncclAllReduce(barrier)");
  cuda_check(cudaStreamSynchronize(stream_), "barrier sync");
}

void Comm::barrier_on(cudaStream_t s, int channel) {
  int* buf = static_cast<int*>(bar_buf_) + 4 * (channel + 1);
  nccl_check(ncclAllReduce(buf, buf + 1, 1, ncclInt32, ncclSum,
                           static_cast<ncclComm_t>(channels_.at(channel)), s),
             "ncclAllReduce(device barrier)");
}

std::vector<std::uint8_t> Comm::allgather(const void* data, std::size_t bytes) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const std::size_t need = bytes * (static_cast<std::size_t>(world_) + 1);
  if (need > dev_buf_bytes_) {
    cudaFree(dev_buf_);
    dev_buf_bytes_ = need;
    cuda_check(cudaMalloc(&dev_buf_, dev_buf_bytes_), "cudaMalloc(comm)");
  }
  auto* base = static_cast<std::uint8_t*>(dev_buf_);
  std::uint8_t* send = base + bytes * world_;
  cuda_check(cudaMemcpyAsync(send, data, bytes, cudaMemcpyHostToDevice, stream_), "H2D(allgather)");
  nccl_check(ncclAllGather(send, base, bytes, ncclUint8, static_cast<ncclComm_t>(comm_), stream_),
             "ncclAllGather");
  std::vector<std::uint8_t> out(bytes * world_);
  cuda_check(cudaMemcpyAsync(out.data(), base, out.size(), cudaMemcpyDeviceToHost, stream_),
             "D2H(allgather)");
  cuda_check(cudaStreamSynchronize(stream_), "allgather sync");
  return out;
}

void Comm::publish(MatrixId id, const LayoutSpec& layout,
                   const std::map<BlockKey, StoredBlock>& owned) {
  std::map<BlockKey, void*> mine;
  for (BlockCoord c : owned_coords(layout, rank_)) mine[{id, c}] = owned.at({id, c}).mem.data();
  publish_raw(id, layout, mine);
}

void Comm::publish_raw(MatrixId id, const LayoutSpec& layout, const std::map<BlockKey, void*>& mine_ptrs) {
  std::size_t max_owned = 0;
  std::vector<std::vector<BlockCoord>> coords(world_);
  for (int r = 0; r < world_; ++r) {
    coords[r] = owned_coords(layout, r);
    max_owned = std::max(max_owned, coords[r].size());
  }
  if (max_owned == 0) return;
  constexpr std::size_t kRec = sizeof(cudaIpcMemHandle_t);
  std::vector<std::uint8_t> mine(max_owned * kRec, 0);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  for (std::size_t i = 0; i < coords[rank_].size(); ++i) {
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, mine_ptrs.at({id, coords[rank_][i]})), "cudaIpcGetMemHandle");
    std::memcpy(mine.data() + i * kRec, &h, kRec);
  }
  const std::vector<std::uint8_t> all = allgather(mine.data(), mine.size());
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    for (std::size_t i = 0; i < coords[r].size(); ++i) {
      std::string key(reinterpret_cast<const char*>(all.data() + r * mine.size() + i * kRec), kRec);
      Mapping& m = opened_[key];
      if (m.refs == 0) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, key.data(), kRec);
        cuda_check(cudaIpcOpenMemHandle(&m.ptr, h, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
      }
      m.refs += 1;
      dir_[{id, coords[r][i]}] = {key, static_cast<const float*>(m.ptr)};
    }
  }
}

void Comm::unpublish(MatrixId id) {
  cudaSetDevice(device_);
  auto it = dir_.lower_bound({id, {0, 0}});
  while (it != dir_.end() && it->first.matrix == id) {
    auto m = opened_.find(it->second.first);
    if (m != opened_.end() && --m->second.refs == 0) {
      cudaIpcCloseMemHandle(m->second.ptr);
      opened_.erase(m);
    }
    it = dir_.erase(it);
  }
}

const float* Comm::remote_ptr(MatrixId id, BlockCoord c) const {
  auto it = dir_.find({id, c});
  if (it == dir_.end())
    throw ProtocolError("peer block " + std::to_string(c.row) + "," + std::to_string(c.col) +
                        " of matrix " + std::to_string(id) + " was never published");
  return it->second.second;
}

}  // namespace dm
