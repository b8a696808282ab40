// Session implementation.  See session.hpp for the architecture; reference
// citations are to /root/reference/proj/include/gridgemm/.
#include "session.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../kernels/tf32x3_gemm.h"
#include "comm.hpp"

namespace dm {

namespace {

std::uint64_t table_digest(const std::map<MatrixId, MatrixDescriptor>& t) {
  Fnv1a h;
  for (const auto& [id, d] : t) hash_descriptor(h, d);
  return h.digest();
}

}  // namespace

// ------------------------------------------------------------------ lifecycle

Session::Session(const dm_session_config& cfg) {
  if (cfg.worker_count < 1) throw UsageError("init: worker_count must be >= 1");
  P_ = cfg.worker_count;
  mode_ = cfg.mode;
  rank_ = cfg.rank;
  coherence_ = cfg.coherence_checks != 0;
  root_seed_ = cfg.root_seed;
  if (cfg.gemm_mode == DM_GEMM_TF32X3) {
    gemm_mode_ = kModeTf32x3;
  } else if (cfg.gemm_mode == DM_GEMM_MIXED) {
    gemm_mode_ = kModeMixed;
  } else if (cfg.gemm_mode == DM_GEMM_AUTO) {
    gemm_mode_ = kModeAuto;
  } else if (cfg.gemm_mode == DM_GEMM_F16X2) {
    gemm_mode_ = kModeF16x2;
  } else if (cfg.gemm_mode == DM_GEMM_DEFAULT) {
    gemm_mode_ = env_gemm_mode();
  } else {
    throw ConfigError("init: unknown gemm_mode");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("init: no CUDA device visible (the B200 path has no CPU fallback)");
  }
  workers_.resize(P_);
  auto make_worker = [&](int w, int dev) {
    if (dev < 0 || dev >= ndev) throw ConfigError("init: device id out of range");
    DeviceGuard g(dev);
    auto wk = std::make_unique<Worker>();
    wk->id = w;
    wk->device = dev;
    cuda_check(cudaStreamCreateWithFlags(&wk->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&wk->side, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&wk->h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&wk->d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&wk->pull, cudaStreamNonBlocking), "cudaStreamCreate");
    wk->pool = std::make_unique<DevicePool>(dev);
    wk->seed = mix64(root_seed_, static_cast<std::uint64_t>(w));  // exec_seed, ops.hpp:1140
    workers_[w] = std::move(wk);
  };
  if (mode_ == DM_MODE_LOCAL) {
    std::set<int> devs;
    for (int w = 0; w < P_; ++w) {
      const int dev = cfg.devices ? cfg.devices[w] : w % ndev;
      make_worker(w, dev);
      devs.insert(dev);
    }
    for (int i : devs)
      for (int j : devs) {
        if (i == j) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, i, j);
        if (!can) throw ConfigError("init: devices without peer access cannot share a session");
        DeviceGuard g(i);
        cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          cuda_check(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
  } else if (mode_ == DM_MODE_SPMD) {
    if (rank_ < 0 || rank_ >= P_) throw UsageError("init: rank out of range");
    const int dev = cfg.devices ? cfg.devices[0] : rank_ % ndev;
    make_worker(rank_, dev);
    comm_ = std::make_unique<Comm>(P_, rank_, cfg.nccl_id, dev);
  } else {
    throw ConfigError("init: unknown session mode");
  }
  if (const char* t = std::getenv("DM_TRACE")) trace_path_ = t;
  live_ = true;
}

Session::~Session() {
  try {
    shutdown();
  } catch (...) {
  }
  comm_.reset();
  for (auto& w : workers_) {
    if (!w) continue;
    cudaSetDevice(w->device);
    for (auto& [a, b] : w->timing_events) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    for (cudaEvent_t e : w->markers)
      if (e) cudaEventDestroy(e);
    drop_graphs(*w, 0);
    w->owned.clear();
    w->cache.clear();
    w->replicas.clear();
    w->arena = DeviceBuffer();
    w->plane_arena = DeviceBuffer();
    for (cudaEvent_t e : {w->plane_reads, w->presplit_done, w->presplit_order, w->maxima_done})
      if (e) cudaEventDestroy(e);
    w->pull_flag = DeviceBuffer();
    w->inflight.clear();
    for (auto* v : {&w->event_pool, &w->events_used})
      for (cudaEvent_t e : *v) cudaEventDestroy(e);
    w->pool.reset();
    cudaStreamDestroy(w->stream);
    cudaStreamDestroy(w->side);
    cudaStreamDestroy(w->h2d);
    cudaStreamDestroy(w->d2h);
    cudaStreamDestroy(w->pull);
  }
}

void Session::shutdown() {
  if (!live_) return;
  if (async_) drain();
  async_ = false;
  sync_local();
  if (comm_) {
    for (const auto& [id, d] : table_) comm_->unpublish(id);
    comm_->unpublish(0);  // exchange arenas
    comm_->barrier();
  }
  arena_ptrs_.clear();
  arena_bytes_ = 0;
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard g(w->device);
    drop_graphs(*w, 0);
    w->owned.clear();
    w->cache.clear();
    w->replicas.clear();
    w->arena = DeviceBuffer();
    w->pull_flag = DeviceBuffer();
    w->descriptors.clear();
    w->pool->trim();
  }
  if (comm_) comm_->barrier();
  table_.clear();
  cache_meta_.clear();
  live_ = false;
}

std::vector<int> Session::local_worker_ids() const {
  std::vector<int> out;
  for (int w = 0; w < P_; ++w)
    if (workers_[w]) out.push_back(w);
  return out;
}

Worker& Session::worker(int w) {
  if (w < 0 || w >= P_) throw UsageError("unknown worker id");
  if (!workers_[w]) throw UsageError("worker " + std::to_string(w) + " is not local to this process");
  return *workers_[w];
}
const Worker& Session::worker(int w) const { return const_cast<Session*>(this)->worker(w); }

Worker* Session::local(int w) { return workers_[w].get(); }
const Worker* Session::local(int w) const { return workers_[w].get(); }

void Session::require_live() const {
  if (!live_) throw UsageError("session has been shut down");
}

void Session::validate_layout_workers(const LayoutSpec& l) const {
  if (l.worker_count < 1) throw UsageError("layout: worker set must not be empty");
  for (int r = 0; r < l.grid.n_block_rows(); ++r)
    for (int c = 0; c < l.grid.n_block_cols(); ++c) {
      const int o = l.owner({r, c});
      if (o < 0 || o >= P_) throw UsageError("layout: block owner outside the session worker set");
    }
}

const MatrixDescriptor& Session::descriptor(MatrixId id) const {
  auto it = table_.find(id);
  if (it == table_.end()) throw UsageError("unknown matrix id " + std::to_string(id));
  return it->second;
}

void Session::sync_local() {
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard g(w->device);
    for (cudaStream_t st : {w->h2d, w->pull, w->side, w->stream, w->d2h})
      cuda_check(cudaStreamSynchronize(st), "stream sync");
  }
}

// ------------------------------------------------------ asynchronous mode

cudaEvent_t Session::ev_get(Worker& w) {
  cudaEvent_t e;
  if (w.event_pool.empty()) {
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  } else {
    e = w.event_pool.back();
    w.event_pool.pop_back();
  }
  w.events_used.push_back(e);
  return e;
}

void Session::mark_write(Worker& w, cudaStream_t s, MatrixId id) {
  Track& t = w.tracks[id];
  t.write = ev_get(w);
  cuda_check(cudaEventRecord(t.write, s), "cudaEventRecord");
  t.reads.clear();
}

void Session::mark_read(Worker& w, cudaStream_t s, MatrixId id) {
  cudaEvent_t e = ev_get(w);
  cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
  w.tracks[id].reads.push_back(e);
}

// `s` waits for the last write of `id` on every local worker (cross-device
// waits are legal inside one process).
void Session::wait_writes(cudaStream_t s, MatrixId id) {
  for (auto& v : workers_) {
    if (!v) continue;
    auto it = v->tracks.find(id);
    if (it != v->tracks.end() && it->second.write)
      cuda_check(cudaStreamWaitEvent(s, it->second.write, 0), "cudaStreamWaitEvent");
  }
}

// ... and for every read of `id` issued since (before overwriting it).
void Session::wait_all(cudaStream_t s, MatrixId id) {
  wait_writes(s, id);
  for (auto& v : workers_) {
    if (!v) continue;
    auto it = v->tracks.find(id);
    if (it == v->tracks.end()) continue;
    for (cudaEvent_t e : it->second.reads) cuda_check(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent");
  }
}

// SPMD: every rank's work issued on `s` so far completes before anything
// issued on `s` afterwards (NCCL all-reduce on the stream, no host wait).
void Session::device_barrier(cudaStream_t s, int channel) {
  if (comm_) comm_->barrier_on(s, channel);
}

void Session::reap_inflight(Worker& w) {
  while (!w.inflight.empty() && cudaEventQuery(w.inflight.front().done) == cudaSuccess) {
    for (cudaEvent_t e : w.inflight.front().events) cudaEventDestroy(e);
    w.inflight.pop_front();
  }
  cudaGetLastError();  // cudaErrorNotReady is not an error here
}

void Session::bound_inflight(Worker& w) {
  reap_inflight(w);
  // Bound the device memory held by queued GEMMs' panel planes: at most
  // DM_MAX_INFLIGHT (default 2) commands in flight per worker.  Waiting here
  // cannot deadlock: every rank already issued the older command waited on.
  const std::size_t cap = static_cast<std::size_t>(std::max<std::int64_t>(1, env_int("DM_MAX_INFLIGHT", 2)));
  while (w.inflight.size() >= cap) {
    cuda_check(cudaEventSynchronize(w.inflight.front().done), "cudaEventSynchronize(inflight)");
    for (cudaEvent_t e : w.inflight.front().events) cudaEventDestroy(e);
    w.inflight.pop_front();
  }
}

// Complete every outstanding asynchronous command on every rank.
void Session::drain() {
  sync_local();
  remote_read_.clear();  // (every rank drains; the barrier below ends the epoch)
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard g(w->device);
    for (auto& f : w->inflight)
      for (cudaEvent_t e : f.events) cudaEventDestroy(e);
    w->inflight.clear();
    w->tracks.clear();
    w->event_pool.insert(w->event_pool.end(), w->events_used.begin(), w->events_used.end());
    w->events_used.clear();
  }
  collect_timing();
  if (comm_) comm_->barrier();
}

SyncScope::SyncScope(Session* ss) : s(ss), prev(ss != nullptr && ss->async_mode()) {
  if (prev) s->set_async(false);
}
SyncScope::~SyncScope() {
  if (prev) {
    try {
      s->set_async(true);
    } catch (...) {
    }
  }
}

void Session::set_async(bool on) {
  require_live();
  if (async_ && !on) {
    drain();
    async_ = false;
    end_command();  // coherence check of everything issued asynchronously
    return;
  }
  if (!async_ && on) sync_local();
  async_ = on;
}

void Session::end_command() {
  if (async_) return;  // stream-ordered; completed by barrier()/drain()
  HostScope hs("end_command");
  if (!streams_drained_) sync_local();
  remote_read_.clear();  // synchronous: every rank's reads finished before the digest exchange
  streams_drained_ = false;
  collect_timing();
  if (comm_) {
    if (coherence_) {
      const std::uint64_t mine = table_digest(workers_[rank_]->descriptors);
      const std::uint64_t master = table_digest(table_);
      if (mine != master) throw ProtocolError("descriptor tables diverged (worker vs master)");
      const auto all = comm_->allgather(&master, sizeof(master));  // doubles as the barrier
      for (int r = 0; r < P_; ++r) {
        std::uint64_t v;
        std::memcpy(&v, all.data() + r * sizeof(v), sizeof(v));
        if (v != master) throw ProtocolError("descriptor tables diverged across ranks");
      }
    } else {
      comm_->barrier();
    }
  } else if (coherence_) {
    const std::uint64_t master = table_digest(table_);
    for (auto& w : workers_)
      if (w && table_digest(w->descriptors) != master)
        throw ProtocolError("descriptor tables diverged");
  }
}

void Session::barrier() {
  if (async_) {
    drain();
    return;
  }
  sync_local();
  if (comm_) comm_->barrier();
}

void Session::marker_record(int w, int slot) {
  Worker& wk = worker(w);
  if (slot < 0 || slot >= 16) throw UsageError("marker slot out of range");
  DeviceGuard g(wk.device);
  if (!wk.markers[slot]) cuda_check(cudaEventCreate(&wk.markers[slot]), "cudaEventCreate");
  cuda_check(cudaEventRecord(wk.markers[slot], wk.stream), "cudaEventRecord");
}

float Session::marker_elapsed(int w, int a, int b) {
  Worker& wk = worker(w);
  if (a < 0 || a >= 16 || b < 0 || b >= 16 || !wk.markers[a] || !wk.markers[b])
    throw UsageError("marker slot not recorded");
  DeviceGuard g(wk.device);
  cuda_check(cudaEventSynchronize(wk.markers[b]), "cudaEventSynchronize");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, wk.markers[a], wk.markers[b]), "cudaEventElapsedTime");
  return ms;
}

// --------------------------------------------------------------- matrices

MatrixId Session::create_matrix(const LayoutSpec& layout, Precision p, FillKind fill,
                                const void* host) {
  require_live();
  SyncScope scope(this);
  validate_layout_workers(layout);
  if (fill == FillKind::FromHost && host == nullptr)
    throw UsageError("create_matrix: FromHost requires host data");
  MatrixDescriptor d;
  d.matrix_id = next_matrix_id_++;
  d.layout = layout;
  d.precision = p;
  d.seed = mix64(root_seed_, d.matrix_id);  // session.hpp:142
  materialize(d, fill == FillKind::SeededRandom);
  end_command();
  if (fill == FillKind::FromHost)
    scatter(d.matrix_id, host, layout.grid.global_rows, layout.grid.global_cols);
  return d.matrix_id;
}

// Allocate (and fill) the blocks every local worker owns under `d`, register
// the descriptor everywhere and export the blocks to the peers (SPMD).
void Session::materialize(const MatrixDescriptor& d, bool seeded) {
  const std::size_t esz = byte_width(d.precision);
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard g(w->device);
    for (BlockCoord c : owned_coords(d.layout, w->id)) {
      auto [br, bc] = block_extent(d.layout.grid, c);
      StoredBlock blk;
      blk.rows = br;
      blk.cols = bc;
      blk.precision = d.precision;
      blk.version_seen = d.version;
      blk.mem = w->pool->acquire(static_cast<std::size_t>(br * bc) * esz);
      if (seeded) {
        const std::uint64_t key =
            mix64(d.seed, (static_cast<std::uint64_t>(static_cast<std::uint32_t>(c.row)) << 32) |
                              static_cast<std::uint32_t>(c.col));
        cuda_check(fill_seeded(blk.mem.data(), static_cast<int>(d.precision), br * bc, key, w->stream),
                   "fill_seeded");
      } else {
        cuda_check(cudaMemsetAsync(blk.mem.data(), 0, static_cast<std::size_t>(br * bc) * esz,
                                   w->stream),
                   "cudaMemsetAsync");
      }
      w->owned[{d.matrix_id, c}] = std::move(blk);
    }
    w->descriptors[d.matrix_id] = d;
  }
  table_[d.matrix_id] = d;
  sync_local();
  if (comm_) comm_->publish(d.matrix_id, d.layout, workers_[rank_]->owned);
}

void Session::destroy_matrix(MatrixId id) {
  require_live();
  SyncScope scope(this);
  descriptor(id);
  sync_local();
  if (comm_) {
    comm_->barrier();
    comm_->unpublish(id);
  }
  for (auto& w : workers_) {
    if (!w) continue;
    {
      DeviceGuard g(w->device);
      drop_graphs(*w, id);
    }
    for (auto* m : {&w->owned, &w->cache, &w->replicas}) {
      auto it = m->lower_bound({id, {0, 0}});
      while (it != m->end() && it->first.matrix == id) it = m->erase(it);
    }
    w->descriptors.erase(id);
  }
  table_.erase(id);
  cache_meta_.erase(id);
  end_command();
}

void Session::bump_version(MatrixId id) {
  const std::uint64_t v = ++table_.at(id).version;
  for (auto& w : workers_) {
    if (!w) continue;
    w->descriptors.at(id).version = v;
    auto it = w->owned.lower_bound({id, {0, 0}});
    for (; it != w->owned.end() && it->first.matrix == id; ++it) it->second.version_seen = v;
  }
}

void Session::scatter(MatrixId id, const void* host, std::int64_t rows, std::int64_t cols) {
  require_live();
  const MatrixDescriptor d = descriptor(id);
  const BlockGrid& g = d.layout.grid;
  if (rows != g.global_rows || cols != g.global_cols)
    throw ShapeError("scatter: host data shape does not match the matrix");
  if (host == nullptr) throw UsageError("scatter: null host pointer");
  const std::size_t esz = byte_width(d.precision);
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard guard(w->device);
    cudaStream_t st = w->stream;
    if (async_) {
      // copy engine stream; wait until nobody (here or on a peer) still reads
      // or writes the blocks we are about to overwrite
      reap_inflight(*w);
      st = w->h2d;
      wait_all(st, id);
      if (remote_read_.count(id)) device_barrier(st, 0);
    }
    for (BlockCoord c : owned_coords(d.layout, w->id)) {
      StoredBlock& blk = w->owned.at({id, c});
      const char* src = static_cast<const char*>(host) +
                        (static_cast<std::int64_t>(c.row) * g.block_rows * g.global_cols +
                         static_cast<std::int64_t>(c.col) * g.block_cols) * esz;
      cuda_check(cudaMemcpy2DAsync(blk.mem.data(), static_cast<std::size_t>(blk.cols) * esz, src,
                                   static_cast<std::size_t>(g.global_cols) * esz,
                                   static_cast<std::size_t>(blk.cols) * esz,
                                   static_cast<std::size_t>(blk.rows), cudaMemcpyHostToDevice,
                                   st),
                 "scatter H2D");
    }
    if (async_) mark_write(*w, st, id);
  }
  remote_read_.erase(id);
  bump_version(id);  // runtime_types.hpp:289-292
  end_command();
}

const void* Session::block_src(MatrixId id, BlockCoord c, const Worker& reader) const {
  const MatrixDescriptor& d = table_.at(id);
  const int owner = d.layout.owner(c);
  if (const Worker* ow = local(owner)) return ow->owned.at({id, c}).mem.data();
  (void)reader;
  return comm_->remote_ptr(id, c);
}

void Session::gather(MatrixId id, void* host, std::int64_t rows, std::int64_t cols, int root) {
  require_live();
  const MatrixDescriptor d = descriptor(id);
  const BlockGrid& g = d.layout.grid;
  if (rows != g.global_rows || cols != g.global_cols)
    throw ShapeError("gather: host buffer shape does not match the matrix");
  if (root < -1 || root >= P_) throw UsageError("gather: root out of range");
  // SPMD gathers to a root read peer blocks through IPC: run synchronously
  SyncScope scope(async_ && comm_ && root != -1 ? this : nullptr);
  const bool all_blocks = !comm_ || root == rank_;
  const bool any = !comm_ || root == -1 || root == rank_;
  if (any && host == nullptr) throw UsageError("gather: null host pointer");
  const std::size_t esz = byte_width(d.precision);
  if (any) {
    Worker& me = comm_ ? *workers_[rank_] : *workers_[0];
    for (int r = 0; r < g.n_block_rows(); ++r)
      for (int c = 0; c < g.n_block_cols(); ++c) {
        const int owner = d.layout.owner({r, c});
        Worker* ow = local(owner);
        if (!all_blocks && ow == nullptr) continue;
        auto [br, bc] = block_extent(g, {r, c});
        const void* src = block_src(id, {r, c}, me);
        Worker& issuer = ow ? *ow : me;
        DeviceGuard guard(issuer.device);
        cudaStream_t st = issuer.stream;
        if (async_) {
          st = issuer.d2h;
          wait_writes(st, id);
        }
        char* dst = static_cast<char*>(host) +
                    (static_cast<std::int64_t>(r) * g.block_rows * g.global_cols +
                     static_cast<std::int64_t>(c) * g.block_cols) * esz;
        cuda_check(cudaMemcpy2DAsync(dst, static_cast<std::size_t>(g.global_cols) * esz, src,
                                     static_cast<std::size_t>(bc) * esz,
                                     static_cast<std::size_t>(bc) * esz,
                                     static_cast<std::size_t>(br), cudaMemcpyDefault, st),
                   "gather D2H");
        if (async_) mark_read(issuer, st, id);
      }
  }
  end_command();
}

// ----------------------------------------------------------------- GEMMs

GemmArgs Session::gemm_command(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c,
                               bool ta, bool tb, bool cache_a) const {
  if (c == a || c == b) throw UsageError("gemm: destination must be distinct from the operands");
  GemmArgs g;
  g.alpha = alpha;
  g.beta = beta;
  g.a = a;
  g.b = b;
  g.c = c;
  g.trans_a = ta;
  g.trans_b = tb;
  g.cache_a = cache_a;
  return g;
}

// Session::validate_general_gemm (session.hpp:531-545).
void Session::validate_general(const GemmArgs& g) const {
  const MatrixDescriptor& da = descriptor(g.a);
  const MatrixDescriptor& db = descriptor(g.b);
  const MatrixDescriptor& dc = descriptor(g.c);
  if (da.precision != db.precision || da.precision != dc.precision)
    throw UsageError("gemm: operands must share a precision; reshape to convert first");
  if (dc.replicated) throw UsageError("gemm: destination matrix may not be replicated");
  const std::int64_t kk = g.trans_a ? da.layout.grid.global_rows : da.layout.grid.global_cols;
  const std::int64_t m = g.trans_a ? da.layout.grid.global_cols : da.layout.grid.global_rows;
  const std::int64_t kb = g.trans_b ? db.layout.grid.global_cols : db.layout.grid.global_rows;
  const std::int64_t n = g.trans_b ? db.layout.grid.global_rows : db.layout.grid.global_cols;
  if (kk != kb) throw ShapeError("gemm: inner dimensions do not conform");
  if (dc.layout.grid.global_rows != m || dc.layout.grid.global_cols != n)
    throw ShapeError("gemm: output dimensions do not conform");
}

// Ring-plan preconditions of build_cyclic_plan (ops.hpp:84-169).
void Session::validate_cyclic(const GemmArgs& g, std::vector<WorkerId>* strip_owners) const {
  validate_general(g);
  const MatrixDescriptor& da = descriptor(g.a);
  const MatrixDescriptor& db = descriptor(g.b);
  const MatrixDescriptor& dc = descriptor(g.c);
  const BlockGrid& ga = da.layout.grid;
  if ((da.layout.kind != LayoutKind::RowBlocks1D && da.layout.kind != LayoutKind::RowCyclic1D) ||
      ga.n_block_cols() != 1)
    throw PlanError("cyclic_gemm: A must use a 1D row-blocked decomposition");
  if (da.layout.worker_count != P_)
    throw PlanError("cyclic_gemm: A must be laid out over all session workers");
  const int nbr = ga.n_block_rows();
  if (nbr % P_ != 0) throw PlanError("cyclic_gemm: A block-rows must divide evenly over the ring");
  const int inner = nbr / P_;
  for (int w = 0; w < P_; ++w)
    for (int i = 0; i < inner; ++i) {
      const int row = da.layout.kind == LayoutKind::RowBlocks1D ? w * inner + i : w + i * P_;
      if (da.layout.owner({row, 0}) != w)
        throw PlanError("cyclic_gemm: A assignment does not match the ring plan");
    }
  const BlockGrid& gb = db.layout.grid;
  const int strips = g.trans_b ? gb.n_block_rows() : gb.n_block_cols();
  if ((g.trans_b ? gb.n_block_cols() : gb.n_block_rows()) != 1)
    throw PlanError("cyclic_gemm: B must be a single line of stationary strips");
  const BlockGrid& gc = dc.layout.grid;
  if (gc.n_block_rows() != 1 || gc.n_block_cols() != strips)
    throw PlanError("cyclic_gemm: C strips must match op(B) strips");
  const std::int64_t m = g.trans_a ? ga.global_cols : ga.global_rows;
  for (int s = 0; s < strips; ++s) {
    const BlockCoord bcd = g.trans_b ? BlockCoord{s, 0} : BlockCoord{0, s};
    auto [br, bc] = block_extent(gb, bcd);
    const std::int64_t width = g.trans_b ? br : bc;
    auto [cr, cc] = block_extent(gc, {0, s});
    if (cc != width || cr != m) throw PlanError("cyclic_gemm: C strip extents must match op(B) strips");
    const int owner = db.layout.owner(bcd);
    if (dc.layout.owner({0, s}) != owner)
      throw PlanError("cyclic_gemm: C strips must be co-located with op(B) strips");
    if (strip_owners) strip_owners->push_back(owner);
  }
}

const void* Session::source_ptr(const Worker& reader, MatrixId m, BlockCoord c, SourcePolicy pol,
                                bool* remote) const {
  const MatrixDescriptor& d = table_.at(m);
  const int owner = d.layout.owner(c);
  *remote = false;
  if (owner == reader.id) return reader.owned.at({m, c}).mem.data();
  // A version-fresh cached copy (CyclicGemmExec cache, ops.hpp:278-289) or
  // replica (ReplicateExec, ops.hpp:660-702) holds the owner's exact bytes:
  // read it instead of crossing the link again.
  for (const auto* store : {&reader.cache, &reader.replicas}) {
    auto hit = store->find({m, c});
    if (hit != store->end() && hit->second.version_seen == d.version) return hit->second.mem.data();
  }
  if (pol == SourcePolicy::LocalOnly)
    throw CacheMissError("cached_backward_gemm: stale or missing cached blocks", {{c.row, c.col}});
  *remote = true;
  if (const Worker* ow = local(owner)) return ow->owned.at({m, c}).mem.data();
  return comm_->remote_ptr(m, c);
}

// Pieces of op(M) covering range rg (op rows of A, or op cols of B) for every
// K panel.  A piece is the intersection of one stored block with the range and
// a panel -- the B200 form of GeneralGemmExec::add_needed + assemble_op_rows /
// assemble_op_cols (ops.hpp:503-524, 177-208, 534-558).
void Session::add_range_pieces(Range& rg, const MatrixDescriptor& d, bool trans, bool is_a,
                               const std::vector<std::int64_t>& k0) const {
  const BlockGrid& grid = d.layout.grid;
  const bool range_on_rows = is_a ? !trans : trans;
  const int np = static_cast<int>(k0.size()) - 1;
  rg.panels.assign(np, {});
  for (int br = 0; br < grid.n_block_rows(); ++br)
    for (int bc = 0; bc < grid.n_block_cols(); ++bc) {
      const std::int64_t sr0 = static_cast<std::int64_t>(br) * grid.block_rows;
      const std::int64_t sc0 = static_cast<std::int64_t>(bc) * grid.block_cols;
      auto [srows, scols] = block_extent(grid, {br, bc});
      const std::int64_t o0 = range_on_rows ? sr0 : sc0, olen = range_on_rows ? srows : scols;
      const std::int64_t q0 = range_on_rows ? sc0 : sr0, qlen = range_on_rows ? scols : srows;
      const std::int64_t lo_o = std::max(o0, rg.start), hi_o = std::min(o0 + olen, rg.start + rg.len);
      if (lo_o >= hi_o) continue;
      for (int p = 0; p < np; ++p) {
        const std::int64_t lo_k = std::max(q0, k0[p]), hi_k = std::min(q0 + qlen, k0[p + 1]);
        if (lo_k >= hi_k) continue;
        Piece pc;
        pc.matrix = d.matrix_id;
        pc.coord = {br, bc};
        pc.lds = scols;
        pc.rows = hi_o - lo_o;
        pc.kcols = hi_k - lo_k;
        pc.dst_row = lo_o - rg.start;
        pc.dst_k = lo_k - k0[p];
        if (range_on_rows) {
          pc.src_off = (lo_o - sr0) * scols + (lo_k - sc0);
          pc.trans = 0;
        } else {
          pc.src_off = (lo_k - sr0) * scols + (lo_o - sc0);
          pc.trans = 1;
        }
        rg.panels[p].push_back(pc);
      }
    }
}

Session::WorkerPlan Session::plan_worker(const GemmArgs& g, int w, SourcePolicy pol, bool presplit) const {
  const MatrixDescriptor& da = table_.at(g.a);
  const MatrixDescriptor& db = table_.at(g.b);
  const MatrixDescriptor& dc = table_.at(g.c);
  const std::int64_t K = g.trans_a ? da.layout.grid.global_rows : da.layout.grid.global_cols;
  WorkerPlan plan;
  const BlockGrid& gc = dc.layout.grid;
  std::map<int, int> row_idx, col_idx;
  for (BlockCoord c : owned_coords(dc.layout, w)) {
    auto [mb, nb] = block_extent(gc, c);
    if (!row_idx.count(c.row)) {
      row_idx[c.row] = static_cast<int>(plan.ar.size());
      Range r;
      r.start = static_cast<std::int64_t>(c.row) * gc.block_rows;
      r.len = mb;
      plan.ar.push_back(std::move(r));
    }
    if (!col_idx.count(c.col)) {
      col_idx[c.col] = static_cast<int>(plan.br.size());
      Range r;
      r.start = static_cast<std::int64_t>(c.col) * gc.block_cols;
      r.len = nb;
      plan.br.push_back(std::move(r));
    }
    plan.tasks.push_back({c, row_idx[c.row], col_idx[c.col]});
  }
  if (plan.tasks.empty()) return plan;

  // Single panel first; pipeline K only when some piece has to cross a link.
  plan.k0 = {0, K};
  for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
  for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
  if (pol == SourcePolicy::Peer) {
    for (const auto* ranges : {&plan.ar, &plan.br})
      for (const Range& r : *ranges)
        for (const Piece& pc : r.panels[0])
          if (table_.at(pc.matrix).layout.owner(pc.coord) != w) {
            bool remote = false;
            source_ptr(*local(w), pc.matrix, pc.coord, pol, &remote);
            if (remote) plan.has_remote = true;
          }
  }
  if (presplit) {
    // Panels start at K-block edges of A or B where they can (a panel inside
    // one block whose range is one local piece is read in place from the
    // owner's arena): the segments between edges are merged up to
    // DM_PRESPLIT_PANEL wide, wider ones cut evenly (256-aligned).  Every
    // plane row carries its whole op row's scale, so a panel may span blocks.
    // Wide panels: every panel after the first re-reads C (beta = 1), and
    // fewer, longer launches measured faster (4 GPUs: 16384-wide 1615 vs
    // 8192-wide 1575 TFLOP/s; 2 GPUs: 855 vs 798); at least two (config 5,
    // N=16384 on 2x2: one 16384-wide panel exposes every pull, 15.8 vs
    // 11.7 ms per chain).
    plan.k0 = presplit_panels(K, g.trans_a ? da.layout.grid.block_rows : da.layout.grid.block_cols,
                              g.trans_b ? db.layout.grid.block_cols : db.layout.grid.block_rows,
                              env_int("DM_PRESPLIT_PANEL", 16384));
    for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
    for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
    // A worker whose every panel needs a pull waits for the first one before
    // its first GEMM: DM_PRESPLIT_LEAD cuts a narrow lead panel off the
    // least-remote panel (it runs first), so only its pull is exposed
    // (4 GPUs: 1618 with a 2048 lead vs 1595 TFLOP/s without).
    const std::int64_t lead = (env_int("DM_PRESPLIT_LEAD", 2048) + 255) / 256 * 256;
    if (lead > 0 && pol == SourcePolicy::Peer) {
      const int n = static_cast<int>(plan.k0.size()) - 1;
      std::vector<std::uint64_t> rb(n, 0);
      for (int p = 0; p < n; ++p)
        for (const auto* ranges : {&plan.ar, &plan.br})
          for (const Range& r : *ranges)
            for (const Piece& pc : r.panels[p])
              if (table_.at(pc.matrix).layout.owner(pc.coord) != w) rb[p] += pc.bytes();
      const int best = static_cast<int>(std::min_element(rb.begin(), rb.end()) - rb.begin());
      if (rb[best] > 0 && plan.k0[best + 1] - plan.k0[best] >= 2 * lead) {
        plan.k0.insert(plan.k0.begin() + best + 1, plan.k0[best] + lead);
        for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
        for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
      }
    }
    return plan;
  }
  const std::int64_t target = env_int("DM_PANEL_K", 8192);
  const std::int64_t local_lead = env_int("DM_PANEL_LOCAL", 0);
  // Only Single32 may cut K into panels: Double64 runs the bit-exact SIMT
  // kernel whose single k-ascending accumulation per output cannot be split,
  // and Half16 C is rounded once from the fp32 sum (AccumOf<Half> then
  // narrow_store, kernels.hpp:29-35, 72) -- a launch per panel would round it
  // once per panel.
  const bool one_panel = da.precision != Precision::Single32;
  if (!plan.has_remote && local_lead > 0 && K >= 4 * local_lead && !one_panel) {
    // All operands local: geometric panels.  Only the narrow lead panel's
    // split is exposed; every later panel is split by the previous panel's
    // GEMM (a GEMM of width w hides the split of ~3.7 w, tf32x3_gemm.cu).
    const std::int64_t growth = std::max<std::int64_t>(2, env_int("DM_PANEL_GROWTH", 3));
    plan.k0.clear();
    std::int64_t k = 0, width = (local_lead + 31) / 32 * 32;
    while (k < K) {
      plan.k0.push_back(k);
      if (K - k < width + width * growth / 2) break;  // last panel absorbs a short tail
      k += width;
      width *= growth;
    }
    plan.k0.push_back(K);
    for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
    for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
    return plan;
  }
  // Pipelining pays only when there is enough math to hide pulls behind;
  // small GEMMs (latency-bound) take one panel.
  double work = 0;
  for (const Task& t : plan.tasks) {
    auto [mb, nb] = block_extent(gc, t.c);
    work += 2.0 * mb * nb * static_cast<double>(K);
  }
  const double min_work = static_cast<double>(env_int("DM_PIPELINE_MIN_GFLOP", 200)) * 1e9;
  if (plan.has_remote && K > 2 * 256 && target != 0 && work >= min_work && !one_panel) {
    // Uniform panels of about `tgt`; per panel: remote and total piece bytes.
    std::vector<std::uint64_t> rb, tb;
    auto build = [&](std::int64_t tgt) {
      std::int64_t np = std::max<std::int64_t>(2, (K + tgt - 1) / tgt);
      np = std::min<std::int64_t>(np, K / 256);
      std::int64_t width = (K + np - 1) / np;
      width = (width + 31) / 32 * 32;
      plan.k0.clear();
      for (std::int64_t k = 0; k < K; k += width) plan.k0.push_back(k);
      plan.k0.push_back(K);
      for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
      for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
      const int n = static_cast<int>(plan.k0.size()) - 1;
      rb.assign(n, 0);
      tb.assign(n, 0);
      for (int p = 0; p < n; ++p)
        for (const auto* ranges : {&plan.ar, &plan.br})
          for (const Range& r : *ranges)
            for (const Piece& pc : r.panels[p]) {
              bool remote = false;
              source_ptr(*local(w), pc.matrix, pc.coord, pol, &remote);
              if (remote) rb[p] += pc.bytes();
              tb[p] += pc.bytes();
            }
    };
    if (target > 0 && std::getenv("DM_PANEL_K") != nullptr) {  // forced width (-1: the model)
      build(target);
    } else {
      // Widest panels whose exposed start -- the least-remote panel's pull
      // (~400 GB/s) and split (~1.5 TB/s of input) before the first GEMM --
      // stays within 3% of this worker's GEMM time (~320 TFLOP/s): fewer
      // panels mean fewer beta=1 passes over C (measured at 2 GPUs: 16384-wide
      // 608 vs 8192-wide 595 TFLOP/s), but a wide all-remote first panel
      // stalls the start (8 GPUs: 2x4 grid).
      for (std::int64_t tgt : {std::int64_t{16384}, std::int64_t{8192}}) {
        build(tgt);
        const int b = static_cast<int>(std::min_element(rb.begin(), rb.end()) - rb.begin());
        const double exposed = static_cast<double>(rb[b]) / 400e9 + static_cast<double>(tb[b]) / 1.5e12;
        if (exposed <= 0.03 * work / 320e12) break;
      }
    }
    // If even the least-remote panel must cross a link, optionally cut a
    // ramp of narrow lead panels off it (DM_LEAD_PANEL_K; off by default).
    const std::int64_t lead = env_int("DM_LEAD_PANEL_K", 0);
    const int best = static_cast<int>(std::min_element(rb.begin(), rb.end()) - rb.begin());
    if (lead > 0 && rb[best] > 0 && plan.k0[best + 1] - plan.k0[best] > 2 * lead) {
      // Ramp: lead, lead, 2 lead, 4 lead, ... so each sub-panel's GEMM is long
      // enough to hide the pull and fused split of the next one.
      const std::int64_t start = plan.k0[best], end = plan.k0[best + 1];
      std::vector<std::int64_t> cuts;
      for (std::int64_t c = lead; start + c < end && end - (start + c) >= lead; c *= 2) cuts.push_back(start + c);
      plan.k0.insert(plan.k0.begin() + best + 1, cuts.begin(), cuts.end());
      for (auto& r : plan.ar) add_range_pieces(r, da, g.trans_a, true, plan.k0);
      for (auto& r : plan.br) add_range_pieces(r, db, g.trans_b, false, plan.k0);
    }
  }
  return plan;
}

void Session::record_timing(Worker& w, bool start) {
  if (!timing_) return;
  if (start) {
    if (w.timing_used == w.timing_events.size()) {
      cudaEvent_t a, b;
      cuda_check(cudaEventCreate(&a), "cudaEventCreate");
      cuda_check(cudaEventCreate(&b), "cudaEventCreate");
      w.timing_events.push_back({a, b});
    }
    cuda_check(cudaEventRecord(w.timing_events[w.timing_used].first, w.stream), "cudaEventRecord");
  } else {
    cuda_check(cudaEventRecord(w.timing_events[w.timing_used].second, w.stream), "cudaEventRecord");
    ++w.timing_used;
  }
}

void Session::collect_timing() {
  for (auto& w : workers_) {
    if (!w) continue;
    for (std::size_t i = 0; i < w->timing_used; ++i) {
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, w->timing_events[i].first, w->timing_events[i].second),
                 "cudaEventElapsedTime");
      w->stats.gemm_ms += ms;
    }
    w->timing_used = 0;
  }
}

cudaEvent_t Session::trace_event(cudaStream_t s) {
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
  return e;
}

// Append the recorded timeline of the last command as JSON lines (one per
// record: worker, what, panel, start/end ms relative to the command start).
void Session::flush_trace(const char* op) {
  if (!tracing()) return;
  ++trace_cmd_;
  FILE* f = std::fopen(trace_path_.c_str(), "a");
  for (auto& wp : workers_) {
    if (!wp || !wp->trace_t0) continue;
    Worker& w = *wp;
    DeviceGuard g(w.device);
    for (auto& r : w.trace) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, w.trace_t0, r.a);
      cudaEventElapsedTime(&b, w.trace_t0, r.b);
      if (f)
        std::fprintf(f,
                     "{\"cmd\":%llu,\"op\":\"%s\",\"rank\":%d,\"worker\":%d,\"what\":\"%s\","
                     "\"panel\":%d,\"t0_ms\":%.4f,\"t1_ms\":%.4f,\"bytes\":%llu,\"flops\":%.6g}\n",
                     static_cast<unsigned long long>(trace_cmd_), op, rank_, w.id, r.what.c_str(), r.panel,
                     a, b, static_cast<unsigned long long>(r.bytes), r.flops);
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    w.trace.clear();
    cudaEventDestroy(w.trace_t0);
    w.trace_t0 = nullptr;
  }
  if (f) std::fclose(f);
}

void Session::cache_foreign_a(const GemmArgs& g) {
  const MatrixDescriptor& da = table_.at(g.a);
  remote_read_.insert(g.a);
  bool copied = false;
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DeviceGuard guard(w.device);
    for (int r = 0; r < da.layout.grid.n_block_rows(); ++r) {
      if (da.layout.owner({r, 0}) == w.id) continue;
      auto cached = w.cache.find({g.a, {r, 0}});
      if (cached != w.cache.end() && cached->second.version_seen == da.version) continue;
      auto [br, bc] = block_extent(da.layout.grid, {r, 0});
      bool remote = false;
      const void* src = block_src(g.a, {r, 0}, w);
      StoredBlock blk;
      blk.rows = br;
      blk.cols = bc;
      blk.precision = da.precision;
      blk.version_seen = da.version;
      blk.mem = w.pool->acquire(blk.bytes());
      cuda_check(cudaMemcpyAsync(blk.mem.data(), src, blk.bytes(), cudaMemcpyDefault, w.side),
                 "cache copy");
      (void)remote;
      w.stats.peer_bytes_read += blk.bytes();
      log_transfer(da.layout.owner({r, 0}), w.id, g.a, {r, 0}, blk.bytes());
      w.cache[{g.a, {r, 0}}] = std::move(blk);
      copied = true;
    }
  }
  if (copied) sync_local();  // a fresh cache: the copies land before the GEMM reads them
}

void Session::general_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta,
                           bool tb) {
  HostScope hs("general_gemm (total)");
  require_live();
  op_tag_ = "general_gemm";
  GemmArgs g = gemm_command(alpha, a, b, beta, c, ta, tb, false);
  validate_general(g);
  run_gemm(g, SourcePolicy::Peer);
  bump_version(c);  // runtime_types.hpp:296-301
  end_command();
  flush_trace("general_gemm");
}

void Session::cyclic_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta,
                          bool tb, bool cache_a) {
  require_live();
  SyncScope scope(this);
  op_tag_ = "cyclic_gemm";
  GemmArgs g = gemm_command(alpha, a, b, beta, c, ta, tb, cache_a);
  g.plane_cache_a = cache_a;  // the FC weight: keep its split planes while its version holds
  validate_cyclic(g, nullptr);
  if (cache_a) {
    // Keep what you've seen (CyclicGemmExec::finish, ops.hpp:278-289): fill the
    // cache first, so the GEMM reads the fresh copies and every foreign block
    // crosses the link once per version instead of twice.
    cache_foreign_a(g);
    cache_meta_[a] = table_.at(a).version;
    run_gemm(g, SourcePolicy::Peer);
  } else {
    run_gemm(g, SourcePolicy::Peer);
    for (auto& w : workers_) {
      if (!w) continue;
      auto it = w->cache.lower_bound({a, {0, 0}});
      while (it != w->cache.end() && it->first.matrix == a) it = w->cache.erase(it);
    }
    cache_meta_.erase(a);
  }
  bump_version(c);
  end_command();
}

void Session::broadcast_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta,
                             bool tb) {
  require_live();
  SyncScope scope(this);
  op_tag_ = "broadcast_gemm";
  GemmArgs g = gemm_command(alpha, a, b, beta, c, ta, tb, false);
  validate_cyclic(g, nullptr);  // build_cyclic_plan preconditions (session.hpp:239)
  // Same pulls as the ring form: every strip owner reads every foreign A block
  // whole from its owner (a fresh cached copy or replica serves instead).  No
  // cache effects either way (session.hpp:236-242 leaves cache_meta_ alone).
  run_gemm(g, SourcePolicy::Peer);
  bump_version(c);
  end_command();
}

void Session::cached_backward_gemm(MatrixId w_id, MatrixId dy, MatrixId dx) {
  require_live();
  SyncScope scope(this);
  op_tag_ = "cached_backward_gemm";
  GemmArgs g = gemm_command(1.0, w_id, dy, 0.0, dx, false, false, false);
  std::vector<WorkerId> strip_owners;
  validate_cyclic(g, &strip_owners);
  // Session::backward_missing_coords (session.hpp:547-559)
  const MatrixDescriptor& dw = table_.at(w_id);
  auto meta = cache_meta_.find(w_id);
  const bool fresh = meta != cache_meta_.end() && meta->second == dw.version;
  std::set<std::pair<int, int>> missing;
  for (WorkerId cw : std::set<WorkerId>(strip_owners.begin(), strip_owners.end()))
    for (int r = 0; r < dw.layout.grid.n_block_rows(); ++r)
      if (dw.layout.owner({r, 0}) != cw && !fresh) missing.insert({r, 0});
  if (!missing.empty())
    throw CacheMissError("cached_backward_gemm: blocks not cached at the current version",
                         {missing.begin(), missing.end()});
  g.plane_cache_a = true;  // W's split planes serve every backward until W changes
  run_gemm(g, SourcePolicy::LocalOnly);
  bump_version(dx);
  end_command();
}

// ----------------------------------------------------------- introspection

DevicePool::Stats Session::pool_stats(int w) const { return worker(w).pool->stats(); }

std::uint64_t Session::pool_trim(int w) {
  Worker& wk = worker(w);
  DeviceGuard g(wk.device);
  cuda_check(cudaStreamSynchronize(wk.stream), "sync");
  return wk.pool->trim();
}

dm_worker_stats Session::worker_stats(int w) const { return worker(w).stats; }

void Session::reset_worker_stats() {
  for (auto& w : workers_)
    if (w) w->stats = dm_worker_stats{};
}

std::uint64_t Session::worker_seed(int w) const {
  if (w < 0 || w >= P_) throw UsageError("unknown worker id");
  return mix64(root_seed_, static_cast<std::uint64_t>(w));
}

std::vector<std::uint64_t> Session::seed_workers(std::uint64_t root) {
  require_live();
  SyncScope scope(this);
  root_seed_ = root;
  std::vector<std::uint64_t> seeds;
  for (int w = 0; w < P_; ++w) {
    seeds.push_back(mix64(root, static_cast<std::uint64_t>(w)));
    if (workers_[w]) workers_[w]->seed = seeds.back();  // OpCode::Seed on each worker
  }
  end_command();
  return seeds;
}

std::uint64_t Session::master_digest() const { return table_digest(table_); }

std::vector<std::uint64_t> Session::worker_digests() const {
  std::vector<std::uint64_t> out;
  for (const auto& w : workers_)
    if (w) out.push_back(table_digest(w->descriptors));
  return out;
}

void* Session::block_device_ptr(MatrixId id, BlockCoord c, int* device) const {
  const MatrixDescriptor& d = descriptor(id);
  const int owner = d.layout.owner(c);
  const Worker* w = local(owner);
  if (w == nullptr) throw UsageError("block is not owned by a local worker");
  *device = w->device;
  return w->owned.at({id, c}).mem.data();
}

}  // namespace dm
