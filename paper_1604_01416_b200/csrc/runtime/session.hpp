// Session: the master facade of the distributed-matrix runtime on B200.
//
// Reference: gridgemm::Session (session.hpp:53-725) with WorkerContext
// (runtime_types.hpp:167-260) and the GEMM executors of ops.hpp.  The
// reference emulates workers as threads exchanging memcpy'd messages; here a
// worker is a GPU:
//   * owned / cached blocks live in HBM, allocated from a per-worker caching
//     DevicePool (pool.hpp);
//   * a GEMM is executed by every worker (owner of C blocks) as a pipeline
//     of K panels over split operand planes (scaled fp16 pair by default,
//     tf32/bf16 or 3xTF32 selectable) the tcgen05 GEMM consumes.  Large
//     f16x2 commands are "presplit": every owner splits its own A / B blocks
//     once into an IPC-exported plane arena and the consumers pull plane
//     rectangles on the copy engines while the previous panel multiplies
//     (session_presplit.cpp); otherwise each worker pulls the fp32 pieces
//     (copy engines into landing buffers, or the split kernel's own peer
//     loads) and splits them itself (session_gemm.cpp);
//   * LOCAL mode: one process drives all P workers (tests, 1-GPU parity at
//     any P);  SPMD mode: one process per GPU (torchrun), every rank issues
//     the same calls in the same order, NCCL provides the barrier and the
//     IPC-handle exchange.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "layout.hpp"
#include "pool.hpp"

namespace dm {

enum class FillKind : std::uint8_t { Zeros = 0, SeededRandom = 1, FromHost = 2 };

struct StoredBlock {
  std::int64_t rows = 0, cols = 0;
  Precision precision = Precision::Single32;
  std::uint64_t version_seen = 0;
  DeviceBuffer mem;
  std::size_t bytes() const { return static_cast<std::size_t>(rows * cols) * byte_width(precision); }
};

struct BlockKey {
  MatrixId matrix = 0;
  BlockCoord coord;
  friend bool operator<(const BlockKey& a, const BlockKey& b) {
    return a.matrix != b.matrix ? a.matrix < b.matrix : a.coord < b.coord;
  }
};

// One worker-to-worker block transfer (the reference's TransferRecord,
// transport.hpp:27-38): `bytes` is the payload this worker read from `src`'s
// block (a GEMM may read part of a block), op the command that moved it.
struct TransferRecord {
  std::uint64_t seq = 0;
  int src = 0, dst = 0;
  MatrixId matrix = 0;
  BlockCoord coord;
  std::uint64_t bytes = 0;
  std::string op;
};

struct GemmArgs {
  double alpha = 1.0, beta = 0.0;
  MatrixId a = 0, b = 0, c = 0;
  bool trans_a = false, trans_b = false, cache_a = false;
  // keep op(A)'s split planes across commands while A's version holds (the
  // FC weight of cyclic_gemm(cache_a) / cached_backward_gemm)
  bool plane_cache_a = false;
};

enum class SourcePolicy { Peer, LocalOnly };

// Outstanding device work on one matrix (asynchronous command mode): the last
// write and the reads issued since, as events on whichever stream ran them.
struct Track {
  cudaEvent_t write = nullptr;
  std::vector<cudaEvent_t> reads;
};

struct Worker {
  int id = 0;
  int device = 0;
  cudaStream_t stream = nullptr;  // GEMM stream
  cudaStream_t side = nullptr;    // split stream
  cudaStream_t pull = nullptr;    // copy engine, peer -> local landing buffers
  cudaStream_t h2d = nullptr;     // copy engine, host -> device (async scatter)
  cudaStream_t d2h = nullptr;     // copy engine, device -> host (async gather)
  std::map<MatrixId, Track> tracks;
  std::vector<cudaEvent_t> event_pool, events_used;
  struct Inflight {  // buffers of an asynchronous GEMM, released once `done` fires
    cudaEvent_t done = nullptr;
    std::vector<DeviceBuffer> bufs;
    std::vector<cudaEvent_t> events;
  };
  std::deque<Inflight> inflight;
  struct TraceRec {  // device timeline of one command (DM_TRACE)
    std::string what;
    int panel = -1;
    std::uint64_t bytes = 0;
    double flops = 0;
    cudaEvent_t a = nullptr, b = nullptr;
  };
  std::vector<TraceRec> trace;
  cudaEvent_t trace_t0 = nullptr;
  std::unique_ptr<DevicePool> pool;
  std::map<MatrixId, MatrixDescriptor> descriptors;
  std::map<BlockKey, StoredBlock> owned;
  std::map<BlockKey, StoredBlock> cache;
  std::map<BlockKey, StoredBlock> replicas;
  // Split planes of an FC weight (GemmArgs::plane_cache_a), keyed by the
  // operand geometry, valid while the matrix version equals `version`.
  struct PlaneCache {
    bool filled = false;  // holds the planes of `version`
    std::uint64_t version = 0;
    DeviceBuffer hi, second, rmax;  // rmax: kModeF16x2 row maxima
  };
  std::map<std::vector<std::int64_t>, PlaneCache> plane_cache;
  // Captured command graphs of small single-panel GEMMs (session_gemm.cpp):
  // a repeated command replays one graph instead of re-issuing its launches.
  struct GraphEntry {
    std::vector<std::uint64_t> sig;
    cudaGraphExec_t exec = nullptr;
    std::vector<DeviceBuffer> bufs;
    dm_worker_stats delta{};
    std::vector<std::pair<BlockKey, std::uint64_t>> pulls;
    std::uint64_t last_use = 0;
    MatrixId ids[3] = {0, 0, 0};
  };
  std::deque<GraphEntry> graphs;
  std::uint64_t graph_clock = 0;
  DeviceBuffer pull_flag;  // landing-copy sequence number (written by the pull stream)
  unsigned pull_seq = 0;
  DeviceBuffer arena;  // exchange buffer peers read (row/col partials, narrowed reshape payloads)
  // Owner-split planes (scaled fp16 pair) of this worker's A / B blocks for a
  // pipelined GEMM: peers pull plane rectangles from it instead of splitting
  // fp32 pieces themselves (session_gemm.cpp, "presplit").  `plane_reads`:
  // this worker's last GEMM that (with its pulls) read any worker's plane
  // arena -- the owner split of the next such command waits for it.
  DeviceBuffer plane_arena;
  cudaEvent_t plane_reads = nullptr;
  cudaEvent_t presplit_done = nullptr;  // this command's owner split (+ barrier) finished
  cudaEvent_t maxima_done = nullptr;    // this command's partial row maxima (+ barrier) finished
  cudaEvent_t presplit_order = nullptr;  // sync commands: the owner split after the compute stream
  std::uint64_t seed = 0;
  dm_worker_stats stats{};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timing_events;
  cudaEvent_t markers[16] = {};
  std::size_t timing_used = 0;
};

class Comm;  // NCCL bootstrap + IPC directory (comm.cpp)

class Session {
 public:
  explicit Session(const dm_session_config& cfg);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  int worker_count() const { return P_; }
  bool spmd() const { return mode_ == DM_MODE_SPMD; }
  int rank() const { return rank_; }
  std::vector<int> local_worker_ids() const;

  MatrixId create_matrix(const LayoutSpec& layout, Precision p, FillKind fill, const void* host);
  void destroy_matrix(MatrixId id);
  void scatter(MatrixId id, const void* host, std::int64_t rows, std::int64_t cols);
  void gather(MatrixId id, void* host, std::int64_t rows, std::int64_t cols, int root);
  void update_block(MatrixId id, BlockCoord c, const void* host, std::int64_t rows, std::int64_t cols);
  // replication, reshape, row/col sums, checkpoint
  void replicate(MatrixId id, bool enable);
  void replica_read(MatrixId id, int reader, void* host, std::int64_t rows, std::int64_t cols);
  MatrixId reshape(MatrixId src, const LayoutSpec& layout, Precision p);
  MatrixId add_row_col_sum(MatrixId id, int axis, bool deterministic);
  void checkpoint(const std::string& path);
  void restore_image(const std::string& path);  // into a fresh session
  std::uint64_t next_matrix_id() const { return next_matrix_id_; }
  std::uint64_t root_seed() const { return root_seed_; }
  int gemm_mode() const { return gemm_mode_; }  // kModeMixed / kModeTf32x3 / kModeAuto
  void general_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta,
                    bool tb);
  void cyclic_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta, bool tb,
                   bool cache_a);
  // broadcast_gemm_reference (session.hpp:236-242, BroadcastGemmExec
  // ops.hpp:578-651): the ring's preconditions and result, every A block read
  // whole by every strip owner; A's block cache and cache_meta_ are untouched.
  void broadcast_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta, bool tb);
  void cached_backward_gemm(MatrixId w, MatrixId dy, MatrixId dx);
  void shutdown();
  bool live() const { return live_; }

  const MatrixDescriptor& descriptor(MatrixId id) const;
  DevicePool::Stats pool_stats(int w) const;
  std::uint64_t pool_trim(int w);
  dm_worker_stats worker_stats(int w) const;
  void reset_worker_stats();
  void set_gemm_timing(bool on) { timing_ = on; }
  std::uint64_t worker_seed(int w) const;
  // Session::seed_workers (session.hpp:115-125): new root seed for the worker
  // seeds and for every matrix created afterwards; returns mix64(root, w).
  std::vector<std::uint64_t> seed_workers(std::uint64_t root);
  std::uint64_t master_digest() const;
  std::vector<std::uint64_t> worker_digests() const;
  void* block_device_ptr(MatrixId id, BlockCoord c, int* device) const;
  void barrier();
  // Asynchronous command mode: create/scatter/gather/general_gemm enqueue
  // stream-ordered work and return; dependencies are tracked per matrix with
  // events (device-side NCCL barriers between ranks in SPMD).  Host buffers
  // must stay valid and unmodified until barrier()/set_async(false).
  void set_async(bool on);
  bool async_mode() const { return async_; }
  void marker_record(int w, int slot);
  float marker_elapsed(int w, int a, int b);

 private:
  struct Piece {
    MatrixId matrix = 0;
    BlockCoord coord;
    std::int64_t src_off = 0, lds = 0;
    int trans = 0;
    std::int64_t rows = 0, kcols = 0;
    std::int64_t dst_row = 0, dst_k = 0;
    std::size_t bytes() const { return static_cast<std::size_t>(rows * kcols) * 4; }
  };
  struct Range {
    std::int64_t start = 0, len = 0;
    std::vector<std::vector<Piece>> panels;  // [panel] -> pieces
  };
  struct Task {
    BlockCoord c;
    int ra = 0, rb = 0;
  };
  struct WorkerPlan {
    std::vector<Range> ar, br;
    std::vector<Task> tasks;
    std::vector<std::int64_t> k0;  // panel starts, size np+1
    bool has_remote = false;
  };

  void materialize(const MatrixDescriptor& d, bool seeded);
  const void* block_src(MatrixId id, BlockCoord c, const Worker& reader) const;
  void sync_replicas(MatrixId id);
  void* arena(int w, std::size_t* bytes);
  void ensure_arenas(std::size_t bytes);
  void mid_barrier();
  void drain();
  void reap_inflight(Worker& w);
  void bound_inflight(Worker& w);  // reap, then wait while >= DM_MAX_INFLIGHT GEMMs queued
  cudaEvent_t ev_get(Worker& w);
  void mark_write(Worker& w, cudaStream_t s, MatrixId id);
  void mark_read(Worker& w, cudaStream_t s, MatrixId id);
  void wait_writes(cudaStream_t s, MatrixId id);
  void wait_all(cudaStream_t s, MatrixId id);
  void device_barrier(cudaStream_t s, int channel);
  Worker& worker(int w);
  const Worker& worker(int w) const;
  Worker* local(int w);
  const Worker* local(int w) const;
  void require_live() const;
  void validate_layout_workers(const LayoutSpec& l) const;
  void apply_effects_create(const MatrixDescriptor& d);
  void bump_version(MatrixId id);
  void end_command();
  void sync_local();

  GemmArgs gemm_command(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool ta,
                        bool tb, bool cache_a) const;
  void validate_general(const GemmArgs& g) const;
  void validate_cyclic(const GemmArgs& g, std::vector<WorkerId>* strip_owners) const;

  WorkerPlan plan_worker(const GemmArgs& g, int w, SourcePolicy pol, bool presplit = false) const;
  // Presplit GEMM (scaled fp16 pair, pipelined): every owner splits its own A
  // and B blocks once into its plane arena; consumers pull plane rectangles.
  // Decided from replicated state only (every rank agrees: it adds a barrier).
  bool presplit_eligible(const GemmArgs& g, SourcePolicy pol) const;
  struct ArenaBlock {  // one owned block's planes in its owner's plane arena
    // byte offsets: fp16 planes, this block's row maxima, the whole op row's
    // maxima (max over the blocks of its band -- the scale the planes carry)
    std::size_t h0 = 0, h1 = 0, rmax = 0, grmax = 0;
    std::int64_t oprows = 0, kext = 0, ld = 0;
    int trans = 0;
  };
  // role 0: A blocks (op(A) rows), role 1: B blocks (op(B)^T rows)
  std::map<std::pair<int, BlockKey>, ArenaBlock> plane_arena_map(const GemmArgs& g, int owner,
                                                                 std::size_t* total) const;
  void ensure_plane_arenas(std::size_t bytes);
  void presplit_owners(const GemmArgs& g);
  void add_range_pieces(Range& rg, const MatrixDescriptor& d, bool op_rows_trans, bool is_a,
                        const std::vector<std::int64_t>& k0) const;
  const void* source_ptr(const Worker& reader, MatrixId m, BlockCoord c, SourcePolicy pol,
                         bool* remote) const;
  void run_gemm(const GemmArgs& g, SourcePolicy pol);
  void drop_graphs(Worker& w, MatrixId id);  // id 0: all
  struct GemmRun;  // one worker's K-panel pipeline of one GEMM command (session_gemm.cpp)
  friend struct GemmRun;
  void cache_foreign_a(const GemmArgs& g);
  void record_timing(Worker& w, bool start);
  void collect_timing();
  // device timeline (DM_TRACE=<file>): events around each panel's pulls and GEMMs
  bool tracing() const { return !trace_path_.empty(); }
  cudaEvent_t trace_event(cudaStream_t s);
  void flush_trace(const char* op);

  int P_ = 1;
  int mode_ = DM_MODE_LOCAL;
  int gemm_mode_ = 2;  // kModeAuto
  int rank_ = 0;
  bool coherence_ = true;
  bool live_ = false;
  bool timing_ = false;
  bool async_ = false;
  // Set when a command already drained every stream it used (run_gemm's
  // per-worker sync: its split / pull streams all feed the GEMM stream), so
  // end_command need not synchronise the idle ones again (~1.5 us each).
  bool streams_drained_ = false;
  std::string trace_path_;
  std::uint64_t trace_cmd_ = 0;
  std::uint64_t root_seed_ = 0;
  std::uint64_t next_matrix_id_ = 1;
  std::vector<std::unique_ptr<Worker>> workers_;  // index = worker id; null if not local
  std::map<MatrixId, MatrixDescriptor> table_;
  std::map<MatrixId, std::uint64_t> cache_meta_;
  // Asynchronous mode: matrices whose blocks a peer GPU may have read since
  // their last write (operands of GEMMs whose consumers pull fp32 pieces,
  // cache fills).  Replicated -- every rank issues the same commands.  A
  // scatter needs the cross-rank barrier only for these; presplit GEMMs read
  // A / B only on their owners (peers pull the plane arenas), so a resident
  // operand refreshed every step is overwritten without waiting for a
  // barrier that could only run after the GEMM freed the SMs.
  std::set<MatrixId> remote_read_;
  std::uint64_t nondet_counter_ = 0;
  // trace() (transport.hpp:56-71): this process's pulls, the newest
  // DM_TRACE_CAP (default 2^20) records -- bounded so long runs do not grow it
  std::deque<TransferRecord> transfers_;
  std::uint64_t transfer_seq_ = 0;
  const char* op_tag_ = "";  // command being executed (TransferRecord::op)
 public:
  const std::deque<TransferRecord>& transfers() const { return transfers_; }
  void log_transfer(int src, int dst, MatrixId m, BlockCoord c, std::uint64_t bytes) {
    static const std::size_t cap = static_cast<std::size_t>(std::max<std::int64_t>(1, env_int("DM_TRACE_CAP", 1 << 20)));
    // BroadcastGemmExec tags each fan-out with the block row (ops.hpp:600-603)
    std::string op = op_tag_;
    if (op == "broadcast_gemm") op += ":r" + std::to_string(c.row);
    transfers_.push_back({++transfer_seq_, src, dst, m, c, bytes, std::move(op)});
    while (transfers_.size() > cap) transfers_.pop_front();
  }
 private:
  std::size_t arena_bytes_ = 0;               // replicated: every worker's arena size
  std::vector<void*> arena_ptrs_;             // per worker (peer-readable)
  std::size_t plane_arena_bytes_ = 0;         // same for the presplit plane arenas
  std::vector<char*> plane_arena_ptrs_;
  std::unique_ptr<Comm> comm_;
};

// Commands without an asynchronous form drain outstanding work first and run
// synchronously (their end_command syncs and checks coherence).
struct SyncScope {
  Session* s;
  bool prev;
  explicit SyncScope(Session* ss);
  ~SyncScope();
  SyncScope(const SyncScope&) = delete;
  SyncScope& operator=(const SyncScope&) = delete;
};

}  // namespace dm
