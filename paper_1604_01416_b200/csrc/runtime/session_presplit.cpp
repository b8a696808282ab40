// Presplit GEMM commands: the owner of each A / B block splits it ONCE into
// the scaled fp16 pair (kModeF16x2) in its plane arena; every worker whose
// C blocks need a piece of it pulls the plane rectangle (4 B / element, the
// same bytes as the fp32 piece) instead of pulling fp32 and splitting it
// itself.  Same pieces and the same pull plan as GeneralGemmExec
// (ops.hpp:406-503); what changes is WHO splits:
//   consumer split: every worker splits op(A) rows + op(B) columns of its C
//                   blocks -- N^2 (1/pr + 1/pc) elements per worker per GEMM,
//                   between its GEMM launches (the split kernels cannot run
//                   beside the persistent GEMM);
//   owner split:    every worker splits its own A and B blocks -- 2 N^2 / P
//                   elements, once, before the first panel; the pulls then
//                   move planes on the copy engines while the GEMMs run.
// At P = 4 (2x2) that halves the split work, at P = 8 (2x4) it is a third.
//
// The row scale of a plane row is the power of two of its |x| maximum over
// the WHOLE op(X) row, as in a one-GPU split: the owners first write their
// blocks' partial row maxima, then (after a barrier) each combines the
// partials of its row band -- the blocks sharing its op rows, on any GPU --
// and splits with that.  Every piece of a plane row therefore carries the
// same scale, so K panels may span several owners' blocks.
#include <algorithm>

#include "../kernels/tf32x3_gemm.h"
#include "comm.hpp"
#include "session.hpp"

namespace dm {

namespace {
constexpr MatrixId kPlaneArenaId = ~MatrixId{0};  // never a matrix id
constexpr std::size_t kAlign = 256;
std::size_t align_up(std::size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
}  // namespace

bool Session::presplit_eligible(const GemmArgs& g, SourcePolicy pol) const {
  if (P_ < 2 || pol != SourcePolicy::Peer || g.cache_a || g.plane_cache_a) return false;
  if (env_int("DM_PRESPLIT", 1) == 0) return false;
  const MatrixDescriptor& da = table_.at(g.a);
  const MatrixDescriptor& db = table_.at(g.b);
  const MatrixDescriptor& dc = table_.at(g.c);
  for (const MatrixDescriptor* d : {&da, &db, &dc})
    if (d->precision != Precision::Single32) return false;
  const std::int64_t K = g.trans_a ? da.layout.grid.global_rows : da.layout.grid.global_cols;
  if (K <= 512) return false;
  // every source must be the owner's block: fresh caches / replicas (read in
  // place by the consumer split path) keep that path
  if (da.replicated || db.replicated) return false;
  for (MatrixId id : {g.a, g.b}) {
    auto it = cache_meta_.find(id);
    if (it != cache_meta_.end() && it->second == table_.at(id).version) return false;
  }
  // plane rows start 16-B aligned at every panel start: K-block edges % 8
  const std::int64_t ka = g.trans_a ? da.layout.grid.block_rows : da.layout.grid.block_cols;
  const std::int64_t kb = g.trans_b ? db.layout.grid.block_cols : db.layout.grid.block_rows;
  if (ka % 8 != 0 || kb % 8 != 0) return false;
  // a row band's partial maxima are combined in one launch
  const int band_a = g.trans_a ? da.layout.grid.n_block_rows() : da.layout.grid.n_block_cols();
  const int band_b = g.trans_b ? db.layout.grid.n_block_cols() : db.layout.grid.n_block_rows();
  if (band_a > RowmaxSources::kMax || band_b > RowmaxSources::kMax) return false;
  // only pipelined commands (enough math per worker to hide the pulls)
  const double min_work = static_cast<double>(env_int("DM_PIPELINE_MIN_GFLOP", 200)) * 1e9;
  bool any = false;
  for (int w = 0; w < P_; ++w) {
    double work = 0;
    for (BlockCoord c : owned_coords(dc.layout, w)) {
      auto [mb, nb] = block_extent(dc.layout.grid, c);
      work += 2.0 * mb * nb * static_cast<double>(K);
    }
    if (work == 0) continue;
    if (work < min_work || resolve_split_mode(gemm_mode_, K, work) != kModeF16x2) return false;
    any = true;
  }
  return any;
}

// Planes of `owner`'s A blocks (role 0, op(A) rows, K-major) then B blocks
// (role 1, op(B)^T rows), block-row-major; per block h0 | h1 | rmax | grmax.
std::map<std::pair<int, BlockKey>, Session::ArenaBlock> Session::plane_arena_map(const GemmArgs& g, int owner,
                                                                                 std::size_t* total) const {
  std::map<std::pair<int, BlockKey>, ArenaBlock> out;
  std::size_t off = 0;
  for (int role = 0; role < 2; ++role) {
    const MatrixDescriptor& d = table_.at(role == 0 ? g.a : g.b);
    const int trans = role == 0 ? (g.trans_a ? 1 : 0) : (g.trans_b ? 0 : 1);
    for (BlockCoord c : owned_coords(d.layout, owner)) {
      auto [rows, cols] = block_extent(d.layout.grid, c);
      ArenaBlock ab;
      ab.trans = trans;
      ab.oprows = trans ? cols : rows;
      ab.kext = trans ? rows : cols;
      ab.ld = (ab.kext + 7) / 8 * 8;
      const std::size_t plane = static_cast<std::size_t>(ab.oprows * ab.ld) * 2;
      ab.h0 = off;
      ab.h1 = off = align_up(off + plane);
      ab.rmax = off = align_up(off + plane);
      ab.grmax = off = align_up(off + static_cast<std::size_t>(ab.oprows) * 4);
      off = align_up(off + static_cast<std::size_t>(ab.oprows) * 4);
      out[{role, BlockKey{d.matrix_id, c}}] = ab;
    }
  }
  *total = off;
  return out;
}

// Collective (every rank passes the same size): plane arenas only grow and
// are exported once per growth, like the exchange arenas (session_ops.cpp).
void Session::ensure_plane_arenas(std::size_t bytes) {
  if (bytes <= plane_arena_bytes_ && !plane_arena_ptrs_.empty()) return;
  sync_local();
  if (comm_) {
    comm_->barrier();
    comm_->unpublish(kPlaneArenaId);
  }
  plane_arena_ptrs_.assign(P_, nullptr);
  for (auto& w : workers_) {
    if (!w) continue;
    DeviceGuard guard(w->device);
    w->plane_arena = DeviceBuffer();
    w->plane_arena = w->pool->acquire(bytes);
    plane_arena_ptrs_[w->id] = static_cast<char*>(w->plane_arena.data());
  }
  if (comm_) {
    const LayoutSpec lay = make_layout(LayoutKind::RowBlocks1D, P_, 1, 1, 1, P_);
    comm_->publish_raw(kPlaneArenaId, lay,
                       {{BlockKey{kPlaneArenaId, {rank_, 0}}, workers_[rank_]->plane_arena.data()}});
    for (int r = 0; r < P_; ++r)
      if (r != rank_)
        plane_arena_ptrs_[r] = reinterpret_cast<char*>(const_cast<float*>(comm_->remote_ptr(kPlaneArenaId, {r, 0})));
  }
  plane_arena_bytes_ = bytes;
}

// Every local worker splits its own A / B blocks into its plane arena on its
// split stream, in two barrier-separated phases: (1) partial row maxima of
// each owned block; (2) the whole-row maxima of each owned block's row band
// (read from every band member's arena, peers included), then the split.
// Pulls ordered after `presplit_done` (phase 2's barrier) see every owner's
// planes.  The caller has ordered the split stream after the operands' writes
// and after every earlier reader of the arenas (Worker::plane_reads, plus the
// async preamble's barrier).
void Session::presplit_owners(const GemmArgs& g) {
  std::map<int, std::map<std::pair<int, BlockKey>, ArenaBlock>> maps;
  std::size_t need = kAlign;
  for (int w = 0; w < P_; ++w) {
    std::size_t t = 0;
    maps[w] = plane_arena_map(g, w, &t);
    need = std::max(need, t);
  }
  ensure_plane_arenas(need);
  for (auto& wp : workers_) {  // phase 1: partial maxima
    if (!wp) continue;
    Worker& w = *wp;
    DeviceGuard guard(w.device);
    for (auto& o : workers_)
      if (o && o->plane_reads) cuda_check(cudaStreamWaitEvent(w.side, o->plane_reads, 0), "wait plane readers");
    char* base = plane_arena_ptrs_.at(w.id);
    for (const auto& [key, ab] : maps.at(w.id)) {
      if (ab.oprows <= 0 || ab.kext <= 0) continue;
      const StoredBlock& blk = w.owned.at(key.second);
      unsigned* rmax = reinterpret_cast<unsigned*>(base + ab.rmax);
      cuda_check(cudaMemsetAsync(rmax, 0, static_cast<std::size_t>(ab.oprows) * 4, w.side), "memset row maxima");
      cuda_check(absmax_rows(blk.mem.f32(), blk.cols, ab.trans, ab.oprows, ab.kext, rmax, w.side), "absmax_rows");
      w.stats.split_launches += 1;
    }
    device_barrier(w.side, 1);  // every owner's partial maxima exist
    if (!w.maxima_done) cuda_check(cudaEventCreateWithFlags(&w.maxima_done, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(w.maxima_done, w.side), "event");
  }
  for (auto& wp : workers_) {  // phase 2: whole-row maxima, split
    if (!wp) continue;
    Worker& w = *wp;
    DeviceGuard guard(w.device);
    for (auto& o : workers_)  // (LOCAL mode: the other workers' phase 1)
      if (o && o.get() != &w) cuda_check(cudaStreamWaitEvent(w.side, o->maxima_done, 0), "wait maxima");
    cudaEvent_t ta = (tracing() && !async_) ? trace_event(w.side) : nullptr;
    std::uint64_t bytes = 0;
    char* base = plane_arena_ptrs_.at(w.id);
    for (const auto& [key, ab] : maps.at(w.id)) {
      if (ab.oprows <= 0 || ab.kext <= 0) continue;
      const int role = key.first;
      const MatrixDescriptor& d = table_.at(key.second.matrix);
      const BlockCoord c = key.second.coord;
      // the band: blocks sharing this block's op rows (same block row when
      // op rows are stored rows, same block column otherwise)
      RowmaxSources src;
      const int nb = ab.trans ? d.layout.grid.n_block_rows() : d.layout.grid.n_block_cols();
      for (int i = 0; i < nb; ++i) {
        const BlockCoord y = ab.trans ? BlockCoord{i, c.col} : BlockCoord{c.row, i};
        const int oy = d.layout.owner(y);
        const ArenaBlock& aby = maps.at(oy).at({role, BlockKey{d.matrix_id, y}});
        if (aby.kext <= 0) continue;
        src.p[src.n++] = reinterpret_cast<const unsigned*>(plane_arena_ptrs_.at(oy) + aby.rmax);
      }
      unsigned* grmax = reinterpret_cast<unsigned*>(base + ab.grmax);
      cuda_check(rowmax_combine(src, grmax, ab.oprows, w.side), "rowmax_combine");
      const StoredBlock& blk = w.owned.at(key.second);
      cuda_check(split_f16x2(blk.mem.f32(), blk.cols, ab.trans, ab.oprows, ab.kext, base + ab.h0, base + ab.h1, ab.ld,
                             grmax, w.side),
                 "split_f16x2");
      w.stats.split_launches += 2;
      bytes += static_cast<std::uint64_t>(ab.oprows * ab.kext) * 4;
    }
    if (ta) w.trace.push_back({"presplit", -1, bytes, 0.0, ta, trace_event(w.side)});
    device_barrier(w.side, 1);  // every owner's planes exist before any peer pulls them
    if (!w.presplit_done) cuda_check(cudaEventCreateWithFlags(&w.presplit_done, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(w.presplit_done, w.side), "event");
  }
}

}  // namespace dm
