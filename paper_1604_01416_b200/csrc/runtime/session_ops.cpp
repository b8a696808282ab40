// Session commands beside the GEMM: update_block, replication,
// reshape with precision change, distributed row/column sums and the DMTH
// checkpoint.  Citations are to /root/reference/proj/include/gridgemm/.
//
// Data movement follows the same B200 pattern as the GEMM: every worker pulls
// what it needs straight from the owner's HBM (peer access / CUDA IPC); when a
// producer must transform data first (narrowing before the link, row/column
// partials) it writes into its exchange arena -- a per-worker buffer exported
// once like a block -- and the consumers pull from there after one barrier.
#include <algorithm>
#include <cstring>
#include <fstream>
#include <set>

#include "../kernels/dataops.h"
#include "comm.hpp"
#include "session.hpp"

namespace dm {

namespace {

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

constexpr MatrixId kArenaId = 0;  // matrix ids start at 1 (session.hpp:717)

// Upload a small host table to a pooled device buffer (stream-ordered).
template <typename T>
const T* upload(Worker& w, std::vector<DeviceBuffer>& keep, const std::vector<T>& v) {
  keep.push_back(w.pool->acquire(std::max<std::size_t>(v.size() * sizeof(T), 64)));
  cuda_check(cudaMemcpyAsync(keep.back().data(), v.data(), v.size() * sizeof(T),
                             cudaMemcpyHostToDevice, w.stream),
             "upload table");
  return static_cast<const T*>(keep.back().data());
}

void put_le(std::vector<unsigned char>& out, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<unsigned char>(v >> (8 * i)));
}

std::uint64_t get_le(const unsigned char* p, int bytes) {
  std::uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
  return v;
}

}  // namespace

// ------------------------------------------------------------ exchange arena

void Session::mid_barrier() {
  sync_local();
  if (comm_) comm_->barrier();
}

// Collective: every rank passes the same byte count (computed from the
// replicated descriptors).  Arenas only grow; they are exported once.
void Session::ensure_arenas(std::size_t bytes) {
  if (bytes <= arena_bytes_ && !arena_ptrs_.empty()) return;
  const std::size_t cap = DevicePool::size_class(std::max<std::size_t>(bytes, 2 * arena_bytes_));
  sync_local();
  if (comm_) {
    comm_->barrier();
    comm_->unpublish(kArenaId);
  }
  arena_ptrs_.assign(P_, nullptr);
  for (auto& w : workers_) {
    if (!w) continue;
    w->arena = DeviceBuffer();
    w->arena = w->pool->acquire(cap);
    arena_ptrs_[w->id] = w->arena.data();
  }
  if (comm_) {
    // each worker owns row block w of a P x 1 "matrix" whose blocks are arenas
    const LayoutSpec lay = make_layout(LayoutKind::RowBlocks1D, P_, 1, 1, 1, P_);
    comm_->publish_raw(kArenaId, lay, {{BlockKey{kArenaId, {rank_, 0}}, workers_[rank_]->arena.data()}});
    for (int r = 0; r < P_; ++r)
      if (r != rank_) arena_ptrs_[r] = const_cast<float*>(comm_->remote_ptr(kArenaId, {r, 0}));
  }
  arena_bytes_ = cap;
}

void* Session::arena(int w, std::size_t* bytes) {
  if (bytes) *bytes = arena_bytes_;
  return arena_ptrs_.at(w);
}

// ------------------------------------------------------------ update_block

// Session::update_block (session.hpp:203-222): replace one block from host
// data of the matrix's precision; version += 1 (runtime_types.hpp:293-295).
void Session::update_block(MatrixId id, BlockCoord c, const void* host, std::int64_t rows,
                           std::int64_t cols) {
  require_live();
  SyncScope scope(this);
  const MatrixDescriptor d = descriptor(id);
  auto [br, bc] = block_extent(d.layout.grid, c);
  if (rows != br || cols != bc)
    throw ShapeError("update_block: data shape does not match the block extent");
  const int owner = d.layout.owner(c);
  if (Worker* w = local(owner)) {
    if (host == nullptr) throw UsageError("update_block: null host pointer");
    DevGuard g(w->device);
    StoredBlock& blk = w->owned.at({id, c});
    cuda_check(cudaMemcpyAsync(blk.mem.data(), host, blk.bytes(), cudaMemcpyHostToDevice, w->stream),
               "update_block H2D");
  }
  bump_version(id);
  end_command();
}

// ------------------------------------------------------------ replication

void Session::sync_replicas(MatrixId id) {
  const MatrixDescriptor& d = table_.at(id);
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DevGuard g(w.device);
    for (int r = 0; r < d.layout.grid.n_block_rows(); ++r)
      for (int c = 0; c < d.layout.grid.n_block_cols(); ++c) {
        if (d.layout.owner({r, c}) == w.id) continue;
        auto it = w.replicas.find({id, {r, c}});
        if (it != w.replicas.end() && it->second.version_seen == d.version) continue;
        auto [br, bc] = block_extent(d.layout.grid, {r, c});
        StoredBlock blk;
        blk.rows = br;
        blk.cols = bc;
        blk.precision = d.precision;
        blk.version_seen = d.version;
        blk.mem = w.pool->acquire(blk.bytes());
        cuda_check(cudaMemcpyAsync(blk.mem.data(), block_src(id, {r, c}, w), blk.bytes(),
                                   cudaMemcpyDefault, w.side),
                   "replica pull");
        w.stats.peer_bytes_read += blk.bytes();
        log_transfer(d.layout.owner({r, c}), w.id, id, {r, c}, blk.bytes());
        w.replicas[{id, {r, c}}] = std::move(blk);
      }
  }
  sync_local();
}

// ReplicateExec (ops.hpp:660-702) + descriptor effects (runtime_types.hpp:302-307).
void Session::replicate(MatrixId id, bool enable) {
  op_tag_ = "replicate";
  require_live();
  SyncScope scope(this);
  descriptor(id);
  if (enable && P_ > 1) sync_replicas(id);
  if (!enable)
    for (auto& w : workers_) {
      if (!w) continue;
      auto it = w->replicas.lower_bound({id, {0, 0}});
      while (it != w->replicas.end() && it->first.matrix == id) it = w->replicas.erase(it);
    }
  auto apply = [&](MatrixDescriptor& d) {
    d.replicated = enable;
    d.replica_version = enable ? d.version : 0;
  };
  apply(table_.at(id));
  for (auto& w : workers_)
    if (w) apply(w->descriptors.at(id));
  end_command();
}

// Session::replica_read (session.hpp:270-297): lazy version-checked resync,
// then the full matrix from worker `reader`'s owned blocks + replicas.
void Session::replica_read(MatrixId id, int reader, void* host, std::int64_t rows,
                           std::int64_t cols) {
  require_live();
  SyncScope scope(this);
  const MatrixDescriptor d0 = descriptor(id);
  if (!d0.replicated) throw UsageError("replica_read: matrix is not replicated");
  if (reader < 0 || reader >= P_) throw UsageError("unknown worker id");
  const BlockGrid& g = d0.layout.grid;
  if (rows != g.global_rows || cols != g.global_cols)
    throw ShapeError("replica_read: host buffer shape does not match the matrix");
  if (d0.replica_version < d0.version && P_ > 1) sync_replicas(id);
  if (Worker* w = local(reader)) {
    if (host == nullptr) throw UsageError("replica_read: null host pointer");
    DevGuard gd(w->device);
    const std::size_t esz = byte_width(d0.precision);
    for (int r = 0; r < g.n_block_rows(); ++r)
      for (int c = 0; c < g.n_block_cols(); ++c) {
        const StoredBlock& blk = d0.layout.owner({r, c}) == reader ? w->owned.at({id, {r, c}})
                                                                   : w->replicas.at({id, {r, c}});
        if (blk.version_seen < d0.version) throw ProtocolError("replica_read: stale replica after sync");
        char* dst = static_cast<char*>(host) +
                    (static_cast<std::int64_t>(r) * g.block_rows * g.global_cols +
                     static_cast<std::int64_t>(c) * g.block_cols) * esz;
        cuda_check(cudaMemcpy2DAsync(dst, static_cast<std::size_t>(g.global_cols) * esz, blk.mem.data(),
                                     static_cast<std::size_t>(blk.cols) * esz,
                                     static_cast<std::size_t>(blk.cols) * esz,
                                     static_cast<std::size_t>(blk.rows), cudaMemcpyDeviceToHost,
                                     w->stream),
                   "replica_read D2H");
      }
  }
  auto apply = [&](MatrixDescriptor& d) {
    if (d.replicated) d.replica_version = d.version;
  };
  apply(table_.at(id));
  for (auto& w : workers_)
    if (w) apply(w->descriptors.at(id));
  end_command();
}

// ------------------------------------------------------------ reshape

// ReshapeExec (ops.hpp:772-944): same row-major linear index, any layout and
// worker set, precision change; narrowing runs before the link (payload at the
// narrower precision), widening at the receiver.
MatrixId Session::reshape(MatrixId src, const LayoutSpec& layout, Precision p) {
  require_live();
  SyncScope scope(this);
  const MatrixDescriptor sd = descriptor(src);
  validate_layout_workers(layout);
  const BlockGrid& gs = sd.layout.grid;
  if (gs.global_rows * gs.global_cols != layout.grid.global_rows * layout.grid.global_cols)
    throw ShapeError("reshape: element count must be preserved");
  MatrixDescriptor nd;
  nd.matrix_id = next_matrix_id_++;
  nd.layout = layout;
  nd.precision = p;
  nd.seed = mix64(root_seed_, nd.matrix_id);
  materialize(nd, false);

  const Precision pay = byte_width(sd.precision) > byte_width(p) ? p : sd.precision;
  const int nbr = gs.n_block_rows(), nbc = gs.n_block_cols();
  // per-source-block payload offsets inside its owner's arena (narrowing only)
  std::vector<std::size_t> off(static_cast<std::size_t>(nbr) * nbc, 0);
  if (pay != sd.precision) {
    std::vector<std::size_t> used(P_, 0);
    for (int r = 0; r < nbr; ++r)
      for (int c = 0; c < nbc; ++c) {
        const int o = sd.layout.owner({r, c});
        auto [br, bc] = block_extent(gs, {r, c});
        off[static_cast<std::size_t>(r) * nbc + c] = used[o];
        used[o] += (static_cast<std::size_t>(br * bc) * byte_width(pay) + 255) / 256 * 256;
      }
    ensure_arenas(*std::max_element(used.begin(), used.end()));
    for (auto& w : workers_) {
      if (!w) continue;
      DevGuard g(w->device);
      for (BlockCoord c : owned_coords(sd.layout, w->id)) {
        const StoredBlock& blk = w->owned.at({src, c});
        char* dst = static_cast<char*>(w->arena.data()) + off[static_cast<std::size_t>(c.row) * nbc + c.col];
        cuda_check(convert_copy(blk.mem.data(), static_cast<int>(sd.precision), dst, static_cast<int>(pay),
                                blk.rows * blk.cols, w->stream),
                   "reshape narrow");
      }
    }
    mid_barrier();
  }
  std::vector<std::vector<DeviceBuffer>> keep(P_);
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DevGuard g(w.device);
    std::vector<const void*> table(static_cast<std::size_t>(nbr) * nbc);
    for (int r = 0; r < nbr; ++r)
      for (int c = 0; c < nbc; ++c) {
        const std::size_t k = static_cast<std::size_t>(r) * nbc + c;
        table[k] = pay != sd.precision
                       ? static_cast<const char*>(arena_ptrs_[sd.layout.owner({r, c})]) + off[k]
                       : block_src(src, {r, c}, w);
      }
    const void* const* dtable = upload(w, keep[w.id], table);
    for (BlockCoord c : owned_coords(layout, w.id)) {
      StoredBlock& blk = w.owned.at({nd.matrix_id, c});
      RemapGeometry geo;
      geo.dst_rows = blk.rows;
      geo.dst_cols = blk.cols;
      geo.r0 = static_cast<std::int64_t>(c.row) * layout.grid.block_rows;
      geo.c0 = static_cast<std::int64_t>(c.col) * layout.grid.block_cols;
      geo.dst_gcols = layout.grid.global_cols;
      geo.src_grows = gs.global_rows;
      geo.src_gcols = gs.global_cols;
      geo.src_brows = gs.block_rows;
      geo.src_bcols = gs.block_cols;
      geo.src_nbc = nbc;
      cuda_check(remap_gather(dtable, static_cast<int>(pay), blk.mem.data(), static_cast<int>(p), geo,
                              w.stream),
                 "reshape remap");
    }
  }
  sync_local();
  keep.clear();
  end_command();
  return nd.matrix_id;
}

// ------------------------------------------------------------ row/col sums

// Session::add_row_col_sum (session.hpp:321-348) + RowColSumExec
// (ops.hpp:954-1119): each contributing worker folds its blocks of a segment
// lane-ascending at the accumulation precision; the segment owner folds the
// partials in worker-id order (deterministic) or in the reference's salted
// permutation (fast mode), so both modes are bit-exact with the reference.
MatrixId Session::add_row_col_sum(MatrixId id, int axis, bool deterministic) {
  require_live();
  SyncScope scope(this);
  const MatrixDescriptor d = descriptor(id);
  const BlockGrid& g = d.layout.grid;
  const bool rows_axis = axis == 0;
  const int segments = rows_axis ? g.n_block_rows() : g.n_block_cols();
  const int lanes = rows_axis ? g.n_block_cols() : g.n_block_rows();
  MatrixDescriptor od;
  od.matrix_id = next_matrix_id_++;
  od.precision = d.precision;
  od.seed = mix64(root_seed_, od.matrix_id);
  std::vector<WorkerId> owners;
  for (int s = 0; s < segments; ++s)
    owners.push_back(d.layout.owner(rows_axis ? BlockCoord{s, 0} : BlockCoord{0, s}));
  od.layout = rows_axis ? make_custom_layout(make_grid(g.global_rows, 1, g.block_rows, 1),
                                             d.layout.worker_count, owners)
                        : make_custom_layout(make_grid(1, g.global_cols, 1, g.block_cols),
                                             d.layout.worker_count, owners);
  const std::uint64_t salt = mix64(root_seed_, ++nondet_counter_);
  materialize(od, false);

  const std::size_t esz = byte_width(d.precision);
  auto seg_len = [&](int s) {
    auto [r, c] = block_extent(g, rows_axis ? BlockCoord{s, 0} : BlockCoord{0, s});
    return rows_axis ? r : c;
  };
  auto contributors = [&](int s) {
    std::set<WorkerId> out;
    for (int l = 0; l < lanes; ++l)
      out.insert(d.layout.owner(rows_axis ? BlockCoord{s, l} : BlockCoord{l, s}));
    return std::vector<WorkerId>(out.begin(), out.end());
  };
  // arena offsets: worker w's partial of segment s
  std::vector<std::vector<std::size_t>> off(P_, std::vector<std::size_t>(segments, 0));
  std::vector<std::size_t> used(P_, 0);
  for (int s = 0; s < segments; ++s)
    for (WorkerId c : contributors(s)) {
      off[c][s] = used[c];
      used[c] += (static_cast<std::size_t>(seg_len(s)) * esz + 255) / 256 * 256;
    }
  ensure_arenas(std::max<std::size_t>(64, *std::max_element(used.begin(), used.end())));

  std::vector<std::vector<DeviceBuffer>> keep(P_);
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DevGuard gd(w.device);
    for (int s = 0; s < segments; ++s) {
      std::vector<const void*> ptrs;
      std::vector<std::int64_t> inner, pitch;
      for (int l = 0; l < lanes; ++l) {
        const BlockCoord c = rows_axis ? BlockCoord{s, l} : BlockCoord{l, s};
        if (d.layout.owner(c) != w.id) continue;
        const StoredBlock& blk = w.owned.at({id, c});
        ptrs.push_back(blk.mem.data());
        inner.push_back(rows_axis ? blk.cols : blk.rows);
        pitch.push_back(blk.cols);
      }
      if (ptrs.empty()) continue;
      cuda_check(segment_partial(upload(w, keep[w.id], ptrs), upload(w, keep[w.id], inner),
                                 upload(w, keep[w.id], pitch), static_cast<int>(ptrs.size()),
                                 rows_axis ? 0 : 1, static_cast<int>(d.precision), seg_len(s),
                                 static_cast<char*>(w.arena.data()) + off[w.id][s], w.stream),
                 "row/col partial");
    }
  }
  mid_barrier();
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DevGuard gd(w.device);
    for (int s = 0; s < segments; ++s) {
      if (owners[s] != w.id) continue;
      std::vector<WorkerId> order = contributors(s);
      if (!deterministic) {  // permuted fold order (ops.hpp:1079-1086)
        std::uint64_t st = mix64(salt, static_cast<std::uint64_t>(s));
        for (std::size_t i = order.size(); i > 1; --i) {
          st = mix64(st);
          std::swap(order[i - 1], order[st % i]);
        }
      }
      std::vector<const void*> parts;
      for (WorkerId c : order) {
        parts.push_back(static_cast<const char*>(arena_ptrs_[c]) + off[c][s]);
        if (c != w.id) w.stats.peer_bytes_read += static_cast<std::uint64_t>(seg_len(s)) * esz;
      }
      StoredBlock& out = w.owned.at({od.matrix_id, rows_axis ? BlockCoord{s, 0} : BlockCoord{0, s}});
      cuda_check(fold_partials(upload(w, keep[w.id], parts), static_cast<int>(parts.size()),
                               static_cast<int>(d.precision), seg_len(s), out.mem.data(), w.stream),
                 "row/col fold");
    }
  }
  sync_local();
  keep.clear();
  end_command();
  return od.matrix_id;
}

// ------------------------------------------------------------ checkpoint

namespace {
std::vector<int> checkpoint_block_order(const LayoutSpec& layout) {
  const int nbr = layout.grid.n_block_rows(), nbc = layout.grid.n_block_cols();
  std::vector<int> order;
  for (WorkerId w = 0; w < layout.worker_count; ++w)
    for (int r = 0; r < nbr; ++r)
      for (int c = 0; c < nbc; ++c)
        if (layout.owner({r, c}) == w) order.push_back(r * nbc + c);
  return order;
}
}  // namespace

// Session::checkpoint (session.hpp:395-423) writing the "DMTH" v1 image of
// checkpoint.hpp:1-12, 61-88: owner-major, block-row-major payloads and a
// trailing FNV-1a.  Blocks stream device -> host straight into the image; in
// SPMD rank 0 reads every peer block through its IPC mapping and writes.
void Session::checkpoint(const std::string& path) {
  require_live();
  SyncScope scope(this);
  const bool writer = !comm_ || rank_ == 0;
  if (writer) {
    std::vector<unsigned char> out;
    out.insert(out.end(), {'D', 'M', 'T', 'H'});
    put_le(out, 1, 4);
    put_le(out, static_cast<std::uint64_t>(P_), 4);
    put_le(out, root_seed_, 8);
    put_le(out, next_matrix_id_, 8);
    put_le(out, table_.size(), 4);
    Worker& me = comm_ ? *workers_[rank_] : *workers_[0];
    for (const auto& [id, d] : table_) {
      put_le(out, d.matrix_id, 8);
      put_le(out, d.version, 8);
      put_le(out, d.seed, 8);
      out.push_back(d.replicated ? 1 : 0);
      out.push_back(static_cast<unsigned char>(d.precision));
      const std::string ls = layout_to_string(d.layout);
      put_le(out, ls.size(), 2);
      out.insert(out.end(), ls.begin(), ls.end());
      const auto order = checkpoint_block_order(d.layout);
      put_le(out, order.size(), 4);
      const int nbc = d.layout.grid.n_block_cols();
      for (int key : order) {
        const BlockCoord c{key / nbc, key % nbc};
        auto [br, bc] = block_extent(d.layout.grid, c);
        const std::size_t bytes = static_cast<std::size_t>(br * bc) * byte_width(d.precision);
        put_le(out, bytes, 4);
        const std::size_t at = out.size();
        out.resize(at + bytes);
        Worker* ow = local(d.layout.owner(c));
        Worker& issuer = ow ? *ow : me;
        DevGuard g(issuer.device);
        cuda_check(cudaMemcpy(out.data() + at, block_src(id, c, me), bytes, cudaMemcpyDefault),
                   "checkpoint D2H");
      }
    }
    Fnv1a h;
    h.update(out.data(), out.size());
    put_le(out, h.digest(), 8);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw ConfigError("checkpoint: cannot open " + path + " for writing");
    f.write(reinterpret_cast<const char*>(out.data()), static_cast<std::streamsize>(out.size()));
    if (!f) throw ConfigError("checkpoint: write failed for " + path);
  }
  end_command();
}

// Session::restore (session.hpp:425-465) into this (fresh) session: every rank
// reads the image, recreates each descriptor (id, version, seed, layout,
// precision) and loads the blocks it owns bit-exactly; replication re-enabled.
void Session::restore_image(const std::string& path) {
  require_live();
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ConfigError("checkpoint: cannot open " + path);
  const std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(f)),
                                         std::istreambuf_iterator<char>());
  if (bytes.size() < 16 || std::memcmp(bytes.data(), "DMTH", 4) != 0)
    throw IntegrityError("checkpoint: bad magic or truncated file");
  Fnv1a h;
  h.update(bytes.data(), bytes.size() - 8);
  if (h.digest() != get_le(bytes.data() + bytes.size() - 8, 8))
    throw IntegrityError("checkpoint: checksum mismatch");
  std::size_t pos = 4;
  const std::size_t limit = bytes.size() - 8;
  auto read_u = [&](int n) {
    if (pos + static_cast<std::size_t>(n) > limit) throw IntegrityError("checkpoint: truncated record");
    const std::uint64_t v = get_le(bytes.data() + pos, n);
    pos += static_cast<std::size_t>(n);
    return v;
  };
  if (read_u(4) != 1) throw IntegrityError("checkpoint: unsupported format version");
  const int workers = static_cast<int>(read_u(4));
  const std::uint64_t root = read_u(8);
  const std::uint64_t next_id = read_u(8);
  if (workers != P_) throw ConfigError("restore: image worker count does not match the session");
  if (!table_.empty()) throw UsageError("restore: session already holds matrices");
  root_seed_ = root;
  const std::uint64_t nmat = read_u(4);
  std::vector<MatrixId> replicated;
  for (std::uint64_t i = 0; i < nmat; ++i) {
    MatrixDescriptor d;
    d.matrix_id = read_u(8);
    d.version = read_u(8);
    d.seed = read_u(8);
    const bool was_replicated = read_u(1) != 0;
    d.precision = static_cast<Precision>(read_u(1));
    const std::size_t lslen = read_u(2);
    if (pos + lslen > limit) throw IntegrityError("checkpoint: truncated record");
    d.layout = layout_from_string(std::string(reinterpret_cast<const char*>(bytes.data() + pos), lslen));
    pos += lslen;
    validate_layout_workers(d.layout);
    materialize(d, false);
    const auto order = checkpoint_block_order(d.layout);
    if (read_u(4) != order.size()) throw IntegrityError("checkpoint: block count mismatch");
    const int nbc = d.layout.grid.n_block_cols();
    for (int key : order) {
      const std::size_t plen = read_u(4);
      if (pos + plen > limit) throw IntegrityError("checkpoint: truncated record");
      const BlockCoord c{key / nbc, key % nbc};
      if (Worker* w = local(d.layout.owner(c))) {
        StoredBlock& blk = w->owned.at({d.matrix_id, c});
        if (plen != blk.bytes()) throw IntegrityError("checkpoint: block payload size mismatch");
        DevGuard g(w->device);
        cuda_check(cudaMemcpy(blk.mem.data(), bytes.data() + pos, plen, cudaMemcpyHostToDevice),
                   "restore H2D");
      }
      pos += plen;
    }
    if (was_replicated) replicated.push_back(d.matrix_id);
    end_command();
  }
  if (pos != limit) throw IntegrityError("checkpoint: trailing bytes");
  next_matrix_id_ = next_id;
  for (MatrixId id : replicated) replicate(id, true);
}

}  // namespace dm
