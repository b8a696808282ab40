// TEST INFRASTRUCTURE ONLY -- the checker, never the product.
//
// C-ABI shim over the UNMODIFIED reference implementation (gridgemm, header
// only), compiled from the sources where they lie under
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/.  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs load it.
//
// Build flags mirror the reference's Release build (proj/CMakeLists.txt:3-8:
// -O3 -DNDEBUG, no -march) plus -ffp-contract=off, which keeps the
// reference's unfused fp32 multiply-add in kernels.hpp:61-72 bit-exact.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "gridgemm/kernels.hpp"
#include "gridgemm/session.hpp"

using namespace gridgemm;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 3;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 4;
  } catch (const DeadlockError& e) {
    g_err = e.what();
    return 5;
  } catch (const IntegrityError& e) {
    g_err = e.what();
    return 6;
  } catch (const PlanError& e) {
    g_err = e.what();
    return 7;
  } catch (const CacheMissError& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

LayoutSpec mk_layout(int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc, int workers) {
  return make_layout(static_cast<LayoutKind>(kind), gr, gc, br, bc, workers);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix64_2(uint64_t a, uint64_t b) { return mix64(a, b); }

int ref_session_create(int workers, uint64_t root_seed, int deterministic, void** out) {
  return guarded([&] {
    Session::Config cfg;
    cfg.worker_count = workers;
    cfg.root_seed = root_seed;
    cfg.deterministic = deterministic != 0;
    *out = new Session(cfg);
  });
}

int ref_session_destroy(void* s) {
  return guarded([&] { delete static_cast<Session*>(s); });
}

int ref_create_matrix(void* s, int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc,
                      int workers, int fill, const float* host, uint64_t* out) {
  return guarded([&] {
    const LayoutSpec l = mk_layout(kind, gr, gc, br, bc, workers);
    if (fill == 2) {
      HostMatrix hm(gr, gc, Precision::Single32);
      std::memcpy(hm.raw(), host, hm.byte_size());
      *out = static_cast<Session*>(s)->create_matrix(l, Precision::Single32, FillKind::FromHost, &hm);
    } else {
      *out = static_cast<Session*>(s)->create_matrix(l, Precision::Single32,
                                                     static_cast<FillKind>(fill));
    }
  });
}

int ref_gather(void* s, uint64_t id, float* out, int64_t n_elems) {
  return guarded([&] {
    HostMatrix hm = static_cast<Session*>(s)->gather(id);
    if (static_cast<int64_t>(hm.byte_size()) != n_elems * 4) throw UsageError("ref_gather: size");
    std::memcpy(out, hm.raw(), hm.byte_size());
  });
}

int ref_scatter(void* s, uint64_t id, const float* host, int64_t rows, int64_t cols) {
  return guarded([&] {
    HostMatrix hm(rows, cols, Precision::Single32);
    std::memcpy(hm.raw(), host, hm.byte_size());
    static_cast<Session*>(s)->scatter(id, hm);
  });
}

int ref_general_gemm(void* s, double alpha, uint64_t a, uint64_t b, double beta, uint64_t c, int ta,
                     int tb) {
  return guarded([&] { static_cast<Session*>(s)->general_gemm(alpha, a, b, beta, c, ta, tb); });
}

int ref_cyclic_gemm(void* s, double alpha, uint64_t a, uint64_t b, double beta, uint64_t c, int ta,
                    int tb, int cache_a) {
  return guarded(
      [&] { static_cast<Session*>(s)->cyclic_gemm(alpha, a, b, beta, c, ta, tb, cache_a); });
}

int ref_broadcast_gemm(void* s, double alpha, uint64_t a, uint64_t b, double beta, uint64_t c, int ta,
                       int tb) {
  return guarded(
      [&] { static_cast<Session*>(s)->broadcast_gemm_reference(alpha, a, b, beta, c, ta, tb); });
}

// trace() records (TraceLog::snapshot, transport.hpp:56-71) from index `from`:
// per record src, dst, payload bytes and the op tag (NUL-padded, 48 bytes).
int ref_trace_records(void* s, uint64_t from, int64_t* out3, char* tags, int cap, int* count) {
  return guarded([&] {
    const auto recs = static_cast<Session*>(s)->trace().snapshot();
    int n = 0;
    for (std::size_t i = from; i < recs.size(); ++i, ++n) {
      if (n >= cap) continue;
      out3[3 * n] = recs[i].src;
      out3[3 * n + 1] = recs[i].dst;
      out3[3 * n + 2] = static_cast<int64_t>(recs[i].payload_bytes);
      std::memset(tags + 48 * n, 0, 48);
      std::strncpy(tags + 48 * n, recs[i].op_tag.c_str(), 47);
    }
    *count = n;
  });
}

int ref_cached_backward_gemm(void* s, uint64_t w, uint64_t dy, uint64_t dx) {
  return guarded([&] { static_cast<Session*>(s)->cached_backward_gemm(w, dy, dx); });
}

int ref_descriptor(void* s, uint64_t id, uint64_t* version, uint64_t* seed) {
  return guarded([&] {
    const MatrixDescriptor& d = static_cast<Session*>(s)->descriptor(id);
    *version = d.version;
    *seed = d.seed;
  });
}

int ref_pool_stats(void* s, int w, uint64_t* out5) {
  return guarded([&] {
    const Pool::Stats st = static_cast<Session*>(s)->worker_pool_stats(w);
    out5[0] = st.fresh_allocations;
    out5[1] = st.reuses;
    out5[2] = st.bytes_live;
    out5[3] = st.bytes_pooled;
    out5[4] = st.high_water;
  });
}

int ref_trace_count(void* s, uint64_t* transfers, uint64_t* bytes) {
  return guarded([&] {
    const auto recs = static_cast<Session*>(s)->trace().snapshot();
    *transfers = recs.size();
    uint64_t b = 0;
    for (const auto& r : recs) b += r.payload_bytes;
    *bytes = b;
  });
}

int ref_layout_owner(int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc, int workers, int row,
                     int col, int* owner) {
  return guarded([&] { *owner = mk_layout(kind, gr, gc, br, bc, workers).owner({row, col}); });
}

int ref_layout_string(int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc, int workers,
                      char* buf, int cap) {
  return guarded([&] {
    const std::string s = layout_to_string(mk_layout(kind, gr, gc, br, bc, workers));
    std::strncpy(buf, s.c_str(), static_cast<size_t>(cap));
    buf[cap - 1] = 0;
  });
}

// local_gemm (kernels.hpp:81-89) on host row-major fp32 arrays.
int ref_local_gemm_f32(double alpha, const float* a, int64_t ar, int64_t ac, int ta, const float* b,
                       int64_t br, int64_t bc, int tb, double beta, float* c, int64_t cr,
                       int64_t cc) {
  return guarded([&] {
    DynConstView va{reinterpret_cast<const std::byte*>(a), ar, ac, Precision::Single32};
    DynConstView vb{reinterpret_cast<const std::byte*>(b), br, bc, Precision::Single32};
    DynView vc{reinterpret_cast<std::byte*>(c), cr, cc, Precision::Single32};
    local_gemm(alpha, va, ta != 0, vb, tb != 0, beta, vc);
  });
}

// Sampled rows of C = alpha op(A) op(B) + beta C0 through the reference's
// local_gemm on 1 x K row slices: each output row is bit-identical to the
// reference's distributed result (k ascending over the full K in every
// executor, ops.hpp:274, 485).  `a_rows` holds op(A)[i, :] for each sampled
// row i (nrows x K, already extracted), `bfull` the full op(B) storage.
int ref_sampled_rows(double alpha, const float* a_rows, int64_t nrows, int64_t k, const float* b,
                     int64_t br, int64_t bc, int tb, double beta, const float* c0_rows,
                     float* out_rows, int64_t n, int threads) {
  return guarded([&] {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(threads));
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (int64_t i = next++; i < nrows; i = next++) {
            DynConstView va{reinterpret_cast<const std::byte*>(a_rows + i * k), 1, k,
                            Precision::Single32};
            DynConstView vb{reinterpret_cast<const std::byte*>(b), br, bc, Precision::Single32};
            float* row = out_rows + i * n;
            if (beta != 0.0) std::memcpy(row, c0_rows + i * n, static_cast<size_t>(n) * 4);
            DynView vc{reinterpret_cast<std::byte*>(row), 1, n, Precision::Single32};
            local_gemm(alpha, va, false, vb, tb != 0, beta, vc);
          }
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw UsageError(e);
  });
}

// Sampled columns of C = alpha op(A) op(B) + beta C0: column j of C depends
// only on op(A) and column j of op(B) (k ascending in every executor,
// ops.hpp:274, 485), so local_gemm on a K x 1 column view reproduces the
// reference's distributed result for that column bit for bit.  `a` is the
// full A storage (ar x ac, op via ta), `b_cols` holds op(B)[:, j] for each
// sampled column (ncols x K), c0_cols / out_cols are ncols x m.
int ref_sampled_cols(double alpha, const float* a, int64_t ar, int64_t ac, int ta, const float* b_cols,
                     int64_t ncols, int64_t k, double beta, const float* c0_cols, float* out_cols, int64_t m,
                     int threads) {
  return guarded([&] {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(threads));
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (int64_t j = next++; j < ncols; j = next++) {
            DynConstView va{reinterpret_cast<const std::byte*>(a), ar, ac, Precision::Single32};
            DynConstView vb{reinterpret_cast<const std::byte*>(b_cols + j * k), k, 1, Precision::Single32};
            float* col = out_cols + j * m;
            if (beta != 0.0) std::memcpy(col, c0_cols + j * m, static_cast<size_t>(m) * 4);
            DynView vc{reinterpret_cast<std::byte*>(col), m, 1, Precision::Single32};
            local_gemm(alpha, va, ta != 0, vb, false, beta, vc);
          }
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw UsageError(e);
  });
}

// ---- precision-generic entry points (SURVEY 8(f) operations) ----
int ref_create_matrix_p(void* s, int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc,
                        int workers, int precision, int fill, const void* host, uint64_t* out) {
  return guarded([&] {
    const LayoutSpec l = mk_layout(kind, gr, gc, br, bc, workers);
    const Precision p = static_cast<Precision>(precision);
    if (fill == 2) {
      HostMatrix hm(gr, gc, p);
      std::memcpy(hm.raw(), host, hm.byte_size());
      *out = static_cast<Session*>(s)->create_matrix(l, p, FillKind::FromHost, &hm);
    } else {
      *out = static_cast<Session*>(s)->create_matrix(l, p, static_cast<FillKind>(fill));
    }
  });
}

int ref_gather_bytes(void* s, uint64_t id, void* out, int64_t nbytes) {
  return guarded([&] {
    HostMatrix hm = static_cast<Session*>(s)->gather(id);
    if (static_cast<int64_t>(hm.byte_size()) != nbytes) throw UsageError("ref_gather_bytes: size");
    std::memcpy(out, hm.raw(), hm.byte_size());
  });
}

int ref_update_block(void* s, uint64_t id, int row, int col, int precision, const void* host,
                     int64_t rows, int64_t cols) {
  return guarded([&] {
    HostMatrix hm(rows, cols, static_cast<Precision>(precision));
    std::memcpy(hm.raw(), host, hm.byte_size());
    static_cast<Session*>(s)->update_block(id, {row, col}, hm);
  });
}

int ref_reshape(void* s, uint64_t src, int kind, int64_t gr, int64_t gc, int64_t br, int64_t bc,
                int workers, int precision, uint64_t* out) {
  return guarded([&] {
    *out = static_cast<Session*>(s)->reshape(src, mk_layout(kind, gr, gc, br, bc, workers),
                                             static_cast<Precision>(precision));
  });
}

int ref_add_row_col_sum(void* s, uint64_t id, int axis, int deterministic, uint64_t* out) {
  return guarded([&] {
    *out = static_cast<Session*>(s)->add_row_col_sum(id, axis == 0 ? Axis::Rows : Axis::Cols,
                                                     deterministic != 0);
  });
}

int ref_replicate(void* s, uint64_t id, int enable) {
  return guarded([&] { static_cast<Session*>(s)->replicate(id, enable != 0); });
}

int ref_replica_read(void* s, uint64_t id, int reader, void* out, int64_t nbytes) {
  return guarded([&] {
    HostMatrix hm = static_cast<Session*>(s)->replica_read(id, reader);
    if (static_cast<int64_t>(hm.byte_size()) != nbytes) throw UsageError("ref_replica_read: size");
    std::memcpy(out, hm.raw(), hm.byte_size());
  });
}

int ref_checkpoint(void* s, const char* path) {
  return guarded([&] { static_cast<Session*>(s)->checkpoint(path); });
}

int ref_restore(const char* path, void** out) {
  return guarded([&] { *out = Session::restore(path).release(); });
}

int ref_descriptor_full(void* s, uint64_t id, uint64_t* out6, char* layout, int cap) {
  return guarded([&] {
    const MatrixDescriptor& d = static_cast<Session*>(s)->descriptor(id);
    out6[0] = d.version;
    out6[1] = d.replica_version;
    out6[2] = d.replicated ? 1 : 0;
    out6[3] = static_cast<uint64_t>(d.precision);
    out6[4] = d.seed;
    out6[5] = static_cast<uint64_t>(d.layout.grid.global_rows) << 32 |
              static_cast<uint64_t>(d.layout.grid.global_cols);
    const std::string ls = layout_to_string(d.layout);
    std::strncpy(layout, ls.c_str(), static_cast<size_t>(cap));
    layout[cap - 1] = 0;
  });
}

// WorkerContext::fill_seeded (runtime_types.hpp:208-218) for one block.
int ref_fill_block(float* out, int64_t rows, int64_t cols, uint64_t matrix_seed, int brow, int bcol) {
  return guarded([&] {
    Pool p;  // declared first: the block's buffer must return to a live pool
    StoredBlock b;
    b.rows = rows;
    b.cols = cols;
    b.precision = Precision::Single32;
    b.mem = p.acquire(static_cast<size_t>(rows * cols) * 4);
    WorkerContext::fill_seeded(b, matrix_seed, {brow, bcol});
    std::memcpy(out, b.mem.data(), static_cast<size_t>(rows * cols) * 4);
  });
}

uint64_t ref_fnv1a(const void* data, int64_t n) {
  Fnv1a h;
  h.update(data, static_cast<size_t>(n));
  return h.digest();
}

}  // extern "C"
