// extern "C" boundary (include/dmath_b200.h).  Every entry point converts
// exceptions into dm_status codes 1:1 with the reference's exception classes
// (gridgemm/common.hpp:22-78) and records the message for dm_last_error().
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <string>

#include "../../include/dmath_b200.h"
#include "kernels/tf32x3_gemm.h"
#include "runtime/layout.hpp"
#include "runtime/pool.hpp"
#include "runtime/session.hpp"

struct dm_session {
  std::unique_ptr<dm::Session> impl;
  std::map<dm::MatrixId, std::vector<int32_t>> custom_tables;  // backing for dm_descriptor
};

namespace {

thread_local std::string g_last_error;
thread_local std::vector<std::pair<int, int>> g_last_missing;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    g_last_missing.clear();
    return DM_OK;
  } catch (const dm::CacheMissError& e) {
    g_last_error = e.what();
    g_last_missing = e.missing_coords;
    return e.code();
  } catch (const dm::Error& e) {
    g_last_error = e.what();
    g_last_missing.clear();
    return e.code();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return DM_ERR_USAGE;
  }
}

dm::Session& S(dm_session* s) {
  if (s == nullptr || !s->impl) throw dm::UsageError("null session");
  return *s->impl;
}

// Split-product mode: explicit (dm_gemm_mode) or, for DM_GEMM_DEFAULT, the
// DM_GEMM_MODE environment variable (0 = 3xTF32), else mixed.
int resolve_gemm_mode(int requested, int64_t m, int64_t n, int64_t k) {
  int mode;
  if (requested == DM_GEMM_TF32X3) mode = dm::kModeTf32x3;
  else if (requested == DM_GEMM_MIXED) mode = dm::kModeMixed;
  else if (requested == DM_GEMM_AUTO) mode = dm::kModeAuto;
  else if (requested == DM_GEMM_F16X2) mode = dm::kModeF16x2;
  else if (requested == DM_GEMM_DEFAULT) mode = dm::env_gemm_mode();
  else throw dm::UsageError("unknown gemm_mode");
  return dm::resolve_split_mode(mode, k, 2.0 * static_cast<double>(m) * static_cast<double>(n) * static_cast<double>(k));
}

// Scratch layout of one local_gemm call: the split planes of op(A) and op(B)
// -- hi fp32 + (lo fp32 | bf16 hi, bf16 lo) = 8 B per element either way --
// then the split-K partials; each region 256-B aligned.  An operand whose
// storage is M/N-contiguous (transposed A, non-transposed B) gets MN-major
// planes -- split row by row, no transpose -- when the other extent (its
// reuse) is below DM_MN_REUSE (session_gemm.cpp range_mn).
struct SeamLayout {
  bool f16x2 = false;  // kModeF16x2: fp16 h0 | h1 planes (4 B / element) + row maxima, K-major
  bool a_mn = false, b_mn = false;
  int64_t lda = 8, ldb = 8;  // plane pitches (elements): K-major kp, MN-major m / n rounded to 32
  int64_t a_elems = 0, b_elems = 0;
  size_t off[5] = {0, 0, 0, 0, 0};  // a_hi, a_second, b_hi, b_second, splitk ws
  size_t off_max = 0;                // kModeF16x2: A row maxima [m], then B^T row maxima [n]
  size_t ws_bytes = 0;
  size_t total = 0;
};

SeamLayout seam_layout(const dm::Tf32x3Args& shape, int ta, int tb) {
  SeamLayout l;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const int64_t thr = dm::env_int("DM_MN_REUSE", 2048);
  l.f16x2 = shape.mode == dm::kModeF16x2;
  l.a_mn = !l.f16x2 && ta != 0 && shape.n < thr;
  l.b_mn = !l.f16x2 && tb == 0 && shape.m < thr;
  const int64_t kp = std::max<int64_t>(8, (shape.k + 7) / 8 * 8);
  l.lda = l.a_mn ? (shape.m + 31) / 32 * 32 : kp;
  l.ldb = l.b_mn ? (shape.n + 31) / 32 * 32 : kp;
  if (shape.m <= 0 || shape.n <= 0 || shape.k <= 0) return l;
  l.a_elems = l.a_mn ? shape.k * l.lda : shape.m * kp;
  l.b_elems = l.b_mn ? shape.k * l.ldb : shape.n * kp;
  const size_t a = up(static_cast<size_t>(l.a_elems) * 4), b = up(static_cast<size_t>(l.b_elems) * 4);
  l.off[1] = a;
  l.off[2] = 2 * a;
  l.off[3] = 2 * a + b;
  l.off[4] = 2 * a + 2 * b;
  l.ws_bytes = dm::tf32x3_splitk_bytes(shape);
  l.off_max = l.off[4] + up(l.ws_bytes);
  l.total = l.off_max + (l.f16x2 ? up(static_cast<size_t>(shape.m + shape.n) * 4) : 0);
  return l;
}

// Scratch of the pool-backed seam: one pool per device; buffers of a call go
// back to the pool only once an event recorded after its kernels fired, so
// the call is stream-ordered (no host wait) and calls on several streams can
// run concurrently.
struct SeamScratch {
  std::mutex mu;
  std::unique_ptr<dm::DevicePool> pool;
  struct Pending {
    cudaEvent_t done;
    dm::DeviceBuffer buf;
  };
  std::deque<Pending> pending;
  void reap() {
    while (!pending.empty() && cudaEventQuery(pending.front().done) == cudaSuccess) {
      cudaEventDestroy(pending.front().done);
      pending.pop_front();
    }
    cudaGetLastError();  // cudaErrorNotReady is not an error here
  }
};

SeamScratch& seam_scratch(int dev) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<SeamScratch>> all;
  std::lock_guard<std::mutex> lk(mu);
  auto& p = all[dev];
  if (!p) {
    p = std::make_unique<SeamScratch>();
    p->pool = std::make_unique<dm::DevicePool>(dev);
  }
  return *p;
}

dm::Tf32x3Args seam_shape(int64_t m, int64_t n, int64_t k, int cta_group, int mode) {
  dm::Tf32x3Args a;
  a.m = m;
  a.n = n;
  a.k = k;
  a.cta_group = cta_group;
  a.mode = mode;
  return a;
}

// local_gemm (kernels.hpp:81-89) on device memory: split op(A) / op(B) into
// planes in `ws`, then the tcgen05 GEMM; everything on `st`.
void local_gemm_run(double alpha, const float* a, int64_t lda, int ta, const float* b, int64_t ldb, int tb,
                    double beta, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int cta_group, int mode,
                    char* ws, const SeamLayout& L, cudaStream_t st) {
  dm::Tf32x3Args args = seam_shape(m, n, k, cta_group, mode);
  if (k > 0 && m > 0 && n > 0) {
    args.a_mn = L.a_mn ? 1 : 0;
    args.b_mn = L.b_mn ? 1 : 0;
    args.a_hi = reinterpret_cast<const float*>(ws + L.off[0]);
    args.b_hi = reinterpret_cast<const float*>(ws + L.off[2]);
    args.lda = args.lda16 = L.lda;
    args.ldb = args.ldb16 = L.ldb;
    if (L.f16x2) {
      // fp16 h0 | h1 in the first half of each operand region (4 B / element)
      args.a_hi = args.b_hi = nullptr;
      args.a_hi16 = ws + L.off[0];
      args.a_lo16 = ws + L.off[0] + L.a_elems * 2;
      args.b_hi16 = ws + L.off[2];
      args.b_lo16 = ws + L.off[2] + L.b_elems * 2;
      unsigned* amax = reinterpret_cast<unsigned*>(ws + L.off_max);
      unsigned* bmax = amax + m;
      args.a_max = amax;
      args.b_max = bmax;
      dm::cuda_check(cudaMemsetAsync(amax, 0, static_cast<size_t>(m + n) * 4, st), "memset maxima");
      dm::cuda_check(dm::absmax_rows(a, lda, ta, m, k, amax, st), "absmax A");
      dm::cuda_check(dm::absmax_rows(b, ldb, tb ? 0 : 1, n, k, bmax, st), "absmax B");
      dm::cuda_check(dm::split_f16x2(a, lda, ta, m, k, const_cast<void*>(args.a_hi16),
                                     const_cast<void*>(args.a_lo16), L.lda, amax, st), "split A");
      dm::cuda_check(dm::split_f16x2(b, ldb, tb ? 0 : 1, n, k, const_cast<void*>(args.b_hi16),
                                     const_cast<void*>(args.b_lo16), L.ldb, bmax, st), "split B");
    } else if (mode == dm::kModeMixed) {
      args.a_hi16 = ws + L.off[1];
      args.a_lo16 = ws + L.off[1] + L.a_elems * 2;
      args.b_hi16 = ws + L.off[3];
      args.b_lo16 = ws + L.off[3] + L.b_elems * 2;
    } else {
      args.a_lo = reinterpret_cast<const float*>(ws + L.off[1]);
      args.b_lo = reinterpret_cast<const float*>(ws + L.off[3]);
    }
    // split_tf32 writes x[r][q] at plane + r * pitch + q with x[r][q] = trans ?
    // src[q * lds + r] : src[r * lds + q]; a K-major plane is op(X) [mn x k], an
    // MN-major plane its transpose [k x mn] (rows and columns swapped, trans flipped)
    auto split = [&](const float* src, int64_t lds, int trans, int64_t mn_len, bool mn, const float* hi,
                     const float* lo, const void* hi16, const void* lo16, int64_t pitch, const char* what) {
      dm::cuda_check(dm::split_tf32(src, 0, lds, mn ? !trans : trans, mn ? k : mn_len, mn ? mn_len : k,
                                    const_cast<float*>(hi), const_cast<float*>(lo), pitch, const_cast<void*>(hi16),
                                    const_cast<void*>(lo16), pitch, st),
                     what);
    };
    if (!L.f16x2) {
      split(a, lda, ta, m, L.a_mn, args.a_hi, args.a_lo, args.a_hi16, args.a_lo16, L.lda, "split A");
      split(b, ldb, tb ? 0 : 1, n, L.b_mn, args.b_hi, args.b_lo, args.b_hi16, args.b_lo16, L.ldb, "split B");
    }
    if (L.ws_bytes > 0) {
      args.ws = reinterpret_cast<float*>(ws + L.off[4]);
      args.ws_bytes = L.ws_bytes;
    }
  }
  args.c = c;
  args.ldc = ldc;
  args.alpha = static_cast<float>(alpha);
  args.beta = static_cast<float>(beta);
  args.read_c = beta != 0.0 ? 1 : 0;
  args.flush_k = dm::env_int("DM_FLUSH_K", 0);
  dm::cuda_check(dm::tf32x3_gemm(args, st), "tf32x3_gemm");
}

void local_gemm_validate(const float* a, int64_t lda, int ta, const float* b, int64_t ldb, int tb, float* c,
                         int64_t ldc, int64_t m, int64_t n, int64_t k, int cta_group) {
  if (m < 0 || n < 0 || k < 0) throw dm::ShapeError("local_gemm: negative dimension");
  if ((m > 0 && n > 0) && c == nullptr) throw dm::UsageError("local_gemm: null C");
  if (k > 0 && (a == nullptr || b == nullptr)) throw dm::UsageError("local_gemm: null operand");
  if (ldc < n) throw dm::ShapeError("local_gemm: ldc < n");
  if (lda < (ta ? m : k) || ldb < (tb ? k : n)) throw dm::ShapeError("local_gemm: bad pitch");
  if (cta_group < 0 || cta_group > 2) throw dm::UsageError("local_gemm: cta_group must be 0, 1 or 2");
}

int local_gemm_impl(double alpha, const float* a, int64_t lda, int ta, const float* b, int64_t ldb,
                    int tb, double beta, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
                    int cta_group, int gemm_mode, void* stream) {
  return guarded([&] {
    local_gemm_validate(a, lda, ta, b, ldb, tb, c, ldc, m, n, k, cta_group);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    dm::cuda_check(cudaStreamIsCapturing(st, &cap), "cudaStreamIsCapturing");
    if (cap != cudaStreamCaptureStatusNone)
      throw dm::UsageError(
          "local_gemm: a captured call must own its scratch for the graph's lifetime: use "
          "dm_local_gemm_f32_ws with a caller workspace");
    int dev = 0;
    dm::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const int mode = resolve_gemm_mode(gemm_mode, m, n, k);
    const SeamLayout L = seam_layout(seam_shape(m, n, k, cta_group, mode), ta, tb);
    SeamScratch& sc = seam_scratch(dev);
    dm::DeviceBuffer buf;
    {
      std::lock_guard<std::mutex> lk(sc.mu);
      sc.reap();
      if (L.total > 0) buf = sc.pool->acquire(L.total);
    }
    // the scratch returns to the pool once the kernels that use it ran (also
    // when a later launch of this call failed: earlier ones may still read it)
    auto release = [&] {
      if (L.total == 0) return;
      cudaEvent_t done = nullptr;
      if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord(done, st) != cudaSuccess) {
        cudaStreamSynchronize(st);  // cannot defer: drain, then release
        if (done) cudaEventDestroy(done);
        std::lock_guard<std::mutex> lk(sc.mu);
        buf = dm::DeviceBuffer();
        return;
      }
      std::lock_guard<std::mutex> lk(sc.mu);
      sc.pending.push_back({done, std::move(buf)});
    };
    try {
      local_gemm_run(alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, m, n, k, cta_group, mode,
                     static_cast<char*>(buf.data()), L, st);
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

}  // namespace

extern "C" {

const char* dm_last_error(void) { return g_last_error.c_str(); }

int dm_last_error_missing(int32_t* coords, int cap) {
  const int n = static_cast<int>(g_last_missing.size());
  for (int i = 0; i < n && i < cap; ++i) {
    coords[2 * i] = g_last_missing[i].first;
    coords[2 * i + 1] = g_last_missing[i].second;
  }
  return n;
}

int dm_abi_version(void) { return DMATH_B200_ABI_VERSION; }

int dm_checkerboard_dims(int workers, int* pr, int* pc) {
  return guarded([&] {
    if (workers < 1) throw dm::UsageError("checkerboard_dims: workers must be >= 1");
    auto [r, c] = dm::checkerboard_dims(workers);
    *pr = r;
    *pc = c;
  });
}

int dm_layout_owner(const dm_layout* layout, int row, int col, int* owner) {
  return guarded([&] { *owner = dm::layout_from_abi(layout).owner({row, col}); });
}

int dm_layout_grid(const dm_layout* layout, int* nbr, int* nbc, int* clamped) {
  return guarded([&] {
    const dm::LayoutSpec l = dm::layout_from_abi(layout);
    *nbr = l.grid.n_block_rows();
    *nbc = l.grid.n_block_cols();
    *clamped = l.grid.clamped ? 1 : 0;
  });
}

int dm_block_extent(const dm_layout* layout, int row, int col, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    auto [r, c] = dm::block_extent(dm::layout_from_abi(layout).grid, {row, col});
    *rows = r;
    *cols = c;
  });
}

int dm_layout_to_string(const dm_layout* layout, char* buf, int cap) {
  std::string s;
  const int rc = guarded([&] { s = dm::layout_to_string(dm::layout_from_abi(layout)); });
  if (rc != DM_OK) return -rc;
  if (buf != nullptr && cap > 0) {
    std::strncpy(buf, s.c_str(), static_cast<size_t>(cap));
    buf[cap - 1] = 0;
  }
  return static_cast<int>(s.size()) + 1;
}

uint64_t dm_pool_size_class(uint64_t bytes) { return dm::DevicePool::size_class(bytes); }

int dm_plan_general_gemm(const dm_layout* a, int ta, const dm_layout* b, int tb,
                         const dm_layout* c, int worker, int64_t* peer_blocks, int64_t* peer_bytes) {
  return guarded([&] {
    const dm::LayoutSpec la = dm::layout_from_abi(a), lb = dm::layout_from_abi(b),
                         lc = dm::layout_from_abi(c);
    std::set<std::pair<int, std::pair<int, int>>> need;  // (matrix 0/1, block)
    auto add = [&](const dm::LayoutSpec& l, bool trans, bool along_rows, int64_t lo, int64_t len,
                   int tag) {
      for (int br = 0; br < l.grid.n_block_rows(); ++br)
        for (int bc = 0; bc < l.grid.n_block_cols(); ++bc) {
          const int64_t ar0 = br * l.grid.block_rows, ac0 = bc * l.grid.block_cols;
          auto [ar, ac] = dm::block_extent(l.grid, {br, bc});
          int64_t o0, olen;
          if (along_rows) {
            o0 = trans ? ac0 : ar0;
            olen = trans ? ac : ar;
          } else {
            o0 = trans ? ar0 : ac0;
            olen = trans ? ar : ac;
          }
          if (o0 + olen <= lo || o0 >= lo + len) continue;
          if (l.owner({br, bc}) != worker) need.insert({tag, {br, bc}});
        }
    };
    for (dm::BlockCoord cc : dm::owned_coords(lc, worker)) {
      auto [mb, nb] = dm::block_extent(lc.grid, cc);
      add(la, ta != 0, true, cc.row * lc.grid.block_rows, mb, 0);
      add(lb, tb != 0, false, cc.col * lc.grid.block_cols, nb, 1);
    }
    int64_t bytes = 0;
    for (const auto& [tag, rc] : need) {
      auto [r, cc] = dm::block_extent((tag == 0 ? la : lb).grid, {rc.first, rc.second});
      bytes += r * cc * 4;
    }
    *peer_blocks = static_cast<int64_t>(need.size());
    *peer_bytes = bytes;
  });
}

int dm_nccl_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw dm::NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int dm_session_create(const dm_session_config* cfg, dm_session** out) {
  return guarded([&] {
    if (cfg == nullptr || out == nullptr) throw dm::UsageError("session_create: null argument");
    auto s = std::make_unique<dm_session>();
    s->impl = std::make_unique<dm::Session>(*cfg);
    *out = s.release();
  });
}

int dm_session_destroy(dm_session* s) {
  return guarded([&] {
    if (s == nullptr) return;
    s->impl.reset();
    delete s;
  });
}

int dm_session_shutdown(dm_session* s) { return guarded([&] { S(s).shutdown(); }); }

int dm_create_matrix(dm_session* s, const dm_layout* layout, int precision, int fill,
                     const void* host, dm_matrix_id* out) {
  return guarded([&] {
    if (precision < 0 || precision > 2) throw dm::ConfigError("unknown precision");
    if (fill < 0 || fill > 2) throw dm::UsageError("unknown fill kind");
    dm::Session& ss = S(s);
    const dm::LayoutSpec l = dm::layout_from_abi(layout);
    *out = ss.create_matrix(l, static_cast<dm::Precision>(precision),
                            static_cast<dm::FillKind>(fill), host);
  });
}

int dm_destroy_matrix(dm_session* s, dm_matrix_id id) {
  return guarded([&] {
    S(s).destroy_matrix(id);
    s->custom_tables.erase(id);
  });
}

int dm_scatter(dm_session* s, dm_matrix_id id, const void* host, int64_t rows, int64_t cols) {
  return guarded([&] { S(s).scatter(id, host, rows, cols); });
}

int dm_gather(dm_session* s, dm_matrix_id id, void* host, int64_t rows, int64_t cols, int root) {
  return guarded([&] { S(s).gather(id, host, rows, cols, root); });
}

int dm_update_block(dm_session* s, dm_matrix_id id, int row, int col, const void* host,
                    int64_t rows, int64_t cols) {
  return guarded([&] { S(s).update_block(id, {row, col}, host, rows, cols); });
}

int dm_replicate(dm_session* s, dm_matrix_id id, int enable) {
  return guarded([&] { S(s).replicate(id, enable != 0); });
}

int dm_replica_read(dm_session* s, dm_matrix_id id, int reader, void* host, int64_t rows,
                    int64_t cols) {
  return guarded([&] { S(s).replica_read(id, reader, host, rows, cols); });
}

int dm_reshape(dm_session* s, dm_matrix_id src, const dm_layout* layout, int precision,
               dm_matrix_id* out) {
  return guarded([&] {
    if (precision < 0 || precision > 2) throw dm::ConfigError("unknown precision");
    *out = S(s).reshape(src, dm::layout_from_abi(layout), static_cast<dm::Precision>(precision));
  });
}

int dm_add_row_col_sum(dm_session* s, dm_matrix_id id, int axis, int deterministic,
                       dm_matrix_id* out) {
  return guarded([&] {
    if (axis != 0 && axis != 1) throw dm::UsageError("add_row_col_sum: axis must be 0 (rows) or 1 (cols)");
    *out = S(s).add_row_col_sum(id, axis, deterministic != 0);
  });
}

int dm_checkpoint(dm_session* s, const char* path) {
  return guarded([&] {
    if (path == nullptr) throw dm::UsageError("checkpoint: null path");
    S(s).checkpoint(path);
  });
}

int dm_restore(const char* path, const dm_session_config* cfg, dm_session** out) {
  return guarded([&] {
    if (path == nullptr || cfg == nullptr || out == nullptr)
      throw dm::UsageError("restore: null argument");
    // the image decides worker count and root seed (session.hpp:427-432)
    std::FILE* f = std::fopen(path, "rb");
    if (f == nullptr) throw dm::ConfigError(std::string("checkpoint: cannot open ") + path);
    unsigned char hdr[20] = {};
    const std::size_t got = std::fread(hdr, 1, sizeof(hdr), f);
    std::fclose(f);
    if (got < sizeof(hdr) || std::memcmp(hdr, "DMTH", 4) != 0)
      throw dm::IntegrityError("checkpoint: bad magic or truncated file");
    auto le = [&](int at, int n) {
      uint64_t v = 0;
      for (int i = 0; i < n; ++i) v |= static_cast<uint64_t>(hdr[at + i]) << (8 * i);
      return v;
    };
    dm_session_config c = *cfg;
    c.worker_count = static_cast<int32_t>(le(8, 4));
    c.root_seed = le(12, 8);
    auto sess = std::make_unique<dm_session>();
    sess->impl = std::make_unique<dm::Session>(c);
    sess->impl->restore_image(path);
    *out = sess.release();
  });
}

int dm_general_gemm(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b, double beta,
                    dm_matrix_id c, int ta, int tb) {
  return guarded([&] { S(s).general_gemm(alpha, a, b, beta, c, ta != 0, tb != 0); });
}

int dm_cyclic_gemm(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b, double beta,
                   dm_matrix_id c, int ta, int tb, int cache_a) {
  return guarded([&] { S(s).cyclic_gemm(alpha, a, b, beta, c, ta != 0, tb != 0, cache_a != 0); });
}

int dm_broadcast_gemm_reference(dm_session* s, double alpha, dm_matrix_id a, dm_matrix_id b,
                                double beta, dm_matrix_id c, int ta, int tb) {
  return guarded([&] { S(s).broadcast_gemm(alpha, a, b, beta, c, ta != 0, tb != 0); });
}

int dm_cached_backward_gemm(dm_session* s, dm_matrix_id w, dm_matrix_id dy, dm_matrix_id dx) {
  return guarded([&] { S(s).cached_backward_gemm(w, dy, dx); });
}

int dm_session_gemm_mode(dm_session* s, int* out) {
  return guarded([&] {
    const int m = S(s).gemm_mode();
    *out = m == dm::kModeTf32x3  ? DM_GEMM_TF32X3
           : m == dm::kModeMixed ? DM_GEMM_MIXED
           : m == dm::kModeF16x2 ? DM_GEMM_F16X2
                                 : DM_GEMM_AUTO;
  });
}

int dm_presplit_panels(int64_t k, int64_t a_kblock, int64_t b_kblock, int64_t max_width, int64_t* out, int cap,
                       int* n) {
  return guarded([&] {
    if (out == nullptr || n == nullptr) throw dm::UsageError("presplit_panels: null output");
    if (k <= 0 || a_kblock <= 0 || b_kblock <= 0) throw dm::ShapeError("presplit_panels: non-positive extent");
    const std::vector<int64_t> k0 = dm::presplit_panels(k, a_kblock, b_kblock, max_width);
    if (static_cast<int64_t>(k0.size()) > cap) throw dm::UsageError("presplit_panels: output too small");
    std::copy(k0.begin(), k0.end(), out);
    *n = static_cast<int>(k0.size());
  });
}

int dm_split_mode_for(int gemm_mode, int64_t k, double work, int* out) {
  return guarded([&] {
    if (out == nullptr) throw dm::UsageError("split_mode_for: null output");
    int mode;
    if (gemm_mode == DM_GEMM_TF32X3) mode = dm::kModeTf32x3;
    else if (gemm_mode == DM_GEMM_MIXED) mode = dm::kModeMixed;
    else if (gemm_mode == DM_GEMM_AUTO) mode = dm::kModeAuto;
    else if (gemm_mode == DM_GEMM_F16X2) mode = dm::kModeF16x2;
    else if (gemm_mode == DM_GEMM_DEFAULT) mode = dm::env_gemm_mode();
    else throw dm::UsageError("unknown gemm_mode");
    const int m = dm::resolve_split_mode(mode, k, work);
    *out = m == dm::kModeTf32x3 ? DM_GEMM_TF32X3 : m == dm::kModeMixed ? DM_GEMM_MIXED : DM_GEMM_F16X2;
  });
}

int dm_worker_count(dm_session* s, int* out) {
  return guarded([&] { *out = S(s).worker_count(); });
}

int dm_local_workers(dm_session* s, int32_t* ids, int cap) {
  std::vector<int> v;
  const int rc = guarded([&] { v = S(s).local_worker_ids(); });
  if (rc != DM_OK) return -rc;
  for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) ids[i] = v[i];
  return static_cast<int>(v.size());
}

int dm_descriptor_get(dm_session* s, dm_matrix_id id, dm_descriptor* out) {
  return guarded([&] {
    const dm::MatrixDescriptor& d = S(s).descriptor(id);
    out->matrix_id = d.matrix_id;
    out->precision = static_cast<int32_t>(d.precision);
    out->replicated = d.replicated ? 1 : 0;
    out->version = d.version;
    out->replica_version = d.replica_version;
    out->seed = d.seed;
    out->layout.kind = static_cast<int32_t>(d.layout.kind);
    out->layout.worker_count = d.layout.worker_count;
    out->layout.global_rows = d.layout.grid.global_rows;
    out->layout.global_cols = d.layout.grid.global_cols;
    out->layout.block_rows = d.layout.grid.block_rows;
    out->layout.block_cols = d.layout.grid.block_cols;
    auto& tbl = s->custom_tables[id];
    tbl.assign(d.layout.custom.begin(), d.layout.custom.end());
    out->layout.custom = tbl.empty() ? nullptr : tbl.data();
    out->layout.custom_len = static_cast<int64_t>(tbl.size());
  });
}

int dm_pool_stats_get(dm_session* s, int worker, dm_pool_stats* out) {
  return guarded([&] {
    const dm::DevicePool::Stats st = S(s).pool_stats(worker);
    out->fresh_allocations = st.fresh_allocations;
    out->reuses = st.reuses;
    out->bytes_live = st.bytes_live;
    out->bytes_pooled = st.bytes_pooled;
    out->high_water = st.high_water;
  });
}

int dm_pool_trim(dm_session* s, int worker, uint64_t* freed) {
  return guarded([&] {
    const uint64_t f = S(s).pool_trim(worker);
    if (freed) *freed = f;
  });
}

int dm_worker_stats_get(dm_session* s, int worker, dm_worker_stats* out) {
  return guarded([&] { *out = S(s).worker_stats(worker); });
}

int dm_worker_stats_reset(dm_session* s) { return guarded([&] { S(s).reset_worker_stats(); }); }

int dm_set_gemm_timing(dm_session* s, int enable) {
  return guarded([&] { S(s).set_gemm_timing(enable != 0); });
}

int dm_worker_seed(dm_session* s, int worker, uint64_t* out) {
  return guarded([&] { *out = S(s).worker_seed(worker); });
}

int dm_transfer_log(dm_session* s, dm_transfer_record* out, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    const auto& log = S(s).transfers();
    n = static_cast<int>(log.size());
    for (int i = 0; i < cap && i < n; ++i) {
      const dm::TransferRecord& r = log[static_cast<std::size_t>(i)];
      dm_transfer_record& o = out[i];
      o.seq = r.seq;
      o.src = r.src;
      o.dst = r.dst;
      o.matrix_id = r.matrix;
      o.row = r.coord.row;
      o.col = r.coord.col;
      o.bytes = r.bytes;
      std::memset(o.op, 0, sizeof o.op);
      std::strncpy(o.op, r.op.c_str(), sizeof o.op - 1);
    }
  });
  return rc != DM_OK ? -rc : n;
}

int dm_root_seed(dm_session* s, uint64_t* out) {
  return guarded([&] { *out = S(s).root_seed(); });
}

int dm_seed_workers(dm_session* s, uint64_t root, uint64_t* seeds, int cap) {
  return guarded([&] {
    const std::vector<uint64_t> v = S(s).seed_workers(root);
    for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) seeds[i] = v[i];
  });
}

int dm_descriptor_digest(dm_session* s, uint64_t* master, uint64_t* workers, int cap) {
  std::vector<uint64_t> v;
  const int rc = guarded([&] {
    *master = S(s).master_digest();
    v = S(s).worker_digests();
  });
  if (rc != DM_OK) return -rc;
  for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) workers[i] = v[i];
  return static_cast<int>(v.size());
}

int dm_block_device_ptr(dm_session* s, dm_matrix_id id, int row, int col, void** ptr, int* device) {
  return guarded([&] { *ptr = S(s).block_device_ptr(id, {row, col}, device); });
}

int dm_barrier(dm_session* s) { return guarded([&] { S(s).barrier(); }); }

int dm_set_async(dm_session* s, int on) { return guarded([&] { S(s).set_async(on != 0); }); }

int dm_marker_record(dm_session* s, int worker, int slot) {
  return guarded([&] { S(s).marker_record(worker, slot); });
}

int dm_marker_elapsed(dm_session* s, int worker, int slot_a, int slot_b, float* ms) {
  return guarded([&] { *ms = S(s).marker_elapsed(worker, slot_a, slot_b); });
}

int dm_local_gemm_f32(double alpha, const float* a, int64_t lda, int ta, const float* b,
                      int64_t ldb, int tb, double beta, float* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, void* stream) {
  return local_gemm_impl(alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, m, n, k, 0, DM_GEMM_DEFAULT, stream);
}

int dm_local_gemm_f32_ex(double alpha, const float* a, int64_t lda, int ta, const float* b,
                         int64_t ldb, int tb, double beta, float* c, int64_t ldc, int64_t m,
                         int64_t n, int64_t k, int cta_group, int gemm_mode, void* stream) {
  return local_gemm_impl(alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, m, n, k, cta_group, gemm_mode, stream);
}

int dm_local_gemm_f32_workspace_size(int64_t m, int64_t n, int64_t k, int cta_group, int gemm_mode,
                                     size_t* bytes) {
  return guarded([&] {
    if (bytes == nullptr) throw dm::UsageError("local_gemm_workspace_size: null output");
    if (m < 0 || n < 0 || k < 0) throw dm::ShapeError("local_gemm: negative dimension");
    const int mode = resolve_gemm_mode(gemm_mode, m, n, k);
    *bytes = 0;
    for (int ta : {0, 1})
      for (int tb : {0, 1}) *bytes = std::max(*bytes, seam_layout(seam_shape(m, n, k, cta_group, mode), ta, tb).total);
  });
}

int dm_local_gemm_f32_ws(double alpha, const float* a, int64_t lda, int ta, const float* b, int64_t ldb,
                         int tb, double beta, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
                         int cta_group, int gemm_mode, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    local_gemm_validate(a, lda, ta, b, ldb, tb, c, ldc, m, n, k, cta_group);
    const int mode = resolve_gemm_mode(gemm_mode, m, n, k);
    const SeamLayout L = seam_layout(seam_shape(m, n, k, cta_group, mode), ta, tb);
    if (workspace_bytes < L.total || (L.total > 0 && workspace == nullptr))
      throw dm::UsageError("local_gemm: workspace smaller than dm_local_gemm_f32_workspace_size");
    if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
      throw dm::UsageError("local_gemm: workspace must be 256-byte aligned");
    local_gemm_run(alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, m, n, k, cta_group, mode,
                   static_cast<char*>(workspace), L, static_cast<cudaStream_t>(stream));
  });
}

int dm_fill_seeded_f32(float* dst, int64_t count, uint64_t matrix_seed, int block_row,
                       int block_col, void* stream) {
  return guarded([&] {
    const uint64_t key =
        dm::mix64(matrix_seed, (static_cast<uint64_t>(static_cast<uint32_t>(block_row)) << 32) |
                                   static_cast<uint32_t>(block_col));
    dm::cuda_check(dm::fill_seeded(dst, 1, count, key, static_cast<cudaStream_t>(stream)),
                   "fill_seeded");
  });
}

}  // extern "C"
