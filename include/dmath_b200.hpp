// dmath_b200.hpp -- header-only C++17 host API over the C ABI (dmath_b200.h).
//
// Mirrors the reference's user-facing interface so a `gridgemm` caller swaps
// the include and namespace and keeps its call sites:
//   gridgemm::Session            session.hpp:53-485   -> dmath_b200::Session
//   gridgemm::LayoutSpec / make_layout / make_custom_layout / checkerboard_dims
//                                layout.hpp:69-220    -> same names
//   gridgemm::HostMatrix         dense.hpp:68-112     -> dmath_b200::HostMatrix
//   UsageError ... CacheMissError common.hpp:22-78    -> same names, same hierarchy
//   Precision / FillKind / Axis  precision.hpp:14, runtime_types.hpp:68, kernels.hpp:17
// Every call goes through libdmath_b200.so; failures throw the exception class
// the reference throws for the same condition (status codes map 1:1).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dmath_b200.h"

namespace dmath_b200 {

using MatrixId = std::uint64_t;
using WorkerId = int;

enum class LayoutKind : std::uint8_t { RowBlocks1D = 0, ColBlocks1D = 1, RowCyclic1D = 2, Checkerboard2D = 3, Custom = 4 };
enum class Precision : std::uint8_t { Half16 = 0, Single32 = 1, Double64 = 2 };
enum class FillKind : std::uint8_t { Zeros = 0, SeededRandom = 1, FromHost = 2 };
enum class Axis : std::uint8_t { Rows = 0, Cols = 1 };

inline std::size_t byte_width(Precision p) { return p == Precision::Half16 ? 2 : p == Precision::Single32 ? 4 : 8; }

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct ProtocolError : Error { using Error::Error; };
struct DeadlockError : Error { using Error::Error; };
struct IntegrityError : Error { using Error::Error; };
struct PlanError : Error { using Error::Error; };
struct CacheMissError : Error {
  CacheMissError(const std::string& m, std::vector<std::pair<int, int>> coords)
      : Error(m), missing_coords(std::move(coords)) {}
  std::vector<std::pair<int, int>> missing_coords;  // common.hpp:72-78
};
struct CudaError : Error { using Error::Error; };
struct NcclError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };

inline void check(int rc) {
  if (rc == DM_OK) return;
  const std::string msg = dm_last_error();
  switch (rc) {
    case DM_ERR_USAGE: throw UsageError(msg);
    case DM_ERR_CONFIG: throw ConfigError(msg);
    case DM_ERR_SHAPE: throw ShapeError(msg);
    case DM_ERR_PROTOCOL: throw ProtocolError(msg);
    case DM_ERR_DEADLOCK: throw DeadlockError(msg);
    case DM_ERR_INTEGRITY: throw IntegrityError(msg);
    case DM_ERR_PLAN: throw PlanError(msg);
    case DM_ERR_CACHE_MISS: {
      std::vector<int32_t> raw(2 * 4096);
      const int n = dm_last_error_missing(raw.data(), static_cast<int>(raw.size() / 2));
      std::vector<std::pair<int, int>> coords;
      for (int i = 0; i < n; ++i) coords.emplace_back(raw[2 * i], raw[2 * i + 1]);
      throw CacheMissError(msg, std::move(coords));
    }
    case DM_ERR_CUDA: throw CudaError(msg);
    case DM_ERR_NCCL: throw NcclError(msg);
    case DM_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw Error(msg);
  }
}

// ------------------------------------------------------------------ layout
struct BlockCoord {
  int row = 0, col = 0;
};

// LayoutSpec (layout.hpp:116-220): the value type; custom owner tables are
// held here so the C struct's pointer stays valid for the object's lifetime.
class LayoutSpec {
 public:
  LayoutSpec() = default;
  LayoutSpec(LayoutKind kind, std::int64_t gr, std::int64_t gc, std::int64_t br, std::int64_t bc, int workers,
             std::vector<int32_t> custom = {})
      : custom_(std::move(custom)) {
    l_.kind = static_cast<int32_t>(kind);
    l_.worker_count = workers;
    l_.global_rows = gr;
    l_.global_cols = gc;
    l_.block_rows = br;
    l_.block_cols = bc;
  }
  LayoutSpec(const LayoutSpec& o) : l_(o.l_), custom_(o.custom_) {}
  LayoutSpec& operator=(const LayoutSpec& o) {
    l_ = o.l_;
    custom_ = o.custom_;
    return *this;
  }

  const dm_layout* c() const {
    l_.custom = custom_.empty() ? nullptr : custom_.data();
    l_.custom_len = static_cast<int64_t>(custom_.size());
    return &l_;
  }
  LayoutKind kind() const { return static_cast<LayoutKind>(l_.kind); }
  int worker_count() const { return l_.worker_count; }
  std::int64_t global_rows() const { return l_.global_rows; }
  std::int64_t global_cols() const { return l_.global_cols; }
  std::int64_t block_rows() const { return l_.block_rows; }
  std::int64_t block_cols() const { return l_.block_cols; }

  WorkerId owner(BlockCoord b) const {
    int o = -1;
    check(dm_layout_owner(c(), b.row, b.col, &o));
    return o;
  }
  std::pair<int, int> grid() const {
    int r = 0, cc = 0, clamped = 0;
    check(dm_layout_grid(c(), &r, &cc, &clamped));
    return {r, cc};
  }
  std::pair<std::int64_t, std::int64_t> block_extent(BlockCoord b) const {
    std::int64_t r = 0, cc = 0;
    check(dm_block_extent(c(), b.row, b.col, &r, &cc));
    return {r, cc};
  }
  std::string to_string() const {  // returns -status on error, else the length + 1
    const int need = dm_layout_to_string(c(), nullptr, 0);
    if (need < 0) check(-need);
    std::string out(static_cast<std::size_t>(need), '\0');
    dm_layout_to_string(c(), &out[0], need);
    out.resize(static_cast<std::size_t>(need - 1));
    return out;
  }

 private:
  mutable dm_layout l_{};
  std::vector<int32_t> custom_;
};

inline std::pair<int, int> checkerboard_dims(int workers) {
  int pr = 0, pc = 0;
  check(dm_checkerboard_dims(workers, &pr, &pc));
  return {pr, pc};
}
inline LayoutSpec make_layout(LayoutKind kind, std::int64_t gr, std::int64_t gc, std::int64_t br, std::int64_t bc,
                              int workers) {
  return LayoutSpec(kind, gr, gc, br, bc, workers);
}
inline LayoutSpec make_custom_layout(std::int64_t gr, std::int64_t gc, std::int64_t br, std::int64_t bc,
                                     int workers, std::vector<int32_t> owners) {
  return LayoutSpec(LayoutKind::Custom, gr, gc, br, bc, workers, std::move(owners));
}

// ------------------------------------------------------------------ host data
namespace detail {
// Round-to-nearest-even double -> binary16 with the reference's rules
// (half.hpp:19-76): saturate to infinity past the half range, NaN keeps its
// top payload bits (a zero payload becomes the quiet bit).
inline std::uint16_t half_from_double(double v) {
  std::uint64_t b;
  std::memcpy(&b, &v, 8);
  const std::uint16_t sign = static_cast<std::uint16_t>((b >> 48) & 0x8000u);
  if ((b & 0x7FF0000000000000ull) == 0x7FF0000000000000ull) {
    if ((b & 0xFFFFFFFFFFFFFull) == 0) return sign | 0x7C00u;  // infinity
    std::uint16_t pay = static_cast<std::uint16_t>((b >> 42) & 0x3FFu);
    return sign | 0x7C00u | (pay ? pay : 0x200u);
  }
  const double a = std::fabs(v);
  if (a >= 65520.0) return sign | 0x7C00u;           // rounds past 65504
  if (a >= 6.103515625e-05) {                         // normal: 2^-14 <= a
    int e = 0;
    const double m = std::frexp(a, &e);               // a = m 2^e, m in [0.5, 1)
    double r = std::nearbyint(std::ldexp(m, 11));     // 11-bit significand, RNE
    if (r == 2048.0) {
      r = 1024.0;
      ++e;
    }
    return sign | static_cast<std::uint16_t>(((e + 14) << 10) | (static_cast<int>(r) - 1024));
  }
  return sign | static_cast<std::uint16_t>(std::nearbyint(std::ldexp(a, 24)));  // subnormal (or 0x400)
}
inline double half_to_double(std::uint16_t h) {
  const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
  const double s = (h & 0x8000) ? -1.0 : 1.0;
  if (e == 0) return s * std::ldexp(m, -24);
  if (e == 31) return m ? NAN : s * INFINITY;
  return s * std::ldexp(1024 + m, e - 25);
}
}  // namespace detail

// HostMatrix (dense.hpp:68-112): row-major bytes at a runtime precision.
class HostMatrix {
 public:
  HostMatrix() = default;
  HostMatrix(std::int64_t rows, std::int64_t cols, Precision p)
      : rows_(rows), cols_(cols), precision_(p),
        bytes_(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols) * byte_width(p)) {}
  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  Precision precision() const { return precision_; }
  std::size_t byte_size() const { return bytes_.size(); }
  const void* raw() const { return bytes_.data(); }
  void* raw() { return bytes_.data(); }

  double get(std::int64_t r, std::int64_t c) const {
    const unsigned char* p = bytes_.data() + off(r, c);
    if (precision_ == Precision::Single32) {
      float f;
      std::memcpy(&f, p, 4);
      return f;
    }
    if (precision_ == Precision::Double64) {
      double d;
      std::memcpy(&d, p, 8);
      return d;
    }
    std::uint16_t h;
    std::memcpy(&h, p, 2);
    return detail::half_to_double(h);
  }
  void set(std::int64_t r, std::int64_t c, double v) {  // narrowed once, RNE (precision.hpp:83-89)
    unsigned char* p = bytes_.data() + off(r, c);
    if (precision_ == Precision::Single32) {
      const float f = static_cast<float>(v);
      std::memcpy(p, &f, 4);
    } else if (precision_ == Precision::Double64) {
      std::memcpy(p, &v, 8);
    } else {
      const std::uint16_t h = detail::half_from_double(v);
      std::memcpy(p, &h, 2);
    }
  }
  // Element-wise conversion through double, as scatter_payloads (session.hpp:568-576).
  HostMatrix converted(Precision p) const {
    if (p == precision_) return *this;
    HostMatrix out(rows_, cols_, p);
    for (std::int64_t r = 0; r < rows_; ++r)
      for (std::int64_t c = 0; c < cols_; ++c) out.set(r, c, get(r, c));
    return out;
  }
  bool bitwise_equal(const HostMatrix& o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && precision_ == o.precision_ && bytes_ == o.bytes_;
  }

 private:
  std::size_t off(std::int64_t r, std::int64_t c) const {
    return static_cast<std::size_t>(r * cols_ + c) * byte_width(precision_);
  }
  std::int64_t rows_ = 0, cols_ = 0;
  Precision precision_ = Precision::Single32;
  std::vector<unsigned char> bytes_;
};

// ------------------------------------------------------------------ session
struct PoolStats {  // Pool::Stats, pool.hpp:63-69
  std::uint64_t fresh_allocations = 0, reuses = 0, bytes_live = 0, bytes_pooled = 0, high_water = 0;
};

struct MatrixDescriptor {  // layout.hpp:224-236
  MatrixId matrix_id = 0;
  LayoutSpec layout;
  Precision precision = Precision::Single32;
  bool replicated = false;
  std::uint64_t version = 0, replica_version = 0, seed = 0;
};

class Session {
 public:
  struct Config {  // session.hpp:55-62 (+ the B200 placement fields)
    int worker_count = 1;
    std::uint64_t root_seed = 0;
    bool coherence_checks = true;
    int mode = DM_MODE_LOCAL;        // DM_MODE_SPMD: one process per GPU
    int rank = 0;                    // SPMD: this process's worker id
    std::vector<int32_t> devices;    // LOCAL: device of each worker (empty: w % device_count)
    std::vector<unsigned char> nccl_id;  // SPMD: 128 bytes from dm_nccl_unique_id on rank 0
    int gemm_mode = DM_GEMM_DEFAULT;     // dm_gemm_mode: split-product scheme of the GEMMs
  };

  explicit Session(Config cfg) : cfg_(std::move(cfg)) { check(dm_session_create(&c_config(), &s_)); }
  ~Session() {
    if (s_) dm_session_destroy(s_);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  static std::unique_ptr<Session> restore(const std::string& path) { return restore(path, Config()); }
  static std::unique_ptr<Session> restore(const std::string& path, Config base) {
    std::unique_ptr<Session> s(new Session());
    s->cfg_ = std::move(base);
    check(dm_restore(path.c_str(), &s->c_config(), &s->s_));
    check(dm_worker_count(s->s_, &s->cfg_.worker_count));
    return s;
  }

  int worker_count() const { return cfg_.worker_count; }
  std::uint64_t root_seed() const {  // session.hpp:92
    std::uint64_t v = 0;
    check(dm_root_seed(s_, &v));
    return v;
  }

  MatrixId create_matrix(const LayoutSpec& layout, Precision precision, FillKind fill,
                         const HostMatrix* host = nullptr) {
    if (fill == FillKind::FromHost && host == nullptr) throw UsageError("create_matrix: FromHost requires host data");
    if (fill == FillKind::FromHost &&
        (host->rows() != layout.global_rows() || host->cols() != layout.global_cols()))
      throw ShapeError("create_matrix: host data shape does not match the layout");
    HostMatrix conv;
    const HostMatrix* h = fill == FillKind::FromHost ? host : nullptr;
    if (h && h->precision() != precision) {
      conv = h->converted(precision);
      h = &conv;
    }
    MatrixId id = 0;
    check(dm_create_matrix(s_, layout.c(), static_cast<int>(precision), static_cast<int>(fill),
                           h ? h->raw() : nullptr, &id));
    return id;
  }
  void destroy_matrix(MatrixId id) { check(dm_destroy_matrix(s_, id)); }

  void scatter(MatrixId id, const HostMatrix& host) {
    const Precision p = descriptor(id).precision;
    if (host.precision() != p) {
      const HostMatrix conv = host.converted(p);
      check(dm_scatter(s_, id, conv.raw(), conv.rows(), conv.cols()));
    } else {
      check(dm_scatter(s_, id, host.raw(), host.rows(), host.cols()));
    }
  }
  HostMatrix gather(MatrixId id) {
    const MatrixDescriptor d = descriptor(id);
    HostMatrix h(d.layout.global_rows(), d.layout.global_cols(), d.precision);
    check(dm_gather(s_, id, h.raw(), h.rows(), h.cols(), 0));
    return h;
  }
  void update_block(MatrixId id, BlockCoord coord, const HostMatrix& data) {
    const HostMatrix conv = data.converted(descriptor(id).precision);  // convert_precision, session.hpp:214-216
    check(dm_update_block(s_, id, coord.row, coord.col, conv.raw(), conv.rows(), conv.cols()));
  }

  void general_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool trans_a, bool trans_b) {
    check(dm_general_gemm(s_, alpha, a, b, beta, c, trans_a, trans_b));
  }
  void cyclic_gemm(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool trans_a, bool trans_b,
                   bool cache_a) {
    check(dm_cyclic_gemm(s_, alpha, a, b, beta, c, trans_a, trans_b, cache_a));
  }
  void broadcast_gemm_reference(double alpha, MatrixId a, MatrixId b, double beta, MatrixId c, bool trans_a,
                                bool trans_b) {
    check(dm_broadcast_gemm_reference(s_, alpha, a, b, beta, c, trans_a, trans_b));
  }
  void cached_backward_gemm(MatrixId w, MatrixId dy, MatrixId dx) { check(dm_cached_backward_gemm(s_, w, dy, dx)); }

  void replicate(MatrixId id, bool enable) { check(dm_replicate(s_, id, enable)); }
  HostMatrix replica_read(MatrixId id, WorkerId reader) {
    const MatrixDescriptor d = descriptor(id);
    HostMatrix h(d.layout.global_rows(), d.layout.global_cols(), d.precision);
    check(dm_replica_read(s_, id, reader, h.raw(), h.rows(), h.cols()));
    return h;
  }
  MatrixId reshape(MatrixId src, const LayoutSpec& layout, Precision precision) {
    MatrixId out = 0;
    check(dm_reshape(s_, src, layout.c(), static_cast<int>(precision), &out));
    return out;
  }
  MatrixId add_row_col_sum(MatrixId id, Axis axis, bool deterministic_reduce) {
    MatrixId out = 0;
    check(dm_add_row_col_sum(s_, id, static_cast<int>(axis), deterministic_reduce, &out));
    return out;
  }
  void checkpoint(const std::string& path) { check(dm_checkpoint(s_, path.c_str())); }
  void shutdown() { check(dm_session_shutdown(s_)); }

  MatrixDescriptor descriptor(MatrixId id) const {
    dm_descriptor d{};
    check(dm_descriptor_get(s_, id, &d));
    MatrixDescriptor out;
    out.matrix_id = d.matrix_id;
    std::vector<int32_t> custom(d.layout.custom, d.layout.custom + (d.layout.custom ? d.layout.custom_len : 0));
    out.layout = LayoutSpec(static_cast<LayoutKind>(d.layout.kind), d.layout.global_rows, d.layout.global_cols,
                            d.layout.block_rows, d.layout.block_cols, d.layout.worker_count, std::move(custom));
    out.precision = static_cast<Precision>(d.precision);
    out.replicated = d.replicated != 0;
    out.version = d.version;
    out.replica_version = d.replica_version;
    out.seed = d.seed;
    return out;
  }
  PoolStats worker_pool_stats(WorkerId w) const {
    dm_pool_stats p{};
    check(dm_pool_stats_get(s_, w, &p));
    return {p.fresh_allocations, p.reuses, p.bytes_live, p.bytes_pooled, p.high_water};
  }
  std::uint64_t worker_seed(WorkerId w) const {
    std::uint64_t v = 0;
    check(dm_worker_seed(s_, w, &v));
    return v;
  }
  // Session::trace() (session.hpp:94): worker-to-worker block transfers pulled by
  // this process's workers, oldest first (TransferRecord, transport.hpp:27-38).
  std::vector<dm_transfer_record> trace() const {
    const int n = dm_transfer_log(s_, nullptr, 0);
    if (n < 0) check(-n);
    std::vector<dm_transfer_record> out(static_cast<std::size_t>(n));
    const int m = dm_transfer_log(s_, out.data(), n);
    if (m < 0) check(-m);
    out.resize(static_cast<std::size_t>(std::min(m, n)));
    return out;
  }
  std::vector<std::uint64_t> seed_workers(std::uint64_t root) {  // session.hpp:115-125
    std::vector<std::uint64_t> v(static_cast<std::size_t>(worker_count()));
    check(dm_seed_workers(s_, root, v.data(), static_cast<int>(v.size())));
    return v;
  }
  dm_worker_stats worker_stats(WorkerId w) const {
    dm_worker_stats st{};
    check(dm_worker_stats_get(s_, w, &st));
    return st;
  }
  void reset_worker_stats() { check(dm_worker_stats_reset(s_)); }
  dm_session* handle() const { return s_; }

 private:
  Session() = default;
  const dm_session_config& c_config() {
    cc_.worker_count = cfg_.worker_count;
    cc_.mode = cfg_.mode;
    cc_.rank = cfg_.rank;
    cc_.coherence_checks = cfg_.coherence_checks ? 1 : 0;
    cc_.root_seed = cfg_.root_seed;
    cc_.devices = cfg_.devices.empty() ? nullptr : cfg_.devices.data();
    cc_.nccl_id = cfg_.nccl_id.empty() ? nullptr : cfg_.nccl_id.data();
    cc_.gemm_mode = cfg_.gemm_mode;
    return cc_;
  }
  Config cfg_;
  dm_session_config cc_{};
  dm_session* s_ = nullptr;
};

// The per-worker BLAS seam (kernels.hpp:81-89) on device pointers, stream-ordered.
inline void local_gemm(double alpha, const float* a, std::int64_t lda, bool trans_a, const float* b,
                       std::int64_t ldb, bool trans_b, double beta, float* c, std::int64_t ldc, std::int64_t m,
                       std::int64_t n, std::int64_t k, void* stream = nullptr) {
  check(dm_local_gemm_f32(alpha, a, lda, trans_a, b, ldb, trans_b, beta, c, ldc, m, n, k, stream));
}

// The same with caller-owned scratch (capturable in a CUDA graph).
inline std::size_t local_gemm_workspace_size(std::int64_t m, std::int64_t n, std::int64_t k,
                                             int gemm_mode = DM_GEMM_DEFAULT) {
  std::size_t bytes = 0;
  check(dm_local_gemm_f32_workspace_size(m, n, k, 0, gemm_mode, &bytes));
  return bytes;
}
inline void local_gemm(double alpha, const float* a, std::int64_t lda, bool trans_a, const float* b,
                       std::int64_t ldb, bool trans_b, double beta, float* c, std::int64_t ldc, std::int64_t m,
                       std::int64_t n, std::int64_t k, void* workspace, std::size_t workspace_bytes,
                       void* stream, int gemm_mode = DM_GEMM_DEFAULT) {
  check(dm_local_gemm_f32_ws(alpha, a, lda, trans_a, b, ldb, trans_b, beta, c, ldc, m, n, k, 0, gemm_mode,
                             workspace, workspace_bytes, stream));
}

}  // namespace dmath_b200
