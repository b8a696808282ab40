// C++ parity tests through include/dmath_b200.hpp -- the reference user's view.
//
// Each case restates a check from the reference's own suites against the same
// inputs: the Appendix-A known answers (tests/acceptance.cpp:61-108),
// distribute/collect bitwise (tests/test_runtime.cpp:106-141), transposes and
// alpha/beta (tests/test_dist_ops.cpp:136-147, 267-282), the FC zero-transfer
// backward (tests/test_dist_ops.cpp:206-249), pool steady state
// (tests/acceptance.cpp:437-457), reshape narrowing (tests/acceptance.cpp:336-388)
// and the error taxonomy (common.hpp:22-78).  fp32 GEMMs are held to the
// reference's relFro <= 1e-5 against a double oracle (harness.hpp:114-120).
//
// usage: test_session [host]   "host": only the checks that need no GPU.
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>

#include "dmath_b200.hpp"

using namespace dmath_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(x)                                                              \
  do {                                                                        \
    if (x) {                                                                  \
      ++g_pass;                                                               \
    } else {                                                                  \
      ++g_fail;                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);       \
    }                                                                         \
  } while (0)

template <class E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "  wrong exception: %s\n", e.what());
    return false;
  }
  return false;
}

// FNV-1a 64 over the row-major bytes (common.hpp:83-103).
static std::uint64_t fnv1a(const HostMatrix& m) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  const auto* p = static_cast<const unsigned char*>(m.raw());
  for (std::size_t i = 0; i < m.byte_size(); ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// double oracle: alpha * op(A) op(B) + beta * C0
static std::vector<double> oracle(double alpha, const HostMatrix& A, bool ta, const HostMatrix& B, bool tb,
                                  double beta, const HostMatrix& C0) {
  const std::int64_t m = ta ? A.cols() : A.rows(), k = ta ? A.rows() : A.cols(), n = tb ? B.rows() : B.cols();
  std::vector<double> out(static_cast<std::size_t>(m * n));
  for (std::int64_t i = 0; i < m; ++i)
    for (std::int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (std::int64_t q = 0; q < k; ++q) acc += (ta ? A.get(q, i) : A.get(i, q)) * (tb ? B.get(j, q) : B.get(q, j));
      out[i * n + j] = alpha * acc + (beta != 0.0 ? beta * C0.get(i, j) : 0.0);
    }
  return out;
}

static double relfro(const HostMatrix& got, const std::vector<double>& want) {
  double num = 0, den = 0;
  for (std::int64_t i = 0; i < got.rows(); ++i)
    for (std::int64_t j = 0; j < got.cols(); ++j) {
      const double w = want[i * got.cols() + j], d = got.get(i, j) - w;
      num += d * d;
      den += w * w;
    }
  return std::sqrt(num / den);
}

static Session::Config local(int workers, std::uint64_t seed) {
  Session::Config c;
  c.worker_count = workers;
  c.root_seed = seed;
  c.devices.assign(workers, 0);  // all workers on GPU 0: the same plans as P GPUs
  return c;
}

static HostMatrix random_host(std::int64_t r, std::int64_t c, unsigned seed) {
  HostMatrix h(r, c, Precision::Single32);
  std::mt19937 g(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (std::int64_t i = 0; i < r; ++i)
    for (std::int64_t j = 0; j < c; ++j) h.set(i, j, u(g));
  return h;
}

// ---------------------------------------------------------------- host only
static void host_checks() {
  CHECK(checkerboard_dims(8) == std::make_pair(2, 4));
  CHECK(checkerboard_dims(6) == std::make_pair(2, 3));
  const LayoutSpec l = make_layout(LayoutKind::Checkerboard2D, 2048, 2048, 1024, 512, 8);
  CHECK(l.to_string() == "checkerboard:2048x2048:1024x512:8");
  CHECK(l.owner({1, 3}) == 7);  // (r % pr) * pc + (c % pc), layout.hpp:131-134
  const LayoutSpec t = make_layout(LayoutKind::RowBlocks1D, 100, 30, 40, 30, 3);
  CHECK(t.block_extent({2, 0}) == std::make_pair(std::int64_t{20}, std::int64_t{30}));  // trimmed edge
  const LayoutSpec cu = make_custom_layout(4, 4, 2, 2, 2, {1, 0, 0, 1});
  CHECK(cu.owner({0, 0}) == 1 && cu.owner({1, 1}) == 1);
  // invalid geometry raises the reference's UsageError (layout.hpp:43-59, 122-139)
  CHECK(throws<UsageError>([] { make_layout(LayoutKind::Checkerboard2D, 10, 10, 0, 5, 4).owner({0, 0}); }));
  CHECK(throws<UsageError>([] { make_layout(LayoutKind::Checkerboard2D, 10, 10, 5, 5, 0).owner({0, 0}); }));
  CHECK(throws<UsageError>([] { make_layout(LayoutKind::Checkerboard2D, 10, 10, 5, 5, 4).owner({5, 0}); }));
  // binary16 narrowing rules of the host conversion (half.hpp)
  HostMatrix h(1, 4, Precision::Half16);
  h.set(0, 0, 1.0);
  h.set(0, 1, 65520.0);        // rounds past the half max -> inf
  h.set(0, 2, 5.960464477539063e-08);  // 2^-24, smallest subnormal
  h.set(0, 3, -0.1);
  CHECK(h.get(0, 0) == 1.0);
  CHECK(std::isinf(h.get(0, 1)));
  CHECK(h.get(0, 2) == 5.960464477539063e-08);
  CHECK(h.get(0, 3) == -0.0999755859375);
  // no GPU: the session refuses loudly (no CPU fallback)
  if (std::getenv("DM_EXPECT_NO_GPU")) CHECK(throws<CudaError>([] { Session s(local(1, 0)); }));
}

// ---------------------------------------------------------------- GPU
static void kat_appendix_a() {
  for (int variant = 0; variant < 2; ++variant) {
    const double alpha = variant ? 1.5 : 1.0, beta = variant ? -0.5 : 0.0;
    Session s(local(4, 42));
    const LayoutSpec l = make_layout(LayoutKind::Checkerboard2D, 256, 256, 128, 128, 4);
    const MatrixId a = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
    const MatrixId b = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
    const MatrixId c = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
    const HostMatrix A = s.gather(a), B = s.gather(b), C0 = s.gather(c);
    CHECK(fnv1a(A) == 0x887fa80ad91cf55full);
    CHECK(fnv1a(B) == 0x05066aab89ecf646ull);
    CHECK(fnv1a(C0) == 0x3e444ea3608a984eull);
    const std::uint64_t v0 = s.descriptor(c).version;
    s.general_gemm(alpha, a, b, beta, c, false, false);
    CHECK(relfro(s.gather(c), oracle(alpha, A, false, B, false, beta, C0)) <= 1e-5);
    CHECK(s.descriptor(c).version == v0 + 1);  // +1 per GEMM on C (runtime_types.hpp:296-301)
  }
}

static void distribute_collect() {
  const LayoutKind kinds[] = {LayoutKind::RowBlocks1D, LayoutKind::ColBlocks1D, LayoutKind::RowCyclic1D,
                              LayoutKind::Checkerboard2D};
  for (LayoutKind k : kinds) {
    Session s(local(3, 5));
    const HostMatrix h = random_host(37, 53, 7 + static_cast<unsigned>(k));
    const MatrixId m = s.create_matrix(make_layout(k, 37, 53, 8, 16, 3), Precision::Single32, FillKind::FromHost, &h);
    CHECK(s.gather(m).bitwise_equal(h));
  }
}

static void transposes_alpha_beta() {
  for (int tr = 0; tr < 4; ++tr) {
    const bool ta = tr & 1, tb = tr & 2;
    Session s(local(3, 900 + tr));
    const MatrixId a = s.create_matrix(make_layout(LayoutKind::RowCyclic1D, 96, 96, 20, 24, 3), Precision::Single32,
                                       FillKind::SeededRandom);
    const MatrixId b = s.create_matrix(make_layout(LayoutKind::Checkerboard2D, 96, 96, 24, 20, 3),
                                       Precision::Single32, FillKind::SeededRandom);
    const MatrixId c = s.create_matrix(make_layout(LayoutKind::ColBlocks1D, 96, 96, 32, 16, 3), Precision::Single32,
                                       FillKind::SeededRandom);
    const HostMatrix A = s.gather(a), B = s.gather(b), C0 = s.gather(c);
    s.general_gemm(1.5, a, b, -0.5, c, ta, tb);
    CHECK(relfro(s.gather(c), oracle(1.5, A, ta, B, tb, -0.5, C0)) <= 1e-5);
  }
}

static void fc_zero_transfer_backward() {
  const int P = 4;
  const std::int64_t fin = 96 * P, fout = 64, batch = 16 * P, strip = batch / P;
  Session s(local(P, 3));
  const MatrixId W = s.create_matrix(make_layout(LayoutKind::RowBlocks1D, fin, fout, fin / P, fout, P),
                                     Precision::Single32, FillKind::SeededRandom);
  const MatrixId X = s.create_matrix(make_layout(LayoutKind::ColBlocks1D, fin, batch, fin, strip, P),
                                     Precision::Single32, FillKind::SeededRandom);
  const MatrixId Y = s.create_matrix(make_layout(LayoutKind::ColBlocks1D, fout, batch, fout, strip, P),
                                     Precision::Single32, FillKind::Zeros);
  const MatrixId dY = s.create_matrix(make_layout(LayoutKind::ColBlocks1D, fout, batch, fout, strip, P),
                                      Precision::Single32, FillKind::SeededRandom);
  const MatrixId dX = s.create_matrix(make_layout(LayoutKind::ColBlocks1D, fin, batch, fin, strip, P),
                                      Precision::Single32, FillKind::Zeros);
  // backward before any forward cached W: stale cache, missing coords reported
  bool missing = false;
  try {
    s.cached_backward_gemm(W, dY, dX);
  } catch (const CacheMissError& e) {
    missing = !e.missing_coords.empty();
  }
  CHECK(missing);
  const HostMatrix Wh = s.gather(W), Xh = s.gather(X), dYh = s.gather(dY);
  s.cyclic_gemm(1.0, W, X, 0.0, Y, true, false, true);  // Y = W^T X, keep W blocks
  CHECK(relfro(s.gather(Y), oracle(1.0, Wh, true, Xh, false, 0.0, Wh)) <= 1e-5);
  s.reset_worker_stats();
  const std::size_t before = s.trace().size();  // as tests/acceptance.cpp:165-171
  s.cached_backward_gemm(W, dY, dX);  // dX = W dY from cached blocks only
  CHECK(s.trace().size() == before);
  for (int w = 0; w < P; ++w) CHECK(s.worker_stats(w).peer_bytes_read == 0);
  CHECK(relfro(s.gather(dX), oracle(1.0, Wh, false, dYh, false, 0.0, Wh)) <= 1e-5);
}

static void pool_steady_state() {
  Session s(local(4, 11));
  const LayoutSpec l = make_layout(LayoutKind::Checkerboard2D, 512, 512, 256, 256, 4);
  const MatrixId a = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
  const MatrixId b = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
  const MatrixId c = s.create_matrix(l, Precision::Single32, FillKind::Zeros);
  s.general_gemm(1.0, a, b, 0.0, c, false, false);
  std::vector<std::uint64_t> fresh;
  for (int w = 0; w < 4; ++w) fresh.push_back(s.worker_pool_stats(w).fresh_allocations);
  for (int it = 0; it < 3; ++it) s.general_gemm(1.0, a, b, 0.0, c, false, false);
  for (int w = 0; w < 4; ++w) CHECK(s.worker_pool_stats(w).fresh_allocations == fresh[w]);
}

static void reshape_narrowing_and_checkpoint(const std::string& dir) {
  Session s(local(4, 21));
  const MatrixId a = s.create_matrix(make_layout(LayoutKind::Checkerboard2D, 64, 48, 32, 24, 4),
                                     Precision::Single32, FillKind::SeededRandom);
  const HostMatrix A = s.gather(a);
  const MatrixId h = s.reshape(a, make_layout(LayoutKind::RowCyclic1D, 64, 48, 8, 48, 4), Precision::Half16);
  CHECK(s.gather(h).bitwise_equal(A.converted(Precision::Half16)));  // narrowed once, RNE
  const MatrixId r = s.add_row_col_sum(a, Axis::Rows, true);
  const HostMatrix R = s.gather(r);
  CHECK(R.rows() * R.cols() == 48 || R.rows() * R.cols() == 64);
  const std::string path = dir + "/cpp_ck.dmth";
  s.checkpoint(path);
  auto back = Session::restore(path, local(4, 0));
  CHECK(back->gather(a).bitwise_equal(A));
  CHECK(back->gather(h).bitwise_equal(A.converted(Precision::Half16)));
}

static void errors() {
  Session s(local(2, 1));
  const LayoutSpec l = make_layout(LayoutKind::RowBlocks1D, 16, 16, 8, 16, 2);
  const MatrixId a = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
  const MatrixId b = s.create_matrix(l, Precision::Single32, FillKind::SeededRandom);
  const MatrixId odd = s.create_matrix(make_layout(LayoutKind::RowBlocks1D, 16, 8, 8, 8, 2), Precision::Single32,
                                       FillKind::Zeros);
  CHECK(throws<UsageError>([&] { s.general_gemm(1, a, b, 0, a, false, false); }));     // C aliases A
  CHECK(throws<ShapeError>([&] { s.general_gemm(1, a, odd, 0, b, false, false); }));   // inner/outer shape
  CHECK(throws<UsageError>([&] { s.general_gemm(1, a, b, 0, 9999, false, false); }));  // unknown id
  const HostMatrix wrong = random_host(5, 5, 1);
  CHECK(throws<ShapeError>([&] { s.scatter(a, wrong); }));
  s.shutdown();
  CHECK(throws<UsageError>([&] { s.gather(a); }));  // session shut down
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "host") == 0;
  host_checks();
  if (!host_only) {
    const std::string dir = argc > 2 ? argv[2] : "/tmp";
    kat_appendix_a();
    distribute_collect();
    transposes_alpha_beta();
    fc_zero_transfer_backward();
    pool_steady_state();
    reshape_narrowing_and_checkpoint(dir);
    errors();
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
