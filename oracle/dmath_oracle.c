/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's hot-path
 * arithmetic, used as the checker by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg.  Never linked into the product.
 *
 * Pinned against the reference itself: tests/test_oracle.py checks every
 * function below bit-for-bit against golden vectors produced by the
 * reference (tests/golden/make_golden.py -> oracle/_ref/libgridgemm_ref.so).
 * Build: -O2 -ffp-contract=off (no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* splitmix64 finalizer, gridgemm/common.hpp:107-112 */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* two-argument mix, gridgemm/common.hpp:114-116 */
uint64_t orc_mix64_2(uint64_t a, uint64_t b) { return orc_mix64(a ^ orc_mix64(b)); }

/* FNV-1a 64, gridgemm/common.hpp:83-103 */
uint64_t orc_fnv1a(const void* data, int64_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 14695981039346656037ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

/* matrix seed, gridgemm/session.hpp:142 */
uint64_t orc_matrix_seed(uint64_t root_seed, uint64_t matrix_id) {
  return orc_mix64_2(root_seed, matrix_id);
}

/* WorkerContext::fill_seeded, gridgemm/runtime_types.hpp:208-218 with
 * u64_to_unit_double, common.hpp:119-121 */
void orc_fill_block(float* out, int64_t rows, int64_t cols, uint64_t matrix_seed, int brow,
                    int bcol) {
  const uint64_t key =
      orc_mix64_2(matrix_seed, ((uint64_t)(uint32_t)brow << 32) | (uint32_t)bcol);
  const int64_t n = rows * cols;
  for (int64_t e = 0; e < n; ++e) {
    const double u = (double)(orc_mix64_2(key, (uint64_t)e) >> 11) * 0x1.0p-53;
    out[e] = (float)(2.0 * u - 1.0);
  }
}

/* Elements [e0, e0+count) of the same block stream (row-major within the
 * block), so a large block can be filled by several threads. */
void orc_fill_range(float* out, int64_t e0, int64_t count, uint64_t matrix_seed, int brow,
                    int bcol) {
  const uint64_t key =
      orc_mix64_2(matrix_seed, ((uint64_t)(uint32_t)brow << 32) | (uint32_t)bcol);
  for (int64_t i = 0; i < count; ++i) {
    const double u = (double)(orc_mix64_2(key, (uint64_t)(e0 + i)) >> 11) * 0x1.0p-53;
    out[i] = (float)(2.0 * u - 1.0);
  }
}

/* detail::checkerboard_dims, gridgemm/layout.hpp:100-105 */
void orc_checkerboard_dims(int workers, int* pr, int* pc) {
  int r = 1;
  for (int d = 1; (int64_t)d * d <= workers; ++d)
    if (workers % d == 0) r = d;
  *pr = r;
  *pc = workers / r;
}

/* LayoutSpec::owner for the four regular kinds, gridgemm/layout.hpp:122-139
 * (grid already clamped: nbr x nbc blocks) */
int orc_owner(int kind, int nbr, int nbc, int workers, int row, int col) {
  switch (kind) {
    case 0: return (int)(((int64_t)row * workers) / nbr); /* RowBlocks1D */
    case 1: return (int)(((int64_t)col * workers) / nbc); /* ColBlocks1D */
    case 2: return row % workers;                          /* RowCyclic1D */
    case 3: {                                              /* Checkerboard2D */
      int pr, pc;
      orc_checkerboard_dims(workers, &pr, &pc);
      return (row % pr) * pc + (col % pc);
    }
  }
  return -1;
}

/* detail::gemm_typed<float>, gridgemm/kernels.hpp:48-75: i, j, k ascending,
 * unfused fp32 multiply then add; alpha/beta narrowed to float; beta == 0
 * never reads C. */
void orc_local_gemm_f32(double alpha, const float* a, int64_t ar, int64_t ac, int ta,
                        const float* b, int64_t br, int64_t bc, int tb, double beta, float* c) {
  const int64_t m = ta ? ac : ar, kk = ta ? ar : ac, n = tb ? br : bc;
  const float al = (float)alpha, be = (float)beta;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (int64_t k = 0; k < kk; ++k) {
        const float av = ta ? a[k * ac + i] : a[i * ac + k];
        const float bv = tb ? b[j * bc + k] : b[k * bc + j];
        const float p = av * bv;
        acc = acc + p;
      }
      float out = al * acc;
      if (beta != 0.0) {
        const float q = be * c[i * n + j];
        out = out + q;
      }
      c[i * n + j] = out;
    }
}

/* relative Frobenius error, tests/oracle.hpp:90-98 */
double orc_rel_frobenius(const float* got, const float* want, int64_t n) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = (double)got[i] - (double)want[i];
    num += d * d;
    den += (double)want[i] * (double)want[i];
  }
  return den == 0 ? sqrt(num) : sqrt(num / den);
}
