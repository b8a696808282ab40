// GEMM-kernel time vs the majorness of op(B)'s planes (K-major / MN-major),
// per plane kind (tf32 hi vs bf16 hi/lo), at N^3 (default 16384), CUDA events
// around the tf32x3_gemm launches only.  Links libdmath_b200.so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1604_01416_b200/csrc \
//     tools/micro/mn_probe.cu -Lpaper_1604_01416_b200/lib -ldmath_b200 -o /tmp/mn_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "kernels/tf32x3_gemm.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 16384;
  const size_t E = static_cast<size_t>(N) * N;
  float *A, *B, *C, *ahi, *bhiK, *bhiM, *scratch;
  char *a16, *b16K, *b16M;
  CK(cudaMalloc(&A, E * 4)); CK(cudaMalloc(&B, E * 4)); CK(cudaMalloc(&C, E * 4));
  CK(cudaMalloc(&ahi, E * 4)); CK(cudaMalloc(&bhiK, E * 4)); CK(cudaMalloc(&bhiM, E * 4));
  CK(cudaMalloc(&scratch, E * 4));
  CK(cudaMalloc(&a16, E * 4)); CK(cudaMalloc(&b16K, E * 4)); CK(cudaMalloc(&b16M, E * 4));
  CK(dm::fill_seeded(A, 1, E, 1, 0)); CK(dm::fill_seeded(B, 1, E, 2, 0));
  // A: K-major (row-major A is M x K); B row-major K x N:
  //   K-major planes = transposing split, MN-major planes = direct split
  CK(dm::split_tf32(A, 0, N, 0, N, N, ahi, nullptr, N, a16, a16 + E * 2, N, 0));
  CK(dm::split_tf32(B, 0, N, 1, N, N, bhiK, nullptr, N, b16K, b16K + E * 2, N, 0));
  CK(dm::split_tf32(B, 0, N, 0, N, N, bhiM, nullptr, N, b16M, b16M + E * 2, N, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const char* names[4] = {"hi K  / bf16 K ", "hi MN / bf16 MN", "hi K  / bf16 MN", "hi MN / bf16 K "};
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 4; ++v) {
      const bool hm = v == 1 || v == 3, bm = v == 1 || v == 2;
      dm::Tf32x3Args a;
      a.mode = dm::kModeMixed;
      a.a_hi = ahi; a.a_hi16 = a16; a.a_lo16 = a16 + E * 2; a.lda = a.lda16 = N;
      a.b_hi = hm ? bhiM : bhiK;
      a.b_hi16 = bm ? b16M : b16K; a.b_lo16 = (bm ? b16M : b16K) + E * 2; a.ldb = a.ldb16 = N;
      a.b_mn = hm; a.b_mn16 = bm;
      a.c = C; a.ldc = N; a.m = a.n = a.k = N;
      CK(dm::tf32x3_gemm(a, 0));
      CK(cudaEventRecord(e0));
      const int reps = 3;
      for (int r = 0; r < reps; ++r) CK(dm::tf32x3_gemm(a, 0));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= reps;
      // checksum of a corner against the all-K-major result
      float c[4];
      CK(cudaMemcpy(c, C, 16, cudaMemcpyDeviceToHost));
      printf("mixed B planes %s : %.2f ms  %.1f TFLOP/s  C[0,0..3]=%.6f %.6f %.6f %.6f\n", names[v], ms,
             2.0 * N * N * N / ms / 1e9, c[0], c[1], c[2], c[3]);
    }
  // 3xTF32: hi/lo both K or both MN
  for (int v = 0; v < 2; ++v) {
    dm::Tf32x3Args a;
    a.mode = dm::kModeTf32x3;
    a.a_hi = ahi; a.a_lo = scratch; a.lda = N;
    a.b_hi = v ? bhiM : bhiK; a.b_lo = v ? bhiM : bhiK; a.ldb = N; a.b_mn = v;
    a.c = C; a.ldc = N; a.m = a.n = a.k = N;
    CK(dm::tf32x3_gemm(a, 0));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 3; ++r) CK(dm::tf32x3_gemm(a, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("3xtf32 B planes %s : %.2f ms  %.1f TFLOP/s\n", v ? "MN" : "K ", ms / 3, 2.0 * N * N * N / (ms / 3) / 1e9);
  }
  return 0;
}
