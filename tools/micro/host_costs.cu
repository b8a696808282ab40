// Host-side cost of the CUDA calls a GEMM command issues (microseconds each).
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

template <class F>
double us(F f, int n = 2000) {
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) f();
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
}
__global__ void noop() {}

int main() {
  cudaFree(0);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  printf("cudaStreamSynchronize(idle)   %.2f us\n", us([&] { cudaStreamSynchronize(s); }));
  printf("cudaStreamQuery(idle)         %.2f us\n", us([&] { cudaStreamQuery(s); }));
  printf("cudaEventCreate+Destroy       %.2f us\n", us([&] {
           cudaEvent_t x;
           cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
           cudaEventDestroy(x);
         }));
  printf("cudaEventRecord               %.2f us\n", us([&] { cudaEventRecord(e, s); }));
  printf("cudaStreamWaitEvent           %.2f us\n", us([&] { cudaStreamWaitEvent(s2, e, 0); }));
  printf("kernel launch (noop)          %.2f us\n", us([&] { noop<<<1, 32, 0, s>>>(); }));
  cudaStreamSynchronize(s);
  printf("launch+sync (noop)            %.2f us\n", us([&] { noop<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }));
  int dev;
  cudaGetDevice(&dev);
  printf("cudaSetDevice(same)           %.2f us\n", us([&] { cudaSetDevice(dev); }));
  printf("cudaGetDevice                 %.2f us\n", us([&] { cudaGetDevice(&dev); }));
  void* p = nullptr;
  cudaMalloc(&p, 1 << 20);
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fp);
  CUtensorMap m;
  cuuint64_t dims[2] = {256, 256}, strides[1] = {1024};
  cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  printf("cuTensorMapEncodeTiled        %.2f us\n", us([&] {
           enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
         }));
  printf("cudaMemsetAsync(16B)          %.2f us\n", us([&] { cudaMemsetAsync(p, 0, 16, s); }));
  cudaStreamSynchronize(s);
  return 0;
}
