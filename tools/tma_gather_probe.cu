// tma_gather_probe.cu -- standalone check of TMA tile::gather4 on sm_100a:
// gathers rows of a [n x 4] fp64 tensor (32-byte node records) into shared
// memory by arbitrary row index and compares with a plain gather.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s), "r"(bytes));
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* m, unsigned phase) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(m));
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(s), "r"(phase));
  return ok != 0;
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, unsigned long long* m,
                                            int r0, int r1, int r2, int r3) {
  const unsigned sd = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned sm = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sd),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(sm)
      : "memory");
}

__global__ void k_probe(const __grid_constant__ CUtensorMap map, const int* idx, int n,
                        double* out) {
  __shared__ __align__(128) double tab[1024][4];
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int groups = (n + 3) / 4;
  if (threadIdx.x == 0) mbar_expect_tx(&mbar, groups * 128);
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    int r[4];
    for (int q = 0; q < 4; ++q) r[q] = idx[min(4 * g + q, n - 1)];
    tma_gather4(&tab[4 * g][0], &map, &mbar, r[0], r[1], r[2], r[3]);
  }
  while (!mbar_try_wait(&mbar, 0)) {
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int c = 0; c < 4; ++c) out[4 * i + c] = tab[i][c];
}

int main() {
  const int nv = 1 << 20, n = 1000;
  std::vector<double> x(4 * static_cast<size_t>(nv));
  for (size_t i = 0; i < x.size(); ++i) x[i] = static_cast<double>(i) * 0.5;
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = static_cast<int>((1103515245u * i + 12345u) % nv);
  double* dx;
  int* didx;
  double* dout;
  CK(cudaMalloc(&dx, x.size() * 8));
  CK(cudaMalloc(&didx, n * 4));
  CK(cudaMalloc(&dout, 4 * n * 8));
  CK(cudaMemcpy(dx, x.data(), x.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, idx.data(), n * 4, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                             cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t gdim[2] = {4, static_cast<cuuint64_t>(nv)};
  cuuint64_t gstride[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dx, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode result %d\n", static_cast<int>(r));
  if (r != CUDA_SUCCESS) return 1;
  k_probe<<<1, 128>>>(map, didx, n, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<double> out(4 * n);
  CK(cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 4; ++c)
      if (out[4 * i + c] != x[4 * static_cast<size_t>(idx[i]) + c]) ++bad;
  std::printf("gather4 probe: %d mismatches of %d\n", bad, 4 * n);
  return bad != 0;
}
