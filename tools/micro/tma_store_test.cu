// Developer microtest: TMA tensor stores with in-bounds / negative / beyond-end
// coordinates and smem source alignments.  nvcc -arch=sm_100a tma_store_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
extern __shared__ float sm[];
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int r0, int soff) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (float)i;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned src = (unsigned)__cvta_generic_to_shared(sm + soff);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n"
                 ::"l"(reinterpret_cast<unsigned long long>(&m)), "r"(src), "r"(c0), "r"(r0) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}
int main(int argc, char** argv) {
  int W = 528, rows = 64, box = argc > 1 ? atoi(argv[1]) : 64;
  int c0 = argc > 2 ? atoi(argv[2]) : 0, soff = argc > 3 ? atoi(argv[3]) : 0;
  float* g; cudaMalloc(&g, W * rows * 4); cudaMemset(g, 0, W * rows * 4);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t bx[2] = {(cuuint32_t)box, 1}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, bx, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128, 8192>>>(m, c0, 3, soff);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(W * rows);
  cudaMemcpy(h.data(), g, W * rows * 4, cudaMemcpyDeviceToHost);
  int nz = 0, first = -1;
  for (int i = 0; i < W; ++i) if (h[3 * W + i] != 0.f) { ++nz; if (first < 0) first = i; }
  printf("box %d c0 %d soff %d: encode %d, kernel %s, nonzero %d first col %d val %g\n", box, c0, soff, (int)r,
         cudaGetErrorString(e), nz, first, first >= 0 ? h[3 * W + first] : -1.f);
  return 0;
}
