// Developer microtest: per-thread TMA tensor stores (64 threads, one row each),
// box X x 1, as the sweep kernel issues them.  nvcc -arch=sm_100a ... -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
extern __shared__ float sm[];
__global__ void k(const __grid_constant__ CUtensorMap m, int X, int c0base, int mode, int nthr) {
  for (int i = threadIdx.x; i < 64 * X; i += blockDim.x) sm[i] = (float)(i + 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  for (int rep = 0; rep < 3; ++rep) {
    if ((mode == 0 && threadIdx.x < nthr) || (mode == 1 && threadIdx.x == 0)) {
      for (int r = (mode == 0 ? threadIdx.x : 0); r < (mode == 0 ? threadIdx.x + 1 : nthr); ++r) {
        unsigned src = (unsigned)__cvta_generic_to_shared(sm + r * X);
        int c0 = c0base + 3 * r;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n"
                     ::"l"(reinterpret_cast<unsigned long long>(&m)), "r"(src), "r"(c0), "r"(r) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    if (threadIdx.x < 64) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x < 64) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
int main(int argc, char** argv) {
  int X = atoi(argv[1]), c0 = atoi(argv[2]), mode = atoi(argv[3]), nthr = atoi(argv[4]);
  int W = 2144, rows = 4096;
  float* g; cudaMalloc(&g, (size_t)W * rows * 4); cudaMemset(g, 0, (size_t)W * rows * 4);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t bx[2] = {(cuuint32_t)X, 1}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, bx, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128, 64 * X * 4>>>(m, X, c0, mode, nthr);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h((size_t)W * rows);
  cudaMemcpy(h.data(), g, (size_t)W * rows * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < nthr && e == cudaSuccess; ++rr)
    for (int i = 0; i < X; ++i) {
      int col = c0 + 3 * rr + i;
      if (col < W && h[(size_t)rr * W + col] != (float)(rr * X + i + 1)) ++bad;
    }
  printf("X %d c0 %d mode %d nthr %d: encode %d kernel %s bad %d\n", X, c0, mode, nthr, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
