// Developer microtest: TMA tensor LOAD at element (non-16-byte-aligned) column coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
extern __shared__ float sm[];
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int r0, float* out, int X) {
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(X * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(reinterpret_cast<unsigned long long>(&m)), "r"(c0), "r"(r0), "r"(b) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(b));
  for (int i = threadIdx.x; i < X; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  int c0 = atoi(argv[1]), X = 64, W = 2144, rows = 16;
  float *g, *o; cudaMalloc(&g, W * rows * 4); cudaMalloc(&o, X * 4);
  float* h = (float*)malloc(W * rows * 4);
  for (int i = 0; i < W * rows; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, W * rows * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t bx[2] = {(cuuint32_t)X, 1}, es[2] = {1, 1};
  cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 64, X * 4>>>(m, c0, 3, o, X);
  cudaError_t e = cudaDeviceSynchronize();
  float r[64];
  cudaMemcpy(r, o, X * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < X; ++i) {
    int col = c0 + i;
    float want = (col >= 0 && col < W) ? (float)(3 * W + col) : 0.f;
    if (r[i] != want) ++bad;
  }
  printf("load c0 %d: %s bad %d first %g\n", c0, cudaGetErrorString(e), bad, r[0]);
  return 0;
}
