// Forward dyadic projection by the Fast Hough Transform (NEXT-1):
//   S[f][t][s] = sum_y G_f[y][s - N + d_t(y)]          PAPER.md:199-202 (Eq.17),
// the four family views G_f of Eq.16 (reading R4), dyadic
// patterns d_t(y) of §4.4 (reading R3), positive shift direction:
//   R_2h[b][t'][u] = R_h[2b][t'/2][u] + R_h[2b+1][t'/2][u + ceil(t'/2)]
// with row y of G_f placed at columns [N, 2N) of a 2N-wide row.  Additions only.
//
// Same two-pass split as the back projection:
//   k_fwd_a: k1 levels on each block b of H = 2^k1 rows of G_f (read straight from
//            the image: row / mirrored row / column / mirrored column), output
//            R_A[sf][b][t'][u] compactly for u in [N - H, 2N) (zero left of it);
//   k_fwd_b: per channel c = t >> m: rows b of R_A[sf][b][c][v + c*b] (the
//            pre-shift, addressing only), m levels, out[sf][c*NB + t_lo][s].
// Both levels loops run in shared memory, one warp per row, lanes over columns
// (coalesced, conflict-free); the ping-pong buffers hold the tile plus the
// right halo the positive shifts read (H - 1, resp. NB - 1 columns).
#include <algorithm>
#include <cstdlib>

#include "fbp_internal.h"

namespace fbp {
namespace {

constexpr int FNT = 256;          // threads per CTA

// FHT levels over R rows x TW = XO + R columns (pitch P), ping-pong a -> b; only
// the columns [0, XO + R - hout) that the remaining levels (and the XO outputs)
// read are computed, and every read lies inside what the previous pass computed.  Level h -> 2h: row blk*2h + tt reads
// rows 2blk*h + tt/2 (at u) and (2blk+1)*h + tt/2 (at u + ceil(tt/2)).
// Two levels per pass (radix 4) where possible: outputs tt = 4 t2 + k of block j
// (rows A0..A3 = sub-blocks 4j..4j+3, row t2 each) are
//   ((A0[u] + A1[u + s1]) + (A2[u + s2] + A3[u + s2 + s1])),
//   s1 = ceil(t1/2), t1 = tt >> 1, s2 = ceil(tt/2)
// -- the recursion's own addition order, from 10 loads for the 4 rows.
// Returns the buffer holding the result.
__device__ float* fwd_levels(float* a, float* b, int R, int TW, int P, int XO) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lg = 0;
  while ((1 << lg) < R) ++lg;
  int h = 1;
  // no bounds guard: a pass from blocks of hin rows to blocks of hout rows computes
  // columns < XO + R - hout and reads at most hout - hin further right, i.e. below
  // XO + R - hin, the width the previous pass (or the fill, TW = XO + R) computed
  auto ld = [&](const float* row, int u) { return row[u]; };
  if (lg & 1) {                                       // one radix-2 level first
    const int need = min(TW, XO + R - 2);
    for (int r = warp; r < R; r += FNT / 32) {
      const int blk = r >> 1, tt = r & 1;
      const float* r0 = a + (2 * blk) * P;
      const float* r1 = a + (2 * blk + 1) * P + tt;
      float* o = b + r * P;
      for (int u = lane; u < need; u += 32) o[u] = r0[u] + r1[u];
    }
    __syncthreads();
    float* t = a;
    a = b;
    b = t;
    h = 2;
  }
  for (; h < R; h *= 4) {
    const int need = min(TW, XO + R - 4 * h);
    const int ngrp = R / 4;                            // (block j, t2) pairs
    for (int gi = warp; gi < ngrp; gi += FNT / 32) {
      const int j = gi / h, t2 = gi - j * h;
      const float* A0 = a + (4 * j * h + t2) * P;
      const float* A1 = A0 + h * P;
      const float* A2 = A1 + h * P;
      const float* A3 = A2 + h * P;
      float* o = b + (4 * j * h + 4 * t2) * P;
      for (int u = lane; u < need; u += 32) {
        const float x0 = A0[u];
        const float q0a = x0 + ld(A1, u + t2), q0b = x0 + ld(A1, u + t2 + 1);
        const float a2a = ld(A2, u + 2 * t2), a2b = ld(A2, u + 2 * t2 + 1), a2c = ld(A2, u + 2 * t2 + 2);
        o[u] = q0a + (a2a + ld(A3, u + 3 * t2));
        o[P + u] = q0a + (a2b + ld(A3, u + 3 * t2 + 1));
        o[2 * P + u] = q0b + (a2b + ld(A3, u + 3 * t2 + 2));
        o[3 * P + u] = q0b + (a2c + ld(A3, u + 3 * t2 + 3));
      }
    }
    __syncthreads();
    float* t = a;
    a = b;
    b = t;
  }
  return a;
}

// grid (u-tiles, NB, slices*4); tile columns u in [u0, u0 + TW), u0 = N - H + tile*FXA
__global__ void __launch_bounds__(FNT) k_fwd_a(const float* __restrict__ img, float* __restrict__ RA, int N,
                                               int H, int NB, int FXA) {
  extern __shared__ float sm[];
  const int TW = FXA + H, P = TW + 1;               // odd pitch: column-wise fills conflict-free
  float* A = sm;
  float* B = sm + H * P;
  const int sf = blockIdx.z, f = sf & 3, b = blockIdx.y;
  const int u0 = N - H + blockIdx.x * FXA;
  const float* im = img + (long long)(sf >> 2) * N * N;
  const int y0 = b * H;
  if (f < 2) {
    // G_0[y][x] = img[y][x], G_1[y][x] = img[y][N-1-x]: rows, lanes over x
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < H; j += FNT / 32) {
      const float* row = im + (long long)(y0 + j) * N;
      for (int ul = lane; ul < TW; ul += 32) {
        const int x = u0 + ul - N;
        float v = 0.f;
        if (x >= 0 && x < N) v = row[f == 0 ? x : N - 1 - x];
        A[j * P + ul] = v;
      }
    }
  } else {
    // G_2[y][x] = img[x][y], G_3[y][x] = img[N-1-x][y]: lanes over y (contiguous in img)
    int lh = 0;
    while ((1 << lh) < H) ++lh;
    for (int e = threadIdx.x; e < H * TW; e += FNT) {
      const int ul = e >> lh, j = e & (H - 1);
      const int x = u0 + ul - N;
      float v = 0.f;
      if (x >= 0 && x < N) v = im[(long long)(f == 2 ? x : N - 1 - x) * N + y0 + j];
      A[j * P + ul] = v;
    }
  }
  __syncthreads();
  const float* res = fwd_levels(A, B, H, TW, P, FXA);
  const int WRF = N + H;
  float* out = RA + ((long long)sf * NB + b) * H * WRF;
  const int j0 = blockIdx.x * FXA;                  // compact column of u0
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < H; t += FNT / 32)
    for (int ul = lane; ul < FXA; ul += 32)
      if (j0 + ul < WRF) out[(long long)t * WRF + j0 + ul] = res[t * P + ul];
}

// grid (s-tiles, H channels, slices*4)
__global__ void __launch_bounds__(FNT) k_fwd_b(const float* __restrict__ RA, float* __restrict__ lin, int N,
                                               int H, int NB, int FXB) {
  extern __shared__ float sm[];
  const int TW = FXB + NB, P = TW + 1;
  float* A = sm;
  float* B = sm + NB * P;
  const int sf = blockIdx.z, c = blockIdx.y;
  const int s0 = blockIdx.x * FXB;
  const int WRF = N + H;
  const float* in = RA + (long long)sf * NB * H * WRF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = warp; b < NB; b += FNT / 32) {
    // G_c[b][v] = R_A[b][c][v + c*b] at compact column v + c*b - (N - H)
    const float* row = in + ((long long)b * H + c) * WRF;
    const int off = c * b - (N - H);
    for (int vl = lane; vl < TW; vl += 32) {
      const int jc = s0 + vl + off;
      A[b * P + vl] = (jc >= 0 && jc < WRF) ? row[jc] : 0.f;
    }
  }
  __syncthreads();
  const float* res = fwd_levels(A, B, NB, TW, P, FXB);
  const int W = 2 * N;
  float* out = lin + ((long long)sf * N + (long long)c * NB) * W;
  for (int t = warp; t < NB; t += FNT / 32)
    for (int vl = lane; vl < FXB; vl += 32)
      if (s0 + vl < W) out[(long long)t * W + s0 + vl] = res[t * P + vl];
}

}  // namespace

size_t fwd_workspace_floats(const Geometry& g) { return (size_t)4 * g.NB * g.H * (g.N + g.H); }

// output columns per tile (a multiple of 32): wide enough that the right halo
// (H - 1, resp. NB - 1 columns) is a small overhead, narrow enough for >= 2 CTAs/SM
static int fwd_tile(int rows, int dflt, const char* env) {
  int x = dflt;                                     // measured best at N = 2048 (r01)
#if FBP_DEV_MASK
  if (const char* ev = std::getenv(env)) x = std::max(32, std::atoi(ev) / 32 * 32);   // developer builds only
#else
  (void)env;
#endif
  while (x > 32 && (size_t)2 * rows * (x + rows + 1) * sizeof(float) > (size_t)227 * 1024) x -= 32;
  return x;
}

cudaError_t launch_fwd_a(const float* img, float* RA, int slices, const Geometry& g, cudaStream_t st,
                         int* launches) {
  const int N = g.N, H = g.H, NB = g.NB;
  const int FXA = fwd_tile(H, 64, "FBP_FXA");
  const size_t smem = (size_t)2 * H * (FXA + H + 1) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((N + H + FXA - 1) / FXA, NB, 4 * slices);
  k_fwd_a<<<grid, FNT, smem, st>>>(img, RA, N, H, NB, FXA);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fwd_b(const float* RA, float* lin, int slices, const Geometry& g, cudaStream_t st,
                         int* launches) {
  const int N = g.N, H = g.H, NB = g.NB;
  const int FXB = fwd_tile(NB, NB <= 32 ? 256 : 128, "FBP_FXB");
  const size_t smem = (size_t)2 * NB * (FXB + NB + 1) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((2 * N + FXB - 1) / FXB, H, 4 * slices);
  k_fwd_b<<<grid, FNT, smem, st>>>(RA, lin, N, H, NB, FXB);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
