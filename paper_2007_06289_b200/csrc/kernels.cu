// sm_100a kernels of the fast-FBP hot path (arXiv 2007.06289).
//
//   K1 k_iir_rows      symmetric recursive ramp filter, one warp per linogram row,
//                      exact chunked scan of the recursion across the warp's lanes
//                      (§3 Eq.12-13).
//   K2 k_fht_pass_a    FHT back-projection levels 1..k1 on blocks of 2^k1 rows
//                      (§4.4, 251-260 §4.5 Eq.19-21), negative
//                      shift direction, additions only.
//   K3 k_fht_pass_b    FHT levels k1+1..n per channel with the channel pre-shift,
//                      plus the family-pair sum and weight of Eq.22.
//
// Level split: with y = c*2^m + r and t = b*2^k1 + r_t,
//   d_y(t) = c*b + d^(m)_r(b) + d^(k1)_c(r_t),
// so pass A is a k1-level FHT of each 2^k1-row block (shift c), and pass B, for a
// channel c, is an m-level FHT of the rows G_c[b][v] = R_A[b][c][v - c*b].
#include "fbp_internal.h"

#include <cuda_runtime.h>

namespace fbp {

// ---------------------------------------------------------------------------
// K1: symmetric IIR, one warp per row.
// ---------------------------------------------------------------------------
// Row staged in shared memory with one pad word per lane chunk (idx = s + s/L)
// so that lane-chunked sequential reads are bank-conflict free.
// Per direction: (1) zero-state sweep over the lane's chunk -> end state v;
// (2) inclusive scan c_i = A^L c_{i-1} + v_i over lanes (Kogge-Stone with
// P[k] = A^(L 2^k)); (3) re-sweep from the exact carry-in, writing the output.
template <int QM>
__device__ __forceinline__ void scan_carry_up(float (&c)[QM], const IirParams& p, int lane) {
#pragma unroll
  for (int k = 0; k < kScanSteps; ++k) {
    const int off = 1 << k;
    float o[QM];
#pragma unroll
    for (int j = 0; j < QM; ++j) o[j] = __shfl_up_sync(0xffffffffu, c[j], off);
    if (lane >= off) {
#pragma unroll
      for (int i = 0; i < QM; ++i) {
        float acc = c[i];
#pragma unroll
        for (int j = 0; j < QM; ++j) acc = fmaf(p.P[k][i * kMaxOrder + j], o[j], acc);
        c[i] = acc;
      }
    }
  }
}

template <int QM>
__device__ __forceinline__ void scan_carry_down(float (&c)[QM], const IirParams& p, int lane) {
#pragma unroll
  for (int k = 0; k < kScanSteps; ++k) {
    const int off = 1 << k;
    float o[QM];
#pragma unroll
    for (int j = 0; j < QM; ++j) o[j] = __shfl_down_sync(0xffffffffu, c[j], off);
    if (lane + off < 32) {
#pragma unroll
      for (int i = 0; i < QM; ++i) {
        float acc = c[i];
#pragma unroll
        for (int j = 0; j < QM; ++j) acc = fmaf(p.P[k][i * kMaxOrder + j], o[j], acc);
        c[i] = acc;
      }
    }
  }
}

// Causal pass over samples [start, start+len) of the staged row X.
//   u[n] = beta x[n] + sum_k c_k D[n-k],   D[n] = x[n] - x[n-1]   (= sum_k b_k x[n-k])
//   y[n] = u[n] - sum_k a_k y[n-k]                                  (Eq.13, upper sign)
// yq holds (y[n-1], y[n-2], ...) on entry (carry) and the end state on exit.
// If Y != nullptr the outputs are stored (WRITE) / accumulated.
template <int QM, bool WRITE>
__device__ __forceinline__ void causal_sweep(const float* X, float* Y, int start, int len, int L,
                                             const IirParams& p, float (&yq)[QM]) {
  if (len <= 0) return;  // idle lane (W < 32): end state stays as given
  auto idx = [L](int s) { return s + s / L; };
  // Difference history dh[k] = D[n-1-k] at the first sample n = start.
  float xm[QM + 1];  // x[start-1-k], k = 0..QM
#pragma unroll
  for (int k = 0; k <= QM; ++k) {
    const int s = start - 1 - k;
    xm[k] = (s >= 0) ? X[idx(s)] : 0.0f;
  }
  float dh[QM];
#pragma unroll
  for (int k = 0; k < QM; ++k) dh[k] = xm[k] - xm[k + 1];
  float xprev = xm[0];
  for (int i = 0; i < len; ++i) {
    const int s = start + i;
    const float x = X[idx(s)];
    const float d = x - xprev;
    xprev = x;
    // feedforward: beta x + c0 d + c1 D[n-1] + ...
    float u = p.beta * x;
    u = fmaf(p.c[0], d, u);
#pragma unroll
    for (int k = 1; k < QM; ++k) u = fmaf(p.c[k], dh[k - 1], u);
#pragma unroll
    for (int k = QM - 1; k > 0; --k) dh[k] = dh[k - 1];
    dh[0] = d;
    // feedback, y[n-1] last (shortest dependency chain)
    float y = u;
#pragma unroll
    for (int k = QM - 1; k >= 0; --k) y = fmaf(-p.a[k], yq[k], y);
#pragma unroll
    for (int k = QM - 1; k > 0; --k) yq[k] = yq[k - 1];
    yq[0] = y;
    if (WRITE) Y[idx(s)] = y;
  }
}

// Anticausal pass over [start, start+len), right to left (Eq.13 lower sign):
//   u[n] = beta x[n] + sum_k c_k E[n+k],   E[n] = x[n] - x[n+1]   (= sum_k b_k x[n+k])
//   y[n] = u[n] - sum_k a_k y[n+k]
// yq holds (y[n+1], y[n+2], ...).  WRITE: Y[n] += y (Y already holds the causal part).
template <int QM, bool WRITE>
__device__ __forceinline__ void anticausal_sweep(const float* X, float* Y, int start, int len,
                                                 int L, int W, const IirParams& p,
                                                 float (&yq)[QM]) {
  if (len <= 0) return;
  auto idx = [L](int s) { return s + s / L; };
  const int end = start + len;  // first sample after the chunk
  float xp[QM + 1];             // x[end+k], k = 0..QM
#pragma unroll
  for (int k = 0; k <= QM; ++k) {
    const int s = end + k;
    xp[k] = (s < W) ? X[idx(s)] : 0.0f;
  }
  float eh[QM];  // E[n+1+k] at the first processed sample n = end-1
#pragma unroll
  for (int k = 0; k < QM; ++k) eh[k] = xp[k] - xp[k + 1];
  float xnext = xp[0];
  for (int i = len - 1; i >= 0; --i) {
    const int s = start + i;
    const float x = X[idx(s)];
    const float e = x - xnext;
    xnext = x;
    float u = p.beta * x;
    u = fmaf(p.c[0], e, u);
#pragma unroll
    for (int k = 1; k < QM; ++k) u = fmaf(p.c[k], eh[k - 1], u);
#pragma unroll
    for (int k = QM - 1; k > 0; --k) eh[k] = eh[k - 1];
    eh[0] = e;
    float y = u;
#pragma unroll
    for (int k = QM - 1; k >= 0; --k) y = fmaf(-p.a[k], yq[k], y);
#pragma unroll
    for (int k = QM - 1; k > 0; --k) yq[k] = yq[k - 1];
    yq[0] = y;
    if (WRITE) Y[idx(s)] += y;
  }
}

template <int QM>
__global__ void __launch_bounds__(256) k_iir_rows(const float* in,  // may alias out
                                                  float* out, long long rows, int W,
                                                  int L, int warps_per_cta, IirParams p) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * warps_per_cta + warp;
  if (row >= rows) return;  // warp-uniform
  const int padded = W + 32;
  float* X = smem + (size_t)warp * 2 * padded;
  float* Y = X + padded;
  const float* src = in + row * (long long)W;
  auto idx = [L](int s) { return s + s / L; };
  for (int s = lane; s < W; s += 32) X[idx(s)] = src[s];
  __syncwarp();

  const int start = lane * L;
  const int len = (start < W) ? L : 0;

  // ---- causal ----
  float c[QM];
#pragma unroll
  for (int j = 0; j < QM; ++j) c[j] = 0.0f;
  causal_sweep<QM, false>(X, nullptr, start, len, L, p, c);
  scan_carry_up<QM>(c, p, lane);
  float cin[QM];
#pragma unroll
  for (int j = 0; j < QM; ++j) {
    const float v = __shfl_up_sync(0xffffffffu, c[j], 1);
    cin[j] = (lane == 0) ? 0.0f : v;
  }
  causal_sweep<QM, true>(X, Y, start, len, L, p, cin);

  // ---- anticausal ----
#pragma unroll
  for (int j = 0; j < QM; ++j) c[j] = 0.0f;
  anticausal_sweep<QM, false>(X, nullptr, start, len, L, W, p, c);
  scan_carry_down<QM>(c, p, lane);
#pragma unroll
  for (int j = 0; j < QM; ++j) {
    const float v = __shfl_down_sync(0xffffffffu, c[j], 1);
    cin[j] = (lane == 31) ? 0.0f : v;
  }
  __syncwarp();
  anticausal_sweep<QM, true>(X, Y, start, len, L, W, p, cin);
  __syncwarp();

  float* dst = out + row * (long long)W;
  for (int s = lane; s < W; s += 32) dst[s] = Y[idx(s)];
}

cudaError_t launch_iir_rows(const float* in, float* out, long long rows, const Geometry& g,
                            const IirParams& p, cudaStream_t st, int* launches) {
  if (rows <= 0) return cudaSuccess;
  const size_t per_warp = (size_t)2 * (g.W + 32) * sizeof(float);
  int wpc = (int)((96 * 1024) / per_warp);
  if (wpc < 1) wpc = 1;
  if (wpc > 8) wpc = 8;
  const size_t smem = per_warp * wpc;
  const long long grid = (rows + wpc - 1) / wpc;
  cudaError_t e;
  if (g.iir_qm == 3) {
    e = cudaFuncSetAttribute(k_iir_rows<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_iir_rows<3><<<(unsigned)grid, 32 * wpc, smem, st>>>(in, out, rows, g.W, g.L, wpc, p);
  } else {
    e = cudaFuncSetAttribute(k_iir_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_iir_rows<8><<<(unsigned)grid, 32 * wpc, smem, st>>>(in, out, rows, g.W, g.L, wpc, p);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FHT levels in shared memory (negative direction), natural row order.
// in/out: `rows` x P tiles; block of height 2h at level with input height h:
//   out[blk + y'][j] = in[blk + y'/2][j] + in[blk + h + y'/2][j - ceil(y'/2)]
// (columns j - s < 0 read as 0: they lie left of the tile and only feed
// columns that are discarded).  Returns the buffer holding the result.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float* fht_levels_smem(float* a, float* b, int rows, int P,
                                                  int levels) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int lvl = 0; lvl < levels; ++lvl) {
    const int h = 1 << lvl;
    for (int y = warp; y < rows; y += nwarps) {
      const int blk = y & ~(2 * h - 1);
      const int yp = y - blk;
      const int lo = yp >> 1;
      const int sh = (yp + 1) >> 1;
      const float* ra = a + (size_t)(blk + lo) * P;
      const float* rb = a + (size_t)(blk + h + lo) * P;
      float* ro = b + (size_t)y * P;
      for (int j = lane; j < P; j += 32) {
        const float vb = (j >= sh) ? rb[j - sh] : 0.0f;
        ro[j] = ra[j] + vb;
      }
    }
    __syncthreads();
    float* t = a;
    a = b;
    b = t;
  }
  return a;
}

// ---------------------------------------------------------------------------
// K2: pass A.  grid (u-tiles, NB blocks, slices*4); block 256.
// Tile: H rows (t = b*H + r) x columns u in [u0-H+1, u0+XA).  After k1 levels row
// c holds R_A[b][c][u] = sum_r F[b*H+r][u - d^(k1)_c(r)].  Stored compactly:
// R[sf][b][c][j'], j' = u + c*b - N + NB, only where pass B reads it,
// u in [N - b(c+1), 2N - c*b).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fht_pass_a(const float* __restrict__ lin,
                                                    float* __restrict__ R, Geometry g) {
  extern __shared__ float smem[];
  const int b = blockIdx.y;
  const long long sf = blockIdx.z;  // slice*4 + family
  const int u0 = blockIdx.x * g.XA;
  const int H = g.H;
  if (u0 + g.XA <= g.N - b * H) return;  // no channel needs these columns
  const int P = g.XA + H - 1;
  float* A = smem;
  float* B = smem + (size_t)H * P;
  const int ubase = u0 - H + 1;
  const float* src = lin + (sf * g.N + (long long)b * H) * g.W;
  for (int r = threadIdx.x >> 5; r < H; r += blockDim.x >> 5) {
    const float* row = src + (long long)r * g.W;
    float* dst = A + (size_t)r * P;
    for (int j = threadIdx.x & 31; j < P; j += 32) {
      const int u = ubase + j;
      dst[j] = (u >= 0) ? __ldg(row + u) : 0.0f;
    }
  }
  __syncthreads();
  const float* res = fht_levels_smem(A, B, H, P, g.k1);
  float* dstR = R + ((sf * g.NB + b) * (long long)H) * g.WR;
  for (int c = threadIdx.x >> 5; c < H; c += blockDim.x >> 5) {
    const int ulo = g.N - b * (c + 1);
    const int uhi = g.W - c * b;
    const float* row = res + (size_t)c * P;
    float* out = dstR + (long long)c * g.WR + (c * b - g.N + g.NB);
    for (int j = (threadIdx.x & 31) + H - 1; j < P; j += 32) {
      const int u = ubase + j;
      if (u >= ulo && u < uhi) out[u] = row[j];
    }
  }
}

cudaError_t launch_fht_pass_a(const float* lin, float* R, int slices, const Geometry& g,
                              cudaStream_t st, int* launches) {
  if (slices <= 0) return cudaSuccess;
  const int P = g.XA + g.H - 1;
  const size_t smem = (size_t)2 * g.H * P * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_fht_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(g.W / g.XA, g.NB, slices * 4);
  k_fht_pass_a<<<grid, 256, smem, st>>>(lin, R, g);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3: pass B + family-pair sum.  grid (N/XB x-tiles, H channels, slices); block 256.
// For family f in {2*pair, 2*pair+1}: rows b in [0,NB) of G_c[b][v] =
// R_A[b][c][v - c*b] (= compact R[..][b][c][v - N + NB]) over v in
// [u0-NB+1, u0+XB), u0 = xs + N; m levels give B_f[c*NB + r][x], x = v - N.
// Family 2p at xs = x0, family 2p+1 at the mirrored tile xs = N - x0 - XB.
//   pair 0 (v): img[y = c*NB + r][x0 + i]  = scale * (B_0[y][x] + B_1[y][N-1-x])
//   pair 1 (h): img[x0 + i][x = c*NB + r] += scale * (B_2[x][y] + B_3[x][N-1-y])
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fht_pass_b(const float* __restrict__ R,
                                                    float* __restrict__ img, int pair,
                                                    float scale, Geometry g) {
  extern __shared__ float smem[];
  const int NB = g.NB;
  const int XB = g.XB;
  const int P = XB + NB - 1;
  const int c = blockIdx.y;
  const long long slice = blockIdx.z;
  const int x0 = blockIdx.x * XB;
  const float* res[2];
  for (int q = 0; q < 2; ++q) {
    const int f = 2 * pair + q;
    const int xs = (q == 0) ? x0 : (g.N - x0 - XB);
    float* A = smem + (size_t)q * 2 * NB * P;
    float* B = A + (size_t)NB * P;
    const float* src = R + (((slice * 4 + f) * NB) * (long long)g.H + c) * g.WR;
    for (int b = threadIdx.x >> 5; b < NB; b += blockDim.x >> 5) {
      const float* row = src + (long long)b * g.H * g.WR + xs + 1;
      float* dst = A + (size_t)b * P;
      for (int j = threadIdx.x & 31; j < P; j += 32) dst[j] = __ldg(row + j);
    }
    __syncthreads();
    res[q] = fht_levels_smem(A, B, NB, P, g.m);
  }
  const long long N = g.N;
  float* out = img + slice * N * N;
  if (pair == 0) {
    for (int r = threadIdx.x >> 5; r < NB; r += blockDim.x >> 5) {
      const float* r0 = res[0] + (size_t)r * P + NB - 1;
      const float* r1 = res[1] + (size_t)r * P + NB - 1;
      float* o = out + (long long)(c * NB + r) * N + x0;
      for (int i = threadIdx.x & 31; i < XB; i += 32) o[i] = scale * (r0[i] + r1[XB - 1 - i]);
    }
  } else {
    // transposed read-modify-write: r fastest for coalesced NB-float runs
    for (int e = threadIdx.x; e < NB * XB; e += blockDim.x) {
      const int r = e % NB;
      const int i = e / NB;
      const float v = res[0][(size_t)r * P + NB - 1 + i] + res[1][(size_t)r * P + NB - 1 + XB - 1 - i];
      float* o = out + (long long)(x0 + i) * N + c * NB + r;
      *o = *o + scale * v;
    }
  }
}

cudaError_t launch_fht_pass_b(const float* R, float* img, int slices, int pair, float scale,
                              const Geometry& g, cudaStream_t st, int* launches) {
  if (slices <= 0) return cudaSuccess;
  const int P = g.XB + g.NB - 1;
  const size_t smem = (size_t)4 * g.NB * P * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_fht_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(g.N / g.XB, g.H, slices);
  k_fht_pass_b<<<grid, 256, smem, st>>>(R, img, pair, scale, g);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
