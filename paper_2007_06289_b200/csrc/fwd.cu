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

#ifndef FBP_FWD_FX6
#define FBP_FWD_FX6 192   // item-path tile width (output columns per CTA), 64-row passes (128, 160: +9 %, 256: +4 %)
#endif
#ifndef FBP_FWD_FX5
#define FBP_FWD_FX5 384   // the same, 32-row passes (measured: 320 +2 %, 448 +9 %, 576 +14 % pass-B time)
#endif

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


// ===========================================================================
// Register-item forward passes (r02), levels split into two radix steps
// R1 + R2 = log2(rows) <= 6, the back projection's item engine with the shift
// direction of Eq.17.  For 2^R consecutive blocks of 2^l rows and a channel c
// (the level-split identity of DESIGN.md §6, positive direction):
//   out[c*2^R + r'][u] = sum_{b' < 2^R} in[b'*2^l + c][u + c*b' + d^(R)_{r'}(b')]
// so step 1 (l = 0) runs R1 levels on row groups of 2^R1, step 2 (l = R1) runs R2
// levels on the rows b'*2^R1 + c, pre-shifted by c*b' (addressing).  Items: 2^R
// rows x 4 columns in registers, windows [v, v + 4 + O) read with LDS.128, levels
// with compile-time shifts (FADD2 where the shift is even), the recursion's own
// addition tree, so the results equal the level-by-level recursion bit for bit.
//
// One shared-memory tile of rows x (4 + W0) floats per CTA (tile of FX outputs plus
// the right halo the shifts read, recomputed per tile).  Step 1 runs IN PLACE in
// rounds of one item per thread: a round loads its windows, synchronises, then
// stores, and rounds advance left to right inside every row group, so a round only
// overwrites columns no later round reads.  Step 1 stores its output rows shifted
// LEFT by their step-2 pre-shift mod 4 (physical = 4 + virtual - (c*b' & 3)), so
// every step-2 window starts on a 16-byte boundary.  Step 2 stores float4 straight
// to HBM.
//   MODE 0 (pass A): rows y0 .. y0 + H of G_f for u-tile columns -> R_A rows.
//           G_0/G_2 are rows of the image / of its transpose (k_transpose, staged
//           in the linogram output, which pass B overwrites later); G_1/G_3 the
//           same rows mirrored: their aligned quads are copied as they are (so
//           each quad lands reversed) and step 1 undoes the reversal in registers.
//           Every fill is a 16-byte cp.async.
//   MODE 1 (pass B): rows b of R_A[b][c][v + c*b] (pass-A channel c) -> linogram
//           rows c*NB + t.
// R_A layout (item path): row (b, t') of width WRF2 = N + H + 4 holds logical
// compact column j (u = N - H + j, j < N + H) at j + ((-t'*b) & 3), zeros in the
// pad, so that pass B's pre-shifted rows start on 16-byte boundaries (every pass-B
// fill quad is one aligned 16-byte copy); pass A stores with the row's alignment
// (STG.128, 2 x STG.64 or 4 x STG.32).
// ===========================================================================
constexpr int FNT2 = 256;

// asynchronous global -> shared copy (LDGSTS, no register round trip); 0 source
// bytes zero-fill the destination (the source address is then not read)
__device__ __forceinline__ void cpa16(float* dst, const float* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
// explicit global stores (the widths chosen from the row's alignment must not be
// merged by the compiler)
__device__ __forceinline__ void stg1(float* g, float a) {
  asm volatile("st.global.f32 [%0], %1;\n" ::"l"(g), "f"(a) : "memory");
}
__device__ __forceinline__ void stg2(float* g, float a, float b) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};\n" ::"l"(g), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void stg4(float* g, float a, float b, float c, float d) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(g), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <int R, int C>
struct ItP {
  static constexpr int NR = 1 << R;
  static constexpr int O = 4 * ((NR - 1 + 3) / 4);   // right halo >= 2^R - 1, whole quads
  static constexpr int T = C + O;
};

__host__ __device__ constexpr int fpitch4(int w) { return (((w + 3) / 4) | 1) * 4; }

template <int T2>
__device__ __forceinline__ float colp(const float2 (&row)[T2], int t) {
  return (t & 1) ? row[t >> 1].y : row[t >> 1].x;
}

// windows of rows b' = 0 .. 2^R - 1 at base + b'*rowstep, virtual start pre-shifted
// by c*b'; the producer stored row b' shifted left by (c*b') & 3
// REV: every quad was stored reversed (mirrored families, see the fill); the
// reversal is undone by register naming.
template <int R, int C, bool REV = false>
__device__ __forceinline__ void itemp_load(const float* base, int rowstep, int c,
                                           float2 (&v)[ItP<R, C>::NR][ItP<R, C>::T / 2]) {
  constexpr int NR = ItP<R, C>::NR, T = ItP<R, C>::T;
  int cb = 0;
#pragma unroll
  for (int b = 0; b < NR; ++b) {
    const float4* w = reinterpret_cast<const float4*>(base + b * rowstep + (cb & ~3));
    cb += c;
#pragma unroll
    for (int q = 0; q < T / 4; ++q) {
      const float4 f = w[q];
      v[b][2 * q] = REV ? make_float2(f.w, f.z) : make_float2(f.x, f.y);
      v[b][2 * q + 1] = REV ? make_float2(f.y, f.x) : make_float2(f.z, f.w);
    }
  }
}

// R levels, positive shifts: level h -> 2h
//   w[blk + y'][t] = v[blk + lo][t] + v[blk + h + lo][t + ceil(y'/2)],  lo = floor(y'/2)
// (the direction of Eq.17), computing after each level only the
// columns [0, C + 2^R - 2^(lvl+1)) the outputs [0, C) still depend on.
template <int R, int C>
__device__ __forceinline__ void itemp_fht(float2 (&v)[ItP<R, C>::NR][ItP<R, C>::T / 2]) {
  constexpr int NR = ItP<R, C>::NR, T2 = ItP<R, C>::T / 2;
#pragma unroll
  for (int lvl = 0; lvl < R; ++lvl) {
    const int h = 1 << lvl;
    const int ub2 = (C + NR - (2 << lvl)) / 2;
    float2 w[NR][T2];
#pragma unroll
    for (int y = 0; y < NR; ++y) {
      const int blk = y & ~(2 * h - 1);
      const int yp = y - blk;
      const int lo = yp >> 1;
      const int sh = (yp + 1) >> 1;
#pragma unroll
      for (int tp = 0; tp < ub2; ++tp) {
        const float2 a = v[blk + lo][tp];
        if ((sh & 1) == 0) {
          w[y][tp] = __fadd2_rn(a, v[blk + h + lo][tp + sh / 2]);
        } else {
          w[y][tp].x = a.x + colp(v[blk + h + lo], 2 * tp + sh);
          w[y][tp].y = a.y + colp(v[blk + h + lo], 2 * tp + 1 + sh);
        }
      }
    }
#pragma unroll
    for (int y = 0; y < NR; ++y)
#pragma unroll
      for (int tp = 0; tp < ub2; ++tp) v[y][tp] = w[y][tp];
  }
}

template <int R1, int R2, int FX>
struct FwdGeo {
  static constexpr int ROWS = 1 << (R1 + R2);
  static constexpr int N1 = 1 << R1, N2 = 1 << R2;
  static constexpr int C = 4;                        // step-1 item columns
  // step-2 item columns (8 for radix 4 measured slower: 1.02 vs 0.77 ms, lanes 32 B
  // apart conflict in LDS.128 and half-fill each store's sectors)
  static constexpr int C2 = 4;
  static constexpr int O1 = ItP<R1, C>::O, O2 = ItP<R2, C2>::O;
  // step-1 output columns step 2 reads: FX + max pre-shift + the step-2 window halo
  static constexpr int W1 = (FX + (N1 - 1) * (N2 - 1) + O2 + 3) / 4 * 4;
  static constexpr int W0 = W1 + O1;                 // input columns step 1 reads
  static constexpr int P = fpitch4(4 + W0);          // 4 columns of room for the left shifts
  static constexpr size_t smem = (size_t)ROWS * P * sizeof(float);
};

template <int R1, int R2, int FX, int MODE>
__global__ void __launch_bounds__(FNT2) k_fwd_item(const float* __restrict__ src, const float* __restrict__ srcT,
                                                   float* __restrict__ dst, int N, int H, int NB) {
  using Gm = FwdGeo<R1, R2, FX>;
  constexpr int ROWS = Gm::ROWS, N1 = Gm::N1, N2 = Gm::N2, C = Gm::C, C2 = Gm::C2, P = Gm::P, W0 = Gm::W0,
                W1 = Gm::W1;
  constexpr int NQ = W0 / 4;
  extern __shared__ float4 fsm4[];
  float* A = reinterpret_cast<float*>(fsm4);
  const int tid = threadIdx.x;
  const int sf = blockIdx.z;
  const int WRF = N + H, WRF2 = N + H + 4;
  // ---- fill: virtual column v of row r at A[r*P + 4 + v], cp.async (zero outside) ----
  if (MODE == 0) {
    const int f = sf & 3, b = blockIdx.y;
    const float* im = (f < 2 ? src : srcT) + (long long)(sf >> 2) * N * N;
    const int x0 = blockIdx.x * FX - H;               // x = u - N of virtual column 0
    const int y0 = b * ROWS;
    for (int e = tid; e < ROWS * NQ; e += FNT2) {
      const int j = e / NQ, q = e - j * NQ;
      const int x = x0 + 4 * q;
      const bool ok = x >= 0 && x < N;
      // G[y][x .. x+3] = row[x .. x+3], or for the mirrored views row[N-4-x .. N-1-x]
      // (reversed)
      const int gx = (f & 1) ? N - 4 - x : x;
      cpa16(A + j * P + 4 + 4 * q, im + (long long)(y0 + j) * N + (ok ? gx : 0), ok);
    }
  } else {
    // rows b of G_c[b][v] = R_A[b][c][v + c*b]: logical column v + c*b - (N - H) at
    // physical v - (N - H) + 4*ceil(c*b/4), a multiple of 4
    const int c = blockIdx.y, s0 = blockIdx.x * FX;
    const float* in = src + (long long)sf * NB * H * WRF2;
    for (int e = tid; e < ROWS * NQ; e += FNT2) {
      const int b = e / NQ, q = e - b * NQ;
      const int pp = s0 + 4 * q - (N - H) + 4 * ((c * b + 3) >> 2);
      const bool ok = pp >= 0 && pp + 4 <= WRF2;
      cpa16(A + b * P + 4 + 4 * q, in + ((long long)b * H + c) * WRF2 + (ok ? pp : 0), ok);
    }
  }
  cpa_wait_all();
  __syncthreads();
  // ---- step 1: R1 levels on row groups g (rows g*N1 ..), in place, in rounds ----
  {
    constexpr int NC1 = W1 / C, G1 = ROWS / N1, NI1 = NC1 * G1;
    for (int base = 0; base < NI1; base += FNT2) {
      const int it = base + tid;
      const bool act = it < NI1;
      const int g = act ? it / NC1 : 0, k = act ? it - g * NC1 : 0;
      float2 v[N1][ItP<R1, C>::T / 2];
      if (act) {
        if (MODE == 0 && (sf & 1))
          itemp_load<R1, C, true>(A + (g * N1) * P + 4 + C * k, P, 0, v);
        else
          itemp_load<R1, C>(A + (g * N1) * P + 4 + C * k, P, 0, v);
        itemp_fht<R1, C>(v);
      }
      __syncthreads();
      if (act) {
#pragma unroll
        for (int r = 0; r < N1; ++r) {
          const int sh = (r * g) & 3;                  // step-2 pre-shift of this row, mod 4
          float* o = A + (g * N1 + r) * P + 4 + C * k - sh;
          if (sh == 0) {
            *reinterpret_cast<float4*>(o) = make_float4(colp(v[r], 0), colp(v[r], 1), colp(v[r], 2), colp(v[r], 3));
          } else if (sh == 2) {
            *reinterpret_cast<float2*>(o) = make_float2(colp(v[r], 0), colp(v[r], 1));
            *reinterpret_cast<float2*>(o + 2) = make_float2(colp(v[r], 2), colp(v[r], 3));
          } else {
#pragma unroll
            for (int tt = 0; tt < C; ++tt) o[tt] = colp(v[r], tt);
          }
        }
      }
      __syncthreads();
    }
  }
  // ---- step 2: R2 levels on rows b'*N1 + c, pre-shift c*b' -> HBM ----
  {
    constexpr int NC2 = FX / C2, NI2 = N1 * NC2;
    for (int it = tid; it < NI2; it += FNT2) {
      const int c = it / NC2, k = it - c * NC2;
      float2 v[N2][ItP<R2, C2>::T / 2];
      itemp_load<R2, C2>(A + c * P + 4 + C2 * k, N1 * P, c, v);
      itemp_fht<R2, C2>(v);
      if (MODE == 0) {
        const int b = blockIdx.y;
        float* out = dst + ((long long)sf * NB + b) * H * WRF2;
#pragma unroll
        for (int hq = 0; hq < C2 / 4; ++hq) {
          const int j = blockIdx.x * FX + C2 * k + 4 * hq;
          if (j < WRF) {
#pragma unroll
            for (int r = 0; r < N2; ++r) {
              const int t = c * N2 + r;
              const int sh = (-(t * b)) & 3;
              float* row = out + (long long)t * WRF2;
              float* o = row + j + sh;
              const float a0 = colp(v[r], 4 * hq), a1 = colp(v[r], 4 * hq + 1), a2 = colp(v[r], 4 * hq + 2),
                          a3 = colp(v[r], 4 * hq + 3);
              if (sh == 0) {
                stg4(o, a0, a1, a2, a3);
              } else if (sh == 2) {
                stg2(o, a0, a1);
                stg2(o + 2, a2, a3);
              } else {
                stg1(o, a0);
                stg1(o + 1, a1);
                stg1(o + 2, a2);
                stg1(o + 3, a3);
              }
              // zero pad: [0, sh) before the row, [WRF + sh, WRF2) after it
              if (j == 0)
                for (int i = 0; i < sh; ++i) stg1(row + i, 0.f);
              if (j + 4 == WRF)
                for (int i = WRF + sh; i < WRF2; ++i) stg1(row + i, 0.f);
            }
          }
        }
      } else {
        const int ca = blockIdx.y, W = 2 * N;
        float* out = dst + ((long long)sf * N + (long long)ca * NB) * W;
#pragma unroll
        for (int hq = 0; hq < C2 / 4; ++hq) {
          const int s = blockIdx.x * FX + C2 * k + 4 * hq;
          if (s < W) {
#pragma unroll
            for (int r = 0; r < N2; ++r)
              stg4(out + (long long)(c * N2 + r) * W + s, colp(v[r], 4 * hq), colp(v[r], 4 * hq + 1),
                   colp(v[r], 4 * hq + 2), colp(v[r], 4 * hq + 3));
          }
        }
      }
    }
  }
}

// tile widths (output columns per CTA), ~64-72 KB of shared memory: 3 CTAs/SM
template <int R1, int R2>
struct FwdFX {
  static constexpr int value = (R1 + R2 == 6) ? FBP_FWD_FX6 : (R1 + R2 == 5) ? FBP_FWD_FX5 : 960;
};

template <int R1, int R2, int MODE>
cudaError_t launch_fwd_item(const float* src, const float* srcT, float* dst, int slices, const Geometry& g,
                            cudaStream_t st) {
  constexpr int FX = FwdFX<R1, R2>::value;
  using Gm = FwdGeo<R1, R2, FX>;
  auto kern = k_fwd_item<R1, R2, FX, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::smem);
  if (e != cudaSuccess) return e;
  const int cols = MODE == 0 ? g.N + g.H : 2 * g.N;
  const dim3 grid((cols + FX - 1) / FX, MODE == 0 ? g.NB : g.H, 4 * slices);
  kern<<<grid, FNT2, Gm::smem, st>>>(src, srcT, dst, g.N, g.H, g.NB);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_fwd_item_rows(int rows, const float* src, const float* srcT, float* dst, int slices,
                                 const Geometry& g, cudaStream_t st) {
  switch (rows) {
    case 16: return launch_fwd_item<2, 2, MODE>(src, srcT, dst, slices, g, st);
    case 32: return launch_fwd_item<3, 2, MODE>(src, srcT, dst, slices, g, st);
    case 64: return launch_fwd_item<3, 3, MODE>(src, srcT, dst, slices, g, st);
    default: return cudaErrorNotSupported;
  }
}

bool fwd_item_rows(int rows) { return rows == 16 || rows == 32 || rows == 64; }

// item path for both passes (N = 512 .. 4096); otherwise the shared-memory kernels
bool fwd_item_path(const Geometry& g) { return fwd_item_rows(g.H) && fwd_item_rows(g.NB); }

// image transpose [slices][N][N] (families 2 and 3 read image columns as rows):
// 32 x 32 tiles through shared memory (odd pitch), coalesced on both sides
__global__ void __launch_bounds__(256) k_transpose(const float* __restrict__ in, float* __restrict__ out, int N) {
  __shared__ float t[32][33];
  const long long off = (long long)blockIdx.z * N * N;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) t[ty + k][tx] = __ldg(in + off + (long long)(y0 + ty + k) * N + x0 + tx);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) out[off + (long long)(x0 + ty + k) * N + y0 + tx] = t[tx][ty + k];
}

}  // namespace

size_t fwd_workspace_floats(const Geometry& g) { return (size_t)4 * g.NB * g.H * (g.N + g.H + 4); }

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

cudaError_t launch_fwd_a(const float* img, float* RA, float* scratch, int slices, const Geometry& g,
                         cudaStream_t st, int* launches) {
  const int N = g.N, H = g.H, NB = g.NB;
  if (fwd_item_path(g)) {
    k_transpose<<<dim3(N / 32, N / 32, slices), 256, 0, st>>>(img, scratch, N);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launches) *launches += 2;
    return launch_fwd_item_rows<0>(H, img, scratch, RA, slices, g, st);
  }
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
  if (fwd_item_path(g)) {
    if (launches) ++*launches;
    return launch_fwd_item_rows<1>(NB, RA, nullptr, lin, slices, g, st);
  }
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
