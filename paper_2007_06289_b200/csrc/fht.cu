// K2/K3: Fast Hough Transform back projection (§4.4, 251-265 §4.5
// Eq.19-22), negative shift direction, additions only.
//
// Level recursion (h -> 2h):  R_2h[b][y'][u] = R_h[2b][y'/2][u] + R_h[2b+1][y'/2][u - ceil(y'/2)].
// Radix-2^R step: after l levels (blocks of 2^l rows, row = block*2^l + c), R more
// levels combine 2^R consecutive blocks; by d_y(t) = c*b' + d^(R)_{r'}(b') + ... :
//   out[G*2^(l+R) + c*2^R + r'][u] = sum_{b'<2^R} in[(G*2^R + b')*2^l + c][u - c*b' - d^(R)_{r'}(b')]
// i.e. a pre-shift c*b' of each input row (addressing only) followed by an R-level
// FHT with compile-time shifts, done in registers on 2^R rows x 8 columns
// (+ 2^R - 1 halo columns).  Shared-memory tiles use a padded layout
// (col + col/8) so that lanes working on consecutive 8-column chunks are
// bank-conflict free.
//
//   pass A (k_fht_a): k1 levels on each block of H = 2^k1 rows of the filtered
//     linogram, tile = H rows x (XA core + H halo) columns; output stored compactly
//     and only where pass B reads it (u in [N - b(c+1), 2N - c b)).
//   pass B (k_fht_b): per channel c, rows b of G_c[b][v] = R_A[b][c][v - c b],
//     m levels, then the family pair of Eq.22 (mirror) and the weight.
#include "fbp_internal.h"

namespace fbp {

namespace {

constexpr int kC = 8;  // output columns per register item

// Padded shared-memory tile layout: 4 pad floats after every 32 columns.  Keeps
// 16-byte alignment of every 4-column group (LDS/STS.128) and makes the
// stride-8-column lane pattern of the radix items bank-conflict free.
__device__ __forceinline__ int pc(int col) { return col + ((col >> 5) << 2); }

// Division by a runtime divisor d (< 2^16) of n (< 2^16) without the integer
// divide sequence: n / d = umulhi(n, ceil(2^32 / d)).
struct FastDiv {
  unsigned m;
  int d;
  __device__ __forceinline__ explicit FastDiv(int dd)
      : m((unsigned)((0x100000000ULL + (unsigned)dd - 1) / (unsigned)dd)), d(dd) {}
  __device__ __forceinline__ int div(int n) const { return (int)__umulhi((unsigned)n, m); }
};

// Register item geometry for radix 2^R: rows NR, halo quads HQ (>= NR-1 columns),
// window width T = kC + 4*HQ, outputs at window offset O = 4*HQ.
template <int R>
struct RT {
  static constexpr int NR = 1 << R;
  static constexpr int HQ = (NR - 1 + 3) / 4;
  static constexpr int O = 4 * HQ;
  static constexpr int T = kC + O;
};

// Register FHT on 2^R rows (natural recursion, compile-time shifts), computing at
// each level only the columns the final outputs [O, T) depend on.
template <int R>
__device__ __forceinline__ void local_fht(float (&v)[RT<R>::NR][RT<R>::T]) {
  constexpr int NR = RT<R>::NR;
  constexpr int T = RT<R>::T;
  // lower column bound needed at the output of level lvl: O - sum_{k>lvl} 2^k
#pragma unroll
  for (int lvl = 0; lvl < R; ++lvl) {
    const int h = 1 << lvl;
    const int lb = RT<R>::O - ((1 << R) - (1 << (lvl + 1)));
    float w[NR][T];
#pragma unroll
    for (int y = 0; y < NR; ++y) {
      const int blk = y & ~(2 * h - 1);
      const int yp = y - blk;
      const int lo = yp >> 1;
      const int sh = (yp + 1) >> 1;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (t >= lb) {
          const float bv = (t >= sh) ? v[blk + h + lo][t - sh] : 0.0f;
          w[y][t] = v[blk + lo][t] + bv;
        }
      }
    }
#pragma unroll
    for (int y = 0; y < NR; ++y)
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (t >= lb) v[y][t] = w[y][t];
  }
}

// Load the window [col0 - O, col0 - O + T) of the 2^R pre-shifted input rows of
// item (G, c, chunk at col0): row b' read at virtual column col - c*b'.
template <int R>
__device__ __forceinline__ void load_item(const float* tile, int P, int l, int G, int c, int col0,
                                          float (&v)[RT<R>::NR][RT<R>::T]) {
  constexpr int NR = RT<R>::NR;
  constexpr int T = RT<R>::T;
#pragma unroll
  for (int b = 0; b < NR; ++b) {
    const int row = ((G << R) + b) * (1 << l) + c;
    const float* rp = tile + (size_t)row * P;
    const int cs = col0 - RT<R>::O - c * b;
    if (cs >= 0) {
      const int ws = cs & ~3;
      const int o = cs & 3;
      float w[T + 4];
#pragma unroll
      for (int q = 0; q < T / 4 + 1; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(rp + pc(ws + 4 * q));
        w[4 * q] = f.x;
        w[4 * q + 1] = f.y;
        w[4 * q + 2] = f.z;
        w[4 * q + 3] = f.w;
      }
      if (o == 0) {
#pragma unroll
        for (int t = 0; t < T; ++t) v[b][t] = w[t];
      } else if (o == 1) {
#pragma unroll
        for (int t = 0; t < T; ++t) v[b][t] = w[t + 1];
      } else if (o == 2) {
#pragma unroll
        for (int t = 0; t < T; ++t) v[b][t] = w[t + 2];
      } else {
#pragma unroll
        for (int t = 0; t < T; ++t) v[b][t] = w[t + 3];
      }
    } else {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int col = cs + t;
        v[b][t] = (col >= 0) ? rp[pc(col)] : 0.0f;
      }
    }
  }
}

// Store 8 outputs at columns [col0, col0 + 8) of a padded row (2 x STS.128).
__device__ __forceinline__ void store8(float* rp, int col0, const float* s) {
  *reinterpret_cast<float4*>(rp + pc(col0)) = make_float4(s[0], s[1], s[2], s[3]);
  *reinterpret_cast<float4*>(rp + pc(col0 + 4)) = make_float4(s[4], s[5], s[6], s[7]);
}

// One radix step in shared memory: tiles in -> out (padded, pitch P), items over
// output chunks [chunk0, chunk0 + nchunks).
template <int R>
__device__ void radix_step_smem(const float* in, float* out, int P, int rows, int l, int chunk0,
                                int nchunks) {
  constexpr int NR = 1 << R;
  const int nch = 1 << l;                  // channels
  const int ngroups = rows >> (l + R);
  const int items = ngroups * nch * nchunks;
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int gc = fd.div(it);
    const int j = chunk0 + it - gc * nchunks;
    const int c = gc & (nch - 1);
    const int G = gc >> l;
    float v[NR][RT<R>::T];
    load_item<R>(in, P, l, G, c, j * kC, v);
    local_fht<R>(v);
#pragma unroll
    for (int r = 0; r < NR; ++r)
      store8(out + (size_t)((G << (l + R)) + c * NR + r) * P, j * kC, &v[r][RT<R>::O]);
  }
}

__device__ __forceinline__ void radix_step_dispatch(int R, const float* in, float* out, int P,
                                                    int rows, int l, int chunk0, int nchunks) {
  if (R == 3) radix_step_smem<3>(in, out, P, rows, l, chunk0, nchunks);
  else if (R == 2) radix_step_smem<2>(in, out, P, rows, l, chunk0, nchunks);
  else radix_step_smem<1>(in, out, P, rows, l, chunk0, nchunks);
}

// Split `levels` into radix steps of at most 3 levels: returns the radix of step s.
__device__ __forceinline__ int step_radix(int levels, int s) {
  // 1->[1] 2->[2] 3->[3] 4->[2,2] 5->[3,2] 6->[3,3] 7->[3,2,2] 8->[3,3,2]
  const int nsteps = (levels + 2) / 3;
  const int base = levels / nsteps, extra = levels % nsteps;
  return base + (s < extra ? 1 : 0);
}

// Run all levels of a pass on a tile whose first buffer is `a`; the last radix step
// is NOT executed (the caller fuses it with its epilogue).  Returns the buffer
// holding the input of the last step and sets *l_last, *R_last.
__device__ __forceinline__ float* run_levels_but_last(float* a, float* b, int P, int rows,
                                                      int levels, int nchunks_all, int* l_last,
                                                      int* R_last) {
  const int nsteps = (levels + 2) / 3;
  int l = 0;
  for (int s = 0; s < nsteps - 1; ++s) {
    const int R = step_radix(levels, s);
    radix_step_dispatch(R, a, b, P, rows, l, 0, nchunks_all);
    __syncthreads();
    float* t = a;
    a = b;
    b = t;
    l += R;
  }
  *l_last = l;
  *R_last = (nsteps > 0) ? step_radix(levels, nsteps - 1) : 0;
  return a;
}

}  // namespace

// ---------------------------------------------------------------------------
// Pass A.  grid (ceil(W/XA) tiles, NB blocks, slices*4), block 256.
// Tile columns u in [u0 - Hp, u0 + XA) -> local col = u - u0 + Hp  (Hp = H rounded
// up to 8 so the core starts on a chunk boundary); F outside [0, W) reads as 0.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void pass_a_last_step(const float* in, int P, int Hp, int l, int XA,
                                                 int u0, int b, const Geometry& g, float* dstR) {
  constexpr int NR = 1 << R;
  const int nch = 1 << l;
  const int nchunks = XA / kC;
  const int chunk0 = Hp / kC;
  const int items = nch * nchunks;   // a single group in the last step
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int c = fd.div(it);
    const int j = chunk0 + it - c * nchunks;
    float v[NR][RT<R>::T];
    load_item<R>(in, P, l, 0, c, j * kC, v);
    local_fht<R>(v);
    const int ubase = u0 - Hp + j * kC;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int cf = c * NR + r;                 // final pass-A channel
      const int ulo = g.N - b * (cf + 1);
      const int uhi = g.W - cf * b;
      float* out = dstR + (long long)cf * g.WR + (cf * b - g.N + g.NB);
      if (ubase >= ulo && ubase + kC <= uhi) {
#pragma unroll
        for (int t = 0; t < kC; ++t) out[ubase + t] = v[r][RT<R>::O + t];
      } else {
#pragma unroll
        for (int t = 0; t < kC; ++t) {
          const int u = ubase + t;
          if (u >= ulo && u < uhi) out[u] = v[r][RT<R>::O + t];
        }
      }
    }
  }
}

// Fill `rows` x D padded tile rows from global rows (pitch gp) starting at global
// column g0 (may be negative); columns outside [0, gw) read as 0.  Each thread
// issues kU independent float4 loads before storing (memory-level parallelism).
__device__ __forceinline__ void fill_tile(float* tile, int P, int rows, int D, const float* src,
                                          long long gp, int g0, int gw) {
  constexpr int kU = 6;
  const int q4 = D >> 2;
  const int total = rows * q4;
  const bool vec = ((g0 & 3) == 0) && ((gp & 3) == 0);
  const FastDiv fq(q4);
  for (int e0 = threadIdx.x; e0 < total; e0 += kU * blockDim.x) {
    float4 v[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int e = e0 + k * blockDim.x;
      if (e < total) {
        const int r = fq.div(e);
        const int u = g0 + (e - r * q4) * 4;
        const float* rp = src + (long long)r * gp;
        if (vec && u >= 0 && u + 3 < gw) {
          v[k] = __ldg(reinterpret_cast<const float4*>(rp + u));
        } else {
          v[k].x = (u >= 0 && u < gw) ? rp[u] : 0.0f;
          v[k].y = (u + 1 >= 0 && u + 1 < gw) ? rp[u + 1] : 0.0f;
          v[k].z = (u + 2 >= 0 && u + 2 < gw) ? rp[u + 2] : 0.0f;
          v[k].w = (u + 3 >= 0 && u + 3 < gw) ? rp[u + 3] : 0.0f;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int e = e0 + k * blockDim.x;
      if (e < total) {
        const int r = fq.div(e);
        const int c4 = (e - r * q4) * 4;
        *reinterpret_cast<float4*>(tile + (size_t)r * P + pc(c4)) = v[k];
      }
    }
  }
}

__global__ void __launch_bounds__(256, 2) k_fht_a(const float* __restrict__ lin,
                                               float* __restrict__ R, Geometry g, int P, int f0,
                                               int nf, long long lin_slice_stride) {
  extern __shared__ float smem[];
  const int b = blockIdx.y;
  const int zs = blockIdx.z / nf, zf = blockIdx.z % nf;
  const long long sf = (long long)zs * 4 + f0 + zf;     // output (slice, family)
  const int XA = g.XA, H = g.H;
  const int Hp = (H + kC - 1) / kC * kC;
  const int u0 = blockIdx.x * XA;
  if (u0 + XA <= g.N - b * H) return;      // no channel needs these columns
  const int D = XA + Hp;
  float* A = smem;
  float* B = smem + (size_t)H * P;
  const float* src = lin + zs * lin_slice_stride + ((long long)zf * g.N + (long long)b * H) * g.W;
  fill_tile(A, P, H, D, src, g.W, u0 - Hp, g.W);
  __syncthreads();
  int l_last, R_last;
  const float* in = run_levels_but_last(A, B, P, H, g.k1, D / kC, &l_last, &R_last);
  float* dstR = R + ((sf * g.NB + b) * (long long)H) * g.WR;
  if (R_last == 3) pass_a_last_step<3>(in, P, Hp, l_last, XA, u0, b, g, dstR);
  else if (R_last == 2) pass_a_last_step<2>(in, P, Hp, l_last, XA, u0, b, g, dstR);
  else pass_a_last_step<1>(in, P, Hp, l_last, XA, u0, b, g, dstR);
}

// ---------------------------------------------------------------------------
// Pass B.  grid (ceil(N/XB) x-tiles, H channels, slices), block 256.
// Family f = 2*pair + q at tile start xs (q = 0: x0; q = 1: mirrored N - x0 - XB).
// Rows b in [0,NB) of G_c[b][v], v in [u0 - NBp, u0 + XB), u0 = xs + N; compact R
// index j' = v - N + NB.  Family 1 runs first and is parked in smem; family 0 then
// adds the mirrored values (Eq.22 pair), scales and stores.
// ---------------------------------------------------------------------------
template <int R, bool PARK>
__device__ __forceinline__ void pass_b_last_step(const float* in, int P, int NBp, int l, int XB,
                                                 float* park, const float* parked, float* out,
                                                 int pair, int c, int NB, int x0, float scale,
                                                 int N, float* stage) {
  constexpr int NR = 1 << R;
  const int nch = 1 << l;
  const int nchunks = XB / kC;
  const int items = nch * nchunks;
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int cc = fd.div(it);
    const int jj = it - cc * nchunks;
    float v[NR][RT<R>::T];
    load_item<R>(in, P, l, 0, cc, NBp + jj * kC, v);
    local_fht<R>(v);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int rf = cc * NR + r;               // final row within the channel block
      if (PARK) {
#pragma unroll
        for (int t = 0; t < kC; ++t) park[rf * XB + jj * kC + t] = v[r][RT<R>::O + t];
      } else {
        float s[kC];
#pragma unroll
        for (int t = 0; t < kC; ++t) {
          const int i = jj * kC + t;
          s[t] = scale * (v[r][RT<R>::O + t] + parked[rf * XB + (XB - 1 - i)]);
        }
        const int y = c * NB + rf;
        const int xb = x0 + jj * kC;
        if (pair == 0) {
          float* o = out + (long long)y * N + xb;
          if (xb + kC <= N) {
            *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
            *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
          } else {
#pragma unroll
            for (int t = 0; t < kC; ++t)
              if (xb + t < N) o[t] = s[t];
          }
        } else {
          // transposed pair: park in the free tile buffer (padded rows), written
          // out coalesced by pass_b_flush_h after the barrier
#pragma unroll
          store8(stage + (size_t)rf * P, jj * kC, s);
        }
      }
    }
  }
}

template <bool PARK>
__device__ __forceinline__ void pass_b_last(int R, const float* in, int P, int NBp, int l, int XB,
                                            float* park, const float* parked, float* out, int pair,
                                            int c, int NB, int x0, float scale, int N, float* stage) {
  if (R == 3) pass_b_last_step<3, PARK>(in, P, NBp, l, XB, park, parked, out, pair, c, NB, x0, scale, N, stage);
  else if (R == 2) pass_b_last_step<2, PARK>(in, P, NBp, l, XB, park, parked, out, pair, c, NB, x0, scale, N, stage);
  else pass_b_last_step<1, PARK>(in, P, NBp, l, XB, park, parked, out, pair, c, NB, x0, scale, N, stage);
}

// h pair: out[x0 + i][c*NB + r] += stage[r][i]  (stage rows padded like the tiles)
__device__ __forceinline__ void pass_b_flush_h(const float* stage, int P, int NB, int XB, int c,
                                               int x0, float* out, int N) {
  if ((NB & 3) == 0) {
    const int q = NB >> 2;
    const FastDiv fq(q);
    for (int e = threadIdx.x; e < XB * q; e += blockDim.x) {
      const int i = fq.div(e);
      const int r = (e - i * q) * 4;
      if (x0 + i >= N) continue;
      float4* o = reinterpret_cast<float4*>(out + (long long)(x0 + i) * N + c * NB + r);
      float4 v = *o;
      v.x += stage[(r + 0) * P + pc(i)];
      v.y += stage[(r + 1) * P + pc(i)];
      v.z += stage[(r + 2) * P + pc(i)];
      v.w += stage[(r + 3) * P + pc(i)];
      *o = v;
    }
  } else {
    const FastDiv fn(NB);
    for (int e = threadIdx.x; e < XB * NB; e += blockDim.x) {
      const int i = fn.div(e);
      const int r = e - i * NB;
      if (x0 + i >= N) continue;
      float* o = out + (long long)(x0 + i) * N + c * NB + r;
      *o = *o + stage[r * P + pc(i)];
    }
  }
}

__global__ void __launch_bounds__(256, 2) k_fht_b(const float* __restrict__ R,
                                               float* __restrict__ img, Geometry g, int P,
                                               int pair, float scale) {
  extern __shared__ float smem[];
  const int NB = g.NB, XB = g.XB, N = g.N;
  const int NBp = (NB + kC - 1) / kC * kC;
  const int c = blockIdx.y;
  const long long slice = blockIdx.z;
  const int x0 = blockIdx.x * XB;
  const int D = XB + NBp;
  float* A = smem;
  float* B = smem + (size_t)NB * P;
  float* park = B + (size_t)NB * P;       // [NB][XB]
  float* out = img + slice * (long long)N * N;
  for (int q = 1; q >= 0; --q) {
    const int f = 2 * pair + q;
    const int xs = (q == 0) ? x0 : (N - x0 - XB);
    const float* src = R + (((slice * 4 + f) * NB) * (long long)g.H + c) * g.WR;
    fill_tile(A, P, NB, D, src, (long long)g.H * g.WR, xs - NBp + NB, g.WR);
    __syncthreads();
    int l_last = 0, R_last = 0;
    const float* in = A;
    if (g.m > 0) in = run_levels_but_last(A, B, P, NB, g.m, D / kC, &l_last, &R_last);
    float* stage = (in == A) ? B : A;     // free buffer during the last step
    if (g.m == 0) {
      // NB == 1: the single row is the result (no levels)
      for (int i = threadIdx.x; i < XB; i += blockDim.x) {
        const float v = in[pc(NBp + i)];
        if (q == 1) {
          park[i] = v;
        } else if (x0 + i < N) {
          const float sv = scale * (v + park[XB - 1 - i]);
          if (pair == 0) out[(long long)c * N + x0 + i] = sv;
          else { float* o = out + (long long)(x0 + i) * N + c; *o = *o + sv; }
        }
      }
    } else if (q == 1) {
      pass_b_last<true>(R_last, in, P, NBp, l_last, XB, park, nullptr, out, pair, c, NB, x0, scale, N, stage);
    } else {
      pass_b_last<false>(R_last, in, P, NBp, l_last, XB, nullptr, park, out, pair, c, NB, x0, scale, N, stage);
      if (pair == 1) {
        __syncthreads();
        pass_b_flush_h(stage, P, NB, XB, c, x0, out, N);
      }
    }
    __syncthreads();
  }
}

static int pitch_for(int D) {
  // widest column read by an item window is D + 3 (see load_item); padded layout,
  // rounded to a multiple of 4 floats (16-byte rows)
  const int w = D + 4;
  return (w + ((w >> 5) << 2) + 3) & ~3;
}

size_t fht_pass_a_smem(const Geometry& g) {
  const int Hp = (g.H + kC - 1) / kC * kC;
  return (size_t)2 * g.H * pitch_for(g.XA + Hp) * sizeof(float);
}

size_t fht_pass_b_smem(const Geometry& g) {
  const int NBp = (g.NB + kC - 1) / kC * kC;
  return ((size_t)2 * g.NB * pitch_for(g.XB + NBp) + (size_t)g.NB * g.XB) * sizeof(float);
}

cudaError_t launch_fht_pass_a(const float* lin, float* R, int slices, int f0, int nf,
                              long long lin_slice_stride, const Geometry& g, cudaStream_t st,
                              int* launches) {
  if (slices <= 0) return cudaSuccess;
  const int Hp = (g.H + kC - 1) / kC * kC;
  const int P = pitch_for(g.XA + Hp);
  const size_t smem = fht_pass_a_smem(g);
  cudaError_t e = cudaFuncSetAttribute(k_fht_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((g.W + g.XA - 1) / g.XA, g.NB, slices * nf);
  k_fht_a<<<grid, 256, smem, st>>>(lin, R, g, P, f0, nf, lin_slice_stride);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fht_pass_b(const float* R, float* img, int slices, int pair, float scale,
                              const Geometry& g, cudaStream_t st, int* launches) {
  if (slices <= 0) return cudaSuccess;
  const int NBp = (g.NB + kC - 1) / kC * kC;
  const int P = pitch_for(g.XB + NBp);
  const size_t smem = fht_pass_b_smem(g);
  cudaError_t e = cudaFuncSetAttribute(k_fht_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((g.N + g.XB - 1) / g.XB, g.H, slices);
  k_fht_b<<<grid, 256, smem, st>>>(R, img, g, P, pair, scale);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
