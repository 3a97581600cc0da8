// K2/K3: Fast Hough Transform back projection (§4.4, 251-265 §4.5
// Eq.19-22), negative shift direction, additions only.
//
// Level recursion (h -> 2h):  R_2h[b][y'][u] = R_h[2b][y'/2][u] + R_h[2b+1][y'/2][u - ceil(y'/2)].
// Radix-2^R step: after l levels (blocks of 2^l rows, row = block*2^l + c), R more
// levels combine 2^R consecutive blocks; by d_y(t) = c*b' + d^(R)_{r'}(b') + ... :
//   out[G*2^(l+R) + c*2^R + r'][u] = sum_{b'<2^R} in[(G*2^R + b')*2^l + c][u - c*b' - d^(R)_{r'}(b')]
// i.e. a pre-shift c*b' of each input row (addressing only) followed by an R-level
// FHT with compile-time shifts, done in registers on 2^R rows x 8 columns (+ halo).
//
//   pass A (k_fht_a): k1 levels on each block of H = 2^k1 rows of the filtered
//     linogram; tile = H rows x (Hp halo + XA core) columns.  Output stored
//     compactly, only where pass B reads it (u in [N - b(c+1), 2N - c b)).
//   pass B (k_fht_b): per channel c, rows b of G_c[b][v] = R_A[b][c][v - c b]
//     (the compact layout already applies the pre-shift), m levels, then the family
//     pair of Eq.22 (mirror), the weight, and the store.
// Both kernels are persistent (grid = resident CTAs) and prefetch the next tile
// with cp.async while computing the current one.
#include "fbp_internal.h"

#include <algorithm>

namespace fbp {

namespace {

constexpr int kC = 8;        // output columns per register item
constexpr int kThreads = 256;

// Padded shared-memory tile layout: 4 pad floats after every 32 columns.  Keeps
// 16-byte alignment of every 4-column group (cp.async / LDS / STS .128) and makes
// the stride-8-column lane pattern of the radix items bank-conflict free.
__device__ __forceinline__ int pc(int col) { return col + ((col >> 5) << 2); }

// Division by a runtime divisor d (< 2^16) of n (< 2^16) without the integer
// divide sequence: n / d = umulhi(n, ceil(2^32 / d)); d = 1 handled separately.
struct FastDiv {
  unsigned m;
  int d;
  __device__ __forceinline__ explicit FastDiv(int dd)
      : m(dd > 1 ? (unsigned)((0x100000000ULL + (unsigned)dd - 1) / (unsigned)dd) : 0u), d(dd) {}
  __device__ __forceinline__ int div(int n) const {
    return d > 1 ? (int)__umulhi((unsigned)n, m) : n;
  }
};

// ---- cp.async (zero-fill when !valid) ----
__device__ __forceinline__ void cp_async16(float* sdst, const float* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gsrc),
               "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NLEFT>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NLEFT));
}

// Asynchronously fill a `rows` x D padded tile (pitch P) from global rows of
// pitch gp, starting at global column g0 (may be negative); columns outside
// [0, gw) are zero-filled.  Rows are spread over warps, 4-column groups over lanes.
// Commits one cp.async group.
__device__ __forceinline__ void fill_async(float* tile, int P, int rows, int D, const float* src,
                                           long long gp, int g0, int gw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q4 = D >> 2;
  const bool vec = ((g0 & 3) == 0) && ((gp & 3) == 0) && ((gw & 3) == 0);
  for (int r = warp; r < rows; r += kThreads / 32) {
    const float* rp = src + (long long)r * gp;
    float* tp = tile + (size_t)r * P;
    for (int q = lane; q < q4; q += 32) {
      const int u = g0 + 4 * q;
      if (vec) {
        const bool ok = (u >= 0) && (u < gw);
        cp_async16(tp + pc(4 * q), ok ? rp + u : rp, ok);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = (u + e >= 0) && (u + e < gw);
          cp_async4(tp + pc(4 * q + e), ok ? rp + u + e : rp, ok);
        }
      }
    }
  }
  cp_async_commit();
}

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

// Intermediate rows are stored shifted right by (their next pre-shift) & 3, so that
// every item window below is 4-column aligned: virtual column x of row rho lives
// at physical column x + sh4(rho), sh4 = (c'*b') & 3 for the step that reads it.

// Load the window [col0 - O, col0 - O + T) of the 2^R pre-shifted input rows of
// item (G, c, chunk at col0): row b read at virtual column col - c*b, i.e. at
// physical col - 4*floor(c*b/4) (aligned LDS.128 quads, no register moves).
template <int R>
__device__ __forceinline__ void load_item(const float* tile, int P, int l, int G, int c, int col0,
                                          float (&v)[RT<R>::NR][RT<R>::T]) {
  constexpr int NR = RT<R>::NR;
  constexpr int T = RT<R>::T;
#pragma unroll
  for (int b = 0; b < NR; ++b) {
    const int row = ((G << R) + b) * (1 << l) + c;
    const float* rp = tile + (size_t)row * P;
    const int s = c * b;
    const int ws = col0 - RT<R>::O - (s & ~3);           // physical, 4-aligned
    if (ws >= 0) {
#pragma unroll
      for (int q = 0; q < T / 4; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(rp + pc(ws + 4 * q));
        v[b][4 * q] = f.x;
        v[b][4 * q + 1] = f.y;
        v[b][4 * q + 2] = f.z;
        v[b][4 * q + 3] = f.w;
      }
    } else {
      const int cs = col0 - RT<R>::O - s;                // virtual window start
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int col = cs + t;
        v[b][t] = (col >= 0) ? rp[pc(ws + t)] : 0.0f;
      }
    }
  }
}

// Process one item: load, R register levels, then the epilogue epi(v) with
// outputs v[r][O + t], t < 8.
template <int R, typename Epi>
__device__ __forceinline__ void item(const float* tile, int P, int l, int G, int c, int col0,
                                     Epi& epi) {
  float v[RT<R>::NR][RT<R>::T];
  load_item<R>(tile, P, l, G, c, col0, v);
  local_fht<R>(v);
  epi(v);
}

// Store 8 outputs at columns [col0, col0 + 8) of a padded row (2 x STS.128).
__device__ __forceinline__ void store8(float* rp, int col0, const float* s) {
  *reinterpret_cast<float4*>(rp + pc(col0)) = make_float4(s[0], s[1], s[2], s[3]);
  *reinterpret_cast<float4*>(rp + pc(col0 + 4)) = make_float4(s[4], s[5], s[6], s[7]);
}

// Store 8 outputs at physical columns [col0 + off, col0 + off + 8), off in 0..3,
// col0 a multiple of 8 (pieces never straddle a 32-column pad boundary).
__device__ __forceinline__ void store8_off(float* rp, int col0, int off, const float* s) {
  float* p = rp + pc(col0);          // 8-aligned group: pc is contiguous over 8 columns
  switch (off) {
    case 0:
      *reinterpret_cast<float4*>(p) = make_float4(s[0], s[1], s[2], s[3]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(s[4], s[5], s[6], s[7]);
      break;
    case 1:
      p[1] = s[0];
      *reinterpret_cast<float2*>(p + 2) = make_float2(s[1], s[2]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(s[3], s[4], s[5], s[6]);
      rp[pc(col0 + 8)] = s[7];
      break;
    case 2:
      *reinterpret_cast<float2*>(p + 2) = make_float2(s[0], s[1]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(s[2], s[3], s[4], s[5]);
      *reinterpret_cast<float2*>(rp + pc(col0 + 8)) = make_float2(s[6], s[7]);
      break;
    default: {
      p[3] = s[0];
      *reinterpret_cast<float4*>(p + 4) = make_float4(s[1], s[2], s[3], s[4]);
      float* q = rp + pc(col0 + 8);
      *reinterpret_cast<float2*>(q) = make_float2(s[5], s[6]);
      q[2] = s[7];
      break;
    }
  }
}

// One intermediate radix step in shared memory: in -> out (padded, pitch P).
// The output row rho is written shifted by (its pre-shift in the next step) & 3;
// the next step has l' = l + R levels done and radix Rn.
template <int R>
__device__ void radix_step_smem(const float* in, float* out, int P, int rows, int l, int Rn,
                                int nchunks) {
  constexpr int NR = 1 << R;
  const int nch = 1 << l;
  const int items = (rows >> (l + R)) * nch * nchunks;
  const int ln = l + R;
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += kThreads) {
    const int gc = fd.div(it);
    const int j = it - gc * nchunks;
    const int c = gc & (nch - 1);
    const int G = gc >> l;
    auto epi = [&](float (&v)[NR][RT<R>::T]) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int rho = (G << (l + R)) + c * NR + r;
        const int cn = rho & ((1 << ln) - 1);                 // next step's channel
        const int bn = (rho >> ln) & ((1 << Rn) - 1);         // next step's block
        store8_off(out + (size_t)rho * P, j * kC, (cn * bn) & 3, &v[r][RT<R>::O]);
      }
    };
    item<R>(in, P, l, G, c, j * kC, epi);
  }
}

__device__ __forceinline__ void radix_step_dispatch(int R, const float* in, float* out, int P,
                                                    int rows, int l, int Rn, int nchunks) {
  if (R == 3) radix_step_smem<3>(in, out, P, rows, l, Rn, nchunks);
  else if (R == 2) radix_step_smem<2>(in, out, P, rows, l, Rn, nchunks);
  else radix_step_smem<1>(in, out, P, rows, l, Rn, nchunks);
}

// Split `levels` into radix steps of at most 3 levels: radix of step s.
// 1->[1] 2->[2] 3->[3] 4->[2,2] 5->[3,2] 6->[3,3] 7->[3,2,2] 8->[3,3,2]
__device__ __forceinline__ int step_radix(int levels, int s) {
  const int nsteps = (levels + 2) / 3;
  const int base = levels / nsteps, extra = levels % nsteps;
  return base + (s < extra ? 1 : 0);
}

// Run all radix steps of a pass except the last, ping-ponging between a and b.
// Returns the buffer holding the last step's input; *l_last, *R_last describe it.
__device__ __forceinline__ float* run_levels_but_last(float* a, float* b, int P, int rows,
                                                      int levels, int nchunks, int* l_last,
                                                      int* R_last) {
  const int nsteps = (levels + 2) / 3;
  int l = 0;
  for (int s = 0; s < nsteps - 1; ++s) {
    const int R = step_radix(levels, s);
    radix_step_dispatch(R, a, b, P, rows, l, step_radix(levels, s + 1), nchunks);
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
// Pass A.  Persistent: each CTA loops over tiles (u-tile, block b, slice*family).
// Tile columns u in [u0 - Hp, u0 + XA) -> local col = u - u0 + Hp (Hp = H rounded
// up to 8 so the core starts on a chunk boundary); F outside [0, W) reads as 0.
// ---------------------------------------------------------------------------
struct PassATile {
  int u0, b;
  long long zs, zf;
};

__device__ __forceinline__ bool pass_a_tile(long long t, const Geometry& g, int nu, int nf,
                                            PassATile* pt) {
  const long long per_z = (long long)nu * g.NB;
  const long long z = t / per_z;
  const int rem = (int)(t - z * per_z);
  pt->b = rem / nu;
  pt->u0 = (rem - pt->b * nu) * g.XA;
  pt->zs = z / nf;
  pt->zf = z - pt->zs * nf;
  return pt->u0 + g.XA > g.N - pt->b * g.H;    // false: no channel needs it
}

template <int R>
__device__ __forceinline__ void pass_a_last(const float* in, int P, int Hp, int l,
                                            const PassATile& pt, const Geometry& g, float* dstR) {
  constexpr int NR = 1 << R;
  const int nchunks = g.XA / kC;
  const int chunk0 = Hp / kC;
  const int items = (1 << l) * nchunks;   // a single group in the last step
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += kThreads) {
    const int c = fd.div(it);
    const int j = chunk0 + it - c * nchunks;
    const int ubase = pt.u0 - Hp + j * kC;
    auto epi = [&](float (&v)[NR][RT<R>::T]) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int cf = c * NR + r;                 // final pass-A channel
        const int ulo = g.N - pt.b * (cf + 1);
        const int uhi = g.W - cf * pt.b;
        float* out = dstR + (long long)cf * g.WR + (cf * pt.b - g.N + g.NB);
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
    };
    item<R>(in, P, l, 0, c, j * kC, epi);
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_fht_a(const float* __restrict__ lin,
                                                       float* __restrict__ R, Geometry g, int P,
                                                       int f0, int nf, long long lin_slice_stride,
                                                       long long ntiles) {
  extern __shared__ float smem[];
  const int H = g.H;
  const int Hp = (H + kC - 1) / kC * kC;
  const int D = g.XA + Hp;
  const int nu = (g.W + g.XA - 1) / g.XA;
  float* buf[2] = {smem, smem + (size_t)H * P};
  auto src_of = [&](const PassATile& pt) {
    return lin + pt.zs * lin_slice_stride + (pt.zf * g.N + (long long)pt.b * H) * g.W;
  };
  long long t = blockIdx.x;
  PassATile cur;
  while (t < ntiles && !pass_a_tile(t, g, nu, nf, &cur)) t += gridDim.x;
  if (t >= ntiles) return;
  int fb = 0;                                       // buffer holding the current fill
  fill_async(buf[fb], P, H, D, src_of(cur), g.W, cur.u0 - Hp, g.W);
  while (true) {
    long long tn = t + gridDim.x;                   // next needed tile
    PassATile nxt;
    while (tn < ntiles && !pass_a_tile(tn, g, nu, nf, &nxt)) tn += gridDim.x;
    cp_async_wait<0>();
    __syncthreads();
    int l_last, R_last;
    float* in = run_levels_but_last(buf[fb], buf[fb ^ 1], P, H, g.k1, D / kC, &l_last, &R_last);
    const int in_idx = (in == buf[0]) ? 0 : 1;
    // the other buffer is free during the last step: prefetch the next tile there
    if (tn < ntiles) fill_async(buf[in_idx ^ 1], P, H, D, src_of(nxt), g.W, nxt.u0 - Hp, g.W);
    const long long sf = cur.zs * 4 + (f0 + cur.zf);
    float* dstR = R + ((sf * g.NB + cur.b) * (long long)H) * g.WR;
    if (R_last == 3) pass_a_last<3>(in, P, Hp, l_last, cur, g, dstR);
    else if (R_last == 2) pass_a_last<2>(in, P, Hp, l_last, cur, g, dstR);
    else pass_a_last<1>(in, P, Hp, l_last, cur, g, dstR);
    if (tn >= ntiles) break;
    __syncthreads();                                 // everyone done reading `in`
    t = tn;
    cur = nxt;
    fb = in_idx ^ 1;
  }
}

// ---------------------------------------------------------------------------
// Pass B.  Persistent: each CTA loops over items (x-tile, channel c, slice).
// Family f = 2*pair + q at tile start xs (q = 0: x0; q = 1: mirrored N - x0 - XB).
// Rows b in [0,NB) of G_c[b][v], v in [u0 - NBp, u0 + XB), u0 = xs + N; compact R
// index j' = v - N + NB.  Family 1 is processed first and parked (padded rows);
// family 0 then adds the mirrored values (Eq.22 pair), scales and stores.
// Buffers: Fb[1], Fb[0] (family fills), Wk (work), PK (park).
// ---------------------------------------------------------------------------
struct PassBItem {
  int x0, c;
  long long slice;
};

__device__ __forceinline__ void pass_b_item(long long t, const Geometry& g, int nx, PassBItem* it) {
  const long long per_s = (long long)nx * g.H;
  it->slice = t / per_s;
  const int rem = (int)(t - it->slice * per_s);
  it->c = rem / nx;
  it->x0 = (rem - it->c * nx) * g.XB;
}

template <int R, bool PARK>
__device__ __forceinline__ void pass_b_last(const float* in, int P, int NBp, int l, int NB,
                                            int XB, float* park, const float* parked, float* out,
                                            int pair, int c, int x0, float scale, int N,
                                            float* stage) {
  constexpr int NR = 1 << R;
  const int nchunks = XB / kC;
  const int items = (1 << l) * nchunks;
  const FastDiv fd(nchunks);
  for (int it = threadIdx.x; it < items; it += kThreads) {
    const int cc = fd.div(it);
    const int jj = it - cc * nchunks;
    auto epi = [&](float (&v)[NR][RT<R>::T]) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int rf = cc * NR + r;                // final row within the channel block
        if (PARK) {
          store8(park + (size_t)rf * P, jj * kC, &v[r][RT<R>::O]);
        } else {
          // mirrored family-1 values: columns XB-1-i for i = jj*8 .. jj*8+7
          const float* pr = parked + (size_t)rf * P;
          const int m0 = XB - kC - jj * kC;
          const float4 a = *reinterpret_cast<const float4*>(pr + pc(m0));
          const float4 bq = *reinterpret_cast<const float4*>(pr + pc(m0 + 4));
          const float mir[kC] = {bq.w, bq.z, bq.y, bq.x, a.w, a.z, a.y, a.x};
          float s[kC];
#pragma unroll
          for (int tt = 0; tt < kC; ++tt) s[tt] = scale * (v[r][RT<R>::O + tt] + mir[tt]);
          const int y = c * NB + rf;
          const int xb = x0 + jj * kC;
          if (pair == 0) {
            float* o = out + (long long)y * N + xb;
            if (xb + kC <= N) {
              *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
              *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
            } else {
#pragma unroll
              for (int tt = 0; tt < kC; ++tt)
                if (xb + tt < N) o[tt] = s[tt];
            }
          } else {
            store8(stage + (size_t)rf * P, jj * kC, s);   // transposed by pass_b_flush_h
          }
        }
      }
    };
    item<R>(in, P, l, 0, cc, NBp + jj * kC, epi);
  }
}

template <bool PARK>
__device__ __forceinline__ void pass_b_last_dispatch(int R, const float* in, int P, int NBp, int l,
                                                     int NB, int XB, float* park,
                                                     const float* parked, float* out, int pair,
                                                     int c, int x0, float scale, int N,
                                                     float* stage) {
  if (R == 3) pass_b_last<3, PARK>(in, P, NBp, l, NB, XB, park, parked, out, pair, c, x0, scale, N, stage);
  else if (R == 2) pass_b_last<2, PARK>(in, P, NBp, l, NB, XB, park, parked, out, pair, c, x0, scale, N, stage);
  else pass_b_last<1, PARK>(in, P, NBp, l, NB, XB, park, parked, out, pair, c, x0, scale, N, stage);
}

// h pair: out[x0 + i][c*NB + r] += stage[r][i]  (stage rows padded like the tiles)
__device__ __forceinline__ void pass_b_flush_h(const float* stage, int P, int NB, int XB, int c,
                                               int x0, float* out, int N) {
  if ((NB & 3) == 0) {
    const int q = NB >> 2;
    const FastDiv fq(q);
    for (int e = threadIdx.x; e < XB * q; e += kThreads) {
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
    for (int e = threadIdx.x; e < XB * NB; e += kThreads) {
      const int i = fn.div(e);
      const int r = e - i * NB;
      if (x0 + i >= N) continue;
      float* o = out + (long long)(x0 + i) * N + c * NB + r;
      *o = *o + stage[r * P + pc(i)];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_fht_b(const float* __restrict__ R,
                                                       float* __restrict__ img, Geometry g, int P,
                                                       int pair, float scale, long long nitems) {
  extern __shared__ float smem[];
  const int NB = g.NB, XB = g.XB, N = g.N;
  const int NBp = (NB + kC - 1) / kC * kC;
  const int D = XB + NBp;
  const int nx = (N + XB - 1) / XB;
  float* Fb[2] = {smem, smem + (size_t)NB * P};       // family fills (q = 0, 1)
  float* Wk = smem + (size_t)2 * NB * P;              // work buffer
  float* PK = smem + (size_t)3 * NB * P;              // park (family 1)
  auto fill = [&](const PassBItem& it, int q) {
    const int f = 2 * pair + q;
    const int xs = (q == 0) ? it.x0 : (N - it.x0 - XB);
    const float* src = R + (((it.slice * 4 + f) * NB) * (long long)g.H + it.c) * g.WR;
    fill_async(Fb[q], P, NB, D, src, (long long)g.H * g.WR, xs - NBp + NB, g.WR);
  };
  long long t = blockIdx.x;
  if (t >= nitems) return;
  PassBItem cur;
  pass_b_item(t, g, nx, &cur);
  fill(cur, 1);
  fill(cur, 0);
  while (true) {
    float* out = img + cur.slice * (long long)N * N;
    const long long tn = t + gridDim.x;
    PassBItem nxt;
    if (tn < nitems) pass_b_item(tn, g, nx, &nxt);
    // ---- family 1 -> park ----
    cp_async_wait<1>();                               // family-1 fill landed
    __syncthreads();
    {
      int l_last = 0, R_last = 0;
      float* in = Fb[1];
      if (g.m > 0) in = run_levels_but_last(Fb[1], Wk, P, NB, g.m, D / kC, &l_last, &R_last);
      if (g.m == 0) {
        for (int i = threadIdx.x; i < XB; i += kThreads) PK[pc(i)] = in[pc(NBp + i)];
      } else {
        pass_b_last_dispatch<true>(R_last, in, P, NBp, l_last, NB, XB, PK, nullptr, out, pair,
                                   cur.c, cur.x0, scale, N, nullptr);
      }
    }
    __syncthreads();
    if (tn < nitems) fill(nxt, 1);                   // Fb[1] free again
    // ---- family 0 + pair sum ----
    if (tn < nitems) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    {
      int l_last = 0, R_last = 0;
      float* in = Fb[0];
      if (g.m > 0) in = run_levels_but_last(Fb[0], Wk, P, NB, g.m, D / kC, &l_last, &R_last);
      float* stage = (in == Wk) ? Fb[0] : Wk;        // free during the last step
      if (g.m == 0) {
        for (int i = threadIdx.x; i < XB; i += kThreads) {
          if (cur.x0 + i >= N) continue;
          const float sv = scale * (in[pc(NBp + i)] + PK[pc(XB - 1 - i)]);
          if (pair == 0) out[(long long)cur.c * N + cur.x0 + i] = sv;
          else { float* o = out + (long long)(cur.x0 + i) * N + cur.c; *o = *o + sv; }
        }
      } else {
        pass_b_last_dispatch<false>(R_last, in, P, NBp, l_last, NB, XB, nullptr, PK, out, pair,
                                    cur.c, cur.x0, scale, N, stage);
        if (pair == 1) {
          __syncthreads();
          pass_b_flush_h(stage, P, NB, XB, cur.c, cur.x0, out, N);
        }
      }
    }
    if (tn >= nitems) break;
    __syncthreads();                                  // Fb[0], Wk, PK reads done
    fill(nxt, 0);
    t = tn;
    cur = nxt;
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
  return (size_t)4 * g.NB * pitch_for(g.XB + NBp) * sizeof(float);
}

static int resident_grid(const void* kernel, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kThreads, smem);
  if (per < 1) per = 1;
  return sms * per;
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
  const long long ntiles = (long long)((g.W + g.XA - 1) / g.XA) * g.NB * slices * nf;
  const long long grid = std::min<long long>(ntiles, resident_grid((const void*)k_fht_a, smem));
  k_fht_a<<<(unsigned)grid, kThreads, smem, st>>>(lin, R, g, P, f0, nf, lin_slice_stride, ntiles);
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
  const long long nitems = (long long)((g.N + g.XB - 1) / g.XB) * g.H * slices;
  const long long grid = std::min<long long>(nitems, resident_grid((const void*)k_fht_b, smem));
  k_fht_b<<<(unsigned)grid, kThreads, smem, st>>>(R, img, g, P, pair, scale, nitems);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
