// Fast path of the hot path:
//
//   k_sweep_a : recursive ramp filter (§3 Eq.12-13) fused with the
//               first k1 FHT levels (§4.4), one CTA per
//               (slice, family, block of H = 2^k1 linogram rows), sweeping along s
//               in tiles of X columns.  The linogram is read from HBM once; the
//               filtered rows F never leave shared memory.
//   k_pair_b  : the last m FHT levels of an Eq.22 family pair,
//               mirror-add, weight and store.
//
// IIR in the sweep.  Every row is split into 32-sample chunks (TPR = X/32 chunks
// of a row per tile, one per thread).  Zero-state sweeps of both directions run
// packed in f32x2 (.x causal at sample i, .y anticausal at sample 31-i); chunk
// carries are combined by a Kogge-Stone scan over the TPR chunks of the row with
// A^32, A^64.  The causal carry into a tile is exact (the sweep goes left to
// right; each row is zero left of N - t, R2 of DESIGN.md).  The anticausal carry
// into tile j is sum_{i=1..D} (A^X)^(i-1) agg[j+i], agg[t] being the anticausal
// state at the left edge of tile t produced by the inputs inside tile t; tiles
// beyond j + D are dropped, and D is chosen by the plan so that the dropped tail
// of the impulse response is below 1e-9 of its l1 norm (R22).
// Delayed finalisation: each raw tile t is landed by TMA once; its "front" step
// runs both recursions with zero anticausal state at the tile's right edge, keeps
// agg[t] (chunk 0's inclusive suffix state) in a shared-memory ring and parks the
// partial output P(t) = y+ + y-_0 in tensor memory (tcgen05.st, 32 columns of the
// thread's own lane).  D steps later its "back" step loads P(t) (tcgen05.ld), adds
// the anticausal homogeneous response of the carry (plan table GA, packed FFMA2)
// and hands F(t) to the FHT steps.  No tile is reduced twice.
//
// FHT items.  A radix-2^R step after l levels computes, for 2^R consecutive
// blocks of 2^l rows and one channel c (PAPER.md recursion):
//   out[G*2^(l+R) + c*2^R + r'][u] = sum_{b'<2^R} in[(G*2^R + b')*2^l + c][u - c*b' - d^(R)_{r'}(b')]
// Each thread owns one item (2^R rows x C columns) per step: it loads the 2^R
// pre-shifted input windows with LDS.128 (rows are stored shifted right by their
// next pre-shift mod 4, so every window is 16-byte aligned), runs R levels in
// registers with compile-time shifts and stores C columns per output row.  Halo
// columns of every step's input are carried from tile to tile, so no level is
// recomputed for halos.
#include "fbp_internal.h"

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

// Developer timing mask (env FBP_DBG, tools/dev_timing.py: skip TMA loads / FHT
// steps / epilogue to attribute time) -- compiled in only with -DFBP_DEV_MASK=1
// (fbp_internal.h).

#ifndef FBP_KS_PFD
#define FBP_KS_PFD 2   // sweep: TMA L2 prefetch distance in tiles (measured: 1-2 best, 4 +1 %, 8 +3 %)
#endif

#ifndef FBP_KB_SKIP
#define FBP_KB_SKIP 1   // pass B step 1: skip halo items no step-2 pre-shift reads
#endif

namespace fbp {

namespace {

extern __shared__ float sm[];

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float4 ld4(int off) { return *reinterpret_cast<const float4*>(sm + off); }
__device__ __forceinline__ void st4(int off, float4 v) { *reinterpret_cast<float4*>(sm + off) = v; }

__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// streaming stores of the compact R rows (read back only by the next launch)
__device__ __forceinline__ void st_ef(float* g, float v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;\n" ::"l"(g), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_ef2(float* g, float a, float b, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(g), "f"(a), "f"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_ef4(float* g, float a, float b, float c, float d, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(g), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}
// ---- TMA (cp.async.bulk.tensor) + mbarrier ----
__device__ __forceinline__ unsigned smem_u32(int off) { return (unsigned)__cvta_generic_to_shared(sm + off); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// 2D tile box (cols c0.., rows r0..) of the linogram -> shared memory, completing on `bar`.
// Out-of-range columns (c0 < 0 or beyond 2N) are zero-filled by the TMA unit.
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int r0, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(r0), "r"(bar)
      : "memory");
}


__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// L2 prefetch of a tensor box (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];\n"
               ::"l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n"
               ::"l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1) : "memory");
}


// Row pitch (floats) for a row of at least w floats: a multiple of 4 whose quad
// count is odd, so that 8 consecutive rows map the same column to 8 distinct
// 4-bank groups (conflict-free LDS/STS.128 for "8 rows x 1 quad" access).
__host__ __device__ constexpr int pitch4(int w) { return (((w + 3) / 4) | 1) * 4; }

// Pass-B step-2 input halo: the window offset O2 plus the largest pre-shift
// (2^R1 - 1)(2^R2 - 1) rounded down to quads, then rounded up to the step-1 item
// width so that step 1 tiles [0, HS + XB) exactly.
__host__ __device__ constexpr int pb_halo(int R1, int R2) {
  return ((((R2 == 3) ? 8 : 4) + 4 * ((((1 << R1) - 1) * ((1 << R2) - 1)) / 4)) + ((R1 == 3) ? 4 : 8) - 1) /
         ((R1 == 3) ? 4 : 8) * ((R1 == 3) ? 4 : 8);
}

// Register item geometry: radix 2^R, C output columns; halo quads HQ >= (2^R-1)/4,
// window T = C + O columns with the outputs at window offset O.
template <int R, int C>
struct It {
  static constexpr int NR = 1 << R;
  static constexpr int HQ = (NR - 1 + 3) / 4;
  static constexpr int O = 4 * HQ;
  static constexpr int T = C + O;
};

// Load the NR pre-shifted windows of an item.  `w0` = float offset of the window
// start (virtual column col0 - O) of input row b' = 0; row b' lives at
// w0 + b'*rowstep, pre-shift c*b' (the physical shift (c*b') & 3 was applied by
// the producer, so the physical window starts 4*floor(c*b'/4) columns left).
// Rows are held as column pairs (float2) so that the levels can add two columns
// per FADD2 where the shift is even.
template <int R, int C>
__device__ __forceinline__ void item_load(int w0, int rowstep, int c,
                                          float2 (&v)[It<R, C>::NR][It<R, C>::T / 2]) {
  constexpr int NR = It<R, C>::NR, T = It<R, C>::T;
  int cb = 0;
#pragma unroll
  for (int b = 0; b < NR; ++b) {
    const int off = w0 + b * rowstep - (cb & ~3);
    cb += c;
#pragma unroll
    for (int q = 0; q < T / 4; ++q) {
      const float4 f = ld4(off + 4 * q);
      v[b][2 * q] = make_float2(f.x, f.y);
      v[b][2 * q + 1] = make_float2(f.z, f.w);
    }
  }
}

template <int T2>
__device__ __forceinline__ float col(const float2 (&row)[T2], int t) {
  return (t & 1) ? row[t >> 1].y : row[t >> 1].x;
}

// R levels in registers (natural recursion, compile-time shifts), computing at each
// level only the window columns the outputs [O, T) depend on.
//   level h -> 2h:  w[blk + y'][t] = v[blk + lo][t] + v[blk + h + lo][t - ceil(y'/2)],
//   lo = floor(y'/2)  (negative shift direction)
// Even shifts: one FADD2 per column pair; odd shifts: two FADDs.
template <int R, int C>
__device__ __forceinline__ void item_fht(float2 (&v)[It<R, C>::NR][It<R, C>::T / 2]) {
  constexpr int NR = It<R, C>::NR, T = It<R, C>::T, O = It<R, C>::O, T2 = T / 2;
#pragma unroll
  for (int lvl = 0; lvl < R; ++lvl) {
    const int h = 1 << lvl;
    const int lb = O - ((1 << R) - (1 << (lvl + 1)));   // even
    float2 w[NR][T2];
#pragma unroll
    for (int y = 0; y < NR; ++y) {
      const int blk = y & ~(2 * h - 1);
      const int yp = y - blk;
      const int lo = yp >> 1;
      const int sh = (yp + 1) >> 1;
#pragma unroll
      for (int tp = lb / 2; tp < T2; ++tp) {
        const int t = 2 * tp;
        const float2 a = v[blk + lo][tp];
        if ((sh & 1) == 0) {
          w[y][tp] = (t >= sh) ? __fadd2_rn(a, v[blk + h + lo][tp - sh / 2]) : a;
        } else {
          w[y][tp].x = (t >= sh) ? a.x + col(v[blk + h + lo], t - sh) : a.x;
          w[y][tp].y = (t + 1 >= sh) ? a.y + col(v[blk + h + lo], t + 1 - sh) : a.y;
        }
      }
    }
#pragma unroll
    for (int y = 0; y < NR; ++y)
#pragma unroll
      for (int tp = lb / 2; tp < T2; ++tp) v[y][tp] = w[y][tp];
  }
}

// ---------------------------------------------------------------- IIR pieces
struct P3 {   // a 3-state pair: .x causal, .y anticausal
  float2 s0, s1, s2;
};

__device__ __forceinline__ P3 mv(const float2 (&M)[9], const P3& v) {
  P3 o;
  o.s0 = __fmul2_rn(M[0], v.s0);
  o.s0 = __ffma2_rn(M[1], v.s1, o.s0);
  o.s0 = __ffma2_rn(M[2], v.s2, o.s0);
  o.s1 = __fmul2_rn(M[3], v.s0);
  o.s1 = __ffma2_rn(M[4], v.s1, o.s1);
  o.s1 = __ffma2_rn(M[5], v.s2, o.s1);
  o.s2 = __fmul2_rn(M[6], v.s0);
  o.s2 = __ffma2_rn(M[7], v.s1, o.s2);
  o.s2 = __ffma2_rn(M[8], v.s2, o.s2);
  return o;
}

// scalar 3x3 matvec using the .x lane of the duplicated matrix: acc + M v
__device__ __forceinline__ void mv1(const float2 (&M)[9], const float (&v)[3], float (&acc)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float s = acc[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) s = fmaf(M[3 * i + j].x, v[j], s);
    acc[i] = s;
  }
}

// Zero-state sweeps of one 32-sample chunk, packed: .x causal at sample i (left to
// right), .y anticausal at sample 31 - i (right to left).  Eq.13 with difference-
// form feedforward (R16): u = beta x + c0 D[n] + c1 D[n-1], D[n] = x[n] - x[n-1]
// (anticausal: E[n] = x[n] - x[n+1], E[n+1]).  xl = x[-1], x[-2]; xr = x[32], x[33].
template <bool BETA>
__device__ __forceinline__ void chunk_sweep(const float (&x)[32], float xl0, float xl1, float xr0,
                                            float xr1, const SweepIir& k, float2 (&yp)[32], float sx0 = 0.f,
                                            float sx1 = 0.f, float sx2 = 0.f) {
  // (sx0, sx1, sx2) = causal state (y[-1], y[-2], y[-3]) at the chunk start (0: zero state)
  float2 dprev = make_float2(xl0 - xl1, xr0 - xr1);
  float2 y1 = make_float2(sx0, 0.f), y2 = make_float2(sx1, 0.f), y3 = make_float2(sx2, 0.f);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float2 d;
    d.x = x[i] - (i == 0 ? xl0 : x[i - 1]);
    d.y = x[31 - i] - (i == 0 ? xr0 : x[32 - i]);
    float2 u = __fmul2_rn(k.c1, dprev);
    u = __ffma2_rn(k.c0, d, u);
    if (BETA) {
      u.x = fmaf(k.beta.x, x[i], u.x);
      u.y = fmaf(k.beta.x, x[31 - i], u.y);
    }
    float2 v = __ffma2_rn(k.na3, y3, u);
    v = __ffma2_rn(k.na2, y2, v);
    v = __ffma2_rn(k.na1, y1, v);
    y3 = y2;
    y2 = y1;
    y1 = v;
    dprev = d;
    yp[i] = v;
  }
}

}  // namespace

// ===========================================================================
// Pass A sweep.  Threads NT = H*X/32 = 128 (thread = one 32-sample chunk of a row
// in the IIR, one register item in the FHT steps).  Shared memory (floats):
//   F      : H x PF  landing target of raw tile t (TMA box, columns tX-8 ..
//            tX+X+4) and, once the IIR has read it, the filtered tile F(t-D):
//            halo [0, HF) = F(t-D-1)'s last HF columns, core [HF, HF+X)
//   (stash : the core's last HF columns, the halo of the next F tile, in registers)
//   S1     : H x PS  step-1 output, core [HS, HS+X), halo [0, HS)
//   ring   : (D+1) x H x 3  anticausal tile aggregates agg[t]
// Tensor memory (IIR): (D+1) slots x 32 columns per thread (its own lane): the
// tile's partial output P(t) = y+(t) + y-_0(t), y-_0 with zero anticausal state at
// the tile's right edge, waiting D tiles for its anticausal carry.
// ===========================================================================
// S1 halo copy plan of the sweep: row (b', c) of step 2 reads S1 virtual columns
// >= HS - O2 - c*b' only, so at the end of a tile only the quads
// qd < (O2 + (c*b' & ~3))/4 + 1 of each row (cols HS - 4 qd ..) move to the halo.
// The needed (row, quad) pairs in row-major order are dealt round-robin to the NT
// threads; v[kk*NT + t] = S1 offset of thread t's kk-th quad, 0xffff for none.
template <int H, int HS, int O2, int PS, int NT>
struct HaloTab {
  static constexpr int MAXQ = (HS + 4) / 4;
  static constexpr int count() {
    int n = 0;
    for (int rr = 0; rr < H; ++rr) {
      const int cb = (rr & 7) * (rr >> 3);
      const int nq = (O2 + (cb & ~3)) / 4 + 1;
      n += nq < MAXQ ? nq : MAXQ;
    }
    return n;
  }
  static constexpr int NKH = (count() + NT - 1) / NT;
  unsigned short v[NKH * NT];
  constexpr HaloTab() : v() {
    for (int i = 0; i < NKH * NT; ++i) v[i] = 0xffff;
    int n = 0;
    for (int rr = 0; rr < H; ++rr) {
      const int cb = (rr & 7) * (rr >> 3);
      int nq = (O2 + (cb & ~3)) / 4 + 1;
      if (nq > MAXQ) nq = MAXQ;
      for (int qd = 0; qd < nq; ++qd, ++n) v[n] = (unsigned short)(rr * PS + HS - 4 * qd);
    }
  }
};
template <int H, int HS, int O2, int PS, int NT>
__device__ constexpr HaloTab<H, HS, O2, PS, NT> kHaloTab{};

// The same plan per step-1 row group G (S1 rows 8G .. 8G+7, written by the step-1
// items of group G): the group's own threads copy its quads, so no CTA barrier is
// needed between this copy and the group's next step 1.
template <int H, int HS, int O2, int PS>
struct HaloTabG {
  static constexpr int MAXQ = (HS + 4) / 4;
  static constexpr int NG = H / 8;
  static constexpr int CAP = 8 * MAXQ;
  unsigned short cnt[NG];
  unsigned short v[NG][CAP];
  constexpr HaloTabG() : cnt(), v() {
    for (int G = 0; G < NG; ++G) {
      int n = 0;
      for (int r = 0; r < 8; ++r) {
        const int rr = 8 * G + r;
        const int cb = (rr & 7) * (rr >> 3);
        int nq = (O2 + (cb & ~3)) / 4 + 1;
        if (nq > MAXQ) nq = MAXQ;
        for (int qd = 0; qd < nq; ++qd) v[G][n++] = (unsigned short)(rr * PS + HS - 4 * qd);
      }
      cnt[G] = (unsigned short)n;
      for (; n < CAP; ++n) v[G][n] = 0xffff;
    }
  }
};
template <int H, int HS, int O2, int PS>
__device__ constexpr HaloTabG<H, HS, O2, PS> kHaloTabG{};

// ---- tensor memory (tcgen05): one 32-column slot of a thread's own lane ----
__device__ __forceinline__ void tmem_st32(unsigned taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]),
        "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]),
        "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

template <int H, int X, bool IIR, bool BETA>
// resident CTAs per SM the register budget is sized for: 4 for the H = 32 sweep (N = 512,
// 1024: 128 registers without spills; r02 s6 A/B: KS -12 % / -8 %), 3 for H = 64
// (N = 2048, 4096: 4 measured 25 % slower, 64 B of spills and no L1 left)
#ifndef FBP_KS_MINB
#define FBP_KS_MINB (H == 32 ? 4 : 3)
#endif
__global__ void __launch_bounds__(H * X / 32, FBP_KS_MINB)
    k_sweep_a(const float* __restrict__ lin, float* __restrict__ Rout, SweepGeom g, SweepIir k, int slices, int f0,
              int nf, long long lin_slice_stride, int nseg, int* __restrict__ counter,
              const __grid_constant__ CUtensorMap tmapF) {
  constexpr int NT = H * X / 32;
  constexpr int TPR = X / 32;                 // chunks (threads) per row in the IIR
  constexpr int R2 = (H == 64) ? 3 : 2;       // k1 = 3 + R2
  constexpr int C1 = 4;
  constexpr int C2 = (R2 == 3) ? 4 : 8;
  constexpr int O2 = It<R2, C2>::O;
  constexpr int NR2 = 1 << R2;
  constexpr int HF = 8;                        // step-1 input halo (>= 7)
  constexpr int HS = O2 + 4 * ((7 * (NR2 - 1)) / 4);   // step-2 input halo
  constexpr int PF = pitch4(HF + X + 4);
  constexpr int PS = pitch4(HS + X + 4);
  // F's last HF columns (the next tile's halo) stay in registers: chunk threads 0, 1
  // of a row keep one quad each (r02 s5: 2 KB less shared memory per CTA puts three
  // CTAs in the 164 KB carveout, doubling L1: KS 0.867 -> 0.839 ms)
  constexpr int oF = 0, oS = H * PF, oRing = oS + H * PS;
  static_assert(X >= HS + 4, "S1 halo copy must not overlap its source");
  static_assert(NT == 128, "TMEM lanes: one per thread");

  const int tid = threadIdx.x;
  const int D = IIR ? g.D : 0;
  const int dbgm = FBP_DEV_MASK ? g.dbg : 0;
  // 1 mbarrier (F landing), the work item, the TMEM base address
  const int oBar = (oRing + (D + 1) * H * 3 + 3) & ~1;
  int* s_item = reinterpret_cast<int*>(sm + oBar + 2);
  unsigned* s_tmem = reinterpret_cast<unsigned*>(sm + oBar + 3);
  if (tid == 0) {
    mbar_init(smem_u32(oBar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (IIR && tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(oBar + 3)),
                 "r"(g.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // this thread's TMEM lane: warp w owns lanes 32w .. 32w + 31
  const unsigned tbase = IIR ? (*s_tmem + ((unsigned)(tid & ~31) << 16)) : 0u;
  unsigned ph = 0;                                       // phase bit of the mbarrier
  const int N = g.N, W = g.W, NB = g.NB, nt = g.nt;
  const long long nsf = (long long)slices * nf;
  const long long nitems = nsf * NB * nseg;
  // IIR roles: a quarter-warp = 8 rows x the same chunk (conflict-free), the TPR
  // chunks of a row sit 8 lanes apart in one warp.
  // Step-1 row group of the thread Gt (rows 8Gt .. 8Gt+7): the IIR threads of a row
  // group are its step-1 threads (no CTA barrier between F and step 1).
  const int Gt = tid / (8 * TPR);
  const int iq = (tid >> 3) % TPR;
  const int ir = (tid & 7) + 8 * Gt;
  const int lane = tid & 31;
  const unsigned long long pol_ef = policy_evict_first();

  while (true) {
    __syncthreads();
    if (tid == 0) *s_item = atomicAdd(counter, 1);
    __syncthreads();
    const long long item = *s_item;
    if (item >= nitems) break;
    // item = (block b, slice*family, segment): longest sweeps first, a sweep's
    // segments adjacent
    const int seg = (int)(item % nseg);
    const long long it2 = item / nseg;
    const int b = NB - 1 - (int)(it2 / nsf);
    const long long sfi = it2 - (long long)(NB - 1 - b) * nsf;
    const long long s = sfi / nf;
    const int fi = (int)(sfi - s * nf);
    const int f = f0 + fi;
    // compact R layout [slice][family][cf][b][WR]: pass B reads, for one channel cf,
    // the NB rows b as one contiguous box
    float* dstR = Rout + (((s * 4 + f) * (long long)H) * NB + b) * g.WR;
    // First tile with an output pass B reads: every stored R column u >= N - b*H
    // depends on F at u - (H-1) >= N - (b+1)H + 1 only.  The IIR starts D tiles
    // earlier (causal warm-up, R22): linogram rows need not be zero left of N - t
    // (noisy inputs, configs 2, 4, 5).
    const int j0 = (N - (b + 1) * H + 1) / X;
    // Segments (small batches): segment seg stores the tiles [ja, jb) of [j0, nt);
    // it runs step 1 from j1 = ja - 1 (the S1 halo of tile ja; segment 0 needs none)
    const int seglen = (nt - j0 + nseg - 1) / nseg;
    const int ja = j0 + seg * seglen, jb = min(nt, ja + seglen);
    if (ja >= jb) continue;
    const int j1 = (seg == 0) ? j0 : ja - 1;
    // front tiles t (IIR of raw tile t) run D tiles ahead of the back tiles j = t - D
    // (anticausal carry of tile j from agg[j+1 .. j+D], R22; F(j) -> FHT)
    const int jst = IIR ? max(0, j1 - D) : j1;
    const int tend = jb + D;

    const int trow = (int)((s * 4 + fi) * N + (long long)b * H);
    auto land = [&](int jt) {
      if (tid == 0 && !(dbgm & 8)) {
        fence_proxy_async();
        const unsigned bar = smem_u32(oBar);
        mbar_expect_tx(bar, H * PF * 4);
        tma_load_2d(smem_u32(oF), &tmapF, jt * X - 8, trow, bar);
      }
    };
    auto tma_wait = [&]() {
      if (!(dbgm & 8)) mbar_wait(smem_u32(oBar), ph & 1);
      ph ^= 1u;
    };
    // L2 prefetch of raw tile jt (TMA, no shared memory): the landing of a tile is
    // issued one step ahead, its first touch of HBM PF tiles ahead
    constexpr int PFD = FBP_KS_PFD;
    auto prefetch = [&](int jt) {
      if (tid == 0 && jt < nt && !(dbgm & 8)) tma_prefetch_2d(&tmapF, jt * X - 8, trow);
    };
    land(jst);
    for (int i = 1; i <= PFD; ++i) prefetch(jst + i);
    // S1 halo of the first stored tile: zero (its outputs are never read, but keep
    // them finite)
    for (int e = tid; e < H * (HS / 4); e += NT) {
      const int r = e / (HS / 4), qd = e - r * (HS / 4);
      st4(oS + r * PS + 4 * qd, make_float4(0.f, 0.f, 0.f, 0.f));
    }
    float cin0 = 0.f, cin1 = 0.f, cin2 = 0.f;           // causal carry of the row
    float4 stash = make_float4(0.f, 0.f, 0.f, 0.f);     // F(j)'s last HF columns, this thread's quad
    int slot_t = 0;                                      // ring / TMEM slot of tile t: (t - jst) mod (D+1)

    for (int t = jst; t < tend; ++t, slot_t = (slot_t == D) ? 0 : slot_t + 1) {
      const int j = t - D;
      const bool back = j >= j1;
      if (IIR) {
        if (t < nt) tma_wait();                          // raw tile t landed
        if (t < nt && !(dbgm & 32)) {
          // ---- front: zero-state sweeps of this thread's chunk ----
          const int rowF = oF + ir * PF + HF + 32 * iq;
          float x[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v = ld4(rowF + 4 * q);
            x[4 * q] = v.x;
            x[4 * q + 1] = v.y;
            x[4 * q + 2] = v.z;
            x[4 * q + 3] = v.w;
          }
          const float4 vl = ld4(rowF - 4);
          const float4 vr = ld4(rowF + 32);
          float2 yp[32];
          if constexpr (TPR == 2) {
            // Two chunks per tile row: chunk 0's causal recursion starts from the exact
            // carry of the previous tile and chunk 1's anticausal one from the tile's
            // right edge (zero state), so only chunk 1 .x and chunk 0 .y need an in-tile
            // carry -- the partner chunk's end state (one exchange, no scan) -- and the
            // fix-up runs on one lane per thread.
            const bool c0 = (iq == 0);
            chunk_sweep<BETA>(x, vl.w, vl.z, vr.x, vr.y, k, yp, c0 ? cin0 : 0.f, c0 ? cin1 : 0.f, c0 ? cin2 : 0.f);
            const float e0 = c0 ? yp[31].x : yp[31].y, e1 = c0 ? yp[30].x : yp[30].y, e2 = c0 ? yp[29].x : yp[29].y;
            // chunk 1 receives chunk 0's exact causal end state, chunk 0 chunk 1's
            // zero-state anticausal state at its left edge
            float h1 = __shfl_xor_sync(0xffffffffu, e0, 8);
            float h2 = __shfl_xor_sync(0xffffffffu, e1, 8);
            float h3 = __shfl_xor_sync(0xffffffffu, e2, 8);
            const float2 msk = c0 ? make_float2(0.f, 1.f) : make_float2(1.f, 0.f);
            const float na1 = k.na1.x, na2 = k.na2.x, na3 = k.na3.x;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              float hh = na3 * h3;
              hh = fmaf(na2, h2, hh);
              hh = fmaf(na1, h1, hh);
              h3 = h2;
              h2 = h1;
              h1 = hh;
              yp[i] = __ffma2_rn(make_float2(hh, hh), msk, yp[i]);
            }
            // causal carry of the next tile: chunk 1's corrected end state; agg[t]:
            // chunk 0's corrected anticausal state at the tile's left edge
            const int src1 = lane | 8;
            cin0 = __shfl_sync(0xffffffffu, yp[31].x, src1);
            cin1 = __shfl_sync(0xffffffffu, yp[30].x, src1);
            cin2 = __shfl_sync(0xffffffffu, yp[29].x, src1);
            if (c0) {
              const int o = oRing + (slot_t * H + ir) * 3;
              sm[o] = yp[31].y;
              sm[o + 1] = yp[30].y;
              sm[o + 2] = yp[29].y;
            }
          } else {
          chunk_sweep<BETA>(x, vl.w, vl.z, vr.x, vr.y, k, yp);
          // carries: inclusive scan over the row's chunks, causal up (seeded with the
          // exact carry of the previous tile), anticausal down with zero state at the
          // tile's right edge (its true carry is added D tiles later)
          P3 S;
          S.s0 = make_float2(yp[31].x, yp[31].y);
          S.s1 = make_float2(yp[30].x, yp[30].y);
          S.s2 = make_float2(yp[29].x, yp[29].y);
          if (iq == 0) {
            P3 E;
            E.s0 = make_float2(cin0, 0.f);
            E.s1 = make_float2(cin1, 0.f);
            E.s2 = make_float2(cin2, 0.f);
            const P3 ME = mv(k.M1, E);
            S.s0.x += ME.s0.x;
            S.s1.x += ME.s1.x;
            S.s2.x += ME.s2.x;
          }
#pragma unroll
          for (int st = 0; (1 << st) < TPR; ++st) {
            const int off = 8 << st;
            P3 o;
            o.s0 = make_float2(__shfl_up_sync(0xffffffffu, S.s0.x, off), __shfl_down_sync(0xffffffffu, S.s0.y, off));
            o.s1 = make_float2(__shfl_up_sync(0xffffffffu, S.s1.x, off), __shfl_down_sync(0xffffffffu, S.s1.y, off));
            o.s2 = make_float2(__shfl_up_sync(0xffffffffu, S.s2.x, off), __shfl_down_sync(0xffffffffu, S.s2.y, off));
            const P3 tt = (st == 0) ? mv(k.M1, o) : mv(k.M2, o);
            if (iq >= (1 << st)) {
              S.s0.x += tt.s0.x;
              S.s1.x += tt.s1.x;
              S.s2.x += tt.s2.x;
            }
            if (iq + (1 << st) < TPR) {
              S.s0.y += tt.s0.y;
              S.s1.y += tt.s1.y;
              S.s2.y += tt.s2.y;
            }
          }
          // exclusive carries of this chunk
          P3 cc;
          {
            const float u0 = __shfl_up_sync(0xffffffffu, S.s0.x, 8);
            const float u1 = __shfl_up_sync(0xffffffffu, S.s1.x, 8);
            const float u2 = __shfl_up_sync(0xffffffffu, S.s2.x, 8);
            const float d0 = __shfl_down_sync(0xffffffffu, S.s0.y, 8);
            const float d1 = __shfl_down_sync(0xffffffffu, S.s1.y, 8);
            const float d2 = __shfl_down_sync(0xffffffffu, S.s2.y, 8);
            cc.s0 = make_float2(iq == 0 ? cin0 : u0, iq == TPR - 1 ? 0.f : d0);
            cc.s1 = make_float2(iq == 0 ? cin1 : u1, iq == TPR - 1 ? 0.f : d1);
            cc.s2 = make_float2(iq == 0 ? cin2 : u2, iq == TPR - 1 ? 0.f : d2);
          }
          // causal carry for the next tile: inclusive state of the row's last chunk;
          // agg[t] (anticausal zero-state state at the tile's left edge) = chunk 0's
          // inclusive suffix state
          {
            const int srcl = (lane & 7) | (8 * (TPR - 1)) | (lane & ~(8 * TPR - 1));
            cin0 = __shfl_sync(0xffffffffu, S.s0.x, srcl);
            cin1 = __shfl_sync(0xffffffffu, S.s1.x, srcl);
            cin2 = __shfl_sync(0xffffffffu, S.s2.x, srcl);
          }
          if (iq == 0) {
            const int o = oRing + (slot_t * H + ir) * 3;
            sm[o] = S.s0.y;
            sm[o + 1] = S.s1.y;
            sm[o + 2] = S.s2.y;
          }
          // fix-up with the in-tile carries: homogeneous response of the recursion
          // from the carry-in state, packed (.x causal, .y anticausal).  (A plan-table
          // form, 3 FFMA2 per sample without the chain, measured slower: r02.)
          {
            float2 h1 = cc.s0, h2 = cc.s1, h3 = cc.s2;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              float2 h = __fmul2_rn(k.na3, h3);
              h = __ffma2_rn(k.na2, h2, h);
              h = __ffma2_rn(k.na1, h1, h);
              h3 = h2;
              h2 = h1;
              h1 = h;
              yp[i] = __fadd2_rn(yp[i], h);
            }
          }
          }   // TPR > 2
          // P(t) = y+ + y-_0 -> tensor memory slot
          // (the slot's previous content, P(t - D - 1), was loaded by the last back step)
          float P[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) P[i] = yp[i].x + yp[31 - i].y;
          tmem_st32(tbase + 32u * slot_t, P);
        } else if (iq == 0) {                            // beyond the row: agg = 0
          const int o = oRing + (slot_t * H + ir) * 3;
          sm[o] = 0.f;
          sm[o + 1] = 0.f;
          sm[o + 2] = 0.f;
        }
        // every read of a row's raw data, and its ring entries, stay inside the row's
        // warp (row r is chunks of threads in one warp; its F and halo writes too)
        __syncwarp();
        if (back && !(dbgm & 64)) {
          // ---- back: F(j) = P(j) + anticausal homogeneous response of the carry ----
          // T_j = sum_{i=1..D} (A^X)^(i-1) agg[j+i] at tile j's right edge (Horner)
          float tm[3];
          {
            int sl = slot_t;                             // slot of tile j + D = t
            tm[0] = sm[oRing + (sl * H + ir) * 3];
            tm[1] = sm[oRing + (sl * H + ir) * 3 + 1];
            tm[2] = sm[oRing + (sl * H + ir) * 3 + 2];
            for (int i = D - 1; i >= 1; --i) {
              sl = (sl == 0) ? D : sl - 1;               // slot of tile j + i
              float acc[3] = {sm[oRing + (sl * H + ir) * 3], sm[oRing + (sl * H + ir) * 3 + 1],
                              sm[oRing + (sl * H + ir) * 3 + 2]};
              mv1(k.MX, tm, acc);
              tm[0] = acc[0];
              tm[1] = acc[1];
              tm[2] = acc[2];
            }
          }
          // carry at this chunk's right edge: A^(32 (TPR-1-iq)) T_j
#pragma unroll
          for (int q = 0; q < TPR - 1; ++q) {
            if (q < TPR - 1 - iq) {
              float acc[3] = {0.f, 0.f, 0.f};
              mv1(k.M1, tm, acc);
              tm[0] = acc[0];
              tm[1] = acc[1];
              tm[2] = acc[2];
            }
          }
          const int slot_j = slot_t == D ? 0 : slot_t + 1;   // slot of tile j = t - D
          float P[32];
          tmem_wait_st();
          tmem_ld32(tbase + 32u * slot_j, P);
          const int rowF = oF + ir * PF + HF + 32 * iq;
          // homogeneous anticausal response at sample i: sum_m (A^(32-i))_{0m} tm_m,
          // adjacent samples packed (plan table k.GA)
          const float2 t0 = make_float2(tm[0], tm[0]), t1 = make_float2(tm[1], tm[1]),
                       t2 = make_float2(tm[2], tm[2]);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float2 a = make_float2(P[4 * q], P[4 * q + 1]);
            float2 c = make_float2(P[4 * q + 2], P[4 * q + 3]);
            a = __ffma2_rn(k.GA[2 * q][0], t0, a);
            a = __ffma2_rn(k.GA[2 * q][1], t1, a);
            a = __ffma2_rn(k.GA[2 * q][2], t2, a);
            c = __ffma2_rn(k.GA[2 * q + 1][0], t0, c);
            c = __ffma2_rn(k.GA[2 * q + 1][1], t1, c);
            c = __ffma2_rn(k.GA[2 * q + 1][2], t2, c);
            st4(rowF + 4 * q, make_float4(a.x, a.y, c.x, c.y));
          }
        }
      } else {
        tma_wait();                                      // raw tile j = F(j) landed
      }
      if (back && iq < 2) {
        // halo: F(j-1)'s last HF columns (zero at the first back tile), written by the
        // row's own chunk threads 0 and 1
        const float4 h = (j == j1) ? make_float4(0.f, 0.f, 0.f, 0.f) : stash;
        st4(oF + ir * PF + 4 * iq, h);
      }
      // F(j) rows 8G .. 8G+7 are complete: they were written by the same threads that
      // run step 1 on them (row group G = the IIR threads of rows 8G..8G+7)
      __syncwarp();
      if (back && !(dbgm & 1)) {
        // ---- FHT step 1 (levels 1-3): F -> S1 ----
        constexpr int NCH = X / C1;
        static_assert(NCH == 8 * TPR, "step-1 row group = the IIR threads of its rows");
        const int jj = tid % NCH, G = Gt;
        float2 v[8][It<3, C1>::T / 2];
        item_load<3, C1>(oF + (G * 8) * PF + C1 * jj, PF, 0, v);   // HF + C1*jj - O(=8)
        item_fht<3, C1>(v);
        const int gb = G & (NR2 - 1);                   // next step's block index
        // outputs shifted by their step-2 pre-shift (r*gb) mod 4 (scalar stores: the
        // aligned-store alternatives measured slower)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int o = oS + (G * 8 + r) * PS + HS + C1 * jj + ((r * gb) & 3);
#pragma unroll
          for (int tt = 0; tt < C1; ++tt) sm[o + tt] = col(v[r], It<3, C1>::O + tt);
        }
      }
      // stash this tile's last HF filtered columns (halo of the next tile), row owners
      if (back && iq < 2) stash = ld4(oF + ir * PF + X + 4 * iq);
      __syncthreads();                                   // F read by all (landing); S1 complete (step 2)
      // F is free: land the next raw tile
      if (IIR) {
        if (t + 1 < nt && t + 1 < tend) land(t + 1);
        prefetch(t + 1 + PFD);
      } else if (j + 1 < jb) {
        land(j + 1);
        if (j + 1 + PFD < jb) prefetch(j + 1 + PFD);
      }
      if (back && j >= ja && !(dbgm & 2)) {
        // ---- FHT step 2 (levels 4..k1): S1 -> R (compact, only the columns pass B reads)
        // Items whose NR2 channels cf = c*NR2 + r need none of their columns (u outside
        // [N - b(cf+1), 2N - cf*b) for every r) are skipped: up to half of them for
        // the high blocks b.
        constexpr int NCH2 = X / C2;
        const int jj = tid % NCH2, c = tid / NCH2;
        const int ubase = j * X + C2 * jj;
        const bool need2 = (ubase + C2 > N - b * (c * NR2 + NR2)) && (ubase < W - c * NR2 * b);
        if (need2) {
          float2 v[NR2][It<R2, C2>::T / 2];
          item_load<R2, C2>(oS + c * PS + HS + C2 * jj - O2, 8 * PS, c, v);
          item_fht<R2, C2>(v);
#pragma unroll
          for (int r = 0; r < NR2; ++r) {
            const int cf = c * NR2 + r;
            const int ulo = N - b * (cf + 1);
            const int uhi = W - cf * b;
            float* o = dstR + (long long)cf * NB * g.WR + (cf * b - N + NB);
            // alignment of the row's pre-shift, (cf*b) mod 4 = (r*b) mod 4: uniform over
            // the CTA item, so the vector width is chosen without divergence
            const int res = (r * b) & 3;
            if (ubase >= ulo && ubase + C2 <= uhi) {
              if (res == 0) {
#pragma unroll
                for (int tt = 0; tt < C2; tt += 4)
                  st_ef4(o + ubase + tt, col(v[r], O2 + tt), col(v[r], O2 + tt + 1), col(v[r], O2 + tt + 2),
                         col(v[r], O2 + tt + 3), pol_ef);
              } else if (res == 2) {
#pragma unroll
                for (int tt = 0; tt < C2; tt += 2)
                  st_ef2(o + ubase + tt, col(v[r], O2 + tt), col(v[r], O2 + tt + 1), pol_ef);
              } else {
#pragma unroll
                for (int tt = 0; tt < C2; ++tt) st_ef(o + ubase + tt, col(v[r], O2 + tt), pol_ef);
              }
            } else if (ubase + C2 > ulo && ubase < uhi) {
#pragma unroll
              for (int tt = 0; tt < C2; ++tt) {
                const int u = ubase + tt;
                if (u >= ulo && u < uhi) st_ef(o + u, col(v[r], O2 + tt), pol_ef);
              }
            }
          }
        }
      }
      __syncthreads();                                   // step 2's S1 reads precede the halo copy
      // ---- S1 halo for the next tile: row (b', c) of step 2 reads virtual columns
      //      >= HS - O2 - c*b' only, so copy just those quads (+ the shift quad) ----
      if (back) {
        constexpr int NCH = X / C1;                      // threads per step-1 row group
        using HG = HaloTabG<H, HS, O2, PS>;
        const int G = Gt, li = tid % NCH;
        const int cnt = kHaloTabG<H, HS, O2, PS>.cnt[G];
#pragma unroll 2
        for (int i = li; i < cnt; i += NCH) {
          const int off = kHaloTabG<H, HS, O2, PS>.v[G][i];
          st4(oS + off, ld4(oS + off + X));
        }
        (void)sizeof(HG);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (IIR && tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(*s_tmem), "r"(g.tmem_cols)
                 : "memory");
}

// ===========================================================================
// Pass B, one family pair (Eq.22): CTA item = (slice, pass-A channel ch, x-tile).
// Family 2p (q = 0) at x0, family 2p+1 (q = 1) at the mirrored tile N - x0 - XB.
// Input rows b of G_ch[b][v] = R_A[b][ch][v - ch*b] (compact layout; the
// pre-shift is addressing).  Step 1 (R1 levels) over [core - HS, core + XB),
// step 2 (R2 levels) over the core; the final rows are parked (aliasing the
// input buffer) and the pair epilogue mirrors, adds, weights and stores:
//   PAIR 0:  img[ch*NB + r][x0 + i]  = w (B0[r][i] + B1[r][XB-1-i])
//   PAIR 1:  img[x0 + i][ch*NB + r] += w (B2[r][i] + B3[r][XB-1-i])
// PAIR 1 adds its tile by a TMA tensor reduce (cp.reduce.async.bulk.tensor .add,
// performed in L2) from a staging tile behind the park; it runs after pair 0 in
// stream order, so every image element is pair 0's value plus one fp32 add, as
// before (bit-identical to a read-modify-write).  Both pairs run 3 CTAs per SM; the
// next item's boxes land while this one computes (double buffer).
// ===========================================================================
// Pass-B item position (slice, channel, x tile).  Items are visited with the grid
// stride; the stride is decomposed once and added with mixed-radix carries, so the
// loop needs no 64-bit division.
struct PbPos {
  int sl, ch, xi;
};
__device__ __forceinline__ PbPos pb_pos(long long t, int nx, int H) {
  const long long per = (long long)nx * H;
  PbPos p;
  p.sl = (int)(t / per);
  const int rem = (int)(t - (long long)p.sl * per);
  p.ch = rem / nx;
  p.xi = rem - p.ch * nx;
  return p;
}
__device__ __forceinline__ PbPos pb_add(PbPos a, const PbPos& d, int nx, int H) {
  a.xi += d.xi;
  if (a.xi >= nx) { a.xi -= nx; ++a.ch; }
  a.ch += d.ch;
  if (a.ch >= H) { a.ch -= H; ++a.sl; }
  a.sl += d.sl;
  return a;
}

__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, unsigned src, int c0, int r0) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];\n"
               ::"l"(reinterpret_cast<unsigned long long>(map)), "r"(src), "r"(c0), "r"(r0)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// First pass-B step-1 item (of C1 columns) of row group G that step 2 reads: the
// step-2 windows of row (G, r) start at virtual column HS - O2 - r*G (pre-shift r*G,
// r < 2^R1), so the items entirely left of HS - O2 - (2^R1 - 1)*G are never read.
template <int R1, int C1, int HS, int O2>
__host__ __device__ constexpr int pb_js(int G) {
  return (HS - O2 - ((1 << R1) - 1) * G) > 0 ? (HS - O2 - ((1 << R1) - 1) * G) / C1 : 0;
}
template <int R1, int C1, int HS, int O2, int NGF>
__host__ __device__ constexpr int pb_items(int nch) {
  int n = 0;
  for (int G = 0; G < NGF; ++G) n += nch - pb_js<R1, C1, HS, O2>(G);
  return n;
}

template <int R1, int R2, int XB, int PAIR, bool DB>
__global__ void __launch_bounds__(256, DB ? 3 : 2)
    k_pair_b(const float* __restrict__ Rin, float* __restrict__ img, SweepGeom g, float scale,
             long long nitems, const __grid_constant__ CUtensorMap tmapR,
             const __grid_constant__ CUtensorMap tmapI) {
  constexpr int NT = 256;
  constexpr int NB = 1 << (R1 + R2);
  constexpr int NR1 = 1 << R1, NR2 = 1 << R2;
  constexpr int C1 = (R1 == 3) ? 4 : 8;
  constexpr int C2 = (R2 == 3 || XB <= 64) ? 4 : 8;
  constexpr bool DIRECT = (R2 == 2);                  // step 2 + epilogue in registers (no park)
  constexpr int O1 = It<R1, C1>::O, O2 = It<R2, C2>::O;
  constexpr int HS = pb_halo(R1, R2);
  constexpr int HI = HS + O1;
  constexpr int RPT = NT / (2 * NB);                  // fill threads per input row
  constexpr int NQF = ((HI + XB) / 4 + RPT - 1) / RPT * RPT;   // filled quads per row
  constexpr int PI = pitch4(4 * NQF);
  constexpr int PS = pitch4(HS + XB + 4);
  constexpr int PK = PAIR == 0 ? XB + 4 : XB + 1;     // pair 1 reads park columns
  // DB: two input buffers, the next item's TMA boxes land while this item computes
  constexpr int NBUF = DB ? 2 : 1;
  // pair 1: reduce staging [XB][NB] behind the park, 128-byte aligned, in the input buffer
  constexpr int oStg = (2 * NB * PK + 31) / 32 * 32;
  constexpr int IN_SZ = (PAIR == 1 && oStg + XB * NB > 2 * NB * PI) ? oStg + XB * NB : 2 * NB * PI;
  constexpr int oIn0 = 0;                             // [NBUF][2 fam][NB][PI]; park aliases it
  constexpr int oS = NBUF * IN_SZ;                    // [2 fam][NB][PS]
  static_assert((HS + XB) % C1 == 0 && XB % C2 == 0, "pass-B item tiling");
  static_assert(2 * NB * PK <= 2 * NB * PI, "park must fit in the input buffer");
  static_assert(PAIR == 0 || oStg + XB * NB <= IN_SZ, "reduce staging must fit in the input buffer");
  static_assert((IN_SZ % 32) == 0, "input buffers 128-byte aligned");
  const int N = g.N, H = g.H;
  const int tid = threadIdx.x;
  const int dbgm = FBP_DEV_MASK ? g.dbg : 0;
  const int nx = (N + XB - 1) / XB;
  constexpr int oBar = oS + 2 * NB * PS;              // NBUF mbarriers (8-byte aligned)
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) mbar_init(smem_u32(oBar + 2 * i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;
  // TMA fills of item tt into buffer bb (thread 0): both families' NB compact rows
  // of channel ch (3D box PI x NB x 1, columns j' = xs - HI + NB.., zero-filled
  // outside the row); plus an L2 prefetch of the boxes of item tt + P*gridDim.x.
  // Pair 1: the buffer's previous reduce must have read its staging first.
  const int nsl = (int)(nitems / ((long long)nx * H));
  const PbPos step = pb_pos(gridDim.x, nx, H);
  const PbPos stepP = pb_pos((long long)g.P * gridDim.x, nx, H);
  auto issue = [&](const PbPos& pt, int bb) {
    if (tid != 0 || pt.sl >= nsl || (dbgm & 4)) return;
    if (g.P > 0) {
      const PbPos pp = pb_add(pt, stepP, nx, H);
      if (pp.sl < nsl) {
        const int x0p = pp.xi * XB;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int xs = (q == 0) ? x0p : (N - x0p - XB);
          tma_prefetch_3d(&tmapR, xs - HI + NB, 0, (pp.sl * 4 + 2 * PAIR + q) * H + pp.ch);
        }
      }
    }
    const int sl2 = pt.sl, ch2 = pt.ch, x02 = pt.xi * XB;
    if (PAIR == 1) bulk_wait_read_all();
    fence_proxy_async();
    const unsigned bar = smem_u32(oBar + 2 * bb);
    mbar_expect_tx(bar, 2u * NB * PI * 4);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int xs = (q == 0) ? x02 : (N - x02 - XB);
      tma_load_3d(smem_u32(oIn0 + bb * IN_SZ + q * NB * PI), &tmapR, xs - HI + NB, 0,
                  (sl2 * 4 + 2 * PAIR + q) * H + ch2, bar);
    }
  };
  PbPos cur = pb_pos(blockIdx.x, nx, H);
  issue(cur, 0);
  int bb = 0;

  for (; cur.sl < nsl; cur = pb_add(cur, step, nx, H)) {
    const int ch = cur.ch;
    const int x0 = cur.xi * XB;
    const int oIn = oIn0 + bb * IN_SZ;
    if (DB) issue(pb_add(cur, step, nx, H), bb ^ 1);   // buffer freed by the previous item
    // ---- fills by TMA: both families' NB compact rows of channel ch (3D box
    //      PI x 1 x NB, columns j' = xs - HI + NB.., zero-filled outside the row) ----
    if (!(dbgm & 4)) mbar_wait(smem_u32(oBar + 2 * bb), (ph >> bb) & 1);
    ph ^= 1u << bb;
    // ---- step 1: both families, output virtual cols [0, HS + XB) ----
    if (!(dbgm & 1)) {
      constexpr int nch = (HS + XB) / C1;
      constexpr int NGF = NB / NR1;                    // row groups per family
#if FBP_KB_SKIP
      // the items of group G left of pb_js(G) (halo columns no step-2 pre-shift
      // reaches) are skipped
      constexpr int per_fam = pb_items<R1, C1, HS, O2, NGF>(nch);
#else
      constexpr int per_fam = NGF * nch;
#endif
      for (int it = tid; it < 2 * per_fam; it += NT) {
        const int q = it / per_fam;
        const int r3 = it - q * per_fam;
#if FBP_KB_SKIP
        int G = 0, rem = r3;
#pragma unroll
        for (int gg = 0; gg + 1 < NGF; ++gg) {
          const int cnt = nch - pb_js<R1, C1, HS, O2>(gg);
          if (G == gg && rem >= cnt) {
            rem -= cnt;
            G = gg + 1;
          }
        }
        int js = 0;
#pragma unroll
        for (int gg = 0; gg < NGF; ++gg)
          if (G == gg) js = pb_js<R1, C1, HS, O2>(gg);
        const int jj = js + rem;
#else
        const int G = r3 / nch, jj = r3 - G * nch;
#endif
        float2 v[NR1][It<R1, C1>::T / 2];
        item_load<R1, C1>(oIn + (q * NB + G * NR1) * PI + C1 * jj, PI, 0, v);
        item_fht<R1, C1>(v);
        // outputs shifted by their step-2 pre-shift (r*G) mod 4
#pragma unroll
        for (int r = 0; r < NR1; ++r) {
          const int o = oS + (q * NB + G * NR1 + r) * PS + C1 * jj + ((r * G) & 3);
#pragma unroll
          for (int tt = 0; tt < C1; ++tt) sm[o + tt] = col(v[r], O1 + tt);
        }
      }
    }
    __syncthreads();
    // ---- step 2, direct (radix-4 step 2): one thread per (channel row group c, column
    //      item jj) runs the item of family 2p at jj and of family 2p+1 at the mirrored
    //      item NCH2-1-jj, so the pair epilogue (mirror, add, weight) happens in
    //      registers: pair 0 stores its NR2 image rows x C2 columns straight to HBM,
    //      pair 1 its transposed 4x4 blocks into the reduce staging -- no park ----
    if (DIRECT) {
      constexpr int NCH2 = XB / C2;
      if (!(dbgm & 1)) {
        for (int it = tid; it < NR1 * NCH2; it += NT) {
          // pair 0: jj fastest (coalesced image rows); pair 1: c fastest (the staging
          // STS.128 of a warp spread over 8 bank quads)
          const int c = PAIR == 0 ? it / NCH2 : it % NR1;
          const int jj = PAIR == 0 ? it - c * NCH2 : it / NR1;
          const int jm = NCH2 - 1 - jj;
          float o[NR2][C2];
          {
            float2 v[NR2][It<R2, C2>::T / 2];
            item_load<R2, C2>(oS + c * PS + HS + C2 * jj - O2, NR1 * PS, c, v);
            item_fht<R2, C2>(v);
#pragma unroll
            for (int r = 0; r < NR2; ++r)
#pragma unroll
              for (int e = 0; e < C2; ++e) o[r][e] = col(v[r], O2 + e);
          }
          {
            float2 v[NR2][It<R2, C2>::T / 2];
            item_load<R2, C2>(oS + (NB + c) * PS + HS + C2 * jm - O2, NR1 * PS, c, v);
            item_fht<R2, C2>(v);
            // column C2*jj + e of family 2p+1 mirrored: XB-1-(C2*jj+e) = C2*jm + C2-1-e
#pragma unroll
            for (int r = 0; r < NR2; ++r)
#pragma unroll
              for (int e = 0; e < C2; ++e) o[r][e] = scale * (o[r][e] + col(v[r], O2 + C2 - 1 - e));
          }
          if (dbgm & 2) continue;
          if (PAIR == 0) {
            // img[ch*NB + c*NR2 + r][x0 + C2*jj + e]
            float* const outc = img + ((long long)cur.sl * N + ch * NB + c * NR2) * N + x0 + C2 * jj;
            if (x0 + C2 * jj < N) {
#pragma unroll
              for (int r = 0; r < NR2; ++r)
#pragma unroll
                for (int e = 0; e < C2; e += 4)
                  *reinterpret_cast<float4*>(outc + (long long)r * N + e) =
                      make_float4(o[r][e], o[r][e + 1], o[r][e + 2], o[r][e + 3]);
            }
          } else {
            // staging [XB image rows x0 + i][NB image columns ch*NB + r], i = C2*jj + e
#pragma unroll
            for (int e = 0; e < C2; ++e)
              st4(oIn + oStg + (C2 * jj + e) * NB + c * NR2, make_float4(o[0][e], o[1][e], o[2][e], o[3][e]));
          }
        }
      }
      if (PAIR == 1) fence_proxy_async();              // staging -> async proxy (each writer)
    } else {
    // ---- step 2: both families, core columns -> park (aliasing the input) ----
    if (!(dbgm & 1)) {
      constexpr int nch = XB / C2;
      constexpr int per_fam = NR1 * nch;
      for (int it = tid; it < 2 * per_fam; it += NT) {
        const int q = it / per_fam;
        const int r3 = it - q * per_fam;
        const int c = r3 / nch, jj = r3 - c * nch;
        float2 v[NR2][It<R2, C2>::T / 2];
        item_load<R2, C2>(oS + (q * NB + c) * PS + HS + C2 * jj - O2, NR1 * PS, c, v);
        item_fht<R2, C2>(v);
#pragma unroll
        for (int r = 0; r < NR2; ++r) {
          const int o = oIn + (q * NB + c * NR2 + r) * PK + C2 * jj;
          if (PAIR == 0) {
#pragma unroll
            for (int tt = 0; tt < C2; tt += 4)
              st4(o + tt, make_float4(col(v[r], O2 + tt), col(v[r], O2 + tt + 1), col(v[r], O2 + tt + 2),
                                      col(v[r], O2 + tt + 3)));
          } else {
#pragma unroll
            for (int tt = 0; tt < C2; ++tt) sm[o + tt] = col(v[r], O2 + tt);
          }
        }
      }
    }
    __syncthreads();
    // ---- epilogue ----
    if (dbgm & 2) {
    } else if (PAIR == 0) {
      constexpr int nq = XB / 4;
      float* const outc = img + ((long long)cur.sl * N + ch * NB) * N + x0;   // image rows ch*NB..
      for (int e = tid; e < NB * nq; e += NT) {
        const int rf = e / nq, kq = e - rf * nq;
        const float4 a = ld4(oIn + rf * PK + 4 * kq);
        const float4 m = ld4(oIn + (NB + rf) * PK + XB - 4 - 4 * kq);
        if (x0 + 4 * kq < N) {
          const float4 o = make_float4(scale * (a.x + m.w), scale * (a.y + m.z), scale * (a.z + m.y),
                                       scale * (a.w + m.x));
          *reinterpret_cast<float4*>(outc + rf * N + 4 * kq) = o;
        }
      }
    } else {
      // staging tile [XB image rows x0 + i][NB image columns ch*NB + r] (the TMA box):
      // lanes = 8 row-quads of one image row x 4 image rows per warp
      constexpr int gq = NB / 4;
      for (int e = tid; e < XB * gq; e += NT) {
        const int i = e / gq, rq = e - i * gq;
        const int rf = 4 * rq;
        float4 o;
        o.x = scale * (sm[oIn + rf * PK + i] + sm[oIn + (NB + rf) * PK + XB - 1 - i]);
        o.y = scale * (sm[oIn + (rf + 1) * PK + i] + sm[oIn + (NB + rf + 1) * PK + XB - 1 - i]);
        o.z = scale * (sm[oIn + (rf + 2) * PK + i] + sm[oIn + (NB + rf + 2) * PK + XB - 1 - i]);
        o.w = scale * (sm[oIn + (rf + 3) * PK + i] + sm[oIn + (NB + rf + 3) * PK + XB - 1 - i]);
        st4(oIn + oStg + i * NB + rf, o);
      }
      fence_proxy_async();                             // staging -> async proxy (each writer)
    }
    }   // !DIRECT
    __syncthreads();                                   // S1 / park / staging reused by the next item
    // pair 1: image[x0 + i][ch*NB + r] += staging (TMA reduce in L2; clipped at row N)
    if (PAIR == 1 && tid == 0 && !(dbgm & 2))
      tma_reduce_add_2d(&tmapI, smem_u32(oIn + oStg), ch * NB, cur.sl * N + x0);
    if (!DB) issue(pb_add(cur, step, nx, H), 0);
    if (DB) bb ^= 1;
  }
  if (PAIR == 1 && tid == 0) bulk_wait_all();          // reduces complete before exit
}

// ---------------------------------------------------------------- host side
bool sweep_supported(int N) { return N == 512 || N == 1024 || N == 2048 || N == 4096; }

size_t sweep_a_smem(const SweepGeom& g) {
  const int H = g.H, X = g.X;
  const int R2 = (H == 64) ? 3 : 2;
  const int HS = (R2 == 3) ? 8 + 4 * ((7 * 7) / 4) : 4 + 4 * ((7 * 3) / 4);
  const int PF = pitch4(8 + X + 4), PS = pitch4(HS + X + 4);
  const size_t fl = (size_t)H * PF + (size_t)H * PS + (size_t)(g.D + 1) * H * 3 + 4 + 8;
  return fl * sizeof(float);
}

size_t pair_b_smem(const SweepGeom& g, int pair) {
  const bool db = g.XB <= 64 && g.NB <= 32;   // NB = 64: single buffer (2 CTAs/SM)
  const int NB = g.NB, XB = g.XB;
  int m = 0;
  while ((1 << m) < NB) ++m;
  const int R1 = (m >= 5) ? 3 : 2, R2 = m - R1;
  const int O1 = (R1 == 3) ? 8 : 4;
  const int HS = pb_halo(R1, R2);
  const int HI = HS + O1;
  const int RPT = 256 / (2 * NB), NQF = ((HI + XB) / 4 + RPT - 1) / RPT * RPT;
  const int PI = pitch4(4 * NQF), PS = pitch4(HS + XB + 4), PG = NB;
  const size_t nbuf = db ? 2 : 1;
  (void)PG;
  const int PK = pair == 0 ? XB + 4 : XB + 1;
  const int oStg = (2 * NB * PK + 31) / 32 * 32;
  const size_t in_sz = (pair == 1 && oStg + XB * NB > 2 * NB * PI) ? (size_t)oStg + XB * NB : (size_t)2 * NB * PI;
  return (nbuf * in_sz + (size_t)2 * NB * PS + 4) * sizeof(float);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D map of the linogram batch: dim0 = s (W columns), dim1 = rows (slices * 4N); box 76 x 64.
static cudaError_t make_lin_map(CUtensorMap* m, const float* lin, int slices, const SweepGeom& g, int box_w,
                                int box_h) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {(cuuint64_t)g.W, (cuuint64_t)slices * 4 * g.N};
  const cuuint64_t strides[1] = {(cuuint64_t)g.W * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(lin), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int H, int X, bool IIR, bool BETA>
static cudaError_t launch_a_t(const float* lin, float* R, int slices, int f0, int nf,
                              long long stride, const SweepGeom& g, const SweepIir& k, int* counter,
                              cudaStream_t st) {
  auto kern = k_sweep_a<H, X, IIR, BETA>;
  size_t smem = sweep_a_smem(g);
  // tensor memory: (D+1) slots of 32 columns per lane; never more CTAs per SM than
  // the 512 columns hold (a CTA waiting in tcgen05.alloc would spin): raise the
  // shared-memory request so that the occupancy limit enforces it
  if (IIR) {
    const int per_tmem = 512 / g.tmem_cols;
    const size_t cap = (size_t)227 * 1024 / (per_tmem + 1) + 1024;
    if (per_tmem < 3) smem = std::max(smem, cap);
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const cudaError_t eo = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, H * X / 32, smem);
  cudaGetLastError();
  {
    // the occupancy calculator reports 1 CTA/SM for kernels that allocate tensor
    // memory; the resident limit is set by shared memory, registers and TMEM columns
    cudaFuncAttributes fa;
    int smem_sm = 0, regs_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && fa.numRegs > 0) {
      const int regs_cta = ((fa.numRegs + 7) / 8 * 8) * (H * X / 32);
      const int by_regs = regs_sm / regs_cta;
      const int by_smem = (int)(smem_sm / (smem + fa.sharedSizeBytes + 1024));
      int manual = std::min(by_regs, by_smem);
      if (IIR) manual = std::min(manual, 512 / g.tmem_cols);
      if (eo != cudaSuccess || per < manual) per = manual;
    }
  }
  if (IIR) per = std::min(per, 512 / g.tmem_cols);
  if (g.ctas_a > 0 && g.ctas_a < per) per = g.ctas_a;   // tuning knob (FBP_SWEEP_CTAS)
  if (per < 1) per = 1;
  // small batches: split every sweep into segments until there are ~1.7 work items
  // per resident CTA slot (measured r01 at N = 2048: B = 1 -> 6 segments, 2 -> 3,
  // 4 -> 2, >= 8 -> 1; FBP_SWEEP_SEG overrides)
  const long long sweeps = (long long)slices * nf * g.NB;
  const long long slots = (long long)sms * per;
  int nseg = (int)std::min<long long>(8, std::max<long long>(1, (17 * slots + 10 * sweeps - 1) / (10 * sweeps)));
  if (g.nseg > 0) nseg = g.nseg;
  const long long nitems = sweeps * nseg;
  const long long grid = std::min<long long>(nitems, (long long)sms * per);
#if FBP_DEV_MASK
  if (std::getenv("FBP_VERBOSE"))
    fprintf(stderr, "sweep: smem %zu per %d tmem_cols %d nseg %d grid %lld D %d\n", smem, per, g.tmem_cols, nseg, grid,
            g.D);
#endif
  CUtensorMap tF;
  e = make_lin_map(&tF, lin, slices, g, pitch4(8 + X + 4), H);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, H * X / 32, smem, st>>>(lin, R, g, k, slices, f0, nf, stride, nseg, counter, tF);
  return cudaGetLastError();
}

cudaError_t launch_sweep_a(const float* lin, float* R, int slices, int f0, int nf,
                           long long lin_slice_stride, const SweepGeom& g, const SweepIir& k,
                           bool iir, int* counter, cudaStream_t st, int* launches) {
  if (slices <= 0 || nf <= 0) return cudaSuccess;
  // the TMA maps address rows (slice*4 + family)*N + t of a contiguous batch
  if (f0 != 0 || nf != 4 || lin_slice_stride != 4LL * g.N * g.W || (reinterpret_cast<uintptr_t>(lin) & 15))
    return cudaErrorInvalidValue;
  if ((long long)slices * 4 * g.H * g.NB > 0x7fffffffLL) return cudaErrorInvalidValue;
  const bool beta = k.beta.x != 0.0f;
  cudaError_t e;
#define FBP_SWEEP_CASE(HH, XX)                                                                     \
  if (g.H == HH) {                                                                                 \
    if (!iir) e = launch_a_t<HH, XX, false, false>(lin, R, slices, f0, nf, lin_slice_stride, g, k, counter, st); \
    else if (beta) e = launch_a_t<HH, XX, true, true>(lin, R, slices, f0, nf, lin_slice_stride, g, k, counter, st); \
    else e = launch_a_t<HH, XX, true, false>(lin, R, slices, f0, nf, lin_slice_stride, g, k, counter, st); \
    if (launches) ++*launches;                                                                     \
    return e;                                                                                      \
  }
  FBP_SWEEP_CASE(64, 64)
  FBP_SWEEP_CASE(32, 128)
#undef FBP_SWEEP_CASE
  return cudaErrorInvalidValue;
}

template <int R1, int R2, int XB, int PAIR>
static cudaError_t launch_b_t(const float* R, float* img, int slices, float scale,
                              const SweepGeom& g, cudaStream_t st) {
  auto kern = k_pair_b<R1, R2, XB, PAIR, (XB <= 64 && R1 + R2 <= 5)>;
  const size_t smem = pair_b_smem(g, PAIR);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, smem);
  if (per < 1) per = 1;
  const long long nitems = (long long)((g.N + g.XB - 1) / g.XB) * g.H * slices;
  const long long grid = std::min<long long>(nitems, (long long)sms * per);
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // compact R viewed as [slices*4*H][NB][WR]; box = one channel's NB rows x PI columns
  constexpr int NB = 1 << (R1 + R2);
  constexpr int O1 = (R1 == 3) ? 8 : 4;
  constexpr int HI = pb_halo(R1, R2) + O1;
  constexpr int RPT = 256 / (2 * NB);
  constexpr int NQF = ((HI + XB) / 4 + RPT - 1) / RPT * RPT;
  constexpr int PI = pitch4(4 * NQF);
  CUtensorMap tR, tI;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)g.WR, (cuuint64_t)NB, (cuuint64_t)slices * 4 * g.H};
    const cuuint64_t strides[2] = {(cuuint64_t)g.WR * 4, (cuuint64_t)NB * g.WR * 4};
    const cuuint32_t box[3] = {(cuuint32_t)PI, (cuuint32_t)NB, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tR, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(R), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)slices * g.N};
    const cuuint64_t strides[1] = {(cuuint64_t)g.N * 4};
    const cuuint32_t box[2] = {(cuuint32_t)NB, (cuuint32_t)XB};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tI, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, img, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  kern<<<(unsigned)grid, 256, smem, st>>>(R, img, g, scale, nitems, tR, tI);
  return cudaGetLastError();
}

cudaError_t launch_pair_b(const float* R, float* img, int slices, int pair, float scale,
                          const SweepGeom& g, cudaStream_t st, int* launches) {
  if (slices <= 0) return cudaSuccess;
  cudaError_t e = cudaErrorInvalidValue;
#define FBP_PAIR_CASE(NBV, R1, R2, XBV)                                                     \
  if (g.NB == NBV && g.XB == XBV)                                                           \
    e = pair == 0 ? launch_b_t<R1, R2, XBV, 0>(R, img, slices, scale, g, st)                \
                  : launch_b_t<R1, R2, XBV, 1>(R, img, slices, scale, g, st);
  FBP_PAIR_CASE(16, 2, 2, 64)    // N = 512: double-buffered, 3 CTAs/SM (r02 s6: KB 0.619 -> 0.425 ms per 256 slices)
#if FBP_DEV_MASK
  FBP_PAIR_CASE(16, 2, 2, 128)   // developer A/B only (FBP_XB=128): the single-buffered r01 tile
#endif
  FBP_PAIR_CASE(32, 3, 2, 128)
  FBP_PAIR_CASE(32, 3, 2, 64)
  FBP_PAIR_CASE(64, 3, 3, 32)
#if FBP_DEV_MASK
  FBP_PAIR_CASE(64, 3, 3, 64)   // developer A/B only (FBP_XB=64): 133 KB per CTA, 1 CTA/SM
#endif
#undef FBP_PAIR_CASE
  if (launches) ++*launches;
  return e;
}

}  // namespace fbp
