// Small-N path (N <= 64, BASELINE config 1): one CTA per slice with the whole slice
// in shared memory, so the IIR pair, every FHT level and the Eq.22 sum run on-chip
// and HBM sees exactly the algorithmic bytes (read the 4 x N x 2N linogram once,
// write the N x N image once).  Replaces the three-kernel general path for these
// sizes, whose cost at N = 64 is launch/latency bound (3 passes through HBM for
// 147 KB per slice).
//
//   per line family f (reading R4):
//     1. TMA bulk copies of its N rows (2N floats each) into a landing buffer (padded
//        pitch), one mbarrier transaction, issued one family ahead (two landing
//        buffers) so the copy overlaps the previous family's compute;
//     2. IIR (Eq.12-13, difference-form feedforward R16, zero state R11): thread r
//        runs the anticausal recursion of row r into the work buffer, then the causal
//        one adding into it (F = p~+ + p~-);
//     3. n = log2 N negative-direction FHT levels (recursion R3)
//        ping-ponging work <-> landing buffer, one warp per row, lanes over columns:
//          R_2h[blk + y'][u] = R_h[blk + y'/2][u] + R_h[blk + h + y'/2][u - ceil(y'/2)];
//     4. Eq.22 (oracle order) in per-thread registers: acc01[y][x] = B0[y][x] +
//        B1[y][N-1-x], acc23[y][x] = B2[x][y] + B3[x][N-1-y], B_f[y][x] = R[y][x + N];
//   then img[y][x] = w * (acc01[y][x] + acc23[y][x]).
// Without the IIR (fbp_fht_backproject) the levels start from X: add-only and
// bit-exact on integer inputs (R21), like the other paths.
#include "fbp_internal.h"

#include <algorithm>

namespace fbp {
namespace {

constexpr int SNT = 256;

__device__ __forceinline__ unsigned s_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int N>
struct SmallGeo {
  static constexpr int W = 2 * N;
  static constexpr int P = W + 4;                    // row pitch: whole quads, odd quad count for N >= 4
  static constexpr int FL = N * P;                   // one family buffer
  static constexpr int floats = 3 * FL;              // landing L0, L1 (alternate per family) + work WK
  static constexpr size_t bytes = (size_t)floats * sizeof(float) + 32;   // + 2 mbarriers
  static constexpr int PX = (N * N + SNT - 1) / SNT;  // image pixels per thread
};

// One FHT level h -> 2h over columns [U0, 2N): one warp per output row (its two
// input rows and the shift are warp-uniform), lanes over the columns, all of a
// lane's columns loaded before any is stored (latency overlap).
template <int N, int U0>
__device__ __forceinline__ void small_level(const float* src, float* dst, int h, int tid) {
  constexpr int W = 2 * N, P = W + 4, NU = (W - U0 + 31) / 32;
  for (int r = tid >> 5; r < N; r += SNT / 32) {
    const int blk = r & ~(2 * h - 1), yp = r - blk, lo = yp >> 1, sh = (yp + 1) >> 1;
    const float* const A = src + (blk + lo) * P;
    const float* const Bs = src + (blk + h + lo) * P - sh;
    float* const Dr = dst + r * P;
    float a[NU], b[NU];
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      const int u = U0 + (tid & 31) + 32 * j;
      a[j] = u < W ? A[u] : 0.f;
      b[j] = (u < W && u >= sh) ? Bs[u] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      const int u = U0 + (tid & 31) + 32 * j;
      if (u < W) Dr[u] = (u >= sh) ? a[j] + b[j] : a[j];
    }
  }
}

template <int N>
__global__ void __launch_bounds__(SNT) k_small(const float* __restrict__ lin, float* __restrict__ img, int slices,
                                               SmallIir k, float scale) {
  using Gm = SmallGeo<N>;
  constexpr int W = Gm::W, P = Gm::P, FL = Gm::FL, PX = Gm::PX;
  extern __shared__ float4 sm4[];
  float* const sm = reinterpret_cast<float*>(sm4);
  float* const WK = sm + 2 * FL;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(sm + Gm::floats);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s_u32(bar + i)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  constexpr int LOGN = (N >= 64) ? 6 : (N >= 32) ? 5 : (N >= 16) ? 4 : (N >= 8) ? 3 : (N >= 4) ? 2 : 1;
  // work items i = (slice, family), this CTA's slices in order; item i lands in L[i & 1],
  // the landing of item i + 1 is issued when item i starts (its buffer was freed by
  // item i - 1's last barrier), so every landing overlaps a whole family's compute
  const int nmine = slices > (int)blockIdx.x ? (slices - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nitems = 4 * nmine;
  auto land = [&](int i) {
    if (tid != 0 || i >= nitems) return;
    const int s = blockIdx.x + (i >> 2) * gridDim.x, f = i & 3;
    float* const L = sm + (i & 1) * FL;
    const unsigned b = s_u32(bar + (i & 1));
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"((unsigned)(N * W * 4))
                 : "memory");
    const float* src = lin + (((long long)s * 4 + f) * N) * W;
    for (int r = 0; r < N; ++r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       s_u32(L + r * P)),
                   "l"(src + (long long)r * W), "r"((unsigned)(W * 4)), "r"(b)
                   : "memory");
  };
  land(0);
  // Eq.22 accumulators in registers: thread owns pixels e = tid + SNT*j, (y, x) = (e / N, e % N)
  float acc01[PX], acc23[PX];
  unsigned phase2 = 0;                                 // parity bits of the two mbarriers
  for (int i = 0; i < nitems; ++i) {
    const int f = i & 3;
    land(i + 1);
    float* const X = sm + (i & 1) * FL;
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
            s_u32(bar + (i & 1))),
        "r"((phase2 >> (i & 1)) & 1u)
        : "memory");
    phase2 ^= 1u << (i & 1);
    // ---- IIR pair, thread = row: anticausal into WK, then causal added ----
    float* src = X;
    float* dst = WK;
    if (k.iir) {
      if (tid < N) {
        const float* xr = X + tid * P;
        float* fr = WK + tid * P;
        // anticausal: E[n] = x[n] - x[n+1], u = beta x + c0 E[n] + c1 E[n+1]
        float x1 = 0.f, e1 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
        float4 vn = *reinterpret_cast<const float4*>(xr + W - 4);
        for (int q = W / 4 - 1; q >= 0; --q) {
          const float4 v = vn;
          if (q > 0) vn = *reinterpret_cast<const float4*>(xr + 4 * q - 4);   // next quad in flight
          float o[4];
          const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 3; j >= 0; --j) {
            const float e = xs[j] - x1;
            float u = k.c1 * e1;
            u = fmaf(k.c0, e, u);
            u = fmaf(k.beta, xs[j], u);
            float y = fmaf(k.na3, y3, u);
            y = fmaf(k.na2, y2, y);
            y = fmaf(k.na1, y1, y);
            y3 = y2;
            y2 = y1;
            y1 = y;
            e1 = e;
            x1 = xs[j];
            o[j] = y;
          }
          *reinterpret_cast<float4*>(fr + 4 * q) = make_float4(o[0], o[1], o[2], o[3]);
        }
        // causal: D[n] = x[n] - x[n-1], u = beta x + c0 D[n] + c1 D[n-1]; F = y+ + y-
        x1 = 0.f;
        e1 = 0.f;
        y1 = y2 = y3 = 0.f;
        vn = *reinterpret_cast<const float4*>(xr);
        float4 an = *reinterpret_cast<const float4*>(fr);
        for (int q = 0; q < W / 4; ++q) {
          const float4 v = vn, a = an;
          if (q + 1 < W / 4) {                         // next quads in flight
            vn = *reinterpret_cast<const float4*>(xr + 4 * q + 4);
            an = *reinterpret_cast<const float4*>(fr + 4 * q + 4);
          }
          const float xs[4] = {v.x, v.y, v.z, v.w};
          float o[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float d = xs[j] - x1;
            float u = k.c1 * e1;
            u = fmaf(k.c0, d, u);
            u = fmaf(k.beta, xs[j], u);
            float y = fmaf(k.na3, y3, u);
            y = fmaf(k.na2, y2, y);
            y = fmaf(k.na1, y1, y);
            y3 = y2;
            y2 = y1;
            y1 = y;
            e1 = d;
            x1 = xs[j];
            o[j] = y + o[j];                           // F = y+ + y- (Eq.12)
          }
          *reinterpret_cast<float4*>(fr + 4 * q) = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
      __syncthreads();
      src = WK;
      dst = X;
    }
    // ---- FHT levels, ping-pong src <-> dst; the last level computes u >= N only ----
#pragma unroll 1
    for (int lv = 0; lv < LOGN; ++lv) {
      if (lv < LOGN - 1)
        small_level<N, 0>(src, dst, 1 << lv, tid);
      else
        small_level<N, N>(src, dst, 1 << lv, tid);
      __syncthreads();
      float* t = src;
      src = dst;
      dst = t;
    }
    // ---- Eq.22 (oracle order): acc01[y][x] = B0[y][x] + B1[y][N-1-x],
    //      acc23[y][x] = B2[x][y] + B3[x][N-1-y], B_f[y][x] = src[y][x + N] ----
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      const int e = tid + SNT * j;
      if (e < N * N) {
        const int y = e / N, x = e - y * N;
        if (f == 0) acc01[j] = src[y * P + N + x];
        else if (f == 1) acc01[j] += src[y * P + N + (N - 1 - x)];
        else if (f == 2) acc23[j] = src[x * P + N + y];
        else acc23[j] += src[x * P + N + (N - 1 - y)];
      }
    }
    if (f == 3) {
      float* const out = img + (long long)(blockIdx.x + (i >> 2) * gridDim.x) * N * N;
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        const int e = tid + SNT * j;
        if (e < N * N) out[e] = scale * (acc01[j] + acc23[j]);
      }
    }
    __syncthreads();   // L[i & 1] and WK free: item i + 2 lands there
  }
}

template <int N>
cudaError_t launch_small_t(const float* lin, float* img, int slices, const SmallIir& k, float scale,
                           cudaStream_t st) {
  using Gm = SmallGeo<N>;
  auto kern = k_small<N>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::bytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, SNT, Gm::bytes);
  const int grid = std::max(1, std::min(slices, sms * std::max(per, 1)));
  kern<<<grid, SNT, Gm::bytes, st>>>(lin, img, slices, k, scale);
  return cudaGetLastError();
}

}  // namespace

bool small_supported(int N) { return N >= 2 && N <= 64; }

cudaError_t launch_small(const float* lin, float* img, int slices, const SmallIir& k, float scale, cudaStream_t st,
                         int* launches) {
  if (slices <= 0) return cudaSuccess;
  if (launches) ++*launches;
  switch (k.N) {
    case 2: return launch_small_t<2>(lin, img, slices, k, scale, st);
    case 4: return launch_small_t<4>(lin, img, slices, k, scale, st);
    case 8: return launch_small_t<8>(lin, img, slices, k, scale, st);
    case 16: return launch_small_t<16>(lin, img, slices, k, scale, st);
    case 32: return launch_small_t<32>(lin, img, slices, k, scale, st);
    case 64: return launch_small_t<64>(lin, img, slices, k, scale, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace fbp
