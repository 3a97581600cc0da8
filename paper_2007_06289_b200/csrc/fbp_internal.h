// Internal declarations shared by the C-ABI layer (api.cu) and the kernels.
// Product code only -- nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

// Developer builds only (FBP_NVCC_FLAGS=-DFBP_DEV_MASK=1): the FBP_DBG timing skip
// mask and the FBP_* tuning environment variables.  Product builds
// read no environment variable.
#ifndef FBP_DEV_MASK
#define FBP_DEV_MASK 0
#endif

namespace fbp {

constexpr int kMaxOrder = 8;       // M, Q <= 8 (fbp.h)
constexpr int kScanSteps = 5;      // log2(32): warp-level carry scan

// Recursive-filter coefficients as the kernels consume them (plan-derived, fp32).
// Feedforward in difference form (reading R16):
//   B(z) = beta + (1 - z^-1) C(z),  C(z) = sum_{k<M-1} c_k z^-k,
//   beta = sum_k b_k,  c_k = -sum_{j>k} b_j.
// Feedback A(z) = 1 + sum_{k=1..Q} a_k z^-k (Eq.9 sign).  Orders are zero-padded
// to the kernel's compile-time order QM (exact: zero taps add nothing).
// P[k] = A^(L*2^k) (companion matrix of A, state (y[n], y[n-1], ...)) for the
// exact chunked scan of the recursion across the 32 lanes of a warp.
// G[i][m] = (A^(i+1))_{0m}: response of y[start+i] to the carry-in state, i < 32.
// AW = A^(32 L): one warp of chunks.
struct IirParams {
  float beta;
  float c[kMaxOrder];
  float a[kMaxOrder];
  float P[kScanSteps][kMaxOrder * kMaxOrder];
  float AW[kMaxOrder * kMaxOrder];
  float G[32][kMaxOrder];
};

struct Geometry {
  int n;       // log2 N
  int N;       // image size
  int W;       // 2N, linogram row length
  int k1;      // FHT levels in pass A
  int m;       // FHT levels in pass B
  int H;       // 2^k1 rows per pass-A block
  int NB;      // 2^m blocks (rows per pass-B channel)
  int WR;      // N + NB: compact pass-A output row width
  int XA;      // pass-A u-tile width
  int XB;      // pass-B x-tile width
  int L;       // IIR per-thread chunk: 32 if W >= 1024, else W/32 (1 if W < 32)
  int iir_qm;  // compile-time padded feedback order of the IIR kernel (3 or 8)
  int iir_mc;  // number of difference-form feedforward taps c_k (M - 1)
};

// ---------------------------------------------------------------------------
// Fast path (sweep.cu): fused IIR + FHT levels 1..k1 as a sweep along s, and the
// pair-wise pass B.  Orders M <= 3, Q <= 3 (the paper's M = Q = 3); all float2
// entries are duplicated (v, v) so that both lanes of an f32x2 op see the same
// coefficient.
struct SweepIir {
  float2 beta, c0, c1;        // difference-form feedforward: beta x + c0 D[n] + c1 D[n-1]
  float2 na1, na2, na3;       // -a_1, -a_2, -a_3
  float2 M1[9];               // A^32 (row-major 3x3, companion matrix of A(z))
  float2 M2[9];               // A^64
  float2 MX[9];               // A^X   (one tile)
  float2 M16[9];              // A^16
  // GA[p][m] = (G^(2p), G^(2p+1)) with G^(i) = (A^(32-i))_{0m}: the anticausal
  // homogeneous response at sample i of a 32-sample chunk to the state at the
  // chunk's right edge (adjacent samples packed for FFMA2)
  float2 GA[16][3];
};

struct SweepGeom {
  int N, W, NB, H, WR;
  int X;      // pass-A tile width (H * X = 4096)
  int nt;     // tiles per linogram row, W / X
  int D;      // look-ahead tiles for the anticausal carry (plan: tail bound)
  int P;      // pass-B L2 prefetch distance in items (env FBP_PREFETCH)
  int XB;     // pass-B x-tile width
  int ctas_a; // cap on resident sweep CTAs per SM (0: occupancy limit); env FBP_SWEEP_CTAS
  int nseg;   // segments per sweep (0: automatic, fill the CTA slots); env FBP_SWEEP_SEG
  int tmem_cols;  // tensor-memory columns per sweep CTA: (D+1) x 32 rounded to a power of two
  int dbg;    // developer timing mask, env FBP_DBG, honoured only in -DFBP_DEV_MASK=1 builds
              // (results invalid when nonzero): pass B bit 0
              // skips the FHT steps, bit 1 the epilogue, bit 2 the fills; sweep bit 3
              // skips every TMA load, bit 4 the R stores
};

// Pass A sweep over `slices` x families [f0, f0+nf) (input family fi of slice s at
// lin + s*lin_slice_stride + fi*N*W), output R[(s*4 + f0 + fi)].  `counter` is a
// device int the launcher zeroes (work queue).  iir=false: plain FHT levels.
cudaError_t launch_sweep_a(const float* lin, float* R, int slices, int f0, int nf,
                           long long lin_slice_stride, const SweepGeom& g, const SweepIir& k,
                           bool iir, int* counter, cudaStream_t st, int* launches);
cudaError_t launch_pair_b(const float* R, float* img, int slices, int pair, float scale,
                          const SweepGeom& g, cudaStream_t st, int* launches);
bool sweep_supported(int N);

// Small-N path (small.cu, N <= 64): one CTA per slice, IIR + FHT + Eq.22 on-chip.
struct SmallIir {
  int N;
  int iir;                     // 0: back projection only (fbp_fht_backproject)
  float beta, c0, c1;          // difference-form feedforward (M <= 3)
  float na1, na2, na3;         // -a_1, -a_2, -a_3 (Q <= 3)
};
bool small_supported(int N);
cudaError_t launch_small(const float* lin, float* img, int slices, const SmallIir& k, float scale, cudaStream_t st,
                         int* launches);
size_t sweep_a_smem(const SweepGeom& g);
size_t pair_b_smem(const SweepGeom& g, int pair);

// Kernel launchers of the general path (iir.cu, fht.cu).  All asynchronous on `st`; return the launch error.
// lane_mats: device [32][8*8], lane_mats[j] = A^(L*j).
cudaError_t launch_iir_rows(const float* in, float* out, long long rows, const Geometry& g,
                            const IirParams& p, const float* lane_mats, cudaStream_t st,
                            int* launches);
size_t fht_pass_a_smem(const Geometry& g);
size_t fht_pass_b_smem(const Geometry& g);
// Pass A over `slices` x families [f0, f0+nf): input family fi of slice s at
// lin + s*lin_slice_stride + fi*N*W; output R[(s*4 + f0 + fi)].
cudaError_t launch_fht_pass_a(const float* lin, float* R, int slices, int f0, int nf,
                              long long lin_slice_stride, const Geometry& g, cudaStream_t st,
                              int* launches);
cudaError_t launch_fht_pass_b(const float* R, float* img, int slices, int pair, float scale,
                              const Geometry& g, cudaStream_t st, int* launches);

// Forward FHT (fwd.cu, Eq.17): image [slices][N][N] -> R_A (workspace of
// fwd_workspace_floats per slice) -> linogram [slices][4][N][2N].  slices <= 16383.
size_t fwd_workspace_floats(const Geometry& g);
// Sinogram -> linogram (resample.cu, Eq.14-15, R23): sino [slices][n_angles][n_bins]
// -> lin [slices][4][N][2N].  slices <= 16383.
cudaError_t launch_resample(const float* sino, float* lin, int slices, int n_angles, int n_bins, double dr,
                            const Geometry& g, cudaStream_t st, int* launches);
cudaError_t launch_fwd_a(const float* img, float* RA, float* scratch, int slices, const Geometry& g, cudaStream_t st,
                         int* launches);
cudaError_t launch_fwd_b(const float* RA, float* lin, int slices, const Geometry& g, cudaStream_t st,
                         int* launches);

}  // namespace fbp
