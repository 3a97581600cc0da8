// Internal declarations shared by the C-ABI layer (api.cu) and the kernels.
// Product code only -- nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

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

// Kernel launchers (kernels.cu).  All asynchronous on `st`; return the launch error.
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

}  // namespace fbp
