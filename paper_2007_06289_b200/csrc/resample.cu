// Sinogram -> linogram resampling (NEXT-2): PAPER.md:172-188
// (Eq.14-15), reading R23.
//
// Linogram sample (f, t, s) is the line of reading R2 (view line X' = A + k Y',
// A = s - N + 0.5 - 0.5 k, k = t/(N-1), mapped to the image per family as in
// Eq.16 / R4).  Its normal angle theta in [0, pi) and signed distance r from the
// image centre select the sinogram sample, linearly interpolated in the angle index
// (row after P-1 = row 0 at -r) and in the bin index (bins outside [0, R) read 0),
// and the value is divided by the Eq.15 stretch |D| = sqrt(1 + k^2) of that line.
//
// One CTA per linogram row (t, family, slice): thread 0 derives the row's geometry
// once in double precision (theta, the angle weight, r as an affine function of s,
// 1/|D|); the threads sweep s, evaluating the bin position in double (|r| reaches
// ~1.5 N, so fp32 would leave ~1e-4-bin errors at N = 2048) and interpolating in
// fp32.  HBM-bound: writes 32 N^2 B per slice, reads two sinogram rows per
// linogram row (mostly from L2).
#include <cmath>

#include "fbp_internal.h"

namespace fbp {
namespace {

constexpr int RNT = 256;

struct RowGeo {
  double a;      // weight of the second angle row
  double w0;     // bin index of s = 0 on row k0 (and k1 unless wrapped)
  double dw;     // d(bin index)/ds
  double wf0;    // bin index of s = 0 on the wrapped row 0 (at -r)
  float inv_len; // 1/|D|
  int k0, k1;    // angle rows; k1 = -1: row 0 at -r
};

__device__ __forceinline__ float interp_row(const float* __restrict__ row, int R, double w) {
  const double fl = floor(w);
  const int j0 = (int)fl;
  const float b = (float)(w - fl);
  float v = 0.f;
  if (j0 >= 0 && j0 < R) v += (1.f - b) * __ldg(row + j0);
  if (j0 + 1 >= 0 && j0 + 1 < R) v += b * __ldg(row + j0 + 1);
  return v;
}

// grid (N rows t, 4 * slices)
__global__ void __launch_bounds__(RNT) k_resample(const float* __restrict__ sino, float* __restrict__ lin,
                                                  int N, int P, int R, double dr) {
  __shared__ RowGeo geo;
  const int t = blockIdx.x, sf = blockIdx.y, f = sf & 3;
  if (threadIdx.x == 0) {
    const double k = (double)t / (N - 1);
    const double A0 = -N + 0.5 - 0.5 * k;              // A at s = 0
    double Dx, Dy, p0x, p0y, dpx, dpy;                 // line point at s = 0, dP0/ds
    switch (f) {
      case 0: Dx = k; Dy = 1.0; p0x = A0; p0y = 0.0; dpx = 1.0; dpy = 0.0; break;
      case 1: Dx = -k; Dy = 1.0; p0x = N - A0; p0y = 0.0; dpx = -1.0; dpy = 0.0; break;
      case 2: Dx = 1.0; Dy = k; p0x = 0.0; p0y = A0; dpx = 0.0; dpy = 1.0; break;
      default: Dx = 1.0; Dy = -k; p0x = 0.0; p0y = N - A0; dpx = 0.0; dpy = -1.0; break;
    }
    const double L = sqrt(Dx * Dx + Dy * Dy);
    double nx = Dy / L, ny = -Dx / L;
    double th = atan2(ny, nx);
    if (th < 0.0 || th >= M_PI) {
      nx = -nx;
      ny = -ny;
      th = atan2(ny, nx);
    }
    const double r0 = (p0x - 0.5 * N) * nx + (p0y - 0.5 * N) * ny;
    const double drs = dpx * nx + dpy * ny;
    const double u = th / (M_PI / P);
    int k0 = (int)floor(u);
    if (k0 > P - 1) k0 = P - 1;
    geo.a = u - k0;
    geo.w0 = r0 / dr + 0.5 * (R - 1);
    geo.dw = drs / dr;
    geo.wf0 = -r0 / dr + 0.5 * (R - 1);
    geo.inv_len = (float)(1.0 / L);
    geo.k0 = k0;
    geo.k1 = (k0 + 1 < P) ? k0 + 1 : -1;
  }
  __syncthreads();
  const float a = (float)geo.a, il = geo.inv_len;
  const float* ps = sino + (long long)(sf >> 2) * P * R;
  const float* row0 = ps + (long long)geo.k0 * R;
  const float* row1 = ps + (long long)(geo.k1 >= 0 ? geo.k1 : 0) * R;
  const bool wrap = geo.k1 < 0;
  float* out = lin + ((long long)sf * N + t) * (2 * N);
  for (int s = threadIdx.x; s < 2 * N; s += RNT) {
    const double w = geo.w0 + s * geo.dw;
    const float v0 = interp_row(row0, R, w);
    const float v1 = interp_row(row1, R, wrap ? geo.wf0 - s * geo.dw : w);
    out[s] = ((1.f - a) * v0 + a * v1) * il;
  }
}

}  // namespace

cudaError_t launch_resample(const float* sino, float* lin, int slices, int n_angles, int n_bins, double dr,
                            const Geometry& g, cudaStream_t st, int* launches) {
  const dim3 grid(g.N, 4 * slices);
  k_resample<<<grid, RNT, 0, st>>>(sino, lin, g.N, n_angles, n_bins, dr);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
