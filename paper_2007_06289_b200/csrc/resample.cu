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
// One CTA per linogram row (t, family) and group of up to 16 slices: thread 0 derives the row's geometry
// once in double precision (theta, the angle weight, r as an affine function of s,
// 1/|D|); each thread takes four consecutive s, evaluating the bin position of the
// first in double (|r| reaches ~1.5 N, so an fp32 position would be off by ~1e-4
// bins at N = 2048) and interpolating in fp32.  HBM-bound in principle: writes
// 32 N^2 B per slice, reads two sinogram rows per linogram row (mostly from L2).
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

// Linear interpolation of one sinogram row at bin position j + b (b in [0, 1) up to
// rounding; bins outside [0, R) read 0).
__device__ __forceinline__ float interp_row(const float* __restrict__ row, int R, int j0, float b) {
  float v = 0.f;
  if (j0 >= 0 && j0 < R) v += (1.f - b) * __ldg(row + j0);
  if (j0 + 1 >= 0 && j0 + 1 < R) v += b * __ldg(row + j0 + 1);
  return v;
}

// grid (N rows t, 4 families, slice groups of SPB): the row geometry does not depend
// on the slice, so each CTA derives it once and sweeps its slices
constexpr int SPB = 16;
__global__ void __launch_bounds__(RNT) k_resample(const float* __restrict__ sino, float* __restrict__ lin,
                                                  int N, int P, int R, double dr, int slices) {
  __shared__ RowGeo geo;
  const int t = blockIdx.x, f = blockIdx.y;
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
  const bool wrap = geo.k1 < 0;
  const float dwf = (float)geo.dw;
  const int sl_end = min(slices, (int)(blockIdx.z + 1) * SPB);
  for (int sl = blockIdx.z * SPB; sl < sl_end; ++sl) {
  const float* ps = sino + (long long)sl * P * R;
  const float* row0 = ps + (long long)geo.k0 * R;
  const float* row1 = ps + (long long)(geo.k1 >= 0 ? geo.k1 : 0) * R;
  float* out = lin + ((long long)(sl * 4 + f) * N + t) * (2 * N);
  // 4 consecutive s per thread (float4 store): the bin position of the quad's first
  // sample in fp64, the next three as fp32 offsets from its integer part (< 4 bins)
  for (int q0 = 4 * threadIdx.x; q0 < 2 * N; q0 += 4 * RNT) {
    const double w = geo.w0 + q0 * geo.dw;
    const double wfl = floor(w);
    const int jw = (int)wfl;
    const float fw = (float)(w - wfl);
    const double x = geo.wf0 - q0 * geo.dw;           // wrapped row: row 0 at -r
    const double xfl = floor(x);
    const int jx = (int)xfl;
    const float fx = (float)(x - xfl);
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float pw = fw + q * dwf, fpw = floorf(pw);
      const float v0 = interp_row(row0, R, jw + (int)fpw, pw - fpw);
      float v1;
      if (wrap) {
        const float px = fx - q * dwf, fpx = floorf(px);
        v1 = interp_row(row1, R, jx + (int)fpx, px - fpx);
      } else {
        v1 = interp_row(row1, R, jw + (int)fpw, pw - fpw);
      }
      o[q] = ((1.f - a) * v0 + a * v1) * il;
    }
    *reinterpret_cast<float4*>(out + q0) = make_float4(o[0], o[1], o[2], o[3]);
  }
  }
}

}  // namespace

cudaError_t launch_resample(const float* sino, float* lin, int slices, int n_angles, int n_bins, double dr,
                            const Geometry& g, cudaStream_t st, int* launches) {
  const dim3 grid(g.N, 4, (slices + SPB - 1) / SPB);
  k_resample<<<grid, RNT, 0, st>>>(sino, lin, g.N, n_angles, n_bins, dr, slices);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace fbp
