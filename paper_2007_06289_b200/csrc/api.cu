// C-ABI layer of libfbp (include/fbp.h): validation, plan (coefficient tables,
// level split, workspace), and stream-ordered orchestration of the kernels.
#include "../../include/fbp.h"
#include "fbp_internal.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: host ranges per entry point and kernel

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace fbp;

struct fbp_plan {
  Geometry g;
  IirParams iir;
  int device = 0;
  int max_batch = 1;
  int group = 1;            // slices per workspace group
  bool per_family = false;  // schedule IIR -> pass A one family at a time (large N)
  float* F = nullptr;       // filtered linogram workspace [group][4][N][2N]
  float* R = nullptr;       // pass-A output workspace [group][4][NB][H][WR]
  float* lane_mats = nullptr;  // [32][8*8] A^(L*j) for the IIR cross-warp carries
  size_t F_bytes = 0, R_bytes = 0;
  // host-path staging (allocated lazily by fbp_reconstruct_host, under host_mu:
  // concurrent host-path calls on one plan are serialised)
  std::mutex host_mu;
  float* d_in[2] = {nullptr, nullptr};
  float* d_out[2] = {nullptr, nullptr};
  float* h_in[2] = {nullptr, nullptr};
  float* h_out[2] = {nullptr, nullptr};
  cudaStream_t s_copy = nullptr, s_comp = nullptr, s_d2h = nullptr;
  // small-N path (small.cu): N <= 64, one CTA per slice; the IIR part needs M, Q <= 3
  bool small = false, small_iir = false;
  SmallIir sk{};
  // fast path (sweep.cu): fused IIR + pass-A sweep and pair-wise pass B
  bool fast = false;
  SweepGeom sg{};
  SweepIir si{};
  int* counter = nullptr;   // sweep work-queue counter (device)
  mutable long long launches = 0;
  // per-kernel event timing (fbp_plan_profile)
  mutable bool profiling = false;
  struct Rec { int kind; cudaEvent_t a, b; };
  mutable std::vector<Rec> recs;
  mutable std::vector<cudaEvent_t> pool;
};

namespace {

thread_local std::string g_last_error;

fbp_status fail(fbp_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

fbp_status cuda_fail(cudaError_t e, const char* where) {
  return fail(FBP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Schur-Cohn / step-down test: all roots of z^Q + a1 z^{Q-1} + ... + aQ strictly
// inside the unit circle iff every reflection coefficient has |k| < 1.
bool stable(int q, const double* a) {
  std::vector<double> c(a, a + q);
  for (int ord = q; ord >= 1; --ord) {
    const double k = c[ord - 1];
    if (!(std::fabs(k) < 1.0)) return false;
    const double den = 1.0 - k * k;
    std::vector<double> nc(ord - 1);
    for (int i = 1; i <= ord - 1; ++i) nc[i - 1] = (c[i - 1] - k * c[ord - i - 1]) / den;
    c.swap(nc);
  }
  return true;
}

// Companion matrix of A(z) acting on the state (y[n], y[n-1], ..., y[n-QM+1]).
void companion(int QM, const double* a_pad, std::vector<double>& A) {
  A.assign((size_t)QM * QM, 0.0);
  for (int j = 0; j < QM; ++j) A[j] = -a_pad[j];
  for (int i = 1; i < QM; ++i) A[(size_t)i * QM + (i - 1)] = 1.0;
}

void matmul(int n, const std::vector<double>& X, const std::vector<double>& Y,
            std::vector<double>& Z) {
  std::vector<double> T((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) T[(size_t)i * n + j] += X[(size_t)i * n + k] * Y[(size_t)k * n + j];
  Z.swap(T);
}

void matpow(int n, const std::vector<double>& X, long long e, std::vector<double>& Z) {
  std::vector<double> R((size_t)n * n, 0.0), B = X;
  for (int i = 0; i < n; ++i) R[(size_t)i * n + i] = 1.0;
  while (e > 0) {
    if (e & 1) matmul(n, R, B, R);
    matmul(n, B, B, B);
    e >>= 1;
  }
  Z.swap(R);
}

Geometry make_geometry(int N, int qm) {
  Geometry g{};
  int n = 0;
  while ((1 << n) < N) ++n;
  g.n = n;
  g.N = N;
  g.W = 2 * N;
  g.k1 = (n + 1) / 2;
  g.m = n - g.k1;
  g.H = 1 << g.k1;
  g.NB = 1 << g.m;
  g.WR = (N + g.NB + 3) / 4 * 4;
  g.XA = std::max(8, std::min(128, g.W));
  while (g.XA > 8 && fht_pass_a_smem(g) > 220 * 1024) g.XA /= 2;
  g.XB = std::max(8, std::min(128, N));
  while (g.XB > 8 && fht_pass_b_smem(g) > 220 * 1024) g.XB /= 2;
  g.L = (g.W >= 1024) ? 32 : (g.W >= 32 ? g.W / 32 : 1);
  g.iir_qm = qm;
  return g;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

fbp_status check_call(const fbp_plan* plan, const void* in, const void* out, int batch) {
  if (!plan) return fail(FBP_ERR_PARAM, "plan is NULL");
  if (batch < 0 || batch > plan->max_batch)
    return fail(FBP_ERR_PARAM, "batch " + std::to_string(batch) + " outside [0, max_batch=" +
                                   std::to_string(plan->max_batch) + "]");
  if (batch == 0) return FBP_OK;
  if (!in || !out) return fail(FBP_ERR_PARAM, "NULL data pointer");
  if (!aligned16(in) || !aligned16(out)) return fail(FBP_ERR_PARAM, "pointer not 16-byte aligned");
  return FBP_OK;
}

cudaEvent_t pool_get(const fbp_plan* p) {
  if (!p->pool.empty()) {
    cudaEvent_t e = p->pool.back();
    p->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Run one kernel launcher; when profiling, bracket it with events on its stream.
// RAII NVTX range (host timeline of each entry point and kernel launch; no cost
// without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <typename Fn>
cudaError_t timed(const fbp_plan* p, int kind, cudaStream_t st, Fn&& fn) {
  static const char* const kNames[] = {"fbp:iir", "fbp:fht_pass_a", "fbp:fht_pass_b", "fbp:fwd_pass_a",
                                       "fbp:fwd_pass_b", "fbp:resample", "fbp:small"};
  NvtxRange range(kind >= 0 && kind < 7 ? kNames[kind] : "fbp:kernel");
  if (!p->profiling) return fn();
  cudaEvent_t a = pool_get(p), b = pool_get(p);
  cudaEventRecord(a, st);
  cudaError_t e = fn();
  cudaEventRecord(b, st);
  p->recs.push_back({kind, a, b});
  return e;
}

// FHT back projection of `slices` linograms (device) into images, via plan->R.
cudaError_t run_backproject(const fbp_plan* p, const float* lin, float* img, int slices,
                            float scale, cudaStream_t st, int* launches) {
  const long long lin_elems = 4LL * p->g.N * p->g.W;
  cudaError_t e = timed(p, 1, st, [&] {
    return launch_fht_pass_a(lin, p->R, slices, 0, 4, lin_elems, p->g, st, launches);
  });
  if (e != cudaSuccess) return e;
  e = timed(p, 2, st, [&] { return launch_fht_pass_b(p->R, img, slices, 0, scale, p->g, st, launches); });
  if (e != cudaSuccess) return e;
  return timed(p, 2, st, [&] { return launch_fht_pass_b(p->R, img, slices, 1, scale, p->g, st, launches); });
}

// Fast path: sweep (IIR fused or not) into plan->R, then the two Eq.22 pairs.
cudaError_t run_fast(const fbp_plan* p, const float* lin, float* img, int batch, float scale,
                     bool iir, cudaStream_t st, int* launches) {
  const Geometry& g = p->g;
  const long long lin_elems = 4LL * g.N * g.W;
  const long long img_elems = (long long)g.N * g.N;
  for (int s0 = 0; s0 < batch; s0 += p->group) {
    const int ns = std::min(p->group, batch - s0);
    cudaError_t e = timed(p, 1, st, [&] {
      return launch_sweep_a(lin + s0 * lin_elems, p->R, ns, 0, 4, lin_elems, p->sg, p->si, iir,
                            p->counter, st, launches);
    });
    if (e != cudaSuccess) return e;
    for (int pair = 0; pair < 2; ++pair) {
      e = timed(p, 2, st, [&] {
        return launch_pair_b(p->R, img + s0 * img_elems, ns, pair, scale, p->sg, st, launches);
      });
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t run_reconstruct(const fbp_plan* p, const float* sino, float* img, int batch,
                            cudaStream_t st, int* launches) {
  const Geometry& g = p->g;
  const long long lin_elems = 4LL * g.N * g.W;
  const long long img_elems = (long long)g.N * g.N;
  const float w = 1.0f / (float)g.N;  // exact power of two (R7)
  const long long fam_elems = (long long)g.N * g.W;
  if (p->fast) return run_fast(p, sino, img, batch, w, true, st, launches);
  if (p->small_iir)
    return timed(p, 6, st, [&] { return launch_small(sino, img, batch, p->sk, w, st, launches); });
  if (p->per_family) {
    // Large N: one line family at a time, so that the filtered family (N x 2N
    // fp32, 32 MiB at N = 2048) is consumed by pass A while it is L2-resident;
    // pass B runs once both families of its Eq.22 pair are done.
    for (int s = 0; s < batch; ++s) {
      const float* S = sino + s * lin_elems;
      for (int f = 0; f < 4; ++f) {
        cudaError_t e = timed(p, 0, st, [&] {
          return launch_iir_rows(S + f * fam_elems, p->F, g.N, g, p->iir, p->lane_mats, st, launches);
        });
        if (e != cudaSuccess) return e;
        e = timed(p, 1, st, [&] {
          return launch_fht_pass_a(p->F, p->R, 1, f, 1, fam_elems, g, st, launches);
        });
        if (e != cudaSuccess) return e;
        if (f & 1) {
          e = timed(p, 2, st, [&] {
            return launch_fht_pass_b(p->R, img + s * img_elems, 1, f >> 1, w, g, st, launches);
          });
          if (e != cudaSuccess) return e;
        }
      }
    }
    return cudaSuccess;
  }
  for (int s0 = 0; s0 < batch; s0 += p->group) {
    const int ns = std::min(p->group, batch - s0);
    cudaError_t e = timed(p, 0, st, [&] {
      return launch_iir_rows(sino + s0 * lin_elems, p->F, (long long)ns * 4 * g.N, g, p->iir,
                             p->lane_mats, st, launches);
    });
    if (e != cudaSuccess) return e;
    e = run_backproject(p, p->F, img + s0 * img_elems, ns, w, st, launches);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

extern "C" {

const char* fbp_status_str(fbp_status s) {
  switch (s) {
    case FBP_OK: return "FBP_OK";
    case FBP_ERR_PLAN: return "FBP_ERR_PLAN: N must be a power of two in [2, 8192]";
    case FBP_ERR_PARAM: return "FBP_ERR_PARAM: invalid argument";
    case FBP_ERR_UNSTABLE: return "FBP_ERR_UNSTABLE: feedback polynomial has a root with |z| >= 1";
    case FBP_ERR_CUDA: return "FBP_ERR_CUDA: CUDA runtime error";
    case FBP_ERR_NOMEM: return "FBP_ERR_NOMEM: workspace allocation failed";
    case FBP_ERR_DEVICE: return "FBP_ERR_DEVICE: device missing or not sm_100";
  }
  return "unknown fbp_status";
}

const char* fbp_last_error(void) { return g_last_error.c_str(); }

fbp_status fbp_plan_create(fbp_plan** out, int n, int max_batch, int m, const double* b, int q,
                           const double* a, int device) {
  g_last_error.clear();
  if (!out) return fail(FBP_ERR_PARAM, "out is NULL");
  *out = nullptr;
  if (n < 2 || n > 8192 || (n & (n - 1)) != 0)
    return fail(FBP_ERR_PLAN, "N=" + std::to_string(n) + " is not a power of two in [2, 8192]");
  if (max_batch < 1) return fail(FBP_ERR_PARAM, "max_batch must be >= 1");
  if (m < 1 || m > kMaxOrder || q < 0 || q > kMaxOrder)
    return fail(FBP_ERR_PARAM, "orders must satisfy 1 <= M <= 8, 0 <= Q <= 8");
  if (!b || (q > 0 && !a)) return fail(FBP_ERR_PARAM, "NULL coefficient pointer");
  for (int i = 0; i < m; ++i)
    if (!std::isfinite(b[i])) return fail(FBP_ERR_PARAM, "non-finite b coefficient");
  for (int i = 0; i < q; ++i)
    if (!std::isfinite(a[i])) return fail(FBP_ERR_PARAM, "non-finite a coefficient");
  if (!stable(q, a)) return fail(FBP_ERR_UNSTABLE, "feedback polynomial is not stable");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(FBP_ERR_DEVICE, "CUDA device " + std::to_string(device) + " not available");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(FBP_ERR_DEVICE, "cudaGetDeviceProperties failed");
  if (prop.major != 10 || prop.minor != 0)
    return fail(FBP_ERR_DEVICE, std::string("device is sm_") + std::to_string(prop.major) +
                                    std::to_string(prop.minor) + ", libfbp is built for sm_100a");
  DeviceGuard guard(device);

  fbp_plan* p = new fbp_plan();
  p->device = device;
  p->max_batch = max_batch;
  const int qm = (std::max(m - 1, q) <= 3) ? 3 : 8;
  p->g = make_geometry(n, qm);
  p->g.iir_mc = std::max(1, m - 1);

  // ---- coefficient tables (double on the host, fp32 for the kernels) ----
  double beta = 0.0;
  for (int i = 0; i < m; ++i) beta += b[i];
  std::memset(&p->iir, 0, sizeof(p->iir));
  p->iir.beta = (float)beta;
  for (int k = 0; k < m - 1; ++k) {
    double s = 0.0;
    for (int j = k + 1; j < m; ++j) s += b[j];
    p->iir.c[k] = (float)(-s);
  }
  std::vector<double> apad(qm, 0.0);
  for (int k = 0; k < q; ++k) {
    apad[k] = a[k];
    p->iir.a[k] = (float)a[k];
  }
  std::vector<double> A, Pk;
  companion(qm, apad.data(), A);
  auto put = [qm](float* dst, const std::vector<double>& M) {
    for (int i = 0; i < qm; ++i)
      for (int j = 0; j < qm; ++j) dst[i * kMaxOrder + j] = (float)M[(size_t)i * qm + j];
  };
  for (int k = 0; k < kScanSteps; ++k) {
    matpow(qm, A, (long long)p->g.L << k, Pk);
    put(p->iir.P[k], Pk);
  }
  matpow(qm, A, 32LL * p->g.L, Pk);
  put(p->iir.AW, Pk);
  for (int i = 0; i < 32; ++i) {   // g_m[i] = (A^(i+1))_{0m}
    matpow(qm, A, i + 1, Pk);
    for (int m2 = 0; m2 < qm; ++m2) p->iir.G[i][m2] = (float)Pk[(size_t)m2];
  }
  std::vector<float> lm((size_t)32 * kMaxOrder * kMaxOrder, 0.0f);
  for (int j = 0; j < 32; ++j) {
    matpow(qm, A, (long long)p->g.L * j, Pk);
    put(lm.data() + (size_t)j * kMaxOrder * kMaxOrder, Pk);
  }

  // ---- fast path: sweep kernels (M, Q <= 3; N in the supported set; the
  //      anticausal look-ahead D tiles long enough for a 1e-9 tail, R22) ----
  if (sweep_supported(n) && m <= 3 && q <= 3) {
    SweepGeom& sg = p->sg;
    sg.N = n;
    sg.W = 2 * n;
    sg.NB = p->g.NB;
    sg.H = p->g.H;
    sg.X = 4096 / sg.H;
    sg.WR = p->g.WR;
    sg.nt = sg.W / sg.X;
    sg.P = 0;   // pass B L2 prefetch distance in items: 0 measured best since pair 0 runs 3 CTAs/SM
                // (0.447 vs 0.453 ms at 1, r01); the TMA double buffer covers the fills
#if FBP_DEV_MASK
    if (const char* ev = std::getenv("FBP_PREFETCH")) sg.P = std::atoi(ev);
#endif
    // pass-B x-tile: 64 for NB = 16 and 32 (double-buffered TMA fills at 3 CTAs/SM; measured
    // 5 % faster than 128 single-buffered at NB = 32 and 31 % faster at NB = 16, N = 512),
    // 32 for NB = 64 (N = 4096: radix 8+8, single-buffered; 64 measured 14 % slower)
    sg.XB = (sg.NB == 64) ? 32 : 64;
#if FBP_DEV_MASK
    // developer tuning knobs: compiled in only with -DFBP_DEV_MASK=1
    if (const char* ev = std::getenv("FBP_XB")) sg.XB = std::atoi(ev);
    if (const char* ev = std::getenv("FBP_SWEEP_CTAS")) sg.ctas_a = std::atoi(ev);
    if (const char* ev = std::getenv("FBP_SWEEP_SEG")) sg.nseg = std::atoi(ev);
    if (const char* ev = std::getenv("FBP_DBG")) sg.dbg = std::atoi(ev);
#endif
    // impulse response of B(z)/A(z) in double; tail bound over lags >= D*X - 2
    const int K = 1 << 16;
    std::vector<double> h(K, 0.0);
    for (int i = 0; i < K; ++i) {
      double v = (i < m) ? b[i] : 0.0;
      for (int k = 1; k <= q && k <= i; ++k) v -= a[k - 1] * h[i - k];
      h[i] = v;
    }
    std::vector<double> tail(K + 1, 0.0);
    for (int i = K - 1; i >= 0; --i) tail[i] = tail[i + 1] + std::fabs(h[i]);
    int D = 0;
    // R22: dropped tail <= 1e-9 of ||h||_1, ~60x below one fp32 ulp (2^-24) of the
    // carried sums (1e-12 gave bit-identical N = 2048 results with one more tile);
    // developer override FBP_TAIL (timing studies only, developer builds only)
    double tail_eps = 1e-9;
#if FBP_DEV_MASK
    if (const char* ev = std::getenv("FBP_TAIL")) tail_eps = std::atof(ev);
#endif
    for (int d = 1; d <= 15; ++d) {   // (D+1) x 32 tensor-memory columns <= 512
      const int lag = std::max(0, d * sg.X - 2);
      if (lag < K && tail[lag] <= tail_eps * tail[0]) {
        D = d;
        break;
      }
    }
    if (D > 0 && std::isfinite(tail[0])) {
      sg.D = D;
      SweepIir& si = p->si;
      auto dup = [](double v) { return make_float2((float)v, (float)v); };
      double bb[3] = {0, 0, 0}, aa[3] = {0, 0, 0};
      for (int i = 0; i < m; ++i) bb[i] = b[i];
      for (int i = 0; i < q; ++i) aa[i] = a[i];
      si.beta = dup(bb[0] + bb[1] + bb[2]);
      si.c0 = dup(-(bb[1] + bb[2]));
      si.c1 = dup(-bb[2]);
      si.na1 = dup(-aa[0]);
      si.na2 = dup(-aa[1]);
      si.na3 = dup(-aa[2]);
      std::vector<double> A3, Pm;
      companion(3, aa, A3);
      auto put = [&](float2* dst, long long e) {
        matpow(3, A3, e, Pm);
        for (int i = 0; i < 9; ++i) dst[i] = dup(Pm[(size_t)i]);
      };
      put(si.M1, 32);
      put(si.M2, 64);
      put(si.MX, sg.X);
      put(si.M16, 16);
      for (int i = 0; i < 32; ++i) {   // anticausal homogeneous response table (sweep back step)
        matpow(3, A3, 32 - i, Pm);
        for (int m2 = 0; m2 < 3; ++m2) {
          if (i & 1) si.GA[i >> 1][m2].y = (float)Pm[(size_t)m2];
          else si.GA[i >> 1][m2].x = (float)Pm[(size_t)m2];
        }
      }
      int cols = 32;
      while (cols < 32 * (D + 1)) cols *= 2;
      sg.tmem_cols = cols;
      p->fast = true;
    }
  }

  // ---- small-N path (N <= 64): one CTA per slice, everything on-chip ----
  if (small_supported(n)) {
    p->small = true;
    p->small_iir = (m <= 3 && q <= 3);
    double bb[3] = {0, 0, 0}, aa[3] = {0, 0, 0};
    for (int i = 0; i < m && i < 3; ++i) bb[i] = b[i];
    for (int i = 0; i < q && i < 3; ++i) aa[i] = a[i];
    p->sk.N = n;
    p->sk.iir = 1;
    p->sk.beta = (float)(bb[0] + bb[1] + bb[2]);   // difference form (R16): beta + (1 - z^-1) C(z)
    p->sk.c0 = (float)(-(bb[1] + bb[2]));
    p->sk.c1 = (float)(-bb[2]);
    p->sk.na1 = (float)(-aa[0]);
    p->sk.na2 = (float)(-aa[1]);
    p->sk.na3 = (float)(-aa[2]);
  }

  // ---- workspace, sized for a group of slices ----
  const Geometry& g = p->g;
  const size_t f_slice = p->fast ? 0 : (size_t)4 * g.N * g.W * sizeof(float);
  // R also serves fbp_fht_forward's pass-A output (fwd_workspace_floats per slice)
  const size_t r_rows = (size_t)4 * g.NB * g.H;
  const size_t r_slice = std::max(r_rows * (p->fast ? (size_t)p->sg.WR : (size_t)g.WR), fwd_workspace_floats(g)) *
                         sizeof(float);
  // fast path: the whole max_batch in one group up to 8 GiB of R (a small trailing
  // group would leave most of the 444 sweep CTA slots idle); general path: 256 MiB
  const size_t budget = p->fast ? ((size_t)8 << 30) : ((size_t)256 << 20);
  long long grp = (long long)(budget / (f_slice + r_slice));
  grp = std::max<long long>(1, std::min<long long>(grp, max_batch));
  grp = std::min<long long>(grp, 16383);
  p->group = (int)grp;
  p->per_family = false;  // measured slower (r01 v2c): launch granularity outweighs L2 reuse
  p->F_bytes = f_slice * p->group;
  p->R_bytes = r_slice * p->group;
  if ((p->F_bytes && cudaMalloc(&p->F, p->F_bytes) != cudaSuccess) ||
      cudaMalloc(&p->R, p->R_bytes) != cudaSuccess ||
      cudaMalloc(&p->counter, 16) != cudaSuccess ||
      cudaMalloc(&p->lane_mats, lm.size() * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();
    fbp_plan_destroy(p);
    return fail(FBP_ERR_NOMEM, "workspace allocation failed");
  }
  // Entries of R that pass A never writes are read (and discarded) by pass B.
  cudaError_t e = cudaMemcpy(p->lane_mats, lm.data(), lm.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p->R, 0, p->R_bytes);
  if (e != cudaSuccess) {
    fbp_plan_destroy(p);
    return cuda_fail(e, "cudaMemset");
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fbp_plan_destroy(p);
    return cuda_fail(e, "plan init");
  }
  *out = p;
  return FBP_OK;
}

void fbp_plan_destroy(fbp_plan* p) {
  if (!p) return;
  DeviceGuard guard(p->device);
  cudaFree(p->F);
  cudaFree(p->R);
  cudaFree(p->counter);
  cudaFree(p->lane_mats);
  for (int i = 0; i < 2; ++i) {
    cudaFree(p->d_in[i]);
    cudaFree(p->d_out[i]);
    cudaFreeHost(p->h_in[i]);
    cudaFreeHost(p->h_out[i]);
  }
  if (p->s_copy) cudaStreamDestroy(p->s_copy);
  if (p->s_comp) cudaStreamDestroy(p->s_comp);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  for (auto& r : p->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : p->pool) cudaEventDestroy(e);
  delete p;
}

fbp_status fbp_iir_filter(const fbp_plan* p, const float* sino, float* filtered, int batch,
                          void* stream) {
  NvtxRange nvtx_range("fbp_iir_filter");
  fbp_status s = check_call(p, sino, filtered, batch);
  if (s != FBP_OK || batch == 0) return s;
  DeviceGuard guard(p->device);
  int launches = 0;
  cudaError_t e = timed(p, 0, (cudaStream_t)stream, [&] {
    return launch_iir_rows(sino, filtered, (long long)batch * 4 * p->g.N, p->g, p->iir,
                           p->lane_mats, (cudaStream_t)stream, &launches);
  });
  p->launches = launches;
  if (e != cudaSuccess) return cuda_fail(e, "fbp_iir_filter");
  return FBP_OK;
}

fbp_status fbp_fht_backproject(const fbp_plan* p, const float* lin, float* image, int batch,
                               float scale, void* stream) {
  NvtxRange nvtx_range("fbp_fht_backproject");
  fbp_status s = check_call(p, lin, image, batch);
  if (s != FBP_OK || batch == 0) return s;
  DeviceGuard guard(p->device);
  int launches = 0;
  const long long lin_elems = 4LL * p->g.N * p->g.W;
  const long long img_elems = (long long)p->g.N * p->g.N;
  if (p->fast) {
    cudaError_t e = run_fast(p, lin, image, batch, scale, false, (cudaStream_t)stream, &launches);
    p->launches = launches;
    if (e != cudaSuccess) return cuda_fail(e, "fbp_fht_backproject");
    return FBP_OK;
  }
  if (p->small) {
    SmallIir k = p->sk;
    k.iir = 0;
    cudaError_t e = timed(p, 6, (cudaStream_t)stream,
                          [&] { return launch_small(lin, image, batch, k, scale, (cudaStream_t)stream, &launches); });
    p->launches = launches;
    if (e != cudaSuccess) return cuda_fail(e, "fbp_fht_backproject");
    return FBP_OK;
  }
  for (int s0 = 0; s0 < batch; s0 += p->group) {
    const int ns = std::min(p->group, batch - s0);
    cudaError_t e = run_backproject(p, lin + s0 * lin_elems, image + s0 * img_elems, ns, scale,
                                    (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) {
      p->launches = launches;
      return cuda_fail(e, "fbp_fht_backproject");
    }
  }
  p->launches = launches;
  return FBP_OK;
}

fbp_status fbp_fht_forward(const fbp_plan* p, const float* image, float* lin, int batch, void* stream) {
  NvtxRange nvtx_range("fbp_fht_forward");
  fbp_status s = check_call(p, image, lin, batch);
  if (s != FBP_OK || batch == 0) return s;
  DeviceGuard guard(p->device);
  int launches = 0;
  const long long lin_elems = 4LL * p->g.N * p->g.W;
  const long long img_elems = (long long)p->g.N * p->g.N;
  // lin also stages the transposed image of pass A: the buffers must not overlap
  if (image < lin + batch * lin_elems && lin < image + batch * img_elems)
    return fail(FBP_ERR_PARAM, "fbp_fht_forward: image and lin overlap");
  const size_t per = fwd_workspace_floats(p->g) * sizeof(float);
  const int grp = (int)std::max<size_t>(1, std::min<size_t>(p->R_bytes / per, 16383));
  const cudaStream_t st = (cudaStream_t)stream;
  for (int s0 = 0; s0 < batch; s0 += grp) {
    const int ns = std::min(grp, batch - s0);
    cudaError_t e = timed(p, 3, st, [&] { return launch_fwd_a(image + s0 * img_elems, p->R, lin + s0 * lin_elems, ns, p->g, st, &launches); });
    if (e == cudaSuccess)
      e = timed(p, 4, st, [&] { return launch_fwd_b(p->R, lin + s0 * lin_elems, ns, p->g, st, &launches); });
    if (e != cudaSuccess) {
      p->launches = launches;
      return cuda_fail(e, "fbp_fht_forward");
    }
  }
  p->launches = launches;
  return FBP_OK;
}

fbp_status fbp_resample_sinogram(const fbp_plan* p, const float* sino, int n_angles, int n_bins, double dr,
                                 float* lin, int batch, void* stream) {
  NvtxRange nvtx_range("fbp_resample_sinogram");
  fbp_status s = check_call(p, sino, lin, batch);
  if (s != FBP_OK || batch == 0) return s;
  if (n_angles < 1 || n_bins < 1) return fail(FBP_ERR_PARAM, "n_angles and n_bins must be >= 1");
  if (!(dr > 0.0) || !std::isfinite(dr)) return fail(FBP_ERR_PARAM, "dr must be finite and > 0");
  DeviceGuard guard(p->device);
  int launches = 0;
  const long long lin_elems = 4LL * p->g.N * p->g.W;
  const long long sino_elems = (long long)n_angles * n_bins;
  const cudaStream_t st = (cudaStream_t)stream;
  for (int s0 = 0; s0 < batch; s0 += 16383) {
    const int ns = std::min(16383, batch - s0);
    cudaError_t e = timed(p, 5, st, [&] {
      return launch_resample(sino + s0 * sino_elems, lin + s0 * lin_elems, ns, n_angles, n_bins, dr, p->g, st,
                             &launches);
    });
    if (e != cudaSuccess) {
      p->launches = launches;
      return cuda_fail(e, "fbp_resample_sinogram");
    }
  }
  p->launches = launches;
  return FBP_OK;
}

fbp_status fbp_reconstruct(const fbp_plan* p, const float* sino, float* image, int batch,
                           void* stream) {
  NvtxRange nvtx_range("fbp_reconstruct");
  fbp_status s = check_call(p, sino, image, batch);
  if (s != FBP_OK || batch == 0) return s;
  DeviceGuard guard(p->device);
  int launches = 0;
  cudaError_t e = run_reconstruct(p, sino, image, batch, (cudaStream_t)stream, &launches);
  p->launches = launches;
  if (e != cudaSuccess) return cuda_fail(e, "fbp_reconstruct");
  return FBP_OK;
}

fbp_status fbp_reconstruct_host(const fbp_plan* cp, const float* sino, float* image, int batch) {
  NvtxRange nvtx_range("fbp_reconstruct_host");
  if (!cp) return fail(FBP_ERR_PARAM, "plan is NULL");
  if (batch < 0) return fail(FBP_ERR_PARAM, "batch < 0");
  if (batch == 0) return FBP_OK;
  if (!sino || !image) return fail(FBP_ERR_PARAM, "NULL data pointer");
  fbp_plan* p = const_cast<fbp_plan*>(cp);
  // the host path owns plan-level staging and streams: one host call at a time
  std::lock_guard<std::mutex> lock(p->host_mu);
  DeviceGuard guard(p->device);
  const Geometry& g = p->g;
  const size_t lin_elems = (size_t)4 * g.N * g.W;
  const size_t img_elems = (size_t)g.N * g.N;
  // pipeline granularity of the host path: at most 4 slices (or 512 MiB of
  // linogram) per stage, so that copies overlap compute and staging stays small
  const int grp = (int)std::max<size_t>(1, std::min<size_t>({(size_t)p->group, (size_t)4,
                                                             ((size_t)512 << 20) / (lin_elems * 4)}));
  cudaError_t e;
  // Are the caller's buffers page-locked?  Then copy directly, else stage.
  auto pinned = [](const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool in_pinned = pinned(sino), out_pinned = pinned(image);
  if (!p->s_copy) {
    if ((e = cudaStreamCreateWithFlags(&p->s_copy, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
  }
  for (int i = 0; i < 2; ++i) {
    if (!p->d_in[i]) {
      if (cudaMalloc(&p->d_in[i], lin_elems * grp * 4) != cudaSuccess ||
          cudaMalloc(&p->d_out[i], img_elems * grp * 4) != cudaSuccess) {
        cudaGetLastError();
        return fail(FBP_ERR_NOMEM, "host-path device buffers");
      }
    }
    if (!in_pinned && !p->h_in[i] && cudaMallocHost(&p->h_in[i], lin_elems * grp * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(FBP_ERR_NOMEM, "pinned staging");
    }
    if (!out_pinned && !p->h_out[i] && cudaMallocHost(&p->h_out[i], img_elems * grp * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(FBP_ERR_NOMEM, "pinned staging");
    }
  }
  cudaEvent_t ev_in[2], ev_done[2], ev_out[2];
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
    cudaEventRecord(ev_out[i], p->s_d2h);
  }
  int launches = 0;
  const int ngroups = (batch + grp - 1) / grp;
  // pending D2H (unpinned output) bookkeeping
  std::vector<int> out_group(2, -1);
  auto flush_out = [&](int slot) {
    if (out_group[slot] < 0) return;
    cudaEventSynchronize(ev_out[slot]);
    const int g0 = out_group[slot] * grp;
    const int ns = std::min(grp, batch - g0);
    std::memcpy(image + (size_t)g0 * img_elems, p->h_out[slot], (size_t)ns * img_elems * 4);
    out_group[slot] = -1;
  };
  e = cudaSuccess;
  for (int gi = 0; gi < ngroups && e == cudaSuccess; ++gi) {
    const int slot = gi & 1;
    const int s0 = gi * grp;
    const int ns = std::min(grp, batch - s0);
    const size_t in_bytes = (size_t)ns * lin_elems * 4, out_bytes = (size_t)ns * img_elems * 4;
    // slot reuse: previous compute on this slot must be done before overwriting d_in
    cudaStreamWaitEvent(p->s_copy, ev_done[slot], 0);
    const float* src = sino + (size_t)s0 * lin_elems;
    if (!in_pinned) {
      cudaEventSynchronize(ev_in[slot]);  // staging buffer free
      std::memcpy(p->h_in[slot], src, in_bytes);
      src = p->h_in[slot];
    }
    if ((e = cudaMemcpyAsync(p->d_in[slot], src, in_bytes, cudaMemcpyHostToDevice, p->s_copy)) != cudaSuccess) break;
    cudaEventRecord(ev_in[slot], p->s_copy);
    cudaStreamWaitEvent(p->s_comp, ev_in[slot], 0);
    cudaStreamWaitEvent(p->s_comp, ev_out[slot], 0);  // d_out[slot] drained
    if ((e = run_reconstruct(p, p->d_in[slot], p->d_out[slot], ns, p->s_comp, &launches)) != cudaSuccess) break;
    cudaEventRecord(ev_done[slot], p->s_comp);
    cudaStreamWaitEvent(p->s_d2h, ev_done[slot], 0);
    flush_out(slot);
    float* dst = out_pinned ? image + (size_t)s0 * img_elems : p->h_out[slot];
    if ((e = cudaMemcpyAsync(dst, p->d_out[slot], out_bytes, cudaMemcpyDeviceToHost, p->s_d2h)) != cudaSuccess) break;
    cudaEventRecord(ev_out[slot], p->s_d2h);
    if (!out_pinned) out_group[slot] = gi;
  }
  // always drain every stream (also after an error: no copy may still touch the
  // caller's buffers when this synchronous call returns)
  {
    const cudaError_t e1 = cudaStreamSynchronize(p->s_copy);
    const cudaError_t e2 = cudaStreamSynchronize(p->s_comp);
    const cudaError_t e3 = cudaStreamSynchronize(p->s_d2h);
    if (e == cudaSuccess) e = (e1 != cudaSuccess) ? e1 : (e2 != cudaSuccess) ? e2 : e3;
  }
  if (e == cudaSuccess)
    for (int i = 0; i < 2; ++i) flush_out(i);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(ev_in[i]);
    cudaEventDestroy(ev_done[i]);
    cudaEventDestroy(ev_out[i]);
  }
  p->launches = launches;
  if (e != cudaSuccess) return cuda_fail(e, "fbp_reconstruct_host");
  return FBP_OK;
}

long long fbp_plan_launch_count(const fbp_plan* p) { return p ? p->launches : -1; }

fbp_status fbp_plan_profile(fbp_plan* p, int enable) {
  if (!p) return fail(FBP_ERR_PARAM, "plan is NULL");
  DeviceGuard guard(p->device);
  for (auto& r : p->recs) {
    cudaEventSynchronize(r.b);
    p->pool.push_back(r.a);
    p->pool.push_back(r.b);
  }
  p->recs.clear();
  p->profiling = enable != 0;
  return FBP_OK;
}

fbp_status fbp_plan_kernel_times(fbp_plan* p, double* ms, long long* launches, int kinds) {
  if (!p || kinds < 0 || kinds > 7 || (kinds > 0 && (!ms || !launches)))
    return fail(FBP_ERR_PARAM, "fbp_plan_kernel_times: bad arguments");
  DeviceGuard guard(p->device);
  for (int k = 0; k < kinds; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
  }
  cudaError_t err = cudaSuccess;
  for (auto& r : p->recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) err = e;
    if (r.kind < kinds) {
      ms[r.kind] += t;
      launches[r.kind] += 1;
    }
    p->pool.push_back(r.a);
    p->pool.push_back(r.b);
  }
  p->recs.clear();
  if (err != cudaSuccess) return cuda_fail(err, "fbp_plan_kernel_times");
  return FBP_OK;
}

fbp_status fbp_plan_path(const fbp_plan* p, int* fast, int* lookahead_tiles, int* tile_width) {
  if (!p) return fail(FBP_ERR_PARAM, "plan is NULL");
  if (fast) *fast = p->fast ? 1 : 0;
  if (lookahead_tiles) *lookahead_tiles = p->fast ? p->sg.D : 0;
  if (tile_width) *tile_width = p->fast ? p->sg.X : 0;
  return FBP_OK;
}

fbp_status fbp_plan_info(const fbp_plan* p, int* n, int* k1, int* m, int* group,
                         long long* workspace_bytes) {
  if (!p) return fail(FBP_ERR_PARAM, "plan is NULL");
  if (n) *n = p->g.N;
  if (k1) *k1 = p->g.k1;
  if (m) *m = p->g.m;
  if (group) *group = p->group;
  if (workspace_bytes) *workspace_bytes = (long long)(p->F_bytes + p->R_bytes);
  return FBP_OK;
}

}  // extern "C"
