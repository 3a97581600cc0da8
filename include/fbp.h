/*
 * fbp.h -- C ABI of the B200-native fast filtered back projection hot path
 *          (arXiv 2007.06289: recursive ramp filter + Fast Hough Transform BP).
 *
 * All entry points are plain C: pointers, sizes and an opaque plan.  No torch
 * (or any C++) type crosses this boundary; no exception crosses it either.
 *
 * Data layout (the paper's (s,t) linogram, §4.1):
 *   linogram  S[batch][4][N][2N]  fp32, row-major, s contiguous.
 *             family f: 0 = L_v+, 1 = L_v-, 2 = L_h+, 3 = L_h-   (SPEC.md:41 order)
 *             row t in [0,N) = |shift|, column s in [0,2N) = x0 + N  (reading R2)
 *   image     img[batch][N][N]   fp32, row-major, img[y][x].
 *
 * Ownership: every data pointer is caller-owned.  Device pointers are CUDA
 * device memory of the plan's device (torch tensors' data_ptr()); host
 * pointers (fbp_reconstruct_host only) are ordinary or pinned host memory.
 * The plan owns its workspace and coefficient tables.  All device pointers
 * must be 16-byte aligned.
 *
 * Streams: device-pointer calls are asynchronous on `cuda_stream` (a
 * cudaStream_t; NULL = legacy default stream).  They never synchronise the
 * host.  The returned status reports argument validation and launch errors;
 * a kernel fault surfaces at the caller's next synchronisation.
 * A plan's workspace is single-stream: concurrent streams need one plan each.
 *
 * Errors: every call returns an fbp_status; fbp_last_error() returns a
 * thread-local human-readable detail of the last failure on this thread.
 */
#ifndef FBP_H_
#define FBP_H_

#if defined(__GNUC__)
#define FBP_API __attribute__((visibility("default")))
#else
#define FBP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fbp_plan fbp_plan; /* opaque; immutable after create */

typedef enum {
  FBP_OK = 0,
  FBP_ERR_PLAN = 1,     /* N not a power of two, N < 2 or N > 8192           */
  FBP_ERR_PARAM = 2,    /* NULL / misaligned pointer, batch < 0 or > max_batch,
                           M < 1, Q < 0, M > 8, Q > 8, non-finite coefficient  */
  FBP_ERR_UNSTABLE = 3, /* a root of z^Q + a_1 z^(Q-1) + ... + a_Q has |z| >= 1 */
  FBP_ERR_CUDA = 4,     /* a CUDA runtime call or kernel launch failed          */
  FBP_ERR_NOMEM = 5,    /* workspace allocation failed                          */
  FBP_ERR_DEVICE = 6    /* device missing or not sm_100 (B200)                  */
} fbp_status;

/*
 * fbp_plan_create -- validate parameters, derive coefficient tables, choose the
 * FHT level split, allocate workspace on `device`.
 *
 *   n         image size N (power of two, 2..8192)            PAPER.md:168 (§4.1)
 *   max_batch largest `batch` any later call may pass (>= 1)
 *   m, b      feedforward order M (1..8) and b_0..b_{M-1}     PAPER.md:112-117 (Eq.9)
 *   q, a      feedback order Q (0..8) and a_1..a_Q with Eq.9's sign:
 *               y[n] = sum_k b_k x[n-k] - sum_k a_k y[n-k]
 *             One coefficient set serves both directions      PAPER.md:153 (§3)
 *   device    CUDA device ordinal
 * Host pointers b, a are read during the call only.  On success *out receives
 * the plan; on failure *out is set to NULL.
 */
FBP_API fbp_status fbp_plan_create(fbp_plan** out, int n, int max_batch, int m, const double* b,
                           int q, const double* a, int device);

/* Free the plan and its workspace (NULL is a no-op).  The caller must ensure no
 * work using the plan is still pending on any stream. */
FBP_API void fbp_plan_destroy(fbp_plan* plan);

/*
 * fbp_iir_filter -- symmetric recursive ramp filter of every linogram row:
 *   filtered = p~+ + p~-     PAPER.md:140-149 (§3, Eq.12-13), per-direction
 *   feedback, zero initial state and zero extension at both row ends (R10, R11).
 *   sino, filtered: device [batch][4][N][2N]; in-place (sino == filtered) allowed.
 *   Unweighted (no 1/N).
 */
FBP_API fbp_status fbp_iir_filter(const fbp_plan* plan, const float* sino, float* filtered, int batch,
                          void* cuda_stream);

/*
 * fbp_fht_backproject -- back projection of a (filtered) linogram by the Fast
 * Hough Transform, four families summed:                PAPER.md:240-265 (§4.4-4.5)
 *   B_f[y][x]  = sum_t lin[f][t][x + N - d_t(y)]        (Eq.19-21, reading R4/R5)
 *   image[y][x] = scale*(B_0[y][x] + B_1[y][N-1-x]) + scale*(B_2[x][y] + B_3[x][N-1-y])
 *                                                        (Eq.22)
 *   lin: device [batch][4][N][2N];  image: device [batch][N][N] (overwritten).
 *   Additions only; bit-exact on integer-valued input when scale is a power of two.
 */
FBP_API fbp_status fbp_fht_backproject(const fbp_plan* plan, const float* lin, float* image, int batch,
                               float scale, void* cuda_stream);

/*
 * fbp_fht_forward -- forward dyadic projection (discrete Radon transform along
 * dyadic patterns) by the Fast Hough Transform, the four families of Eq.16:
 *   lin[f][t][s] = sum_{y<N} G_f[y][s - N + d_t(y)]     PAPER.md:199-202 (Eq.17),
 *   G_0 = image[y][x], G_1 = image[y][N-1-x], G_2 = image[x][y], G_3 = image[N-1-x][y]
 *   (Eq.16, reading R4); terms with a column outside [0, N) are dropped.
 *   image: device [batch][N][N];  lin: device [batch][4][N][2N] (overwritten).
 *   Additions only (bit-exact on integer-valued input); the exact adjoint of
 *   fbp_fht_backproject's per-family sums.  Uses the plan's workspace, so calls on
 *   one plan must not run concurrently; lin doubles as scratch (the transposed
 *   image), so image and lin must not overlap.  Errors: FBP_ERR_PARAM (NULL /
 *   misaligned pointer, batch outside [0, max_batch], overlapping buffers),
 *   FBP_ERR_CUDA.
 */
FBP_API fbp_status fbp_fht_forward(const fbp_plan* plan, const float* image, float* lin, int batch,
                                   void* cuda_stream);

/*
 * fbp_resample_sinogram -- scanner sinogram -> linogram (NEXT-2), the step before
 * the hot path:                                        PAPER.md:172-188 (Eq.14-15)
 *   sino: device [batch][n_angles][n_bins] fp32, p(r_j, theta_k) with theta_k =
 *         k*pi/n_angles the angle of the line normal (cos, sin) in image coordinates
 *         (x = column, y = row) and r_j = (j - (n_bins-1)/2)*dr the signed distance
 *         from the image centre (N/2, N/2) (reading R23);
 *   lin:  device [batch][4][N][2N] (overwritten): sample (f, t, s) = the sinogram
 *         linearly interpolated (angle and bin index; the row after the last angle
 *         is row 0 at -r; bins outside the detector read 0) at the (r, theta) of
 *         its line (Eq.14 for the line model of reading R2), divided by the Eq.15
 *         stretch sqrt(1 + (t/(N-1))^2) of that line.
 *   Errors: FBP_ERR_PARAM (NULL / misaligned pointer, batch outside [0, max_batch],
 *   n_angles or n_bins < 1, dr not finite and > 0), FBP_ERR_CUDA.
 */
FBP_API fbp_status fbp_resample_sinogram(const fbp_plan* plan, const float* sino, int n_angles, int n_bins,
                                         double dr, float* lin, int batch, void* cuda_stream);

/*
 * fbp_reconstruct -- the whole hot path: IIR ramp filter then FHT back
 * projection with weight w = 1/N (reading R7).
 *   sino: device [batch][4][N][2N];  image: device [batch][N][N].
 * Not required to equal fbp_fht_backproject(fbp_iir_filter(.), 1/N) bitwise.
 * On the fused fast path (fbp_plan_path) both recursions are truncated to the
 * same tail bound: the anticausal carry into each tile of X samples sums the
 * next D tiles only, and a sweep (or sweep segment) starts its causal recursion
 * from zero state D tiles before the first tile it needs.  D is the smallest tile
 * count whose dropped impulse-response tail is <= 1e-9 of its l1 norm
 * (reading R22).  The general path's recursions are exact, and so
 * are those of the small-N path (N <= 64 with M, Q <= 3: one CTA per slice runs
 * both recursions over whole rows, every FHT level and the Eq.22 sum on-chip;
 * fbp_fht_backproject uses the same kernel without the IIR for any M, Q).
 */
FBP_API fbp_status fbp_reconstruct(const fbp_plan* plan, const float* sino, float* image, int batch,
                           void* cuda_stream);

/*
 * fbp_reconstruct_host -- fbp_reconstruct on HOST buffers: stages slices to the
 * device (pinned staging, copies overlapped with compute on two internal
 * streams), reconstructs, copies images back.  Synchronous: returns when
 * `image` holds the result.  sino: host [batch][4][N][2N]; image: host [batch][N][N].
 * batch may exceed max_batch (processed in groups).  The plan's host-path staging
 * is created on first use; concurrent host-path calls on one plan are serialised
 * (a plan mutex), and the call drains its streams before returning, also on error.
 */
FBP_API fbp_status fbp_reconstruct_host(const fbp_plan* plan, const float* sino, float* image, int batch);

/* Static description of a status code. */
FBP_API const char* fbp_status_str(fbp_status s);

/* Thread-local detail of the last failure on the calling thread ("" if none). */
FBP_API const char* fbp_last_error(void);

/* Launch statistics of the last call on this plan (kernels launched); for the
 * bench's gpu_launches count.  Returns -1 for a NULL plan. */
FBP_API long long fbp_plan_launch_count(const fbp_plan* plan);

/*
 * Per-kernel device timing (CUDA events recorded on the launching stream around
 * every kernel while enabled).  fbp_plan_profile(plan, 1) clears and enables,
 * 0 disables.  fbp_plan_kernel_times synchronises on the recorded events and
 * writes, for kind k in {0: IIR, 1: FHT pass A, 2: FHT pass B, 3: forward FHT
 * pass A, 4: forward FHT pass B, 5: sinogram resampling, 6: small-N slice kernel
 * (N <= 64: IIR + FHT + Eq.22 in one kernel)}, the summed milliseconds ms[k] and
 * launch count launches[k] (arrays of length `kinds`, at most 7) since the last
 * enable, then clears the record.
 */
FBP_API fbp_status fbp_plan_profile(fbp_plan* plan, int enable);
FBP_API fbp_status fbp_plan_kernel_times(fbp_plan* plan, double* ms, long long* launches, int kinds);

/*
 * Schedule chosen for this plan.  *fast = 1: fused IIR + FHT pass-A sweep and
 * pair-wise pass B (N in {512, 1024, 2048, 4096}, M <= 3, Q <= 3, coefficient tail
 * bound met); 0: separate IIR and two-pass FHT kernels.  *lookahead_tiles = D,
 * *tile_width = X of the sweep (0 when not fast).  Any pointer may be NULL.
 */
FBP_API fbp_status fbp_plan_path(const fbp_plan* plan, int* fast, int* lookahead_tiles, int* tile_width);

/* Level split chosen for this plan: *k1 levels in pass A, *m levels in pass B. */
FBP_API fbp_status fbp_plan_info(const fbp_plan* plan, int* n, int* k1, int* m, int* slices_per_group,
                         long long* workspace_bytes);

#ifdef __cplusplus
}
#endif
#endif /* FBP_H_ */
