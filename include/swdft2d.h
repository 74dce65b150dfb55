/*
 * swdft2d.h — C ABI of libswdft2d.so, the B200 (sm_100a) 2D tree sliding-window DFT.
 *
 * Drop-in boundary for the reference's batch 2D tree SWDFT,
 *   swdft.tree2d.tree_swdft_2d(x, spec, loop_order, counter, budget, threads)
 *   (/root/reference/pkg/src/swdft/tree2d.py:175-202).
 * The reference has no FFI of its own (it is pure Python + numpy); these are the
 * entry points its ctypes binding would call.  Plain
 * pointers and sizes only: no torch types cross this boundary.
 *
 * Output convention (identical to the reference, core.py:258-285, tree2d.py:69):
 *   out[p0, p1, k0, k1], p in window-START coordinates (P_i = N_i - n_i + 1),
 *   = sum_{j0<n0, j1<n1} x[p0+j0, p1+j1] * exp(-2*pi*i*(j0*k0/n0 + j1*k1/n1)),
 *   C-contiguous interleaved (re, im), natural-order k, k0 on axis 2.
 *   Twiddles are core.make_twiddles (core.py:125-138), bitwise.
 *
 * Precision:
 *   SWDFT2D_PREC_FP64 -> complex128 out, every tree node computed with the
 *     reference's DAG and rounding order (core.py:223-246): bitwise equal to
 *     tree_swdft_2d / oracle.swfft_2d.
 *   SWDFT2D_PREC_FP32 -> complex64 out, fp32 arithmetic (FMA allowed);
 *     BASELINE.json tolerance: max |err| / ||window||_2 <= 1e-4.
 *
 * Streams: every launch is stream-ordered on the caller's cudaStream_t (passed
 * as void*).  Device memory: the twiddle tables and the guided K1 schedule's tile
 * counters (one 8-byte slot per stream) are allocated once per device and freed by
 * swdft2d_shutdown; a forward call allocates nothing, except the large-window path
 * when the caller gives it no workspace (see swdft2d_forward_ws).  swdft2d_forward_host
 * owns its device scratch (input rows + a ring of 4 output strips) and a pinned staging
 * ring, both cached between calls and freed by swdft2d_shutdown.
 * Errors: functions return SWDFT2D_OK (0) or a negative code; the message of
 * the last error on the calling thread is swdft2d_last_error().
 */
#ifndef SWDFT2D_H_
#define SWDFT2D_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWDFT2D_ABI_VERSION 1

/* status codes; the Python wrapper maps them onto the reference's exception
 * classes (core.py:23-56). */
#define SWDFT2D_OK 0
#define SWDFT2D_E_INVALID_ARG (-1)       /* ValueError                    */
#define SWDFT2D_E_SHAPE (-2)             /* core.ShapeError               */
#define SWDFT2D_E_WINDOW_TOO_LARGE (-3)  /* core.WindowTooLargeError      */
#define SWDFT2D_E_INVALID_WINDOW (-4)    /* core.InvalidWindowError       */
#define SWDFT2D_E_UNSUPPORTED (-6)       /* shape outside the CUDA paths  */
#define SWDFT2D_E_CUDA (-7)              /* CUDA runtime / launch failure */
#define SWDFT2D_E_NOMEM (-8)             /* device allocation failed      */

/* element type of x */
#define SWDFT2D_IN_F32 0
#define SWDFT2D_IN_F64 1
#define SWDFT2D_IN_C64 2
#define SWDFT2D_IN_C128 3

/* arithmetic precision == output element type */
#define SWDFT2D_PREC_FP32 0 /* complex64 out  */
#define SWDFT2D_PREC_FP64 1 /* complex128 out */

/* kernel selection for swdft2d_forward */
#define SWDFT2D_KERNEL_AUTO 0       /* KR if n0 = 1, else K1 (n <= 64), else KR + KC       */
#define SWDFT2D_KERNEL_STREAM 1     /* K1, input by register prefetch (LDG)               */
#define SWDFT2D_KERNEL_WINDOW 2     /* K0: per-(window, k1) DAG kernel (bring-up)          */
#define SWDFT2D_KERNEL_STREAM_TMA 3 /* K1, input tiles staged by TMA when x is addressable */
#define SWDFT2D_KERNEL_ROWS 4       /* KR: row-tree kernel, windows with n0 = 1 (1D), n1 <= 1024 */
#define SWDFT2D_KERNEL_SEPARABLE 5  /* KR (rows) + KC (columns) over a workspace, any n <= 1024 */

/* Largest window exponent handled by K1 / by K0, KR and KR + KC. */
#ifndef SWDFT2D_K1_MAX_M  /* tuning builds may raise it to try larger K1 windows */
#define SWDFT2D_K1_MAX_M 6
#endif
/* K1 also takes, in fp32, 128-row windows (m0 = 7) of n1 <= 32, 256-row windows of
 * n1 <= 4 and 512-row windows of n1 <= 2 (fp64: 128x1); the stream push (K2) stays at
 * SWDFT2D_K1_MAX_M. */
#ifndef SWDFT2D_K1_MAX_M0
#define SWDFT2D_K1_MAX_M0 9
#endif
#define SWDFT2D_K0_MAX_M 10

int swdft2d_abi_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char *swdft2d_last_error(void);

/* core.WindowSpec.check_fits (core.py:116-122) and P_i = N_i - n_i + 1.
 * Returns SWDFT2D_E_WINDOW_TOO_LARGE when n_i > N_i. */
int swdft2d_output_shape(int64_t N0, int64_t N1, int m0, int m1, int64_t *P0, int64_t *P1);

/* core.lattice_bytes + core.output_bytes (core.py:363-381): the reference's
 * memory accounting at 16 B per complex, used by the wrapper's budget check
 * (tree2d.py:195-196). */
int swdft2d_reference_bytes(int64_t N0, int64_t N1, int m0, int m1, int64_t *lattice_bytes,
                            int64_t *output_bytes);

/* core.make_twiddles(n) (core.py:125-138) into out[2*n] as interleaved float64
 * (re, im).  Same libm formula, bitwise equal to numpy's table on x86-64 glibc. */
int swdft2d_twiddles(int n, double *out_interleaved);

/*
 * Batch 2D tree SWDFT of window rows [p0_begin, p0_end) — replaces the compute of
 * tree_swdft_2d (tree2d.py:197-202: _levels_outer + coefficients() + normalize).
 *   x        device pointer, N0 x N1 elements of in_dtype, row stride ld_x elements
 *   m0, m1   window exponents (n_i = 2^m_i), as WindowSpec.exponents
 *   prec     SWDFT2D_PREC_FP32 / SWDFT2D_PREC_FP64
 *   scale    normalization factor (core.normalization_factor); 1.0 = mode "none"
 *   out      device pointer, (p0_end - p0_begin) x P1 x n0 x n1 complex of prec,
 *            C-contiguous; row p0 of the full output lands at out row p0 - p0_begin
 *   kernel   SWDFT2D_KERNEL_*
 *   stream   cudaStream_t (NULL = legacy default stream)
 * Reads only input rows [p0_begin, p0_end + n0 - 1), so a strip of x (with its
 * n0-1 halo rows) can be passed with p0 relative to the strip.
 */
int swdft2d_forward(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                    int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                    int kernel, void *stream);

/*
 * swdft2d_forward with a caller-owned device workspace.  Only the large-window path
 * (KR + KC: a window side above 64, or SWDFT2D_KERNEL_SEPARABLE) uses one: its stage-R
 * rows of a strip of window rows.  swdft2d_workspace_bytes gives the size the library
 * would pick (0 when the selected path needs none); any size of at least n0 stage-R
 * rows works (smaller = shorter strips).  With workspace == NULL the large-window path
 * takes its workspace stream-ordered from the device's default pool for the call
 * (cudaMallocAsync / cudaFreeAsync); every other path allocates nothing per call.
 */
int swdft2d_forward_ws(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                       int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                       void *workspace, int64_t workspace_bytes, int kernel, void *stream);

/* Workspace bytes swdft2d_forward_ws would use for this call (0: none needed). */
int swdft2d_workspace_bytes(int64_t N0, int64_t N1, int m0, int m1, int prec, int64_t p0_begin,
                            int64_t p0_end, int kernel, int64_t *bytes);

/*
 * Host-to-host forward: the call a numpy-based caller binds (the reference's
 * tree_swdft_2d takes and returns host arrays, tree2d.py:189,201-202).  Same arguments
 * as swdft2d_forward, but
 *   x         host pointer (pageable or pinned; a device pointer also works), N0 x N1
 *             elements of in_dtype, row stride ld_x
 *   out_host  host pointer, (p0_end - p0_begin) x P1 x n0 x n1 complex of prec.  Pinned
 *             memory (swdft2d_host_alloc, cudaHostAlloc, cudaHostRegister) is copied at
 *             the PCIe rate while later strips compute; pageable memory works at the
 *             driver's staged rate
 *   strip_bytes  device bytes per output strip (0: 512 MiB)
 * The input rows the window rows need are copied to the device, the output is computed
 * in strips of window rows into a ring of 4 device strips and copied out on two copy
 * streams while later strips compute, so the device holds at most 4 strips whatever the
 * output size (outputs larger than HBM are fine).  Compute is ordered on `stream`; the
 * call is synchronous: out_host is complete on return.  One host call runs at a time per
 * process (they share the link, the scratch and the staging ring).  Pageable destinations
 * are filled by SWDFT2D_HOST_THREADS worker threads (default: the online cores, at most 16)
 * from SWDFT2D_HOST_CHUNK_MB-sized (default 4) pinned staging chunks.
 */
int swdft2d_forward_host(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                         int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end,
                         void *out_host, int64_t strip_bytes, int kernel, void *stream);

/*
 * Device buffer -> host array, synchronous, ordered after the work queued on `stream`
 * (results that were left resident, the 1D / kD outputs).  Pinned destinations take one
 * cudaMemcpyAsync; pageable ones (a fresh numpy array) go through the same pinned staging
 * ring and worker threads as swdft2d_forward_host.
 */
int swdft2d_download(const void *dev_src, void *host_dst, int64_t bytes, void *stream);

/* Pinned (page-locked, portable) host memory for swdft2d_forward_host's buffers; NULL on
 * failure (swdft2d_last_error).  Free with swdft2d_host_free. */
void *swdft2d_host_alloc(int64_t bytes);
int swdft2d_host_free(void *p);

/*
 * The K1 launch schedule swdft2d_forward would use for window rows [p0_begin, p0_end)
 * on the current device (for tests and tuning; the reference has no equivalent):
 *   info = {mode (0 uniform row chunks on a persistent grid, 1 guided big-first chunks
 *           on a persistent grid with a tile counter, 2 one-shot grid: one CTA per tile,
 *           3 stream-K: grid CTAs each take an equal contiguous share of the
 *           column-block-major (column block, window row) space in cost units — every
 *           column block counted as its n0 - 1 warm-up rows plus its window rows — and
 *           walk it as one tile per column block touched; chunks = 0, no bounds),
 *           rows per tile (uniform), row chunks, tiles, grid CTAs, column blocks,
 *           CTA slots (SMs x occupancy), CTAs per SM}
 *   bounds[c] (c <= chunks, up to max_bounds entries): first window row of chunk c,
 *           relative to p0_begin; bounds[chunks] = p0_end - p0_begin.
 * Honours the SWDFT2D_K1_GUIDED / _ONESHOT / _RCH / _STREAMK overrides like the forward call.
 * SWDFT2D_E_UNSUPPORTED if (m0, m1, prec) has no K1 instantiation.
 */
int swdft2d_k1_schedule(int64_t N0, int64_t N1, int m0, int m1, int prec, int64_t p0_begin,
                        int64_t p0_end, int64_t info[8], int64_t *bounds, int max_bounds);

/* Whether K1 is instantiated for (m0, m1, prec): 1 yes, 0 no. */
int swdft2d_has_stream_kernel(int m0, int m1, int prec);

/* Static shape of the K1 instantiation for (m0, m1, prec):
 * info = {Q (J = 2^Q residue groups), TP1 (window columns per CTA), threads per CTA,
 *         dynamic shared memory bytes (LDG variant), rows per batch NB,
 *         1 if the TMA input-staging variant is used for TMA-addressable inputs}.
 * SWDFT2D_E_UNSUPPORTED if not instantiated. */
int swdft2d_stream_kernel_info(int m0, int m1, int prec, int64_t info[6]);

/*
 * Window-row strip partition for world ranks (single box):
 * rank g of G gets window rows [floor(P0*g/G), floor(P0*(g+1)/G)) and input rows
 * [p0_begin, p0_end + n0 - 1).  range = {p0_begin, p0_end, row_begin, row_end}.
 * Empty ranges are legal (P0 < G).
 */
int swdft2d_strip_range(int64_t P0, int m0, int rank, int world, int64_t range[4]);

/*
 * Single-process multi-GPU forward (SURVEY.md 8b "swdft2d_forward_multi", 8e): the
 * strip partition above over ndev devices driven from one host thread.  The reference
 * has no multi-device path; its axis-0 chunking is tree2d.py:22-27,58-64.
 *   x         device pointer on devs[0] (N0 x N1, row stride ld_x), ready on streams[0]
 *   devs      CUDA device ordinals; slot g owns strip g of ndev (duplicates allowed)
 *   stage[g]  g >= 1: buffer on devs[g] of (row_end - row_begin) x N1 elements of
 *             in_dtype (rows contiguous, ld = N1) that receives strip g with its
 *             n0-1 halo rows; stage[0] (and stage itself when ndev == 1) is unused
 *   outs[g]   buffer on devs[g] of (p0_end - p0_begin) x P1 x n0 x n1 complex of prec
 *   streams[g] cudaStream_t on devs[g]
 * Per slot g >= 1: streams[g] waits for x, copies the strip over NVLink (peer access is
 * enabled on first use; cudaMemcpyDefault), then runs swdft2d_forward on the stage.
 * Slot 0 computes straight from x.  Work later enqueued on streams[0] is ordered after
 * every strip copy, so x may be reused from there.  The library allocates no staging
 * (the caller's stage buffers; per-slot forwards behave as swdft2d_forward); outputs
 * stay on their devices (no gather, no reduction).
 */
int swdft2d_forward_multi(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x,
                          int m0, int m1, int prec, double scale, int ndev, const int *devs,
                          void *const *stage, void *const *outs, void *const *streams);

/*
 * One push of the row-push stream (SlidingRowStream2D.push_row, tree2d.py:205-303,
 * SPEC.md:335-343).  Rows must be pushed in order p0 = 0, 1, 2, ...; once
 * p0 >= n0 - 1 the (P1, n0, n1) slab of window row p0 - n0 + 1 is written to out
 * (equal, bitwise in fp64, to that row of the batch transform).
 *   row    device pointer, N1 elements of in_dtype
 *   state  incremental mode (m0, m1 <= SWDFT2D_K1_MAX_M): the tree's level state,
 *          swdft2d_stream_state_bytes bytes, zero-filled before the first push.  One
 *          K2 launch computes the pushed row's dim-1 tree nodes and the dim-0 levels
 *          from the state — the reference stream's O(n0 n1) work per position.
 *          NULL: recompute mode, K1 (or `kernel`) over the raw ring.
 *   ring   raw row ring, [2 n0, N1] complex of prec (row p at slots p mod n0 and
 *          p mod n0 + n0); required in recompute mode, optional (may be NULL) with state
 *   out    may be NULL while p0 < n0 - 1 (or to only advance the state)
 */
int swdft2d_stream_push(const void *row, int in_dtype, int64_t N1, void *ring, void *state, int m0,
                        int m1, int prec, double scale, int64_t p0, void *out, int kernel,
                        void *stream);

/* Bytes of the incremental stream state: (m0 * n0/2 + n0 - 1) * P1 * n1 complex of prec. */
int swdft2d_stream_state_bytes(int64_t N1, int m0, int m1, int prec, int64_t *bytes);

/*
 * The dim-0 tree down every column of a complex matrix z ([N0][cols], row stride ld_z,
 * complex of prec), written in the layout of the reference's k-D output:
 * out[p0 - p0_begin][c >> m_inner][k0][c & (2^m_inner - 1)].  The last level block of
 * treekd.tree_swdft_kd (treekd.py:102-121, kd_level_step for dimension 0) over the
 * stacked results of the inner dimensions, with the transpose of k0 into place fused
 * (KC).  1 <= m0 <= 10; cols a multiple of 2^m_inner.
 */
int swdft2d_forward_columns(const void *z, int prec, int64_t N0, int64_t cols, int64_t ld_z, int m0,
                            int m_inner, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                            void *stream);

/* Frees cached per-device state (twiddle tables, tile counters, swdft2d_forward_host's
 * device scratch and pinned staging).  Safe to call twice;
 * no call may be in flight on any stream. */
int swdft2d_shutdown(void);

#ifdef __cplusplus
}
#endif

#endif /* SWDFT2D_H_ */
