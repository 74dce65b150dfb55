/*
 * swdft2d_oracle.c — CPU restatement of the reference 2D Tree SWDFT.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  Nothing in the product path
 * (paper_1707_08213_b200/) may link, load or call it.
 *
 * What it restates (reference = /root/reference/pkg/src/swdft):
 *   - core.make_twiddles            core.py:125-138   (Omega[j] = cos(j*fl(2pi/n)) - i sin(...))
 *   - core.butterfly                core.py:223-246   (separately rounded: re=(wr*cr)-(wi*ci),
 *                                                      im=(wr*ci)+(wi*cr), out=shifted+(re,im))
 *   - tree2d.TreeLattice2D          tree2d.py:30-69   (double-buffered [rows, N1, n0, n1] lattice)
 *   - tree2d.row_level_step         tree2d.py:72-93   (levels 1..m1 along dim 1, first)
 *   - tree2d.col_level_step         tree2d.py:96-120  (levels m1+1..m1+m0 along dim 0)
 *   - tree2d._levels_outer          tree2d.py:123-129 (schedule) and coefficients() :66-69
 *   - tree2d._split / _run_chunks   tree2d.py:22-27,58-64 (contiguous axis-0 chunks per level,
 *                                                      barrier between levels -> pthreads here)
 *   - core.normalize                core.py:288-302   (values * float64(factor), per component)
 *
 * Output rows are computed as a *strip*: window rows [p0_begin, p0_end) are
 * produced from input rows [p0_begin, p0_end + n0 - 1) only.  The reference's
 * output for a strip of rows is bitwise identical to the same rows of a full
 * run, so large arrays are processed strip by strip with
 * a bounded lattice.  Compile with -ffp-contract=off (no FMA contraction): the
 * reference's float64 ufuncs round every multiply and add separately.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

/* tree2d._split (tree2d.py:22-27): contiguous chunks of [lo, hi), one per worker,
 * joined before the next level starts (the reference creates a pool per level). */
typedef void (*range_fn)(void *ctx, int64_t a, int64_t b);
typedef struct { range_fn fn; void *ctx; int64_t a, b; } range_job;

static void *range_job_run(void *p) {
    range_job *j = (range_job *)p;
    j->fn(j->ctx, j->a, j->b);
    return NULL;
}

static void par_for(int threads, int64_t lo, int64_t hi, range_fn fn, void *ctx) {
    int64_t span = hi - lo;
    if (span <= 0) return;
    int64_t parts = threads < span ? threads : span;
    if (parts <= 1) { fn(ctx, lo, hi); return; }
    int64_t step = (span + parts - 1) / parts;
    pthread_t tid[256];
    range_job jobs[256];
    int n = 0;
    for (int64_t a = lo; a < hi && n < 256; a += step, ++n) {
        jobs[n].fn = fn; jobs[n].ctx = ctx; jobs[n].a = a;
        jobs[n].b = a + step < hi ? a + step : hi;
    }
    for (int k = 1; k < n; ++k) pthread_create(&tid[k], NULL, range_job_run, &jobs[k]);
    range_job_run(&jobs[0]);
    for (int k = 1; k < n; ++k) pthread_join(tid[k], NULL);
}

#define ORACLE_ABI_VERSION 1

int swdft2d_oracle_abi_version(void) { return ORACLE_ABI_VERSION; }

/* core.py:125-138.  ang = arange(n) * (2.0*pi/n); re = cos(ang); im = -sin(ang). */
void swdft2d_oracle_twiddles(int n, double *re, double *im) {
    const double step = (2.0 * 3.141592653589793) / (double)n;
    for (int j = 0; j < n; ++j) {
        double ang = (double)j * step;
        re[j] = cos(ang);
        im[j] = -sin(ang);
    }
}

/* core.py:238-245, one element. */
static inline void bfly(double sr, double si, double wr, double wi, double cr, double ci,
                        double *outr, double *outi) {
    double re = wr * cr;
    re = re - wi * ci;
    double im = wr * ci;
    im = im + wi * cr;
    *outr = sr + re;
    *outi = si + im;
}

/* Shared state of one strip pass; the per-level bodies below run on chunks of axis 0. */
typedef struct {
    const double *x;
    int64_t ldx, R_in, N1, n0, n1, node, rowstride;
    const double *twr, *twi;  /* table of the level being computed */
    int64_t s, L, H, lo;      /* level shift, node count, modulus, threshold */
    const double *cur;
    double *scr;
    double scale;
    int apply_scale;
    double *out;
} strip_ctx;

/* level 0: cur[:, :, 0, 0] = x  (tree2d.py:51) */
static void level0_body(void *p, int64_t a, int64_t b) {
    strip_ctx *c = (strip_ctx *)p;
    double *cur = (double *)c->cur;
    for (int64_t r = a; r < b; ++r)
        for (int64_t col = 0; col < c->N1; ++col) {
            double *d = cur + 2 * (r * c->rowstride + col * c->node);
            d[0] = c->x[2 * (r * c->ldx + col)];
            d[1] = c->x[2 * (r * c->ldx + col) + 1];
        }
}

/* row level: tree2d.py:84-87.  p1 in [n1 - s, N1), i in [0, L). */
static void row_level_body(void *p, int64_t a, int64_t b) {
    strip_ctx *c = (strip_ctx *)p;
    for (int64_t r = a; r < b; ++r)
        for (int64_t p1 = c->lo; p1 < c->N1; ++p1) {
            const double *sh = c->cur + 2 * (r * c->rowstride + (p1 - c->s) * c->node);
            const double *cu = c->cur + 2 * (r * c->rowstride + p1 * c->node);
            double *o = c->scr + 2 * (r * c->rowstride + p1 * c->node);
            for (int64_t i = 0; i < c->L; ++i) {
                const int64_t ii = i % c->H, w = i * c->s;
                bfly(sh[2 * ii], sh[2 * ii + 1], c->twr[w], c->twi[w], cu[2 * ii], cu[2 * ii + 1],
                     &o[2 * i], &o[2 * i + 1]);
            }
        }
}

/* column level: tree2d.py:109-112.  p0 in [n0 - s, R), p1 in [n1 - 1, N1). */
static void col_level_body(void *p, int64_t a, int64_t b) {
    strip_ctx *c = (strip_ctx *)p;
    const int64_t n1 = c->n1;
    for (int64_t r = a; r < b; ++r)
        for (int64_t p1 = n1 - 1; p1 < c->N1; ++p1) {
            const double *sh = c->cur + 2 * ((r - c->s) * c->rowstride + p1 * c->node);
            const double *cu = c->cur + 2 * (r * c->rowstride + p1 * c->node);
            double *o = c->scr + 2 * (r * c->rowstride + p1 * c->node);
            for (int64_t i0 = 0; i0 < c->L; ++i0) {
                const int64_t ii = i0 % c->H, w = i0 * c->s;
                for (int64_t i1 = 0; i1 < n1; ++i1) {
                    const int64_t q = ii * n1 + i1, d = i0 * n1 + i1;
                    bfly(sh[2 * q], sh[2 * q + 1], c->twr[w], c->twi[w], cu[2 * q], cu[2 * q + 1],
                         &o[2 * d], &o[2 * d + 1]);
                }
            }
        }
}

/* coefficients(): cur[n0-1:, n1-1:] (tree2d.py:69), then normalize (core.py:301). */
static void extract_body(void *p, int64_t a, int64_t b) {
    strip_ctx *c = (strip_ctx *)p;
    const int64_t P1 = c->N1 - c->n1 + 1;
    for (int64_t r = a; r < b; ++r)
        for (int64_t p1 = 0; p1 < P1; ++p1) {
            const double *src =
                c->cur + 2 * ((r + c->n0 - 1) * c->rowstride + (p1 + c->n1 - 1) * c->node);
            double *dst = c->out + 2 * ((r * P1 + p1) * c->node);
            if (c->apply_scale) {
                for (int64_t k = 0; k < 2 * c->node; ++k) dst[k] = src[k] * c->scale;
            } else {
                memcpy(dst, src, (size_t)(2 * c->node) * sizeof(double));
            }
        }
}

/*
 * One strip through the levels-outer schedule.
 * x: interleaved complex128 input rows [row0, row0 + R_in) of an N1-wide array,
 *    leading dimension ldx (in complex elements).
 * out: interleaved complex128 [R_out, P1, n0, n1]; R_out = R_in - n0 + 1.
 * work: 2 * R_in * N1 * n0 * n1 complex (the two lattice buffers).
 */
static void strip_levels_outer(const double *x, int64_t ldx, int64_t R_in, int64_t N1, int m0,
                               int m1, const double *tw0r, const double *tw0i,
                               const double *tw1r, const double *tw1i, double scale,
                               int apply_scale, double *out, double *work, int threads) {
    strip_ctx c;
    memset(&c, 0, sizeof c);
    c.x = x; c.ldx = ldx; c.R_in = R_in; c.N1 = N1;
    c.n0 = (int64_t)1 << m0; c.n1 = (int64_t)1 << m1;
    c.node = c.n0 * c.n1; c.rowstride = N1 * c.node;
    c.scale = scale; c.apply_scale = apply_scale; c.out = out;
    double *cur = work, *scr = work + 2 * R_in * c.rowstride;
    c.cur = cur;
    par_for(threads, 0, R_in, level0_body, &c);

    for (int t = 1; t <= m1; ++t) {           /* _levels_outer, tree2d.py:125-126 */
        c.s = (int64_t)1 << (m1 - t); c.L = (int64_t)1 << t; c.H = c.L / 2; c.lo = c.n1 - c.s;
        c.twr = tw1r; c.twi = tw1i; c.cur = cur; c.scr = scr;
        par_for(threads, 0, R_in, row_level_body, &c);
        double *tmp = cur; cur = scr; scr = tmp;
    }
    for (int q = 1; q <= m0; ++q) {           /* tree2d.py:127-128 */
        c.s = (int64_t)1 << (m0 - q); c.L = (int64_t)1 << q; c.H = c.L / 2; c.lo = c.n0 - c.s;
        c.twr = tw0r; c.twi = tw0i; c.cur = cur; c.scr = scr;
        par_for(threads, c.lo, R_in, col_level_body, &c);
        double *tmp = cur; cur = scr; scr = tmp;
    }
    c.cur = cur;
    par_for(threads, 0, R_in - c.n0 + 1, extract_body, &c);
}

/*
 * Public oracle entry.  x: interleaved complex128 [N0, N1] (ldx = N1); output
 * rows [p0_begin, p0_end) into out (interleaved complex128 [p0_end-p0_begin, P1, n0, n1]).
 * scale: normalization factor (apply_scale=0 means mode "none": identity).
 * max_lattice_bytes bounds the lattice: the strip is split into sub-strips.
 * Returns 0 on success, -1 on bad arguments, -2 on allocation failure.
 */
int swdft2d_oracle_forward(const double *x, int64_t N0, int64_t N1, int m0, int m1,
                           int64_t p0_begin, int64_t p0_end, double scale, int apply_scale,
                           double *out, int threads, int64_t max_lattice_bytes) {
    if (m0 < 0 || m1 < 0 || m0 > 20 || m1 > 20) return -1;
    const int64_t n0 = (int64_t)1 << m0, n1 = (int64_t)1 << m1;
    if (n0 > N0 || n1 > N1) return -1;
    const int64_t P0 = N0 - n0 + 1, P1 = N1 - n1 + 1;
    if (p0_begin < 0 || p0_end > P0 || p0_begin > p0_end) return -1;
    if (p0_begin == p0_end) return 0;
    if (threads < 1) threads = 1;
    const int64_t per_row = 2 * N1 * n0 * n1 * 16; /* two lattice buffers, bytes per input row */
    int64_t chunk = max_lattice_bytes / per_row - (n0 - 1);
    if (chunk < 1) chunk = 1;

    double *tw0r = malloc(sizeof(double) * n0), *tw0i = malloc(sizeof(double) * n0);
    double *tw1r = malloc(sizeof(double) * n1), *tw1i = malloc(sizeof(double) * n1);
    if (!tw0r || !tw0i || !tw1r || !tw1i) { free(tw0r); free(tw0i); free(tw1r); free(tw1i); return -2; }
    swdft2d_oracle_twiddles((int)n0, tw0r, tw0i);
    swdft2d_oracle_twiddles((int)n1, tw1r, tw1i);

    int64_t want = p0_end - p0_begin;
    if (chunk > want) chunk = want;
    double *work = malloc((size_t)((chunk + n0 - 1) * per_row));
    if (!work) { free(tw0r); free(tw0i); free(tw1r); free(tw1i); return -2; }

    for (int64_t a = p0_begin; a < p0_end; a += chunk) {
        int64_t b = a + chunk < p0_end ? a + chunk : p0_end;
        int64_t R_in = (b - a) + n0 - 1;
        strip_levels_outer(x + 2 * a * N1, N1, R_in, N1, m0, m1, tw0r, tw0i, tw1r, tw1i, scale,
                           apply_scale, out + 2 * (a - p0_begin) * P1 * n0 * n1, work, threads);
    }
    free(work); free(tw0r); free(tw0i); free(tw1r); free(tw1i);
    return 0;
}

/*
 * Per-window DIT FFT (the reference's oracle.swfft_2d, oracle.py:118-133,166-187):
 * dim 1 first, then dim 0, residue-major stages.  Bitwise equal to the tree.
 * Computes a single window (p0, p1) into out (interleaved complex128 [n0, n1]).
 * Used by tests as an independent-schedule cross-check of the lattice restatement.
 */
static void fft_residue_major(double *buf, int64_t n, const double *twr, const double *twi,
                              double *tmp) {
    /* buf: n complex in natural sample order; classes of stride n/L hold length-L DFTs. */
    /* layout: cur[class][k], start classes = n, L = 1 */
    int64_t classes = n, L = 1;
    memcpy(tmp, buf, sizeof(double) * 2 * n);
    while (L < n) {
        const int64_t half = classes / 2, L2 = 2 * L, stride = n / L2;
        double *src = tmp, *dst = buf;
        for (int64_t c = 0; c < half; ++c)
            for (int64_t i = 0; i < L2; ++i) {
                const int64_t ii = i % L;
                const double *e = src + 2 * (c * L + ii);
                const double *o = src + 2 * ((c + half) * L + ii);
                bfly(e[0], e[1], twr[i * stride], twi[i * stride], o[0], o[1], &dst[2 * (c * L2 + i)],
                     &dst[2 * (c * L2 + i) + 1]);
            }
        memcpy(tmp, buf, sizeof(double) * 2 * n);
        classes = half;
        L = L2;
    }
    memcpy(buf, tmp, sizeof(double) * 2 * n);
}

int swdft2d_oracle_window_fft(const double *x, int64_t N0, int64_t N1, int m0, int m1, int64_t p0,
                              int64_t p1, double *out) {
    const int64_t n0 = (int64_t)1 << m0, n1 = (int64_t)1 << m1;
    if (p0 < 0 || p1 < 0 || p0 + n0 > N0 || p1 + n1 > N1) return -1;
    double *tw0r = malloc(sizeof(double) * n0), *tw0i = malloc(sizeof(double) * n0);
    double *tw1r = malloc(sizeof(double) * n1), *tw1i = malloc(sizeof(double) * n1);
    int64_t nmax = n0 > n1 ? n0 : n1;
    double *b = malloc(sizeof(double) * 2 * nmax), *t = malloc(sizeof(double) * 2 * nmax);
    swdft2d_oracle_twiddles((int)n0, tw0r, tw0i);
    swdft2d_oracle_twiddles((int)n1, tw1r, tw1i);
    /* rows: z[j0][k1] */
    for (int64_t j0 = 0; j0 < n0; ++j0) {
        for (int64_t j1 = 0; j1 < n1; ++j1) {
            b[2 * j1] = x[2 * ((p0 + j0) * N1 + p1 + j1)];
            b[2 * j1 + 1] = x[2 * ((p0 + j0) * N1 + p1 + j1) + 1];
        }
        fft_residue_major(b, n1, tw1r, tw1i, t);
        for (int64_t k1 = 0; k1 < n1; ++k1) {
            out[2 * (j0 * n1 + k1)] = b[2 * k1];
            out[2 * (j0 * n1 + k1) + 1] = b[2 * k1 + 1];
        }
    }
    /* columns */
    for (int64_t k1 = 0; k1 < n1; ++k1) {
        for (int64_t j0 = 0; j0 < n0; ++j0) {
            b[2 * j0] = out[2 * (j0 * n1 + k1)];
            b[2 * j0 + 1] = out[2 * (j0 * n1 + k1) + 1];
        }
        fft_residue_major(b, n0, tw0r, tw0i, t);
        for (int64_t k0 = 0; k0 < n0; ++k0) {
            out[2 * (k0 * n1 + k1)] = b[2 * k0];
            out[2 * (k0 * n1 + k1) + 1] = b[2 * k0 + 1];
        }
    }
    free(tw0r); free(tw0i); free(tw1r); free(tw1i); free(b); free(t);
    return 0;
}
