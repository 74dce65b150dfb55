// abi.cu — extern "C" boundary of libswdft2d.so (declared in include/swdft2d.h).
//
// Mirrors the validation, accounting and dispatch the reference does around its
// compute (tree2d.py:175-202, core.py:116-122, 363-388) and launches K1 (fused
// streaming tree, k1_stream.cuh) or K0 (per-window DAG, k0_window.cu) on the
// caller's stream.  No torch types, no host threads.  Device memory is allocated
// once per device (twiddle tables, guided-schedule tile counters) and freed by
// swdft2d_shutdown; a forward call allocates nothing, except the large-window path's
// workspace when the caller passes none (swdft2d_forward vs swdft2d_forward_ws).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/swdft2d.h"
#include "swdft2d_internal.h"

namespace swdft2d {

void k1_register_m0_0();
void k1_register_m0_1();
void k1_register_m0_2();
void k1_register_m0_3();
void k1_register_m0_4();
void k1_register_m0_5();
void k1_register_m0_6();
void k1_register_m0_7();
void k1_register_m0_8();
void k1_register_m0_9();

static thread_local std::string g_last_error;
// K1 input path: register prefetch (LDG, default) or TMA tile staging (SWDFT2D_TMA=1).
// Measured on B200 (profiles/TMA_r01.md): the input is ~0.2 % of the traffic and the
// LDG variant is 3-12 % faster on configs 2-4 and level on config 5.
// K1 schedule override: SWDFT2D_K1_GUIDED=1 forces the guided schedule, =0 the uniform
// one; unset = the measured rule in swdft2d_forward
static const int g_k1_guided = [] {
    const char *e = std::getenv("SWDFT2D_K1_GUIDED");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
}();
// K1 grid: SWDFT2D_K1_ONESHOT=1 forces one CTA per tile (no persistence), =0 never;
// unset = the measured rule in swdft2d_forward (one-shot full-height tiles for 64-row
// windows with several waves of column blocks)
static const int g_k1_oneshot = [] {
    const char *e = std::getenv("SWDFT2D_K1_ONESHOT");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
}();
// K1 stream-K schedule: SWDFT2D_K1_STREAMK=k (k >= 1) forces equal contiguous shares of
// the (column block, window row) space over k x slots CTAs, =0 never; unset = the rule
static const int g_k1_streamk = [] {
    const char *e = std::getenv("SWDFT2D_K1_STREAMK");
    return e ? std::atoi(e) : -1;
}();
static const bool g_use_tma = [] {
    const char *e = std::getenv("SWDFT2D_TMA");
    return e && e[0] == '1';
}();

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int set_error(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

// ---- K1 registry ---------------------------------------------------------
// [m0][m1][prec][variant]: 0 LDG input, 1 TMA input, 2 the Z-column kernel (m1 = 0),
// 3 LDG with float32 input folded at compile time (fp32)
static const K1Info *g_k1[SWDFT2D_K1_MAX_M0 + 1][SWDFT2D_K1_MAX_M + 1][2][4];

void register_k1(const K1Info *info) { g_k1[info->m0][info->m1][info->prec][info->tma] = info; }

static void ensure_registered() {
    static std::once_flag once;
    std::call_once(once, [] {
        k1_register_m0_0();
        k1_register_m0_1();
        k1_register_m0_2();
        k1_register_m0_3();
        k1_register_m0_4();
        k1_register_m0_5();
        k1_register_m0_6();
        k1_register_m0_7();
        k1_register_m0_8();
        k1_register_m0_9();
    });
}

const K1Info *find_k1(int m0, int m1, int prec, int tma) {
    ensure_registered();
    if (m0 < 0 || m1 < 0 || m0 > SWDFT2D_K1_MAX_M0 || m1 > SWDFT2D_K1_MAX_M || prec < 0 ||
        prec > 1 || tma < 0 || tma > 3)
        return nullptr;
    return g_k1[m0][m1][prec][tma];
}

// ---- TMA tensor map for the input (driver entry point, no libcuda link) -----
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// Describes x as a 2D tensor of 4- or 8-byte elements (complex128 = 2 elements per
// sample); box = NB rows x (TP1 + n1 - 1) samples rounded up to 16 B.  Returns false
// when TMA cannot address x (alignment, strides, box limits): the LDG path is used.
static bool encode_input_map(const K1Info *k, const void *x, int in_dtype, int64_t N0, int64_t N1,
                             int64_t ldx, CUtensorMap *map, K1Params *P) {
    static const int sample_bytes[4] = {4, 8, 8, 16};
    const int sb = sample_bytes[in_dtype];
    const int elt = in_dtype == SWDFT2D_IN_F32 ? 4 : 8;
    const int per = sb / elt;
    const int n1 = 1 << k->m1;
    // + 16 B: the box starts at the 16-B boundary at or left of the tile's first sample
    const int row_bytes = ((k->tp1 + n1 - 1) * sb + 15) / 16 * 16 + (sb < 16 ? 16 : 0);
    const int box_w = row_bytes / elt;
    P->sample_bytes = sb;
    P->tma_per_sample = per;
    P->tma_row_bytes = row_bytes;
    if (((uintptr_t)x & 15) || ((ldx * sb) & 15) || box_w > 256 || k->nb > 256 ||
        N0 > 0x7fffffffLL || N1 * per > 0xffffffffLL)
        return false;
    auto fn = encode_fn();
    if (!fn) return false;
    const CUtensorMapDataType dt =
        in_dtype == SWDFT2D_IN_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
    const cuuint64_t gdim[2] = {(cuuint64_t)(N1 * per), (cuuint64_t)N0};
    const cuuint64_t gstride[1] = {(cuuint64_t)(ldx * sb)};
    const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)k->nb};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dt, 2, const_cast<void *>(x), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ---- per-device state ----------------------------------------------------
struct DeviceState {
    int sms = 0;
    void *k0_tw64 = nullptr;  // double2[K0_TW_N]
    void *k0_tw32 = nullptr;  // float2[K0_TW_N]
    std::map<const void *, int> occupancy;  // K1 function -> CTAs per SM
    // K1 uniform row-chunk choice per (rows, column blocks, slots, n0): the cost-model
    // scan is thousands of 64-bit divisions, too slow to redo on every call
    std::map<std::tuple<int64_t, int64_t, int64_t, int>, int64_t> rch;
    // guided K1 tile counters: blocks of zeroed 8-byte slots, one slot per stream handle
    std::vector<unsigned long long *> ctr_blocks;
    std::map<cudaStream_t, unsigned long long *> ctr;
};
static std::mutex g_mu;
static std::map<int, DeviceState> g_dev;

// core.make_twiddles (core.py:134-137): ang = j * fl(2*pi/n); (cos, -sin).
static void host_twiddles(int n, double *re, double *im) {
    const double step = (2.0 * 3.141592653589793) / (double)n;
    for (int j = 0; j < n; ++j) {
        const double ang = (double)j * step;
        re[j] = std::cos(ang);
        im[j] = -std::sin(ang);
    }
}


static int device_state(DeviceState **out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState &st = g_dev[dev];
    if (st.sms == 0) {
        e = cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess)
            return fail(SWDFT2D_E_CUDA, "cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
        // The stream-ordered allocations (K1's tile counter, the large-window workspace)
        // come from the device's default pool, whose release threshold is 0: every
        // synchronize would hand the memory back and the next call re-map it (measured:
        // +3.6 ms per config-3 call outside CUDA graphs).  Keep up to 1 GiB cached.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 1ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    *out = &st;
    return SWDFT2D_OK;
}

// Relaxes the calling thread's stream-capture mode for its scope (restores it after).
struct CaptureModeGuard {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    CaptureModeGuard() { cudaThreadExchangeStreamCaptureMode(&mode); }
    ~CaptureModeGuard() { cudaThreadExchangeStreamCaptureMode(&mode); }
};

static int k0_tables(DeviceState *st, const void **tw64, const void **tw32) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!st->k0_tw64) {
        static double re[K0_TW_N], im[K0_TW_N];
        static double2 h64[K0_TW_N];
        static float2 h32[K0_TW_N];
        host_twiddles(K0_TW_N, re, im);
        for (int i = 0; i < K0_TW_N; ++i) {
            h64[i] = make_double2(re[i], im[i]);
            h32[i] = make_float2((float)re[i], (float)im[i]);
        }
        // The first call may come while the caller's stream is being captured into a CUDA
        // graph: allocate with the thread's capture mode relaxed and upload on a private
        // non-blocking stream, so the one-time setup neither joins nor breaks the capture.
        CaptureModeGuard relaxed;
        cudaStream_t up = nullptr;
        cudaError_t e = cudaMalloc(&st->k0_tw64, sizeof h64);
        if (e == cudaSuccess) e = cudaMalloc(&st->k0_tw32, sizeof h32);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(st->k0_tw64, h64, sizeof h64, cudaMemcpyHostToDevice, up);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(st->k0_tw32, h32, sizeof h32, cudaMemcpyHostToDevice, up);
        if (e == cudaSuccess) e = cudaStreamSynchronize(up);
        if (up) cudaStreamDestroy(up);
        if (e != cudaSuccess) {
            cudaFree(st->k0_tw64);
            cudaFree(st->k0_tw32);
            st->k0_tw64 = st->k0_tw32 = nullptr;
            return fail(SWDFT2D_E_NOMEM, "twiddle table: %s", cudaGetErrorString(e));
        }
    }
    *tw64 = st->k0_tw64;
    *tw32 = st->k0_tw32;
    return SWDFT2D_OK;
}

static int k1_occupancy(DeviceState *st, const K1Info *info, int *occ) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = st->occupancy.find(info->func);
    if (it != st->occupancy.end()) {
        *occ = it->second;
        return SWDFT2D_OK;
    }
    cudaError_t e = cudaSuccess;
    if (info->smem_bytes > 48 * 1024)
        e = cudaFuncSetAttribute(info->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)info->smem_bytes);
    int n = 0;
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, info->func, info->threads,
                                                          info->smem_bytes);
    if (e != cudaSuccess)
        return fail(SWDFT2D_E_CUDA, "K1 occupancy (m0=%d m1=%d): %s", info->m0, info->m1,
                    cudaGetErrorString(e));
    if (n < 1)
        return fail(SWDFT2D_E_UNSUPPORTED, "K1 (m0=%d m1=%d) cannot be resident (smem %zu B)",
                    info->m0, info->m1, info->smem_bytes);
    st->occupancy[info->func] = n;
    *occ = n;
    return SWDFT2D_OK;
}

// Row-chunk size for K1 tiles: minimise (waves x rows per tile incl. the n0-1
// warm-up rows); an under-filled single wave is charged as if it ran at the
// fraction of the slots it occupies.
static int64_t k1_rows_per_tile(int64_t rows, int64_t CB, int64_t slots, int n0) {
    int64_t best_rch = rows;
    double best = 1e300;
    const int64_t rc_max = rows < 8192 ? rows : 8192;
    for (int64_t rc = 1; rc <= rc_max; ++rc) {
        const int64_t rch = (rows + rc - 1) / rc;
        const int64_t rca = (rows + rch - 1) / rch;
        const int64_t tiles = CB * rca;
        const double per = (double)(rch + n0 - 1);
        double cost;
        if (tiles >= slots) cost = (double)((tiles + slots - 1) / slots) * per;
        else cost = per * (double)slots / (double)tiles;
        if (cost < best * 0.999) {
            best = cost;
            best_rch = rch;
        }
    }
    return best_rch;
}

// Window rows per strip of the large-window path: the stage-R rows of R window rows
// (plus the n0 - 1 halo rows) fill the workspace; ~512 MB when the library chooses.
static int64_t sep_strip_rows(int64_t zrow, int64_t n0, int64_t rows, int64_t ws_bytes) {
    int64_t R;
    if (ws_bytes > 0) {
        R = ws_bytes / zrow - (n0 - 1);
    } else {
        R = ((int64_t)512 << 20) / zrow - (n0 - 1);
        if (R < 64) R = 64;
    }
    return R > rows ? rows : R;
}

// Large-window path (n0 or n1 above K1's 2^6, up to 2^10): the separable schedule in
// strips of window rows — KR writes the strip's stage-R rows Z (the dim-1 tree of each
// input row, unscaled) into a workspace, KC runs the dim-0 trees down Z's columns into
// the output.  The workspace is the caller's (swdft2d_forward_ws, sized by
// swdft2d_workspace_bytes; a smaller one just means shorter strips); without one the
// library takes <= ~512 MB stream-ordered from the device pool for the call
// (cudaMallocAsync / cudaFreeAsync on the caller's stream).
static int run_k1(DeviceState *ds, const K1Info *k1, K1Params &P, const CUtensorMap &tmap,
                  int64_t p0_begin, int64_t p0_end, const void *tw64, cudaStream_t st);
// Column trees of the large-window path: K1's 1-column Z-column kernel (n0 x 1 over Z,
// columns decomposed as (p1, k1), K1Params::col_m1) or KC.  K1 streams down the rows
// with the tree's reuse along p0 (no halo recompute, no Z re-reads) but pays an n0 - 1
// row warm-up per tile; KC recomputes each tile's halo.  Measured per window
// (scripts/sep_cols_sweep.py, ~4 GB outputs, profiles/sep_cols_r02_{kc,k1}.jsonl), K1 / KC:
// n1 = 128 with n0 = 2..64 1.02-1.22 (fp32 and fp64); 8x1024 1.12; 128x128 1.39 / 1.13
// (fp32 / fp64); 256x16, 256x64 fp32 1.13; 128x32 fp64 0.81 (the fp64 128-row kernel
// runs at 252 registers); 512-row fp32 0.91-0.94.  Short strips of small windows lose to
// K1's per-tile warm-up (8x1024 fp64 on 29 window rows: 0.92; 3-D 16x8x4 on 81: 0.83;
// 64x1024 on 8: 0.45), while tall windows win even on strips shorter than n0 (256x64 on
// 175 rows 1.13, 128x128 fp64 on 119 rows 1.13: KC's halo recompute grows with n0).  So K1
// for fp32 n0 <= 256, fp64 n0 <= 64 (and 128 when n1 >= 64), on strips of >= 32 window
// rows, and >= 8 n0 rows when n0 <= 16.
// SWDFT2D_SEP_COLS=kc / k1 forces one (k1 where instantiated).
static const int g_sep_cols = [] {
    const char *e = std::getenv("SWDFT2D_SEP_COLS");
    return e ? (e[0] == 'k' && e[1] == '1' ? 1 : 0) : -1;
}();

static bool use_k1_columns(int m0, int m_inner, int prec, int64_t rows) {
    if (g_sep_cols >= 0) return g_sep_cols == 1;
    const int64_t n0 = (int64_t)1 << m0;
    if (rows < 32 || (n0 <= 16 && rows < 8 * n0)) return false;
    if (prec == SWDFT2D_PREC_FP64) return m0 <= 6 || (m0 == 7 && m_inner >= 6);
    return m0 <= 8;
}

static int forward_separable(const void *x, int in_dtype, int64_t N1, int64_t ld_x, int m0,
                             int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end,
                             void *out, void *ws, int64_t ws_bytes, cudaStream_t st,
                             DeviceState *ds, const void *tw, const void *tw64) {
    const int64_t n0 = (int64_t)1 << m0, n1 = (int64_t)1 << m1;
    const int64_t P1 = N1 - n1 + 1, cols = P1 * n1;
    const int64_t esz = prec == SWDFT2D_PREC_FP64 ? 16 : 8;
    const int64_t rows = p0_end - p0_begin;
    const int64_t zrow = cols * esz;
    const int64_t R = sep_strip_rows(zrow, n0, rows, ws ? ws_bytes : 0);
    if (R < 1)
        return fail(SWDFT2D_E_INVALID_ARG,
                    "workspace of %lld B is below one strip (%lld B = n0 stage-R rows)",
                    (long long)ws_bytes, (long long)(n0 * zrow));
    void *z = ws;
    if (!z) {
        cudaError_t e = cudaMallocAsync(&z, (size_t)((R + n0 - 1) * zrow), st);
        if (e != cudaSuccess)
            return fail(SWDFT2D_E_NOMEM, "large-window workspace (%lld B): %s",
                        (long long)((R + n0 - 1) * zrow), cudaGetErrorString(e));
    }
    int rc = SWDFT2D_OK;
    cudaError_t ce;
    for (int64_t a = p0_begin; a < p0_end && rc == SWDFT2D_OK; a += R) {
        const int64_t b = a + R < p0_end ? a + R : p0_end;
        KRParams r;
        std::memset(&r, 0, sizeof r);
        r.x = x;
        r.in_dtype = in_dtype;
        r.N1 = N1;
        r.ldx = ld_x;
        r.p0_begin = a;
        r.p0_end = b + n0 - 1;  // input rows of the strip
        r.P1 = P1;
        r.out = z;
        r.scale = 1.0;
        r.tw = tw;
        r.sms = ds->sms;
        KCParams c;
        std::memset(&c, 0, sizeof c);
        c.z = z;
        c.cols = cols;
        c.ldz = cols;
        c.zrows = b - a + n0 - 1;
        c.P0s = b - a;
        c.P1 = P1;
        c.m1 = m1;
        c.apply_scale = scale == 1.0 ? 0 : 1;
        c.scale = scale;
        c.out = static_cast<char *>(out) + (a - p0_begin) * P1 * n0 * n1 * esz;
        c.tw = tw;
        c.sms = ds->sms;
        const K1Info *kz = use_k1_columns(m0, m1, prec, b - a) ? find_k1(m0, 0, prec, 2) : nullptr;
        if (launch_kr(r, m1, prec, st)) {
            rc = fail(SWDFT2D_E_CUDA, "large-window launch setup failed (m0=%d m1=%d)", m0, m1);
        } else if (kz) {
            K1Params Pz;
            std::memset(&Pz, 0, sizeof Pz);
            CUtensorMap tmap;
            std::memset(&tmap, 0, sizeof tmap);
            Pz.x = z;
            Pz.in_dtype = prec == SWDFT2D_PREC_FP64 ? SWDFT2D_IN_C128 : SWDFT2D_IN_C64;
            Pz.N0 = c.zrows;
            Pz.N1 = cols;
            Pz.ldx = cols;
            Pz.P1 = cols;
            Pz.out = c.out;
            Pz.scale = scale;
            Pz.apply_scale = c.apply_scale;
            Pz.col_m1 = m1;
            rc = run_k1(ds, kz, Pz, tmap, 0, b - a, tw64, st);
        } else if (launch_kc(c, m0, prec, st)) {
            rc = fail(SWDFT2D_E_CUDA, "large-window launch setup failed (m0=%d m1=%d)", m0, m1);
        }
        if (rc == SWDFT2D_OK && (ce = cudaGetLastError()) != cudaSuccess)
            rc = fail(SWDFT2D_E_CUDA, "large-window kernel launch: %s", cudaGetErrorString(ce));
    }
    if (!ws) cudaFreeAsync(z, st);
    return rc;
}

// Which kernel family serves (m0, m1, prec, kernel); the error code when none does.
enum Path { PATH_KR, PATH_SEP, PATH_K1, PATH_K0 };

static int select_path(int m0, int m1, int prec, int kernel, Path *path) {
    if (kernel < SWDFT2D_KERNEL_AUTO || kernel > SWDFT2D_KERNEL_SEPARABLE)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown kernel code %d", kernel);
    if (kernel == SWDFT2D_KERNEL_ROWS && m0 != 0)
        return fail(SWDFT2D_E_UNSUPPORTED, "the row-tree kernel needs n0 = 1 (m0 = %d)", m0);
    if ((kernel == SWDFT2D_KERNEL_ROWS || kernel == SWDFT2D_KERNEL_AUTO ||
         kernel == SWDFT2D_KERNEL_SEPARABLE) && m0 == 0) {
        if (m1 > SWDFT2D_K0_MAX_M)
            return fail(SWDFT2D_E_UNSUPPORTED, "window 1 x 2^%d exceeds the CUDA paths (max 2^%d)",
                        m1, SWDFT2D_K0_MAX_M);
        *path = PATH_KR;
        return SWDFT2D_OK;
    }
    const K1Info *k1 = find_k1(m0, m1, prec, 0);
    if ((kernel == SWDFT2D_KERNEL_STREAM || kernel == SWDFT2D_KERNEL_STREAM_TMA) && !k1)
        return fail(SWDFT2D_E_UNSUPPORTED, "no K1 instantiation for m0=%d m1=%d prec=%d", m0, m1, prec);
    if (kernel != SWDFT2D_KERNEL_SEPARABLE && kernel != SWDFT2D_KERNEL_WINDOW && k1) {
        *path = PATH_K1;
        return SWDFT2D_OK;
    }
    if (m0 > SWDFT2D_K0_MAX_M || m1 > SWDFT2D_K0_MAX_M)
        return fail(SWDFT2D_E_UNSUPPORTED, "window 2^%d x 2^%d exceeds the CUDA paths (max 2^%d)",
                    m0, m1, SWDFT2D_K0_MAX_M);
    *path = kernel == SWDFT2D_KERNEL_WINDOW ? PATH_K0 : PATH_SEP;
    return SWDFT2D_OK;
}

// The K1 launch schedule of window rows [p0_begin, p0_end) (filled into P: CB, RCH,
// ntiles, nchunks, chunk[]): uniform row chunks on a persistent grid, guided big-first
// chunks on a persistent grid with a tile counter, or a one-shot grid (one CTA per tile).
struct K1Plan {
    int occ = 0;
    int64_t slots = 0, grid = 0;
    bool oneshot = false, guided = false, streamk = false;
};

static int k1_plan(DeviceState *ds, const K1Info *k1, int64_t P1, int64_t p0_begin,
                   int64_t p0_end, K1Params *P, K1Plan *pl) {
    const int n0 = 1 << k1->m0;
    int rc = k1_occupancy(ds, k1, &pl->occ);
    if (rc) return rc;
    P->p0_begin = p0_begin;
    P->p0_end = p0_end;
    P->CB = (P1 + k1->tp1 - 1) / k1->tp1;
    const int64_t rows = p0_end - p0_begin;
    const int64_t slots = (int64_t)ds->sms * pl->occ;
    pl->slots = slots;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const auto key = std::make_tuple(rows, P->CB, slots, n0);
        auto it = ds->rch.find(key);
        if (it == ds->rch.end()) {
            if (ds->rch.size() > 4096) ds->rch.clear();
            it = ds->rch.emplace(key, k1_rows_per_tile(rows, P->CB, slots, n0)).first;
        }
        P->RCH = it->second;
    }
    // One-shot grid of full-height tiles (one CTA per column block, scheduled by the
    // hardware) for 64-row windows when the column blocks fill >= 3 waves: their 63
    // warm-up rows make short tiles expensive, and short-lived CTAs write faster than
    // a persistent grid (profiles/write_probe3_r01.jsonl).  Config 5: 804-810 ->
    // 825-841 Gcoef/s over three alternations (profiles/k1_oneshot_r01.jsonl).  For
    // n0 <= 32 the gain was within noise (config 4 +0-1.5 %), so they stay persistent.
    const bool oneshot = g_k1_oneshot >= 0 ? g_k1_oneshot == 1 : (n0 >= 64 && P->CB >= 3 * slots);
    if (oneshot && g_k1_oneshot < 0) P->RCH = rows;
    if (const char *e = std::getenv("SWDFT2D_K1_RCH")) {  // tuning / test override (rows per tile)
        const long long v = std::atoll(e);
        if (v > 0) P->RCH = v < rows ? v : rows;
    }
    P->nchunks = 0;
    P->ntiles = P->CB * ((rows + P->RCH - 1) / P->RCH);
    // Guided schedule when there are more column blocks than CTA slots (the uniform
    // chunks then leave a partial last wave: config 4 837 -> 851-857 Gcoef/s, config 3
    // 724 -> 853, 64x4 / 64x8 / 64x16 on ~8 GB outputs 730-758 -> 817-830) for windows
    // below 2048 coefficients; the largest (32x64, 64x64: one to two 256-512-thread CTAs
    // per SM) run 6-9 % slower guided and keep the uniform chunks
    // (profiles/shape_check_r01d.jsonl).  64-row windows with >= 3 waves of column
    // blocks take the one-shot grid above instead (config 5: persistent uniform 786,
    // persistent guided 826-828, one-shot 858-865; profiles/k1_oneshot_r01.jsonl).  Small
    // problems keep the uniform chunks (config 2: guided 687 -> 618).
    // (one-shot grids take the guided chunk sizes only when both are forced: the
    // hardware then hands the big-first tiles out in blockIdx order, no counter)
    const bool guided = oneshot ? (g_k1_oneshot == 1 && g_k1_guided == 1)
                                : (g_k1_guided >= 0 ? g_k1_guided == 1
                                                    : (P->CB >= slots && (n0 << k1->m1) < 2048));
    if (guided) {
        // guided self-scheduling: each row chunk is about half of the remaining work
        // spread over the CTAs, so big tiles (little warm-up) go first and small ones
        // fill the tail
        int64_t R = rows, off = 0;
        int nc = 0;
        const int64_t cmin = n0 > 8 ? n0 : 8;
        P->chunk[0] = 0;
        while (R > 0) {
            int64_t c = (R * P->CB + 2 * slots - 1) / (2 * slots);
            if (c > (R + 1) / 2) c = (R + 1) / 2;
            if (c < cmin) c = cmin;
            if (c > R || nc == K1_MAX_CHUNKS - 1) c = R;
            off += c;
            R -= c;
            P->chunk[++nc] = off;
        }
        P->nchunks = nc;
        P->ntiles = P->CB * nc;
    }
    pl->oneshot = oneshot;
    pl->guided = guided;
    pl->grid = (oneshot || P->ntiles < slots) ? P->ntiles : slots;
    // Stream-K (equal contiguous shares of the column-block-major row space, one
    // tile per column block a share touches) where the tile grids above quantize badly
    // (profiles/sched_sweep_r02*.jsonl, configs 2-5 and their 2-D partition blocks):
    //  * uniform chunks, when a one-wave share is >= 1 warm-up (n0 - 1 rows);
    //  * one-shot grids whose last wave is < 90 % full.
    // In k waves of CTAs: identical shares still finish at very different times (config 2,
    // one wave: 57-91 us per CTA, scripts/tune/k1_timeline.py), and short CTAs let the
    // hardware scheduler even that out, until a share is little more than its warm-up:
    // k = share / (2 warm-ups) in fp32 (3 in fp64), clamped to 1..12 — config 2 k = 2 -> 5:
    // 0.0908 -> 0.0876-0.0891 ms; column blocks of configs 3-4 k = 8-12 vs 1-4: +2-10 %.
    // One CTA per SM (64-row windows, 32x64): k = 1 — their SM idles between successive
    // CTAs (config-5 blocks and 32x64 / 64x64 windows: k = 1 best or within 2 % in 6 of 8
    // cases, k = 12 up to 9 % slower).  profiles/sched_sweep_r02_waves*.jsonl.
    // Guided schedules stay: long-lived stream-K CTAs spread their stores over the whole
    // output, and on large outputs that measured 3-20 % slower than guided chunks.
    int sk = g_k1_streamk;
    if (sk < 0 && g_k1_oneshot < 0 && g_k1_guided < 0 && !std::getenv("SWDFT2D_K1_RCH")) {
        const int64_t warm = n0 - 1 > 0 ? n0 - 1 : 1;
        const double share = (double)P->CB * (double)rows / (double)slots;
        bool use = false;
        if (oneshot) {
            const double waves = (double)P->CB / (double)slots;
            use = waves / std::ceil(waves) < 0.9;
        } else {
            use = !guided && share >= (double)warm;
        }
        sk = 0;
        if (use) {
            const double per = (k1->prec ? 3.0 : 2.0) * (double)warm;
            const int k = (int)(share / per);
            sk = pl->occ == 1 ? 1 : k < 1 ? 1 : k > 12 ? 12 : k;
        }
        // Short launches (at most 2 n0 window rows: push_rows blocks, the first scatter
        // piece, host-output strips of large windows): every tile is mostly warm-up, and
        // guided chunks (>= n0 rows each, every one with its own warm-up) or one CTA per
        // column block waste the most on it.  One wave of equal contiguous shares is the
        // fastest or level in every measured case once a share holds >= half a warm-up:
        // config 3 16/32/64 rows 29.7/42.0/60.4 -> 23.6/31.6/52.1 us, config 4 16/32 rows
        // 35.9/58.4 -> 33.6/52.1, config 5 16..128 rows -2.5..-4 %, config 2 32 rows
        // 17.4 -> 15.4; fp64 config 4 16/32 rows -3/-11 %, but config 3 below n0 rows
        // +4 % (so fp64 needs rows >= n0) (profiles/short_launch_r02.jsonl).
        if (rows <= 2 * (int64_t)n0 && share >= 0.5 * (double)warm &&
            (k1->prec == 0 || rows >= n0))
            sk = 1;
    }
    if (sk > 0) {
        const int64_t L = P->CB * rows;
        pl->streamk = true;
        pl->oneshot = pl->guided = false;
        P->streamk = 1;
        P->nchunks = 0;
        pl->grid = (int64_t)sk * slots < L ? (int64_t)sk * slots : L;
        P->ntiles = pl->grid;
    }
    return SWDFT2D_OK;
}

// The guided K1 tile counter of (current device, stream): one 8-byte slot per stream
// handle, from blocks allocated and zeroed once (the kernel leaves it zeroed after every
// launch), so a forward call allocates nothing.  Launches on one stream are ordered, so
// they can share the slot; distinct streams never do (up to K1_CTR_MAX streams per device,
// after which slots are recycled).
static constexpr int K1_CTR_BLOCK = 256, K1_CTR_MAX = 16 * K1_CTR_BLOCK;

static int k1_counter(DeviceState *ds, cudaStream_t s, unsigned long long **out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = ds->ctr.find(s);
    if (it != ds->ctr.end()) {
        *out = it->second;
        return SWDFT2D_OK;
    }
    const size_t used = ds->ctr.size();
    if (used >= (size_t)K1_CTR_MAX) {  // recycle: every slot is zero between launches
        unsigned long long *p = ds->ctr.begin()->second;
        ds->ctr.erase(ds->ctr.begin());
        ds->ctr[s] = p;
        *out = p;
        return SWDFT2D_OK;
    }
    if (used == ds->ctr_blocks.size() * K1_CTR_BLOCK) {
        CaptureModeGuard relaxed;
        void *blk = nullptr;
        cudaStream_t up = nullptr;
        cudaError_t e = cudaMalloc(&blk, K1_CTR_BLOCK * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMemsetAsync(blk, 0, K1_CTR_BLOCK * sizeof(unsigned long long), up);
        if (e == cudaSuccess) e = cudaStreamSynchronize(up);
        if (up) cudaStreamDestroy(up);
        if (e != cudaSuccess) {
            if (blk) cudaFree(blk);
            return fail(SWDFT2D_E_NOMEM, "K1 tile counters: %s", cudaGetErrorString(e));
        }
        ds->ctr_blocks.push_back(static_cast<unsigned long long *>(blk));
    }
    unsigned long long *p = ds->ctr_blocks[used / K1_CTR_BLOCK] + used % K1_CTR_BLOCK;
    ds->ctr[s] = p;
    *out = p;
    return SWDFT2D_OK;
}

// Plan and launch K1 over window rows [p0_begin, p0_end) with P's input/output fields set.
static int run_k1(DeviceState *ds, const K1Info *k1, K1Params &P, const CUtensorMap &tmap,
                  int64_t p0_begin, int64_t p0_end, const void *tw64, cudaStream_t st) {
    K1Plan pl;
    int rc = k1_plan(ds, k1, P.P1, p0_begin, p0_end, &P, &pl);
    if (rc) return rc;
    P.tw = static_cast<const double2 *>(tw64);
    P.counter = nullptr;  // one-shot grids take one tile per CTA: no counter
    if (pl.guided && !pl.oneshot && (rc = k1_counter(ds, st, &P.counter))) return rc;
    k1->launch(P, tmap, (int)pl.grid, st);
    return SWDFT2D_OK;
}

}  // namespace swdft2d

using namespace swdft2d;

extern "C" {

int swdft2d_abi_version(void) { return SWDFT2D_ABI_VERSION; }

const char *swdft2d_last_error(void) { return g_last_error.c_str(); }

int swdft2d_output_shape(int64_t N0, int64_t N1, int m0, int m1, int64_t *P0, int64_t *P1) {
    if (m0 < 0 || m1 < 0) return fail(SWDFT2D_E_INVALID_WINDOW, "window exponents must be non-negative");
    if (m0 > 62 || m1 > 62) return fail(SWDFT2D_E_INVALID_WINDOW, "window exponent too large");
    const int64_t n0 = (int64_t)1 << m0, n1 = (int64_t)1 << m1;
    if (n0 > N0)
        return fail(SWDFT2D_E_WINDOW_TOO_LARGE, "window size %lld exceeds extent %lld in dimension 0",
                    (long long)n0, (long long)N0);
    if (n1 > N1)
        return fail(SWDFT2D_E_WINDOW_TOO_LARGE, "window size %lld exceeds extent %lld in dimension 1",
                    (long long)n1, (long long)N1);
    if (P0) *P0 = N0 - n0 + 1;
    if (P1) *P1 = N1 - n1 + 1;
    return SWDFT2D_OK;
}

int swdft2d_reference_bytes(int64_t N0, int64_t N1, int m0, int m1, int64_t *lattice_bytes,
                            int64_t *output_bytes) {
    int64_t P0 = 0, P1 = 0;
    int rc = swdft2d_output_shape(N0, N1, m0, m1, &P0, &P1);
    if (rc) return rc;
    // 16 B per complex (core.COMPLEX_BYTES, core.py:17); saturate instead of overflowing.
    const long double win = std::ldexp(1.0L, m0 + m1);
    const long double lat = 2.0L * (long double)N0 * (long double)N1 * win * 16.0L;
    const long double outb = (long double)P0 * (long double)P1 * win * 16.0L;
    const long double lim = 9.2e18L;
    if (lattice_bytes) *lattice_bytes = lat > lim ? INT64_MAX : (int64_t)lat;
    if (output_bytes) *output_bytes = outb > lim ? INT64_MAX : (int64_t)outb;
    return SWDFT2D_OK;
}

int swdft2d_twiddles(int n, double *out) {
    if (n < 1 || (n & (n - 1)) != 0)
        return fail(SWDFT2D_E_INVALID_WINDOW, "twiddle table size %d is not a power of two", n);
    if (!out) return fail(SWDFT2D_E_INVALID_ARG, "null output");
    const double step = (2.0 * 3.141592653589793) / (double)n;
    for (int j = 0; j < n; ++j) {
        const double ang = (double)j * step;
        out[2 * j] = std::cos(ang);
        out[2 * j + 1] = -std::sin(ang);
    }
    return SWDFT2D_OK;
}

int swdft2d_has_stream_kernel(int m0, int m1, int prec) { return find_k1(m0, m1, prec) ? 1 : 0; }

int swdft2d_stream_kernel_info(int m0, int m1, int prec, int64_t info[6]) {
    const K1Info *k = find_k1(m0, m1, prec);
    if (!k) return fail(SWDFT2D_E_UNSUPPORTED, "no K1 instantiation for m0=%d m1=%d prec=%d", m0, m1, prec);
    if (!info) return fail(SWDFT2D_E_INVALID_ARG, "null info");
    info[0] = k->q;
    info[1] = k->tp1;
    info[2] = k->threads;
    info[3] = (int64_t)k->smem_bytes;
    info[4] = k->nb;
    info[5] = (g_use_tma && find_k1(m0, m1, prec, 1)) ? 1 : 0;
    return SWDFT2D_OK;
}

int swdft2d_strip_range(int64_t P0, int m0, int rank, int world, int64_t range[4]) {
    if (world < 1 || rank < 0 || rank >= world || P0 < 0 || m0 < 0 || m0 > 62 || !range)
        return fail(SWDFT2D_E_INVALID_ARG, "bad strip request (P0=%lld rank=%d world=%d)",
                    (long long)P0, rank, world);
    const int64_t n0 = (int64_t)1 << m0;
    // floor(P0*g/G) without overflow for P0 < 2^62 / world
    const int64_t a = (int64_t)(((__int128)P0 * rank) / world);
    const int64_t b = (int64_t)(((__int128)P0 * (rank + 1)) / world);
    range[0] = a;
    range[1] = b;
    range[2] = a;
    range[3] = b > a ? b + n0 - 1 : a;
    return SWDFT2D_OK;
}

// Shared validation of swdft2d_forward* / swdft2d_workspace_bytes.
static int check_forward_args(int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0, int m1,
                              int prec, int64_t p0_begin, int64_t p0_end, int64_t *P1) {
    if (in_dtype < SWDFT2D_IN_F32 || in_dtype > SWDFT2D_IN_C128)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown input dtype code %d", in_dtype);
    if (prec != SWDFT2D_PREC_FP32 && prec != SWDFT2D_PREC_FP64)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown precision code %d", prec);
    if (N0 < 1 || N1 < 1) return fail(SWDFT2D_E_SHAPE, "empty input (%lld x %lld)", (long long)N0, (long long)N1);
    if (ld_x < N1) return fail(SWDFT2D_E_INVALID_ARG, "ld_x %lld < N1 %lld", (long long)ld_x, (long long)N1);
    int64_t P0 = 0;
    int rc = swdft2d_output_shape(N0, N1, m0, m1, &P0, P1);
    if (rc) return rc;
    if (p0_begin < 0 || p0_end > P0 || p0_begin > p0_end)
        return fail(SWDFT2D_E_INVALID_ARG, "window rows [%lld, %lld) outside [0, %lld)",
                    (long long)p0_begin, (long long)p0_end, (long long)P0);
    return SWDFT2D_OK;
}

int swdft2d_workspace_bytes(int64_t N0, int64_t N1, int m0, int m1, int prec, int64_t p0_begin,
                            int64_t p0_end, int kernel, int64_t *bytes) {
    if (!bytes) return fail(SWDFT2D_E_INVALID_ARG, "null output");
    int64_t P1 = 0;
    int rc = check_forward_args(SWDFT2D_IN_F32, N0, N1, N1, m0, m1, prec, p0_begin, p0_end, &P1);
    if (rc) return rc;
    Path path;
    if ((rc = select_path(m0, m1, prec, kernel, &path))) return rc;
    *bytes = 0;
    if (path != PATH_SEP || p0_end == p0_begin) return SWDFT2D_OK;
    const int64_t n0 = (int64_t)1 << m0;
    const int64_t zrow = P1 * ((int64_t)1 << m1) * (prec == SWDFT2D_PREC_FP64 ? 16 : 8);
    const int64_t R = sep_strip_rows(zrow, n0, p0_end - p0_begin, 0);
    *bytes = (R + n0 - 1) * zrow;
    return SWDFT2D_OK;
}

int swdft2d_k1_schedule(int64_t N0, int64_t N1, int m0, int m1, int prec, int64_t p0_begin,
                        int64_t p0_end, int64_t info[8], int64_t *bounds, int max_bounds) {
    if (!info) return fail(SWDFT2D_E_INVALID_ARG, "null info");
    int64_t P1 = 0;
    int rc = check_forward_args(SWDFT2D_IN_F32, N0, N1, N1, m0, m1, prec, p0_begin, p0_end, &P1);
    if (rc) return rc;
    const K1Info *k1 = find_k1(m0, m1, prec, 0);
    if (!k1) return fail(SWDFT2D_E_UNSUPPORTED, "no K1 instantiation for m0=%d m1=%d prec=%d", m0, m1, prec);
    if (p0_end == p0_begin) return fail(SWDFT2D_E_INVALID_ARG, "empty row range");
    CaptureModeGuard relaxed;
    DeviceState *ds = nullptr;
    if ((rc = device_state(&ds))) return rc;
    K1Params P;
    std::memset(&P, 0, sizeof P);
    K1Plan pl;
    if ((rc = k1_plan(ds, k1, P1, p0_begin, p0_end, &P, &pl))) return rc;
    const int64_t rows = p0_end - p0_begin;
    const int64_t nchunks = pl.streamk ? 0 : P.nchunks > 0 ? P.nchunks : (rows + P.RCH - 1) / P.RCH;
    info[0] = pl.streamk ? 3 : pl.oneshot ? 2 : pl.guided ? 1 : 0;
    info[1] = P.RCH;
    info[2] = nchunks;
    info[3] = P.ntiles;
    info[4] = pl.grid;
    info[5] = P.CB;
    info[6] = pl.slots;
    info[7] = pl.occ;
    for (int64_t c = 0; bounds && c <= nchunks && c < max_bounds; ++c) {
        const int64_t v = P.nchunks > 0 ? P.chunk[c] : c * P.RCH;
        bounds[c] = v < rows ? v : rows;
    }
    return SWDFT2D_OK;
}

int swdft2d_forward(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                    int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                    int kernel, void *stream) {
    return swdft2d_forward_ws(x, in_dtype, N0, N1, ld_x, m0, m1, prec, scale, p0_begin, p0_end,
                              out, nullptr, 0, kernel, stream);
}

int swdft2d_forward_ws(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                       int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                       void *workspace, int64_t workspace_bytes, int kernel, void *stream) {
    int64_t P1 = 0;
    int rc = check_forward_args(in_dtype, N0, N1, ld_x, m0, m1, prec, p0_begin, p0_end, &P1);
    if (rc) return rc;
    Path path;
    if ((rc = select_path(m0, m1, prec, kernel, &path))) return rc;
    if (p0_begin == p0_end) return SWDFT2D_OK;
    if (!x || !out) return fail(SWDFT2D_E_INVALID_ARG, "null device pointer");
    if (workspace_bytes < 0 || (workspace_bytes > 0 && !workspace))
        return fail(SWDFT2D_E_INVALID_ARG, "bad workspace (%p, %lld B)", workspace,
                    (long long)workspace_bytes);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // While the caller's stream is captured into a CUDA graph, the one-time setup of a
    // first call (device state, twiddle tables, tile counters, kernel attributes and
    // occupancy, lazy module loading) runs with the thread's capture mode relaxed: in the
    // default global mode those calls invalidated the capture.  The launches are captured.
    CaptureModeGuard relaxed;
    DeviceState *ds = nullptr;
    if ((rc = device_state(&ds))) return rc;
    const void *tw64 = nullptr, *tw32 = nullptr;
    if ((rc = k0_tables(ds, &tw64, &tw32))) return rc;
    const void *tw = prec == SWDFT2D_PREC_FP64 ? tw64 : tw32;
    const bool apply = !(scale == 1.0);

    if (path == PATH_KR) {
        KRParams P;
        std::memset(&P, 0, sizeof P);
        P.x = x;
        P.in_dtype = in_dtype;
        P.apply_scale = apply ? 1 : 0;
        P.N1 = N1;
        P.ldx = ld_x;
        P.p0_begin = p0_begin;
        P.p0_end = p0_end;
        P.P1 = P1;
        P.out = out;
        P.scale = scale;
        P.tw = tw;
        P.sms = ds->sms;
        const int r = launch_kr(P, m1, prec, st);
        if (r != 0) return fail(SWDFT2D_E_CUDA, "row-tree kernel launch setup failed (%d)", r);
    } else if (path == PATH_SEP) {
        if ((rc = forward_separable(x, in_dtype, N1, ld_x, m0, m1, prec, scale, p0_begin, p0_end,
                                    out, workspace, workspace_bytes, st, ds, tw, tw64)))
            return rc;
    } else if (path == PATH_K1) {
        const K1Info *k1 = find_k1(m0, m1, prec, 0);
        K1Params P;
        std::memset(&P, 0, sizeof P);
        CUtensorMap tmap;
        std::memset(&tmap, 0, sizeof tmap);
        // the TMA variant stages input tiles with cp.async.bulk.tensor when x is addressable;
        // the LDG variant needs no tensor map (no driver call on the default path)
        const bool want_tma =
            kernel == SWDFT2D_KERNEL_STREAM_TMA || (kernel == SWDFT2D_KERNEL_AUTO && g_use_tma);
        const K1Info *kt = want_tma ? find_k1(m0, m1, prec, 1) : nullptr;
        if (kt && encode_input_map(kt, x, in_dtype, N0, N1, ld_x, &tmap, &P)) k1 = kt;
        else if (in_dtype == SWDFT2D_IN_F32 && prec == SWDFT2D_PREC_FP32)
            if (const K1Info *kf = find_k1(m0, m1, prec, 3)) k1 = kf;
        P.x = x;
        P.in_dtype = in_dtype;
        P.apply_scale = apply ? 1 : 0;
        P.N0 = N0;
        P.N1 = N1;
        P.ldx = ld_x;
        P.P1 = P1;
        P.out = out;
        P.scale = scale;
        if ((rc = run_k1(ds, k1, P, tmap, p0_begin, p0_end, tw64, st))) return rc;
    } else {
        K0Params P;
        std::memset(&P, 0, sizeof P);
        P.x = x;
        P.in_dtype = in_dtype;
        P.m0 = m0;
        P.m1 = m1;
        P.apply_scale = apply ? 1 : 0;
        P.ldx = ld_x;
        P.p0_begin = p0_begin;
        P.p0_end = p0_end;
        P.P1 = P1;
        P.out = out;
        P.scale = scale;
        P.tw = tw;
        P.tw_n = K0_TW_N;
        if (launch_k0(P, prec, st))
            return fail(SWDFT2D_E_UNSUPPORTED, "K0 grid too large for %lld x %lld outputs",
                        (long long)(p0_end - p0_begin), (long long)P1);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return SWDFT2D_OK;
}

static const int64_t k_in_bytes[4] = {4, 8, 8, 16};  // SWDFT2D_IN_* element sizes

// Peer access from `dev` to `src` (once per pair; a no-op where the pair has no P2P —
// cudaMemcpyDefault then stages through the host).
static void enable_peer(int dev, int src) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(dev, src);
    if (dev == src || done.count(key)) return;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, dev, src);
    if (can) {
        cudaSetDevice(dev);
        if (cudaDeviceEnablePeerAccess(src, 0) == cudaErrorPeerAccessAlreadyEnabled)
            cudaGetLastError();
    }
    done[key] = true;
}

int swdft2d_forward_multi(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x,
                          int m0, int m1, int prec, double scale, int ndev, const int *devs,
                          void *const *stage, void *const *outs, void *const *streams) {
    if (ndev < 1 || !devs || !outs || !streams)
        return fail(SWDFT2D_E_INVALID_ARG, "forward_multi: need ndev >= 1 devices, outs and streams");
    if (in_dtype < SWDFT2D_IN_F32 || in_dtype > SWDFT2D_IN_C128)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown input dtype code %d", in_dtype);
    if (N0 < 1 || N1 < 1) return fail(SWDFT2D_E_SHAPE, "empty input (%lld x %lld)", (long long)N0, (long long)N1);
    if (ld_x < N1) return fail(SWDFT2D_E_INVALID_ARG, "ld_x %lld < N1 %lld", (long long)ld_x, (long long)N1);
    int64_t P0 = 0, P1 = 0;
    int rc = swdft2d_output_shape(N0, N1, m0, m1, &P0, &P1);
    if (rc) return rc;
    if (!x) return fail(SWDFT2D_E_INVALID_ARG, "null device pointer");
    int cur = 0;
    cudaGetDevice(&cur);
    const int64_t es = k_in_bytes[in_dtype];
    // x is ready on devs[0]'s stream: every other device's stream waits for it, copies its
    // strip (with halo) into its own stage buffer, and computes there
    cudaEvent_t ready = nullptr;
    cudaSetDevice(devs[0]);
    cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ready, reinterpret_cast<cudaStream_t>(streams[0]));
    if (e != cudaSuccess) {
        if (ready) cudaEventDestroy(ready);
        cudaSetDevice(cur);
        return fail(SWDFT2D_E_CUDA, "forward_multi: event on device %d: %s", devs[0], cudaGetErrorString(e));
    }
    std::vector<cudaEvent_t> copied;
    for (int g = 0; g < ndev && rc == SWDFT2D_OK; ++g) {
        int64_t r[4];
        if ((rc = swdft2d_strip_range(P0, m0, g, ndev, r))) break;
        if (r[1] == r[0]) continue;
        cudaStream_t st = reinterpret_cast<cudaStream_t>(streams[g]);
        if (g == 0) {
            cudaSetDevice(devs[0]);
            rc = swdft2d_forward(x, in_dtype, N0, N1, ld_x, m0, m1, prec, scale, r[0], r[1],
                                 outs[0], SWDFT2D_KERNEL_AUTO, streams[0]);
            continue;
        }
        if (!stage || !stage[g] || !outs[g]) {
            rc = fail(SWDFT2D_E_INVALID_ARG, "forward_multi: device slot %d needs a stage and an out buffer", g);
            break;
        }
        enable_peer(devs[g], devs[0]);
        cudaSetDevice(devs[g]);
        const int64_t rows = r[3] - r[2];
        e = cudaStreamWaitEvent(st, ready, 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(stage[g], (size_t)(N1 * es),
                                  static_cast<const char *>(x) + r[2] * ld_x * es, (size_t)(ld_x * es),
                                  (size_t)(N1 * es), (size_t)rows, cudaMemcpyDefault, st);
        cudaEvent_t ev = nullptr;
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ev, st);
        if (ev) copied.push_back(ev);
        if (e != cudaSuccess) {
            rc = fail(SWDFT2D_E_CUDA, "forward_multi: strip copy to device %d: %s", devs[g],
                      cudaGetErrorString(e));
            break;
        }
        rc = swdft2d_forward(stage[g], in_dtype, rows, N1, N1, m0, m1, prec, scale, 0, r[1] - r[0],
                             outs[g], SWDFT2D_KERNEL_AUTO, streams[g]);
    }
    // later work on devs[0]'s stream (e.g. overwriting x) is ordered after every strip copy
    cudaSetDevice(devs[0]);
    for (cudaEvent_t ev : copied) {
        cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(streams[0]), ev, 0);
        cudaEventDestroy(ev);
    }
    cudaEventDestroy(ready);
    cudaSetDevice(cur);
    return rc;
}

int swdft2d_stream_state_bytes(int64_t N1, int m0, int m1, int prec, int64_t *bytes) {
    if (prec != SWDFT2D_PREC_FP32 && prec != SWDFT2D_PREC_FP64)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown precision code %d", prec);
    if (!bytes) return fail(SWDFT2D_E_INVALID_ARG, "null output");
    if (m0 < 0 || m1 < 0 || m0 > SWDFT2D_K1_MAX_M || m1 > SWDFT2D_K1_MAX_M)
        return fail(SWDFT2D_E_UNSUPPORTED, "no incremental stream kernel for m0=%d m1=%d", m0, m1);
    int64_t P1 = 0;
    int rc = swdft2d_output_shape((int64_t)1 << m0, N1, m0, m1, nullptr, &P1);
    if (rc) return rc;
    const int64_t eb = prec == SWDFT2D_PREC_FP64 ? 16 : 8;
    const int64_t n0 = (int64_t)1 << m0;
    const int64_t nodes = m0 ? (int64_t)m0 * (n0 / 2) + n0 - 1 : 0;  // per column, k2_push.cu
    *bytes = nodes * P1 * ((int64_t)1 << m1) * eb;
    return SWDFT2D_OK;
}

int swdft2d_stream_push(const void *row, int in_dtype, int64_t N1, void *ring, void *state, int m0,
                        int m1, int prec, double scale, int64_t p0, void *out, int kernel,
                        void *stream) {
    if (in_dtype < SWDFT2D_IN_F32 || in_dtype > SWDFT2D_IN_C128)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown input dtype code %d", in_dtype);
    if (prec != SWDFT2D_PREC_FP32 && prec != SWDFT2D_PREC_FP64)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown precision code %d", prec);
    if (kernel < SWDFT2D_KERNEL_AUTO || kernel > SWDFT2D_KERNEL_SEPARABLE)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown kernel code %d", kernel);
    if (p0 < 0) return fail(SWDFT2D_E_INVALID_ARG, "negative row index %lld", (long long)p0);
    if (m0 < 0 || m1 < 0 || m0 > 30) return fail(SWDFT2D_E_INVALID_WINDOW, "bad window exponents");
    const int64_t n0 = (int64_t)1 << m0;
    int64_t P1 = 0;
    int rc = swdft2d_output_shape(n0, N1, m0, m1, nullptr, &P1);
    if (rc) return rc;
    if (!row || (!ring && !state)) return fail(SWDFT2D_E_INVALID_ARG, "null device pointer");
    CaptureModeGuard relaxed;  // first-call setup must not invalidate a graph capture
    DeviceState *ds = nullptr;
    if ((rc = device_state(&ds))) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (state) {  // K2: incremental push over the level state (and the raw ring, if given)
        if (m0 > SWDFT2D_K1_MAX_M || m1 > SWDFT2D_K1_MAX_M)
            return fail(SWDFT2D_E_UNSUPPORTED, "no incremental stream kernel for m0=%d m1=%d", m0, m1);
        K2Params P;
        std::memset(&P, 0, sizeof P);
        P.row = row;
        P.in_dtype = in_dtype;
        P.apply_scale = scale == 1.0 ? 0 : 1;
        P.N1 = N1;
        P.P1 = P1;
        P.r = p0;
        P.state = state;
        P.ring = ring;
        P.out = p0 >= n0 - 1 ? out : nullptr;
        P.scale = scale;
        const void *tw64 = nullptr, *tw32 = nullptr;
        if ((rc = k0_tables(ds, &tw64, &tw32))) return rc;
        P.tw = static_cast<const double2 *>(tw64);
        launch_k2(P, m0, m1, prec, st);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "K2 push: %s", cudaGetErrorString(e));
        return SWDFT2D_OK;
    }
    launch_ring_store(row, in_dtype, N1, ring, prec, (int)n0, p0, ds->sms, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "ring store: %s", cudaGetErrorString(e));
    if (p0 < n0 - 1) return SWDFT2D_OK;  // warming up: no window row complete yet
    if (!out) return fail(SWDFT2D_E_INVALID_ARG, "null output slab");
    const int64_t first = (p0 + 1) % n0;
    const int64_t eb = prec == SWDFT2D_PREC_FP64 ? 16 : 8;
    const void *win = static_cast<const char *>(ring) + first * N1 * eb;
    return swdft2d_forward(win, prec == SWDFT2D_PREC_FP64 ? SWDFT2D_IN_C128 : SWDFT2D_IN_C64, n0,
                           N1, N1, m0, m1, prec, scale, 0, 1, out, kernel, stream);
}

int swdft2d_forward_columns(const void *z, int prec, int64_t N0, int64_t cols, int64_t ld_z, int m0,
                            int m_inner, double scale, int64_t p0_begin, int64_t p0_end, void *out,
                            void *stream) {
    if (prec != SWDFT2D_PREC_FP32 && prec != SWDFT2D_PREC_FP64)
        return fail(SWDFT2D_E_INVALID_ARG, "unknown precision code %d", prec);
    if (m0 < 1 || m0 > SWDFT2D_K0_MAX_M)
        return fail(SWDFT2D_E_UNSUPPORTED, "column trees need 1 <= m0 <= %d (got %d)",
                    SWDFT2D_K0_MAX_M, m0);
    if (m_inner < 0 || m_inner > 40 || cols < 1 || (cols & (((int64_t)1 << m_inner) - 1)) != 0)
        return fail(SWDFT2D_E_INVALID_ARG, "cols %lld is not a multiple of 2^%d", (long long)cols,
                    m_inner);
    if (ld_z < cols) return fail(SWDFT2D_E_INVALID_ARG, "ld_z %lld < cols %lld", (long long)ld_z, (long long)cols);
    const int64_t n0 = (int64_t)1 << m0;
    if (n0 > N0)
        return fail(SWDFT2D_E_WINDOW_TOO_LARGE, "window size %lld exceeds extent %lld in dimension 0",
                    (long long)n0, (long long)N0);
    const int64_t P0 = N0 - n0 + 1;
    if (p0_begin < 0 || p0_end > P0 || p0_begin > p0_end)
        return fail(SWDFT2D_E_INVALID_ARG, "window rows [%lld, %lld) outside [0, %lld)",
                    (long long)p0_begin, (long long)p0_end, (long long)P0);
    if (p0_begin == p0_end) return SWDFT2D_OK;
    if (!z || !out) return fail(SWDFT2D_E_INVALID_ARG, "null device pointer");
    CaptureModeGuard relaxed;
    DeviceState *ds = nullptr;
    int rc = device_state(&ds);
    if (rc) return rc;
    const void *tw64 = nullptr, *tw32 = nullptr;
    if ((rc = k0_tables(ds, &tw64, &tw32))) return rc;
    const int64_t esz = prec == SWDFT2D_PREC_FP64 ? 16 : 8;
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // the same choice as forward_separable's column trees (use_k1_columns)
    const bool want_kz = m_inner < 31 && use_k1_columns(m0, m_inner, prec, p0_end - p0_begin);
    if (const K1Info *kz = want_kz ? find_k1(m0, 0, prec, 2) : nullptr) {
        K1Params Pz;
        std::memset(&Pz, 0, sizeof Pz);
        CUtensorMap tmap;
        std::memset(&tmap, 0, sizeof tmap);
        Pz.x = static_cast<const char *>(z) + p0_begin * ld_z * esz;
        Pz.in_dtype = prec == SWDFT2D_PREC_FP64 ? SWDFT2D_IN_C128 : SWDFT2D_IN_C64;
        Pz.N0 = p0_end - p0_begin + n0 - 1;
        Pz.N1 = cols;
        Pz.ldx = ld_z;
        Pz.P1 = cols;
        Pz.out = out;
        Pz.scale = scale;
        Pz.apply_scale = scale == 1.0 ? 0 : 1;
        Pz.col_m1 = m_inner;
        if ((rc = run_k1(ds, kz, Pz, tmap, 0, p0_end - p0_begin, tw64, st))) return rc;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "column-tree launch: %s", cudaGetErrorString(e));
        return SWDFT2D_OK;
    }
    KCParams c;
    std::memset(&c, 0, sizeof c);
    c.z = static_cast<const char *>(z) + p0_begin * ld_z * esz;
    c.cols = cols;
    c.ldz = ld_z;
    c.zrows = p0_end - p0_begin + n0 - 1;
    c.P0s = p0_end - p0_begin;
    c.P1 = cols >> m_inner;
    c.m1 = m_inner;
    c.apply_scale = scale == 1.0 ? 0 : 1;
    c.scale = scale;
    c.out = out;
    c.tw = prec == SWDFT2D_PREC_FP64 ? tw64 : tw32;
    c.sms = ds->sms;
    if (launch_kc(c, m0, prec, st))
        return fail(SWDFT2D_E_CUDA, "column-tree launch setup failed (m0=%d)", m0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SWDFT2D_E_CUDA, "column-tree launch: %s", cudaGetErrorString(e));
    return SWDFT2D_OK;
}

int swdft2d_shutdown(void) {
    // the host path first, outside g_mu: a host-to-host call holds its own lock and then
    // takes g_mu inside the forward calls it makes (same order here)
    release_host_pipe();
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_dev) {
        if (kv.second.k0_tw64 || kv.second.k0_tw32) {
            cudaSetDevice(kv.first);
            cudaFree(kv.second.k0_tw64);
            cudaFree(kv.second.k0_tw32);
        }
        if (!kv.second.ctr_blocks.empty()) {
            cudaSetDevice(kv.first);
            for (unsigned long long *b : kv.second.ctr_blocks) cudaFree(b);
        }
    }
    g_dev.clear();
    cudaSetDevice(cur);
    return SWDFT2D_OK;
}

}  // extern "C"
