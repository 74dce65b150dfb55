// swdft2d_internal.h — host/device shared parameter blocks and launcher
// prototypes (internal to libswdft2d.so; the public surface is include/swdft2d.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace swdft2d {

constexpr int K2_TW_N = 64;   // make_twiddles(64): K2 (stream push) windows up to 64
constexpr int K1_MAX_CHUNKS = 48;  // guided K1 schedule: row chunks per launch
// device twiddle table make_twiddles(1024) (fp64 and fp32 copies), allocated once per
// device; every kernel reads it at stride 1024/n (bitwise make_twiddles(n), App. A #4)
constexpr int K0_TW_N = 1024;

struct K0Params {
    const void *x;
    int in_dtype, m0, m1, apply_scale;
    int64_t ldx, p0_begin, p0_end, P1;
    void *out;
    double scale;
    const void *tw;  // device table of K0_TW_N complex (float2 or double2)
    int tw_n;
};

struct K1Params {
    const void *x;
    int in_dtype, apply_scale;
    int64_t N0, N1, ldx;
    int64_t p0_begin, p0_end, P1;
    void *out;
    double scale;
    int64_t CB;      // column blocks of TP1 window positions
    int64_t RCH;     // window rows per tile (uniform chunks, nchunks == 0)
    int64_t ntiles;  // CB * number of row chunks
    // guided schedule (nchunks > 0): row chunk c covers window rows
    // [p0_begin + chunk[c], p0_begin + chunk[c + 1]); tiles past the first wave are
    // handed out by atomicAdd on *counter (zero at launch; the launch's last fetch zeroes
    // it again, so one per-(device, stream) counter serves every launch on that stream)
    int nchunks;
    unsigned long long *counter;
    int64_t chunk[K1_MAX_CHUNKS + 1];
    // stream-K schedule (streamk != 0): the CB x rows (column block, window row) space,
    // column-block major, is cut into gridDim.x equal contiguous ranges; CTA b walks
    // range b as one tile per column block it touches (each with its own warm-up)
    int streamk;
    // 1-column windows (M1 = 0 instantiations) over the large-window path's stage-R rows:
    // column c of x is (p1, k1) = (c >> col_m1, c mod 2^col_m1) of an n1 = 2^col_m1
    // window, written to out[p0][p1][k0][k1] (0: plain n0 x 1 windows)
    int col_m1;
    int sample_bytes;    // bytes per input sample (4, 8, 16)
    int tma_per_sample;  // TMA elements per sample (1, or 2 for complex128)
    int tma_row_bytes;   // bytes of one staged input row (TMA box width, 16-B multiple)
    // device make_twiddles(K0_TW_N) in fp64 (the K0 table), read at stride 1024/NMAX:
    // bitwise make_twiddles(NMAX); a pointer keeps the launch
    // parameters small (the by-value 256-entry table was 4 KB per launch)
    const double2 *tw;
};

// Static shape of one K1 instantiation (filled by the instantiation units).
struct K1Info {
    int m0, m1, prec, q, tp1, threads, nb, tma;
    size_t smem_bytes;
    const void *func;  // kernel symbol for occupancy queries / attribute setting
    int (*launch)(const K1Params &, const CUtensorMap &, int grid, cudaStream_t);
};

// Registry of compiled K1 instantiations; nullptr if (m0, m1, prec, tma) is absent.
const K1Info *find_k1(int m0, int m1, int prec, int tma = 0);
void register_k1(const K1Info *info);

int launch_k0(const K0Params &P, int prec, cudaStream_t stream);

// KR: row-tree kernel for n0 = 1 windows (kr_rows.cu), n1 up to 1024.
struct KRParams {
    const void *x;
    int in_dtype, apply_scale;
    int64_t N1, ldx;
    int64_t p0_begin, p0_end, P1;
    void *out;
    double scale;
    const void *tw;  // device make_twiddles(K0_TW_N) of the precision (float2 / double2)
    int sms;         // SMs of the device (persistent grid = SMs x occupancy)
};
// 0 ok, -2 shared-memory attribute / occupancy refused, -3 m1 out of range
int launch_kr(const KRParams &P, int m1, int prec, cudaStream_t stream);

// KC: column-tree kernel of the large-window path (kc_cols.cu), n0 = 2 .. 1024.
struct KCParams {
    const void *z;     // stage-R rows of the strip: [zrows][cols] complex of the precision
    int64_t cols;      // P1 * n1 (columns transformed)
    int64_t ldz;       // row stride of z, elements (>= cols)
    int64_t zrows;     // P0s + n0 - 1
    int64_t P0s;       // window rows of the strip
    int64_t P1;        // cols >> m1
    int m1;            // output layout [P0s][P1][n0][2^m1]: column c = (c >> m1, c & (2^m1 - 1))
    int apply_scale;
    void *out;         // the strip's first output row: [P0s][P1][n0][n1]
    double scale;
    const void *tw;    // device make_twiddles(K0_TW_N) of the precision
    int sms;
};
int launch_kc(const KCParams &P, int m0, int prec, cudaStream_t stream);

// K2: one incremental stream push (k2_push.cu).
struct K2Params {
    const void *row;  // the pushed row, N1 elements of in_dtype
    int in_dtype, apply_scale;
    int64_t N1, P1;
    int64_t r;    // index of the pushed row
    void *state;  // (m0 * n0/2 + n0 - 1) * P1 * n1 complex (level rings), zero-initialised
    void *ring;   // optional raw ring [2 n0, N1] (nullptr: not stored)
    void *out;    // optional (P1, n0, n1) slab of window row r - n0 + 1
    double scale;
    const double2 *tw;  // device make_twiddles(K0_TW_N), fp64; K2 reads every 16th entry
                        // = make_twiddles(64), bitwise (small launch parameters)
};
int launch_k2(const K2Params &P, int m0, int m1, int prec, cudaStream_t stream);

// Stream ring: store row p0 (N1 elements of in_dtype) at slots p0 mod n0 and
// p0 mod n0 + n0 of ring ([2 n0, N1] complex of prec).
int launch_ring_store(const void *row, int in_dtype, int64_t N1, void *ring, int prec, int n0,
                      int64_t p0, int sms, cudaStream_t stream);

// Sets the calling thread's swdft2d_last_error message; returns code (abi.cu).
int set_error(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
// Frees swdft2d_forward_host's cached device scratch and pinned staging (host_pipe.cu).
void release_host_pipe();

}  // namespace swdft2d
