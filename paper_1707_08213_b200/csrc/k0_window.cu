// k0_window.cu — K0, the bring-up / cross-check kernel.
//
// One thread per (window row p0, window column p1, frequency k1).  The thread
// recomputes its n0 row transforms at frequency k1 along the reference's own
// DAG (only the 2^m1 - 1 butterflies that feed node k1), then runs the full
// n0-point column transform, i.e. exactly oracle.swfft_2d's per-window
// row-column FFT (/root/reference/pkg/src/swdft/oracle.py:118-133,166-187),
// which is bitwise equal to the tree.  No reuse across windows:
// O(n0*n1) butterflies per coefficient.  It exists to bring the boundary up
// and as an independent on-device schedule the fused kernel K1 is checked
// against; it is not the throughput path.
#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"
#include "../../include/swdft2d.h"

namespace swdft2d {

template <typename T, bool EXACT, int MAXN>
__global__ void __launch_bounds__(128) k0_window_kernel(K0Params P) {
    using C = cplx<T>;
    const int n0 = 1 << P.m0, n1 = 1 << P.m1;
    const int64_t rows = P.p0_end - P.p0_begin;
    const int64_t total = rows * P.P1 * n1;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int k1 = (int)(gid % n1);
    const int64_t p1 = (gid / n1) % P.P1;
    const int64_t pr = gid / ((int64_t)n1 * P.P1);
    const int64_t p0 = P.p0_begin + pr;
    const C *tw = reinterpret_cast<const C *>(P.tw);  // make_twiddles(TW_N), strided
    const int st0 = P.tw_n >> P.m0, st1 = P.tw_n >> P.m1;

    C z[MAXN], buf[MAXN];
    // Row transforms at frequency k1 (dim 1 first, tree2d.py:125-126).
    for (int t = 0; t < n0; ++t) {
        const int64_t row = p0 + t;
        for (int c = 0; c < n1; ++c) buf[c] = load_x<T>(P.x, P.in_dtype, row * P.ldx + p1 + c);
        // Residue classes of stride n1/L; class c combines classes c and c + half.
        int cnt = n1;
        for (int L2 = 2; L2 <= n1; L2 <<= 1) {
            const int half = cnt >> 1;
            const int i = k1 & (L2 - 1);                    // node index at this level
            const C w = tw[(int64_t)i * (n1 / L2) * st1];   // Omega1[i * s]
            for (int c = 0; c < half; ++c) buf[c] = bfly<EXACT>(buf[c], w, buf[c + half]);
            cnt = half;
        }
        z[t] = buf[0];
    }
    // Column transform over z[0..n0): all k0 (tree2d.py:127-128), residue-major.
    int classes = n0;
    for (int L = 1; L < n0; L <<= 1) {
        const int half = classes >> 1, L2 = L << 1;
        for (int c = 0; c < half; ++c)
            for (int i = 0; i < L2; ++i) {
                const int ii = i & (L - 1);
                const C w = tw[(int64_t)i * (n0 / L2) * st0];
                buf[c * L2 + i] = bfly<EXACT>(z[c * L + ii], w, z[(c + half) * L + ii]);
            }
        for (int q = 0; q < n0; ++q) z[q] = buf[q];
        classes = half;
    }
    C *out = reinterpret_cast<C *>(P.out) + ((pr * P.P1 + p1) * n0) * n1 + k1;
    for (int k0 = 0; k0 < n0; ++k0) {
        C v = z[k0];
        if (P.apply_scale) v = cscale(v, (T)P.scale);
        st_stream(out + (int64_t)k0 * n1, v);
    }
}

// Windows above 64: the same per-(p0, p1, k1) DAG without per-thread arrays of n
// complex (a MAXN = 1024 instantiation held 32 KB of local memory per thread, which the
// driver reserves for every resident thread: ~9.7 GB of HBM).  The row node k1 of each
// of the n0 rows is evaluated depth-first over the leaves in bit-reversed order with a
// stack of m1 + 1 partial nodes (each node is the same bfly(lower class, w, upper class)
// as the level loop above, so the bits are unchanged); the n0 results go straight into
// the thread's own output column out[p0, p1, :, k1], where the column transform runs in
// place: the element (class c, index i) of sub-length L lives at slot
// c + bitrev_{log2 L}(i) * n0 / L, so each butterfly pair overwrites its own two inputs,
// and a final bit-reversal swap puts k0 in natural order.  Consecutive threads own
// consecutive k1, so every in-place access of a warp is one contiguous run.
template <typename T, bool EXACT>
__global__ void __launch_bounds__(128) k0_window_large_kernel(K0Params P) {
    using C = cplx<T>;
    const int m0 = P.m0, m1 = P.m1, n0 = 1 << m0, n1 = 1 << m1;
    const int64_t rows = P.p0_end - P.p0_begin;
    const int64_t total = rows * P.P1 * n1;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int k1 = (int)(gid % n1);
    const int64_t p1 = (gid / n1) % P.P1;
    const int64_t pr = gid / ((int64_t)n1 * P.P1);
    const int64_t p0 = P.p0_begin + pr;
    const C *tw = reinterpret_cast<const C *>(P.tw);  // make_twiddles(TW_N), strided
    const int st0 = P.tw_n >> m0, st1 = P.tw_n >> m1;
    C *col = reinterpret_cast<C *>(P.out) + ((pr * P.P1 + p1) * n0) * n1 + k1;  // slot t: col[t * n1]

    for (int t = 0; t < n0; ++t) {
        const int64_t row = (p0 + t) * P.ldx + p1;
        C stk[SWDFT2D_K0_MAX_M + 1];
        int lvl[SWDFT2D_K0_MAX_M + 1];
        int sp = 0;
        for (int q = 0; q < n1; ++q) {
            const int c = m1 ? (int)(__brev((unsigned)q) >> (32 - m1)) : 0;
            C v = load_x<T>(P.x, P.in_dtype, row + c);
            int l = 0;
            while (sp > 0 && lvl[sp - 1] == l) {  // combine with the left (lower-class) sibling
                const int L2 = 2 << l;
                const C w = tw[(int64_t)(k1 & (L2 - 1)) * (n1 / L2) * st1];
                v = bfly<EXACT>(stk[sp - 1], w, v);
                --sp;
                ++l;
            }
            stk[sp] = v;
            lvl[sp] = l;
            ++sp;
        }
        col[(int64_t)t * n1] = stk[0];
    }
    for (int L = 1; L < n0; L <<= 1) {
        const int half = n0 / (2 * L), lg = 31 - __clz(L);
        for (int c = 0; c < half; ++c)
            for (int ii = 0; ii < L; ++ii) {
                const int br = lg ? (int)(__brev((unsigned)ii) >> (32 - lg)) : 0;
                C *a = col + (int64_t)(c + br * (n0 / L)) * n1;
                C *b = col + (int64_t)(c + half + br * (n0 / L)) * n1;
                const C A = *a, B = *b;
                const int64_t s = (int64_t)(n0 / (2 * L)) * st0;
                *a = bfly<EXACT>(A, tw[(int64_t)ii * s], B);
                *b = bfly<EXACT>(A, tw[(int64_t)(ii + L) * s], B);
            }
    }
    for (int t = 0; t < n0; ++t) {
        const int u = m0 ? (int)(__brev((unsigned)t) >> (32 - m0)) : 0;
        if (u > t) {
            const C A = col[(int64_t)t * n1], B = col[(int64_t)u * n1];
            col[(int64_t)t * n1] = B;
            col[(int64_t)u * n1] = A;
        }
    }
    if (P.apply_scale)
        for (int t = 0; t < n0; ++t) col[(int64_t)t * n1] = cscale(col[(int64_t)t * n1], (T)P.scale);
}

template <typename T, bool EXACT>
static int launch_k0_t(const K0Params &P, cudaStream_t stream) {
    const int64_t total = (P.p0_end - P.p0_begin) * P.P1 * ((int64_t)1 << P.m1);
    if (total == 0) return 0;
    const int threads = 128;
    const int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 0x7fffffffLL) return -1;
    if (P.m0 <= 6 && P.m1 <= 6)
        k0_window_kernel<T, EXACT, 64><<<(unsigned)blocks, threads, 0, stream>>>(P);
    else
        k0_window_large_kernel<T, EXACT><<<(unsigned)blocks, threads, 0, stream>>>(P);
    return 0;
}

int launch_k0(const K0Params &P, int prec, cudaStream_t stream) {
    return prec == 1 ? launch_k0_t<double, true>(P, stream) : launch_k0_t<float, false>(P, stream);
}

}  // namespace swdft2d
