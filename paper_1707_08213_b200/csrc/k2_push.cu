// K2 — incremental row-push kernel of the stream (SlidingRowStream2D.push_row,
// reference tree2d.py:205-303).
//
// The reference's stream keeps tree levels between pushes so that a push costs
// O(n0 n1) per window position instead of re-running the window.  K2 does the same
// on the device, one thread per output column c = (p1, k1), P1 * n1 threads:
//   1. stage R for the pushed row r alone: Z[r][p1][k1], the dim-1 tree of each window
//      position (the reference's DAG, tree2d.py:72-93: level t, shift s_t = n1 >> t,
//      node k1 mod 2^t, twiddle Omega1[(k1 mod 2^t) s_t]), built cooperatively by the
//      CTA in shared memory, one level per step (n1 log2 n1 / n1 butterflies per column);
//   2. the column levels l = 1..m0 of the dim-0 tree (tree2d.py:96-120):
//      T_l[r][i] = T_{l-1}[r - s_l][i mod h] (+) Omega0[i s_l] (x) T_{l-1}[r][i mod h],
//      s_l = n0 >> l, h = 2^(l-1).  T_{l-1}[r - s_l] comes from a per-level state ring
//      (below), where T_{l-1}[r] is stored for the push s_l rows later;
//   3. level m0 is the (P1, n0, n1) slab of window row r - n0 + 1 (written once r >= n0-1).
// Device state: m0 * n0/2 + n0 - 1 complex per column (level l ring = s_l + 1 slots
// x 2^(l-1) nodes), laid out [level][slot][node][column] so every access is
// coalesced across consecutive columns.  Every node is the same IEEE operation sequence as
// core.butterfly (fp64: bitwise equal to the batch transform); nodes whose rows
// precede row 0 read the zero-initialised state and are never consumed by a valid
// output (a level-l node at row r is valid iff r >= n0 - s_l).
// Per push: (n0 - 1) state reads + (n0 - 1) state writes + n0 output stores per
// column, against K1's n0-row warm-up per emitted row.  Large windows split a column
// over J = 2^max(m0-3, 0) threads (k0 residue classes) to keep registers low.
//
// Also here: the raw-row ring store (rows double-stored at slots p mod n0 and
// p mod n0 + n0) that push_rows and the non-incremental push read.
#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"

namespace swdft2d {

template <typename T>
__device__ __forceinline__ cplx<T> tw64(const K2Params &P, int idx) {
    const double2 w = P.tw[idx * (K0_TW_N / K2_TW_N)];
    return mk<T>((T)w.x, (T)w.y);
}

// State of level l (l = 1..m0): s_l + 1 slots (s_l = n0 >> l) of 2^(l-1) nodes of
// level l - 1, per column.  Push r reads slot (r - s_l) mod (s_l + 1) and writes slot
// r mod (s_l + 1) — never the same slot, so no thread's store can race another
// thread's load of the same node within a push.  Offset of level l, in nodes per column:
template <int M0, int L> __host__ __device__ constexpr int64_t k2_level_base() {
    return (int64_t)(L - 1) * ((1 << M0) / 2) + ((1 << (L - 1)) - 1);
}

// Threads per output column: J = 2^QK, QK = max(m0 - 3, 0); thread t of a column owns
// the final coefficients k0 = t (mod J), at most 8, so its register ring stays small
// and large windows still put enough loads in flight.
template <int M0> __host__ __device__ constexpr int k2_qk() { return M0 > 3 ? M0 - 3 : 0; }

template <typename T, bool EXACT, int M0, int M1>
__global__ void __launch_bounds__(256) k2_push_kernel(const __grid_constant__ K2Params P) {
    using C = cplx<T>;
    constexpr int n0 = 1 << M0, n1 = 1 << M1;
    constexpr int QK = k2_qk<M0>(), J = 1 << QK;
    const int64_t cols = P.P1 * n1;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int t = (int)blockIdx.y;  // k0 residue class of this thread
    // twiddles in shared memory: stage R indexes them by the lane's k1 (divergent)
    __shared__ C stw[K2_TW_N];
    if (threadIdx.x < K2_TW_N) stw[threadIdx.x] = tw64<T>(P, threadIdx.x);
    __syncthreads();
    if (P.ring && t == 0 && c < P.N1) {  // raw ring, both copies
        const C v = load_x<T>(P.row, P.in_dtype, c);
        C *ring = static_cast<C *>(P.ring);
        const int64_t slot = P.r & (n0 - 1);
        ring[slot * P.N1 + c] = v;
        ring[(slot + n0) * P.N1 + c] = v;
    }
    // 1. stage R for the pushed row: the CTA's 256 columns are 256 / n1 whole window
    //    positions (n1 <= 64 divides 256), whose n1-point trees it builds cooperatively in
    //    shared memory, one tree level per step (every node once, instead of each thread
    //    re-evaluating the 2^m1-leaf chain of its own output — 63 butterflies and 64
    //    loads per thread for n1 = 64, times J residue threads).  The nodes and their
    //    operand roles are the reference DAG's (tree2d.py:72-93), as in rnode:
    //      Y_t[a][r] = Y_{t-1}[a + (n1 >> t)][r mod 2^(t-1)] (+) Omega1[r (n1 >> t)] (x)
    //                  Y_{t-1}[a][r mod 2^(t-1)],   a < n1 >> t, r < 2^t,
    //    Y_0[a][0] = x[e - a] (e = the position's last sample), Z[k1] = Y_m1[0][k1].
    constexpr int NPOS = 256 / n1;
    __shared__ C samp[NPOS + n1 - 1];
    __shared__ C ybuf[2][256];
    const int64_t cb0 = blockIdx.x * (int64_t)blockDim.x;
    const int64_t pos0 = cb0 >> M1;
    if constexpr (M1 > 0) {
        for (int i = threadIdx.x; i < NPOS + n1 - 1; i += blockDim.x) {
            const int64_t xi = pos0 + i;
            samp[i] = xi < P.N1 ? load_x<T>(P.row, P.in_dtype, xi) : mk<T>((T)0, (T)0);
        }
        __syncthreads();
        const int lp = threadIdx.x >> M1, idx = threadIdx.x & (n1 - 1);  // (position, node)
        static_for<M1>([&](auto tc) {
            constexpr int t = decltype(tc)::value + 1;
            constexpr int sa = n1 >> t, hr = 1 << (t - 1);
            const int a = idx >> t, r = idx & ((1 << t) - 1), rh = r & (hr - 1);
            C sh, cu;
            if constexpr (t == 1) {  // level-0 operands straight from the samples
                sh = samp[lp + n1 - 1 - (a + sa)];
                cu = samp[lp + n1 - 1 - a];
            } else {
                const C *src = ybuf[(t - 2) & 1] + lp * n1;
                sh = src[(a + sa) * hr + rh];
                cu = src[a * hr + rh];
            }
            ybuf[(t - 1) & 1][lp * n1 + idx] = bfly<EXACT>(sh, stw[r << (6 - t)], cu);
            __syncthreads();
        });
    }
    if (c >= cols) return;
    const int64_t p1 = c >> M1;
    const int k1 = (int)(c & (n1 - 1));
    C z;
    if constexpr (M1 == 0) {
        z = load_x<T>(P.row, P.in_dtype, p1);
    } else {
        z = ybuf[(M1 - 1) & 1][threadIdx.x];
    }

    C *__restrict__ out = static_cast<C *>(P.out);
    const bool emit = out != nullptr && P.r >= n0 - 1;
    const T f = (T)P.scale;
    if constexpr (M0 == 0) {
        if (emit) out[p1 * n1 + k1] = P.apply_scale ? cscale(z, f) : z;
        return;
    } else {
        C *__restrict__ state = static_cast<C *>(P.state);
        // 2a. levels 1..QK (2^l <= J): the thread's one node, index t mod 2^l; the
        //     level-(l-1) node j = t mod h is stored by thread t = j.
        C v = z;
        static_for<QK>([&](auto lc) {
            constexpr int l = decltype(lc)::value + 1;
            constexpr int h = 1 << (l - 1);
            constexpr int s = n0 >> l;
            const int j = t & (h - 1);
            C *lev = state + (k2_level_base<M0, l>() + j) * cols + c;
            const C sh = __ldcg(lev + (int64_t)((P.r + 1) % (s + 1)) * h * cols);  // T_{l-1}[r - s_l][j]
            if (t < h) __stcg(lev + (int64_t)(P.r % (s + 1)) * h * cols, v);      // T_{l-1}[r][j]
            v = bfly<EXACT>(sh, stw[(t & (2 * h - 1)) << (6 - l)], v);
        });
        // 2b. levels QK+1..m0 (2^l > J): the thread holds nodes t + J u, u < 2^l / J
        C cur[n0 / (2 * J) > 1 ? n0 / (2 * J) : 1];
        cur[0] = v;
        static_for<M0 - QK>([&](auto lc) {
            constexpr int l = decltype(lc)::value + QK + 1;
            constexpr int h = 1 << (l - 1);
            constexpr int s = n0 >> l;
            constexpr int nh = h / J;  // nodes held at level l - 1
            C *lev = state + (k2_level_base<M0, l>() + t) * cols + c;
            const C *rd = lev + (int64_t)((P.r + 1) % (s + 1)) * h * cols;
            C *wr = lev + (int64_t)(P.r % (s + 1)) * h * cols;
            C sh[nh];
            static_for<nh>([&](auto uc) {
                constexpr int u = decltype(uc)::value;
                sh[u] = __ldcg(rd + (int64_t)(J * u) * cols);  // T_{l-1}[r - s_l][t + J u]
            });
            static_for<nh>([&](auto uc) {
                constexpr int u = decltype(uc)::value;
                __stcg(wr + (int64_t)(J * u) * cols, cur[u]);  // T_{l-1}[r][t + J u]
            });
            static_for<nh>([&](auto uc) {
                constexpr int u = decltype(uc)::value;
                const int j = t + J * u;
                C lo, hi;
                bfly_pair<EXACT>(sh[u], stw[j << (6 - l)], stw[(j + h) << (6 - l)], cur[u], lo, hi);
                if constexpr (l < M0) {
                    cur[u + nh] = hi;
                    cur[u] = lo;
                } else if (emit) {
                    C *o = out + (p1 * n0) * n1 + k1;
                    o[(int64_t)j * n1] = P.apply_scale ? cscale(lo, f) : lo;
                    o[(int64_t)(j + h) * n1] = P.apply_scale ? cscale(hi, f) : hi;
                }
            });
        });
    }
}

template <typename T, bool EXACT, int M0, int M1>
static void launch_t(const K2Params &P, cudaStream_t st) {
    const int64_t cols = P.P1 * ((int64_t)1 << M1);
    const int64_t work = cols > P.N1 ? cols : P.N1;
    const int threads = 256;
    const dim3 grid((unsigned)((work + threads - 1) / threads), 1u << k2_qk<M0>());
    k2_push_kernel<T, EXACT, M0, M1><<<grid, threads, 0, st>>>(P);
}

template <typename T, bool EXACT, int M0>
static int dispatch_m1(const K2Params &P, int m1, cudaStream_t st) {
    switch (m1) {
    case 0: launch_t<T, EXACT, M0, 0>(P, st); return 0;
    case 1: launch_t<T, EXACT, M0, 1>(P, st); return 0;
    case 2: launch_t<T, EXACT, M0, 2>(P, st); return 0;
    case 3: launch_t<T, EXACT, M0, 3>(P, st); return 0;
    case 4: launch_t<T, EXACT, M0, 4>(P, st); return 0;
    case 5: launch_t<T, EXACT, M0, 5>(P, st); return 0;
    case 6: launch_t<T, EXACT, M0, 6>(P, st); return 0;
    default: return -1;
    }
}

template <typename T, bool EXACT>
static int dispatch(const K2Params &P, int m0, int m1, cudaStream_t st) {
    switch (m0) {
    case 0: return dispatch_m1<T, EXACT, 0>(P, m1, st);
    case 1: return dispatch_m1<T, EXACT, 1>(P, m1, st);
    case 2: return dispatch_m1<T, EXACT, 2>(P, m1, st);
    case 3: return dispatch_m1<T, EXACT, 3>(P, m1, st);
    case 4: return dispatch_m1<T, EXACT, 4>(P, m1, st);
    case 5: return dispatch_m1<T, EXACT, 5>(P, m1, st);
    case 6: return dispatch_m1<T, EXACT, 6>(P, m1, st);
    default: return -1;
    }
}

int launch_k2(const K2Params &P, int m0, int m1, int prec, cudaStream_t stream) {
    return prec == 1 ? dispatch<double, true>(P, m0, m1, stream)
                     : dispatch<float, false>(P, m0, m1, stream);
}

template <typename T>
__global__ void __launch_bounds__(256) ring_store_kernel(const void *__restrict__ row, int in_dtype,
                                                         int64_t N1, cplx<T> *__restrict__ a,
                                                         cplx<T> *__restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const cplx<T> v = load_x<T>(row, in_dtype, i);
        a[i] = v;
        b[i] = v;
    }
}

int launch_ring_store(const void *row, int in_dtype, int64_t N1, void *ring, int prec, int n0,
                      int64_t p0, int sms, cudaStream_t stream) {
    const int64_t slot = p0 % n0;
    const int threads = 256;
    int64_t blocks = (N1 + threads - 1) / threads;
    if (blocks > 4 * (int64_t)sms) blocks = 4 * (int64_t)sms;
    if (prec == 1) {
        double2 *r = static_cast<double2 *>(ring);
        ring_store_kernel<double><<<(unsigned)blocks, threads, 0, stream>>>(
            row, in_dtype, N1, r + slot * N1, r + (slot + n0) * N1);
    } else {
        float2 *r = static_cast<float2 *>(ring);
        ring_store_kernel<float><<<(unsigned)blocks, threads, 0, stream>>>(
            row, in_dtype, N1, r + slot * N1, r + (slot + n0) * N1);
    }
    return 0;
}

}  // namespace swdft2d
