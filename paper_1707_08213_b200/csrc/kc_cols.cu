// KC — column-tree kernel of the large-window path (windows with n0 > 64 or n1 > 64,
// up to 1024 x 1024), the stage-C half of the separable schedule:
//   stage R: KR writes Z[r][p1][k1], the dim-1 tree of every input row of a strip
//            (row_level_step, tree2d.py:72-93) into a stream-ordered workspace;
//   stage C: KC runs the dim-0 tree (col_level_step, tree2d.py:96-120) down every
//            column c = (p1, k1) of Z and writes out[p0][p1][k0][k1].
// The factorisation is exact, so fp64 stays bitwise.
// KC is KR's shared-memory level schedule (radix-4 passes, the middle level in
// registers; one radix-2 pass first when m0 is odd) with a column dimension: a CTA
// owns CW consecutive columns (the fast index, so Z reads and output writes are
// CW-element runs) x TP0 window rows.
#include <cstdlib>

#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"

namespace swdft2d {

// CTA sizes: two 113 KB CTAs per SM of KC_THREADS_STD threads, or one 227 KB CTA (deep
// tiles of n0 >= 512) of KC_THREADS_BIG threads — the passes are loops over thousands of
// independent items, and a lone 256-thread CTA left the SM at 8 warps, latency-bound
// (ncu, 1024 x 8: issue 35 %, profiles/ncu_r02.md)
#ifndef KC_THREADS_STD
#define KC_THREADS_STD 256
#endif
#ifndef KC_THREADS_BIG
#define KC_THREADS_BIG 1024
#endif
constexpr size_t KC_SMEM_CAP = 113 * 1024;  // two CTAs per SM

// nodes of level t for TP0 window rows: (TP0 + s_t - 1) 2^t, per column
__host__ __device__ constexpr int64_t kc_level_nodes(int M0, int TP0, int t) {
    return (int64_t)(TP0 + (1 << (M0 - t)) - 1) << t;
}
// levels stored in shared memory (pass order t = 0, [1 if m0 odd], then every second up
// to m0 - 2), alternating between buffers A (which = 0) and B (which = 1)
__host__ __device__ constexpr int64_t kc_buf(int M0, int TP0, int which) {
    int64_t best = 1;
    int idx = 0;
    for (int t = 0; t <= (M0 > 1 ? M0 - 2 : 0); ++t) {
        const bool stored = t == 0 || (t % 2) == (M0 % 2);
        if (!stored) continue;
        const int64_t v = kc_level_nodes(M0, TP0, t);
        if ((idx & 1) == which && v > best) best = v;
        ++idx;
    }
    return best;
}
// twiddles: Omega_n0[k] (n0 entries), then compact level tables Omega_L[k] = Omega_n0[k n0/L]
// for L = 2 .. n0/4 at offset L - 2 (n0/2 - 2 entries): a pass reads level-L twiddles of
// consecutive k, which at stride n0/L >= 4 in the n0 table all fell in one bank
__host__ __device__ constexpr int kc_tw_entries(int M0) {
    return (1 << M0) + (M0 >= 3 ? (1 << (M0 - 1)) - 2 : 0);
}
__host__ __device__ constexpr size_t kc_smem(int M0, int TP0, int CW, int esz) {
    return (size_t)esz * ((size_t)CW * (kc_buf(M0, TP0, 0) + kc_buf(M0, TP0, 1)) + kc_tw_entries(M0));
}
// level-(l) twiddle k (Omega_{2^l}[k]) from the smem tables above
template <int M0, typename C> __device__ __forceinline__ C kc_tw(const C *stw, int l, int k) {
    return M0 - l <= 1 ? stw[k << (M0 - l)] : stw[(1 << M0) + (1 << l) - 2 + k];
}
// Tile shape (CW columns x TP0 window rows) within the cap, two rules:
//  * wide (DEEP = false): the widest column group, then the most window rows — long
//    contiguous Z reads and output runs;
//  * deep (DEEP = true): the least per-output cost counting the tree nodes the tile
//    computes (its n0 - 1 halo rows are recomputed, so few window rows cost up to 2x
//    more butterflies for tall windows), the Z rows it reads, and stores narrower than a
//    32-byte sector.
// The output run of a column group is at most n1 columns long (the next columns belong
// to the next window position), so narrow windows gain nothing from wide groups: the
// launcher takes the deep rule when n1 x element <= 512 B (measured: 128x8 fp32 3.6 ->
// 5.0 TB/s, 256x64 3.8 -> 4.0; 128x128 fp64 keeps the wide rule, 4.3 vs 3.9).
__host__ __device__ constexpr double kc_cost(int M0, int TP0, int CW, int esz) {
    int64_t nodes = 0;
    for (int t = 1; t <= M0; ++t) nodes += kc_level_nodes(M0, TP0, t);
    const double per = (double)TP0 * (double)(1 << M0);
    const double wide = (double)CW * esz >= 32 ? 1.0 : (double)CW * esz / 32.0;
    return (double)nodes / per + 2.0 * (double)(TP0 + (1 << M0) - 1) / per + 2.0 / wide;
}
template <typename T, int M0, bool DEEP> struct KCShape {
    // deep tiles of the tallest windows (n0 >= 512) may take a whole SM's shared memory:
    // one CTA per SM, but 16 window rows per tile instead of 4 (~40 % fewer nodes)
    static constexpr size_t CAP = (DEEP && M0 >= 9) ? 227 * 1024 : KC_SMEM_CAP;
    static constexpr int pick(int what) {
        const int cws[6] = {32, 16, 8, 4, 2, 1};
        const int tps[4] = {16, 8, 4, 2};
        const int esz = (int)sizeof(T) * 2;
        int bc = 1, bt = 2;
        double best = 1e300;
        for (int a = 0; a < 6; ++a)
            for (int b = 0; b < 4; ++b)
                if (kc_smem(M0, tps[b], cws[a], esz) <= CAP) {
                    if (!DEEP) return what == 0 ? cws[a] : tps[b];
                    const double c = kc_cost(M0, tps[b], cws[a], esz);
                    if (c < best) {
                        best = c;
                        bc = cws[a];
                        bt = tps[b];
                    }
                }
        return what == 0 ? bc : bt;
    }
    static constexpr int CW = pick(0), TP0 = pick(1);
    static constexpr size_t SMEM = kc_smem(M0, TP0, CW, (int)sizeof(T) * 2);
    static constexpr int THREADS = CAP > KC_SMEM_CAP ? KC_THREADS_BIG : KC_THREADS_STD;
};

template <typename T, bool EXACT, int M0, int TP0, int CW, int t, bool LAST, int KC_THREADS>
__device__ __forceinline__ void kc_pass4(const cplx<T> *src, cplx<T> *dst, const cplx<T> *stw,
                                         int npos, int ncol, const KCParams &P, int64_t r0,
                                         int64_t c0) {
    using C = cplx<T>;
    constexpr int n0 = 1 << M0, Lt = 1 << t, s2 = n0 >> (t + 2);
    constexpr int cnt = LAST ? TP0 : TP0 + s2 - 1;
    const int items = (LAST ? npos : cnt) * Lt * CW;
    const T f = (T)P.scale;
    // When the CTA size is a multiple of CW x Lt, every item a thread takes has the same j,
    // so its six twiddles are read once per pass: per item, they were smem reads at a
    // stride of 2^(m0-1-t) entries — all in one bank, up to 8-way conflicts (ncu,
    // 1024 x 8: 40 % of shared-memory wavefronts were conflicts)
    constexpr bool HOIST = KC_THREADS % (CW * Lt) == 0;
    C w[6];
    auto twiddles = [&](int j) {
        w[0] = kc_tw<M0>(stw, t + 1, j);
        w[1] = kc_tw<M0>(stw, t + 1, j + Lt);
#pragma unroll
        for (int u = 0; u < 4; ++u) w[2 + u] = kc_tw<M0>(stw, t + 2, j + u * Lt);
    };
    if constexpr (HOIST) twiddles((threadIdx.x / CW) % Lt);
    for (int it = threadIdx.x; it < items; it += KC_THREADS) {
        const int col = it % CW, q = it / CW, j = q % Lt, p = q / Lt;
        const C a0 = src[(p * Lt + j) * CW + col], a1 = src[((p + s2) * Lt + j) * CW + col];
        const C a2 = src[((p + 2 * s2) * Lt + j) * CW + col];
        const C a3 = src[((p + 3 * s2) * Lt + j) * CW + col];
        if constexpr (!HOIST) twiddles(j);
        C b0, b1, c0v, c1, o[4];
        bfly_pair<EXACT>(a0, w[0], w[1], a2, b0, b1);    // level t+1 at p
        bfly_pair<EXACT>(a1, w[0], w[1], a3, c0v, c1);   // at p + s_{t+2}
        bfly_pair<EXACT>(b0, w[2], w[4], c0v, o[0], o[2]);
        bfly_pair<EXACT>(b1, w[3], w[5], c1, o[1], o[3]);
        if constexpr (LAST) {
            if (col >= ncol) continue;
            const int64_t cc = c0 + col;
            const int64_t p1 = cc >> P.m1, k1 = cc & (((int64_t)1 << P.m1) - 1);
            C *o_ = static_cast<C *>(P.out) +
                    ((((r0 + p) * P.P1 + p1) * n0 + j) << P.m1) + k1;
            if (P.apply_scale) {  // uniform branch: no predicated multiplies when unscaled
#pragma unroll
                for (int u = 0; u < 4; ++u) st_stream(o_ + ((int64_t)(u * Lt) << P.m1), cscale(o[u], f));
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) st_stream(o_ + ((int64_t)(u * Lt) << P.m1), o[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) dst[(p * 4 * Lt + j + u * Lt) * CW + col] = o[u];
        }
    }
}

template <typename T, bool EXACT, int M0, int TP0, int CW, bool LAST, int KC_THREADS>
__device__ __forceinline__ void kc_pass2(const cplx<T> *src, cplx<T> *dst, const cplx<T> *stw,
                                         int npos, int ncol, const KCParams &P, int64_t r0,
                                         int64_t c0) {
    // levels 0 -> 1 (m0 odd), or the whole tree when m0 = 1
    using C = cplx<T>;
    constexpr int n0 = 1 << M0, s1 = n0 >> 1;
    constexpr int cnt = LAST ? TP0 : TP0 + s1 - 1;
    const int items = (LAST ? npos : cnt) * CW;
    const C wa = stw[0], wb = stw[1 << (M0 - 1)];
    const T f = (T)P.scale;
    for (int it = threadIdx.x; it < items; it += KC_THREADS) {
        const int col = it % CW, p = it / CW;
        const C a0 = src[p * CW + col], a1 = src[(p + s1) * CW + col];
        C lo, hi;
        bfly_pair<EXACT>(a0, wa, wb, a1, lo, hi);
        if constexpr (LAST) {
            if (col >= ncol) continue;
            const int64_t cc = c0 + col;
            const int64_t p1 = cc >> P.m1, k1 = cc & (((int64_t)1 << P.m1) - 1);
            C *o_ = static_cast<C *>(P.out) + ((((r0 + p) * P.P1 + p1) * n0) << P.m1) + k1;
            st_stream(o_, P.apply_scale ? cscale(lo, f) : lo);
            st_stream(o_ + ((int64_t)1 << P.m1), P.apply_scale ? cscale(hi, f) : hi);
        } else {
            dst[(p * 2) * CW + col] = lo;
            dst[(p * 2 + 1) * CW + col] = hi;
        }
    }
}

template <typename T, bool EXACT, int M0, bool DEEP>
__global__ void __launch_bounds__(KCShape<T, M0, DEEP>::THREADS)
    kc_cols_kernel(const __grid_constant__ KCParams P) {
    using C = cplx<T>;
    using S = KCShape<T, M0, DEEP>;
    constexpr int KC_THREADS = S::THREADS;
    constexpr int n0 = 1 << M0, TP0 = S::TP0, CW = S::CW;
    constexpr int W = TP0 + n0 - 1;
    extern __shared__ __align__(16) unsigned char kc_smem_raw[];
    C *bufA = reinterpret_cast<C *>(kc_smem_raw);
    C *bufB = bufA + CW * kc_buf(M0, TP0, 0);
    C *stw = bufB + CW * kc_buf(M0, TP0, 1);  // Omega_n0[k] (make_twiddles(1024), stride 1024/n0)
    for (int k = threadIdx.x; k < n0; k += KC_THREADS)
        stw[k] = __ldg(static_cast<const C *>(P.tw) + (k << (10 - M0)));
    for (int e = threadIdx.x; e < kc_tw_entries(M0) - n0; e += KC_THREADS) {
        const int l = 31 - __clz(e + 2), k = e + 2 - (1 << l);  // table L = 2^l, entry k
        stw[n0 + e] = __ldg(static_cast<const C *>(P.tw) + (k << (10 - l)));
    }
    const C *z = static_cast<const C *>(P.z);
    const int64_t ctiles = (P.cols + CW - 1) / CW;
    const int64_t ntiles = ctiles * ((P.P0s + TP0 - 1) / TP0);
    // level 0 (the tile's W Z rows x CW columns) of the NEXT tile is loaded into
    // registers while the current tile's passes run
    constexpr int NLOAD = (W * CW + KC_THREADS - 1) / KC_THREADS;
    // prefetch unless the column group is narrow (scattered 16-32 B row pieces: measured
    // slower for n0 = 1024) or the tile too large for registers
    constexpr bool PF = NLOAD <= 20 && CW >= 8;
    constexpr int NPRE = PF ? NLOAD : 1;
    C pre[NPRE];
    auto fetch = [&](int64_t tile) {
        const int64_t rt = tile / ctiles, ct = tile - rt * ctiles;
        const int64_t r0 = rt * TP0, c0 = ct * CW;
        const int ncol = (int)(P.cols - c0 < CW ? P.cols - c0 : CW);
#pragma unroll
        for (int q = 0; q < NPRE; ++q) {
            const int it = threadIdx.x + q * KC_THREADS;
            const int col = it % CW, p = it / CW;
            const int64_t r = r0 + p;
            pre[q] = (it < W * CW && col < ncol && r < P.zrows) ? z[r * P.ldz + c0 + col]
                                                                : mk<T>((T)0, (T)0);
        }
    };
    if (PF && (int64_t)blockIdx.x < ntiles) fetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t rt = tile / ctiles, ct = tile - rt * ctiles;
        const int64_t r0 = rt * TP0, c0 = ct * CW;
        const int npos = (int)(P.P0s - r0 < TP0 ? P.P0s - r0 : TP0);
        const int ncol = (int)(P.cols - c0 < CW ? P.cols - c0 : CW);
        __syncthreads();  // previous tile done with the buffers (and stw filled)
        if constexpr (PF) {
#pragma unroll
            for (int q = 0; q < NPRE; ++q) {  // level 0 = Z rows
                const int it = threadIdx.x + q * KC_THREADS;
                if (it < W * CW) bufA[it] = pre[q];
            }
            if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
        } else {
            for (int it = threadIdx.x; it < W * CW; it += KC_THREADS) {
                const int col = it % CW, p = it / CW;
                const int64_t r = r0 + p;
                bufA[it] = (col < ncol && r < P.zrows) ? z[r * P.ldz + c0 + col] : mk<T>((T)0, (T)0);
            }
        }
        __syncthreads();
        if constexpr (M0 == 1) {
            kc_pass2<T, EXACT, M0, TP0, CW, true, KC_THREADS>(bufA, nullptr, stw, npos, ncol, P, r0, c0);
        } else {
            constexpr int T0 = M0 % 2;
            C *src = bufA, *dst = bufB;
            if constexpr (T0 == 1) {
                kc_pass2<T, EXACT, M0, TP0, CW, false, KC_THREADS>(src, dst, stw, npos, ncol, P, r0, c0);
                __syncthreads();
                src = bufB;
                dst = bufA;
            }
            static_for<(M0 - T0) / 2>([&](auto kcc) {
                constexpr int t = T0 + 2 * decltype(kcc)::value;
                if constexpr (t + 2 == M0) {
                    kc_pass4<T, EXACT, M0, TP0, CW, t, true, KC_THREADS>(src, nullptr, stw, npos, ncol, P, r0, c0);
                } else {
                    kc_pass4<T, EXACT, M0, TP0, CW, t, false, KC_THREADS>(src, dst, stw, npos, ncol, P, r0, c0);
                    __syncthreads();
                    C *tmp = src;
                    src = dst;
                    dst = tmp;
                }
            });
        }
    }
}

template <typename T, bool EXACT, int M0, bool DEEP>
static int kc_launch_one(const KCParams &P, cudaStream_t st, int64_t *rows_per_strip_hint) {
    using S = KCShape<T, M0, DEEP>;
    auto fn = &kc_cols_kernel<T, EXACT, M0, DEEP>;
    if (S::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM) !=
            cudaSuccess)
        return -2;
    if (rows_per_strip_hint) *rows_per_strip_hint = S::TP0;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, S::THREADS, S::SMEM) != cudaSuccess ||
        occ < 1)
        return -2;
    const int64_t tiles = ((P.cols + S::CW - 1) / S::CW) * ((P.P0s + S::TP0 - 1) / S::TP0);
    if (tiles == 0) return 0;
    const int64_t slots = (int64_t)P.sms * occ;
    static const int force = [] {  // SWDFT2D_KC_ONESHOT=0/1: persistent / one CTA per tile
        const char *e = std::getenv("SWDFT2D_KC_ONESHOT");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    // One CTA per tile for deep tiles (short output runs) below the 227 KB shapes, when the
    // tiles fill >= 3 waves: 128x8 5.0 -> 5.4 TB/s (fp64 5.1 -> 5.7), 256x64 4.0 -> 4.2,
    // 16x16 forced separable 4.6 -> 5.4; wide tiles lose with it (128x128 fp32 -6 %,
    // 64x256 -3 %: their persistent grid prefetches the next tile's Z rows), and so do the
    // one-CTA-per-SM 227 KB tiles of n0 >= 512 (-5 %), and the small trees (n0 <= 8) of the
    // kD path's dim-0 pass (3-D 4x8x8 -11 %, 8x8x8 -4 %; 16x8x4 gains 9-13 %).
    // profiles/bench_large_r01b.jsonl, bench_kd_r01b.jsonl.
    const bool oneshot =
        force >= 0 ? force == 1 : (DEEP && M0 >= 4 && M0 < 9 && tiles >= 3 * slots);
    fn<<<(unsigned)((oneshot || tiles < slots) ? tiles : slots), S::THREADS, S::SMEM, st>>>(P);
    return 0;
}

template <typename T, bool EXACT, int M0>
static int kc_launch_t(const KCParams &P, cudaStream_t st, int64_t *rows_per_strip_hint) {
    // deep tiles when a window position's n1 columns are a short run (<= 512 B)
    const bool deep = ((int64_t)sizeof(cplx<T>) << P.m1) <= 512;
    return deep ? kc_launch_one<T, EXACT, M0, true>(P, st, rows_per_strip_hint)
                : kc_launch_one<T, EXACT, M0, false>(P, st, rows_per_strip_hint);
}

template <typename T, bool EXACT>
static int kc_dispatch(const KCParams &P, int m0, cudaStream_t st) {
    switch (m0) {
    case 1: return kc_launch_t<T, EXACT, 1>(P, st, nullptr);
    case 2: return kc_launch_t<T, EXACT, 2>(P, st, nullptr);
    case 3: return kc_launch_t<T, EXACT, 3>(P, st, nullptr);
    case 4: return kc_launch_t<T, EXACT, 4>(P, st, nullptr);
    case 5: return kc_launch_t<T, EXACT, 5>(P, st, nullptr);
    case 6: return kc_launch_t<T, EXACT, 6>(P, st, nullptr);
    case 7: return kc_launch_t<T, EXACT, 7>(P, st, nullptr);
    case 8: return kc_launch_t<T, EXACT, 8>(P, st, nullptr);
    case 9: return kc_launch_t<T, EXACT, 9>(P, st, nullptr);
    case 10: return kc_launch_t<T, EXACT, 10>(P, st, nullptr);
    default: return -3;
    }
}

int launch_kc(const KCParams &P, int m0, int prec, cudaStream_t stream) {
    return prec == 1 ? kc_dispatch<double, true>(P, m0, stream)
                     : kc_dispatch<float, false>(P, m0, stream);
}

}  // namespace swdft2d
