// KR — row-tree kernel for windows with n0 = 1: the 1D tree (tree1d.py:29-60, the
// m0 = 0 case of the 2D tree) and 2D windows of one row, for n1 = 2 .. 1024.
//
// With n0 = 1 every output row is an independent set of 1D sliding transforms, so K1's
// row ring and column stage have nothing to do; KR instead gives each CTA a tile of
// TPOS consecutive window positions of one row and builds the dim-1 tree level by
// levels in shared memory (row_level_step, tree2d.py:72-93), two levels per pass
// (radix-4 passes, the middle level in registers; one radix-2 pass first if m is odd):
//   L_t[p][i] = L_{t-1}[p][i mod h] (+) Omega[i s_t] (x) L_{t-1}[p + s_t][i mod h],
//   s_t = n >> t, h = 2^(t-1).  L_t[p] holds the 2^t level-t nodes at tile-local end
//   position p + n - s_t: level t is needed at TPOS + s_t - 1 end positions, and the
//   level-(t-1) nodes at end positions e - s_t and e sit at indices p and p + s_t.
// Level 0 = the W = TPOS + n - 1 input samples; the last pass writes straight into the
// output, TPOS x n contiguous coefficients per tile (streaming stores).  The
// same IEEE operation per node as core.butterfly, so fp64 is bitwise equal to the
// reference.  Per coefficient: ~2 + log2(n)/TPOS butterflies; bound by the writes.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"

namespace swdft2d {

// Window positions per tile: ~16 K coefficients per CTA (32 K for fp32 n >= 512 and fp64
// n = 1024), the best of 4 K .. 64 K in the sweep of profiles/kr_sweep_r01.jsonl
// (n = 16 .. 1024); fp64 n = 1024 with 32 positions instead of 16: 3.95 -> 4.88 TB/s.
// Position cap: 512 for n <= 16 (one-shot CTAs of 256 positions were too short: n = 16
// 4.99 -> 5.27 TB/s fp32, 5.53 -> 6.36 fp64; a 1024 cap fell back to 5.04 / 5.91),
// 256 above (n = 32 fp64 spills at 512)
#ifndef KR_TPOS_CAP
#define KR_TPOS_CAP (M1 <= 4 ? 512 : 256)
#endif
template <typename T, int M1> __host__ __device__ constexpr int kr_tpos() {
#if defined(KR_PER32) && defined(KR_PER64)  // tuning builds (scripts/tune/kr)
    const int per = (sizeof(T) == 8 ? KR_PER64 : KR_PER32) >> M1;
#else
    const int per = (sizeof(T) == 4 && M1 >= 9 ? 32768 : sizeof(T) == 8 && M1 >= 10 ? 32768 : 16384) >> M1;
#endif
    const int lo = sizeof(T) == 8 ? 4 : 8;
    return per < lo ? lo : per > KR_TPOS_CAP ? KR_TPOS_CAP : per;
}
// Levels kept in shared memory, in pass order: t = 0, then (odd m) 1, then every second
// level up to m - 2; they alternate between buffer A (even index in that order) and B.
// Nodes of level t in a tile: (TPOS + s_t - 1) 2^t.
template <int M1, int TPOS> __host__ __device__ constexpr int kr_buf(int which) {
    int best = 0, idx = 0;
    for (int t = 0; t <= (M1 > 1 ? M1 - 2 : 0); ++t) {
        const bool stored = t == 0 || (t % 2) == (M1 % 2);
        if (!stored) continue;
        const int v = (TPOS + (1 << (M1 - t)) - 1) << t;
        if ((idx & 1) == which && v > best) best = v;
        ++idx;
    }
    return best > 1 ? best : 1;
}

constexpr int KR_THREADS = 256;

// Radix-2 pass (levels t -> t + 1; used for t = 0 when m is odd, or alone when m = 1):
// per (position p, node j < 2^t) both children j and j + 2^t from the same two reads.
template <typename T, bool EXACT, int M1, int TPOS, int t, bool LAST>
__device__ __forceinline__ void kr_pass2(const cplx<T> *src, cplx<T> *dst, const cplx<T> *stw,
                                         int npos, const KRParams &P) {
    using C = cplx<T>;
    constexpr int n = 1 << M1, Lt = 1 << t, s1 = n >> (t + 1);
    constexpr int cnt = LAST ? TPOS : TPOS + s1 - 1;
    const int items = (LAST ? npos : cnt) * Lt;
    static_assert(Lt <= KR_THREADS, "radix-2 pass only at small t");
    const int j = threadIdx.x & (Lt - 1);
    const C wa = stw[j << (M1 - 1 - t)], wb = stw[(j + Lt) << (M1 - 1 - t)];
    const T f = (T)P.scale;
    for (int it = threadIdx.x; it < items; it += KR_THREADS) {
        const int p = it >> t;
        const C a0 = src[p * Lt + j], a1 = src[(p + s1) * Lt + j];
        C lo, hi;
        bfly_pair<EXACT>(a0, wa, wb, a1, lo, hi);
        if constexpr (LAST) {
            if (P.apply_scale) {  // uniform branch: no predicated multiplies when unscaled
                lo = cscale(lo, f);
                hi = cscale(hi, f);
            }
            st_stream(dst + p * n + j, lo);
            st_stream(dst + p * n + j + Lt, hi);
        } else {
            dst[p * 2 * Lt + j] = lo;
            dst[p * 2 * Lt + j + Lt] = hi;
        }
    }
}

// Radix-4 pass (levels t -> t + 2): per (position p, node j < 2^t) the four level-t
// nodes at p + c s_{t+2}, c = 0..3, give the level-(t+1) nodes j, j + 2^t at p and
// p + s_{t+2} and then the four level-(t+2) nodes j + u 2^t at p — the same butterflies
// as two row_level_step levels, the middle level kept in registers.
template <typename T, bool EXACT, int M1, int TPOS, int t, bool LAST>
__device__ __forceinline__ void kr_pass4(const cplx<T> *src, cplx<T> *dst, const cplx<T> *stw,
                                         int npos, const KRParams &P) {
    using C = cplx<T>;
    constexpr int n = 1 << M1, Lt = 1 << t, s2 = n >> (t + 2);
    constexpr int cnt = LAST ? TPOS : TPOS + s2 - 1;
    const int items = (LAST ? npos : cnt) * Lt;
    const int j = threadIdx.x & (Lt - 1);  // Lt <= 256 = blockDim: fixed per thread
    // Omega_n[k] = stw[k]: level t+1 node i uses k = i s_{t+1}, level t+2 k = i s_{t+2}
    const C w1a = stw[j << (M1 - 1 - t)], w1b = stw[(j + Lt) << (M1 - 1 - t)];
    C w2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w2[u] = stw[(j + u * Lt) << (M1 - 2 - t)];
    const T f = (T)P.scale;
    for (int it = threadIdx.x; it < items; it += KR_THREADS) {
        const int p = it >> t;
        const C a0 = src[p * Lt + j], a1 = src[(p + s2) * Lt + j];
        const C a2 = src[(p + 2 * s2) * Lt + j], a3 = src[(p + 3 * s2) * Lt + j];
        C b0, b1, c0, c1, o[4];
        bfly_pair<EXACT>(a0, w1a, w1b, a2, b0, b1);  // level t+1 at p
        bfly_pair<EXACT>(a1, w1a, w1b, a3, c0, c1);  // at p + s_{t+2}
        bfly_pair<EXACT>(b0, w2[0], w2[2], c0, o[0], o[2]);
        bfly_pair<EXACT>(b1, w2[1], w2[3], c1, o[1], o[3]);
        if constexpr (LAST) {
            C *d = dst + p * n + j;
            if (P.apply_scale) {  // uniform branch: no predicated multiplies when unscaled
#pragma unroll
                for (int u = 0; u < 4; ++u) st_stream(d + u * Lt, cscale(o[u], f));
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) st_stream(d + u * Lt, o[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) dst[p * 4 * Lt + j + u * Lt] = o[u];
        }
    }
}

template <typename T, bool EXACT, int M1>
__global__ void __launch_bounds__(KR_THREADS) kr_rows_kernel(const __grid_constant__ KRParams P) {
    using C = cplx<T>;
    constexpr int n = 1 << M1, TPOS = kr_tpos<T, M1>();
    constexpr int W = TPOS + n - 1;
    constexpr int NPRE = (W + KR_THREADS - 1) / KR_THREADS;
    extern __shared__ __align__(16) unsigned char kr_smem[];
    C *bufA = reinterpret_cast<C *>(kr_smem);
    C *bufB = bufA + kr_buf<M1, TPOS>(0);
    C *stw = bufB + kr_buf<M1, TPOS>(1);  // Omega_n[k], k < n (make_twiddles(1024), stride 1024/n)
    for (int k = threadIdx.x; k < n; k += KR_THREADS)
        stw[k] = __ldg(static_cast<const C *>(P.tw) + (k << (10 - M1)));

    // persistent CTAs over tiles (row, TPOS window positions); the next tile's samples
    // are loaded into registers while the current tile's passes run
    const int64_t tiles_per_row = (P.P1 + TPOS - 1) / TPOS;
    const int64_t ntiles = (P.p0_end - P.p0_begin) * tiles_per_row;
    C pre[NPRE];
    auto fetch = [&](int64_t tile) {
        const int64_t row = tile / tiles_per_row;
        const int64_t q0 = (tile - row * tiles_per_row) * TPOS;
        const int64_t xrow = (P.p0_begin + row) * P.ldx;
#pragma unroll
        for (int r = 0; r < NPRE; ++r) {
            const int p = threadIdx.x + r * KR_THREADS;
            pre[r] = (p < W && q0 + p < P.N1) ? load_raw<T>(P.x, P.in_dtype, xrow + q0 + p)
                                              : mk<T>((T)0, (T)0);
        }
    };
    int64_t tile = blockIdx.x;
    if (tile < ntiles) fetch(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t row = tile / tiles_per_row;
        const int64_t q0 = (tile - row * tiles_per_row) * TPOS;
        const int npos = (int)(P.P1 - q0 < TPOS ? P.P1 - q0 : TPOS);
        C *out = static_cast<C *>(P.out) + (row * P.P1 + q0) * n;
#pragma unroll
        for (int r = 0; r < NPRE; ++r) {  // level 0: samples x[row, q0 .. q0 + W)
            const int p = threadIdx.x + r * KR_THREADS;
            if (p < W) bufA[p] = from_raw<T>(pre[r], P.in_dtype);
        }
        if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
        __syncthreads();
        if constexpr (M1 == 0) {
            const T f = (T)P.scale;
            for (int p = threadIdx.x; p < npos; p += KR_THREADS)
                st_stream(out + p, P.apply_scale ? cscale(bufA[p], f) : bufA[p]);
        } else if constexpr (M1 == 1) {
            kr_pass2<T, EXACT, M1, TPOS, 0, true>(bufA, out, stw, npos, P);
        } else {
            constexpr int T0 = M1 % 2;  // odd m: one radix-2 pass first
            C *src = bufA, *dst = bufB;
            if constexpr (T0 == 1) {
                kr_pass2<T, EXACT, M1, TPOS, 0, false>(src, dst, stw, npos, P);
                __syncthreads();
                src = bufB;
                dst = bufA;
            }
            static_for<(M1 - T0) / 2>([&](auto kc) {
                constexpr int t = T0 + 2 * decltype(kc)::value;
                if constexpr (t + 2 == M1) {
                    kr_pass4<T, EXACT, M1, TPOS, t, true>(src, out, stw, npos, P);
                } else {
                    kr_pass4<T, EXACT, M1, TPOS, t, false>(src, dst, stw, npos, P);
                    __syncthreads();
                    C *tmp = src;
                    src = dst;
                    dst = tmp;
                }
            });
        }
        __syncthreads();  // the next tile overwrites bufA
    }
}

// CTAs per SM of one KR instantiation on the current device (cached).
static int kr_occupancy(const void *fn, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(dev, fn);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, KR_THREADS, smem) != cudaSuccess)
        occ = 0;
    cache[key] = occ;
    return occ;
}

template <typename T, bool EXACT, int M1>
static int kr_launch_t(const KRParams &P, cudaStream_t st) {
    constexpr int TPOS = kr_tpos<T, M1>();
    constexpr size_t smem =
        sizeof(cplx<T>) * (kr_buf<M1, TPOS>(0) + kr_buf<M1, TPOS>(1) + (1 << M1));
    const int64_t tiles = (P.p0_end - P.p0_begin) * ((P.P1 + TPOS - 1) / TPOS);
    if (tiles == 0) return 0;
    auto fn = &kr_rows_kernel<T, EXACT, M1>;
    if (smem > 48 * 1024 &&  // per device, so set on every launch (cheap)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return -2;
    const int occ = kr_occupancy((const void *)fn, smem);
    if (occ < 1) return -2;
    const int64_t slots = (int64_t)P.sms * occ;
    // One CTA per tile (hardware-scheduled, short-lived CTAs) when the tiles fill >= 3
    // waves and the window is <= 256: n = 64..256 write at 6.8-7.2 TB/s instead of
    // 5.9-6.4 as a persistent grid (fp32; fp64 6.4-7.1 vs 5.9-6.4), n = 16 +2 %.  Windows
    // of 512-1024 keep the persistent grid: their tiles are 16-32 positions with a
    // 511-1023-sample halo, which the persistent grid prefetches behind the previous tile
    // (one-shot: n = 1024 5.56 -> 4.82 TB/s).  profiles/bench_1d_r01.jsonl.
    // SWDFT2D_KR_ONESHOT=0/1 forces either grid.
    static const int force = [] {
        const char *e = std::getenv("SWDFT2D_KR_ONESHOT");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool oneshot = force >= 0 ? force == 1 : (M1 <= 8 && tiles >= 3 * slots);
    const int64_t grid = (oneshot || tiles < slots) ? tiles : slots;
    fn<<<(unsigned)grid, KR_THREADS, smem, st>>>(P);
    return 0;
}

template <typename T, bool EXACT>
static int kr_dispatch(const KRParams &P, int m1, cudaStream_t st) {
    switch (m1) {
    case 0: return kr_launch_t<T, EXACT, 0>(P, st);
    case 1: return kr_launch_t<T, EXACT, 1>(P, st);
    case 2: return kr_launch_t<T, EXACT, 2>(P, st);
    case 3: return kr_launch_t<T, EXACT, 3>(P, st);
    case 4: return kr_launch_t<T, EXACT, 4>(P, st);
    case 5: return kr_launch_t<T, EXACT, 5>(P, st);
    case 6: return kr_launch_t<T, EXACT, 6>(P, st);
    case 7: return kr_launch_t<T, EXACT, 7>(P, st);
    case 8: return kr_launch_t<T, EXACT, 8>(P, st);
    case 9: return kr_launch_t<T, EXACT, 9>(P, st);
    case 10: return kr_launch_t<T, EXACT, 10>(P, st);
    default: return -3;
    }
}

int launch_kr(const KRParams &P, int m1, int prec, cudaStream_t stream) {
    return prec == 1 ? kr_dispatch<double, true>(P, m1, stream)
                     : kr_dispatch<float, false>(P, m1, stream);
}

}  // namespace swdft2d
