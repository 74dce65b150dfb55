// k1_stream.cuh — K1, the fused row-streaming 2D tree SWDFT kernel for sm_100a.
//
// The reference computes the tree levels-outer over a double-buffered
// [N0, N1, n0, n1] lattice (tree2d.py:30-129): every level is a full pass over
// HBM-sized slabs.  The tree factorises exactly:
//   stage R  (tree levels 1..m1, dim 1, row_level_step tree2d.py:72-93)
//            Z[r, p1, k1] = n1-point DIT transform of x[r, p1 : p1+n1]
//   stage C  (tree levels m1+1..m1+m0, dim 0, col_level_step tree2d.py:96-120)
//            a[p0, p1, k0, k1] = 1D tree along rows of the column Z[:, p1, k1]
// K1 streams each CTA down a strip of input rows, so no tree level ever
// reaches HBM: only the final coefficients are written (the HBM-write
// roofline of the path).
//
// CTA = TP1 consecutive window columns x all n1 frequencies k1 x J "k0
// residue groups".  Thread (k1, j, pos) owns column (pos, k1) and the output
// frequencies k0 = j + J*u.  The grid walks (column block, row chunk) tiles —
// persistent CTAs with uniform or guided (big-first, atomic counter) chunks, or, for
// 64-row windows with many column blocks, one CTA per full-height column block
// (abi.cu) — and each tile is processed in batches of NB input rows:
//   0. input: the batch's NB x (TP1 + n1 - 1) samples arrive either by per-lane
//      loads issued one batch ahead into registers (default), or (TMA=true) as a
//      cp.async.bulk.tensor tile in a 4-stage shared-memory ring with mbarriers.
//   1. stage R: the warps split the NB x TP1 row transforms; each transform
//      is an n1-point radix-2 DIT on G = min(n1, 32) lanes (V = n1/G values
//      per lane) with warp shuffles for the level exchanges, written into a
//      shared-memory ring Z (D >= n0 - n0/J + NB rows; every row stored twice,
//      at slot and slot + D, so stage C reads at constant offsets).
//   2. __syncthreads
//   3. stage C, per row: the thread rebuilds the level-Q node j of its column
//      tree from J ring rows (2^Q - 1 butterflies, the reference DAG), then
//      advances levels Q+1..m0 with the tree's reuse along p0: the level l-1
//      node of the tree s_l rows back (tree2d.py:110) comes from a register
//      ring, so each row costs 2(n0/J - 1) butterflies per thread.  The n0/J
//      finished coefficients are written with streaming (evict-first) stores;
//      consecutive lanes hold consecutive k1, so each warp store is a
//      contiguous 256-byte (complex64) run of the [P0, P1, n0, n1] output.  The
//      output address is a running row pointer and the scale a uniform branch, so a
//      row's epilogue is a handful of instructions.
//   4. __syncthreads (ring slots are recycled by the next batch's stage R)
//
// EXACT (fp64) instantiations use the reference's operand roles and rounding
// order for every node (core.py:238-245 via bfly_exact, the node's own
// twiddle Omega[i*s] — no +-w pair symmetry, which is not bitwise,
// SURVEY.md App. A #3), so they reproduce tree_swdft_2d bit for bit.  The fp32
// instantiations use FMAs and the pair symmetry w[i + L/2] = -w[i].
#pragma once

#include <type_traits>
#include <utility>

#include <cuda.h>

#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"

namespace swdft2d {

#ifdef K1_TIMELINE  // tuning builds: per-CTA start / end / SM id of the last K1 launch
__device__ unsigned long long g_k1_timeline[8192][3];
#endif

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <int M0, int M1, int Q, int TP1, int NBM = 1> struct K1Shape {
    static constexpr int n0 = 1 << M0, n1 = 1 << M1, J = 1 << Q;
    static constexpr int NT = n1 * J * TP1;               // threads per CTA
    static constexpr int WARPS = NT / 32;
    static constexpr int NB = cmax(n0 / J, 4) * NBM;      // rows per batch
    static constexpr int D = pow2ceil(n0 - n0 / J + NB);  // Z ring depth (rows)
    static constexpr int G = cmin(n1, 32);                // lanes per row transform
    static constexpr int V = n1 / G;                      // values per lane
    static constexpr int GW = 32 / G;                     // transforms per warp task
    static constexpr int TPR = (TP1 + GW - 1) / GW;       // warp tasks per row
    // n1 > 32: after the in-register level(s) the V slots evolve independently, so a
    // row transform splits into V warp tasks (one slot each) to spread stage R evenly
    static constexpr int SPLIT = V > 1 ? V : 1;
    static constexpr int TASKS = NB * TPR * SPLIT;
    static constexpr int TPW = (TASKS + WARPS - 1) / WARPS;
    static constexpr int NMAX = cmax(n0, n1);
    static constexpr int RING = cmax((M0 - Q) * (n0 / (2 * J)), 1);  // register ring, complex
    static constexpr int OUTS = n0 / J;                   // coefficients per thread per row
    static constexpr int UNR = cmin(cmax(n0 / (2 * J), 8), NB);  // stage-C rows per unrolled block
    // TMA staging: NSTAGE stages x NB rows x (TP1 + n1 - 1) samples of <= 16 B, plus up
    // to 16 B in front (the box starts on a 16-B aligned column), rows 16-B padded
    static constexpr int STAGE_ROW_MAX = ((TP1 + n1 - 1) * 16 + 15) / 16 * 16 + 16;
    static constexpr int STAGE_SPAN = (NB * STAGE_ROW_MAX + 127) / 128 * 128;  // 128-B aligned
    static constexpr int NSTAGE = 4;  // TMA tiles in flight: batch b loads while b-3 computes
    static constexpr int STAGE_BYTES = NSTAGE * STAGE_SPAN;
    static_assert(Q <= M0, "J must divide n0");
    static_assert(NT % 32 == 0 && NT <= 1024, "CTA size must be a warp multiple <= 1024");
};

template <typename T, int M0, int M1, int Q, int TP1, int NBM = 1, bool TMA = false>
constexpr size_t k1_smem_bytes() {
    using S = K1Shape<M0, M1, Q, TP1, NBM>;
    return (TMA ? (size_t)S::STAGE_BYTES : 0) +
           sizeof(cplx<T>) * ((size_t)2 * S::D * TP1 * S::n1 + S::NMAX);
}

template <typename C> __device__ __forceinline__ void k1_store(C *p, C v) {
#if defined(K1_DRY)  // tuning builds: no stores (the address test cannot be proven false)
    if (reinterpret_cast<uintptr_t>(p) == 1) *p = v;
#elif defined(K1_PLAIN_STORES)  // tuning builds: default-policy stores instead of evict-first
    *p = v;
#else
    st_stream(p, v);
#endif
}

template <typename T, int M0, int M1, int Q, int TP1, bool EXACT, int MINB = 1, int NBM = 1,
          bool TMA = false, bool COLZ = false, int IND = -1>
__global__ void __launch_bounds__(K1Shape<M0, M1, Q, TP1, NBM>::NT, MINB)
    k1_stream_kernel(const __grid_constant__ K1Params P, const __grid_constant__ CUtensorMap tmap) {
    static_assert(!COLZ || (M1 == 0 && !TMA), "the Z-column variant is a 1-column LDG kernel");
    using S = K1Shape<M0, M1, Q, TP1, NBM>;
    using C = cplx<T>;
    constexpr int n0 = S::n0, n1 = S::n1, J = S::J, NB = S::NB, D = S::D;
    constexpr int G = S::G, V = S::V, GW = S::GW, TPR = S::TPR, NMAX = S::NMAX;
    constexpr int ST0 = NMAX / n0, ST1 = NMAX / n1;  // table strides (exact, App. A #4)

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *stage = smem_raw;  // TMA: NSTAGE x [NB][row] input tiles (128-B aligned)
    // Z ring [2D][TP1][n1]: row r is stored at slot r mod D and again at slot + D, so the
    // J rows stage C reads (r - t*n0/J) sit at constant offsets below slot + D
    C *ring = reinterpret_cast<C *>(smem_raw + (TMA ? S::STAGE_BYTES : 0));
    C *tw = ring + 2 * D * TP1 * n1;  // make_twiddles(NMAX)
    __shared__ __align__(8) uint64_t mbar[S::NSTAGE];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef K1_TIMELINE
    if (tid == 0 && blockIdx.x < 8192) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_k1_timeline[blockIdx.x][0] = t;
        g_k1_timeline[blockIdx.x][2] = smid;
    }
    struct TimelineEnd {
        __device__ ~TimelineEnd() {
            if (threadIdx.x == 0 && blockIdx.x < 8192) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                g_k1_timeline[blockIdx.x][1] = t;
            }
        }
    } timeline_end;
#endif
    // input element type: a compile-time constant in the IND >= 0 variants (the per-sample
    // dtype switch folds away), else the launch's
    const int in_dtype = IND >= 0 ? IND : P.in_dtype;
    for (int i = tid; i < NMAX; i += S::NT) {
        const double2 w = P.tw[i * (K0_TW_N / NMAX)];
        tw[i] = mk<T>((T)w.x, (T)w.y);
    }
    if constexpr (TMA) {
        if (tid == 0) {
            for (int i = 0; i < S::NSTAGE; ++i) mbar_init(&mbar[i], 1);
            fence_mbar_init();
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
        }
    }
    __syncthreads();
    // TMA: one elected thread loads batch gb's [NB x box] input tile into stage gb % NSTAGE
    uint32_t gb = 0;  // batches processed by this CTA (mbarrier phase bookkeeping)
    // The box's first column must sit on a 16-byte boundary of the row (measured: an
    // unaligned inner coordinate faults), so it starts `shift` samples left of pbase.
    auto tma_shift = [&](int64_t pbase) {
        return (int)(((pbase * P.sample_bytes) & 15) / P.sample_bytes);
    };
    auto tma_issue = [&](uint32_t g, int64_t brow, int64_t pbase) {
        const int st = (int)(g % S::NSTAGE);
        mbar_expect_tx(&mbar[st], (uint32_t)(NB * P.tma_row_bytes));
        tma_load_2d(stage + st * S::STAGE_SPAN, &tmap, &mbar[st],
                    (int)((pbase - tma_shift(pbase)) * P.tma_per_sample), (int)brow);
    };

    // stage C identity: column (pos, k1), output residue j.  COLZ (the large-window path's
    // column trees, abi.cu forward_separable): the 1-column kernel runs over the stage-R
    // rows Z, whose column c is (p1, k1) = (c >> col_m1, c mod 2^col_m1) of the real
    // window; consecutive lanes take consecutive columns, i.e. consecutive k1 of the
    // output [p0][p1][k0][k1] (coalesced stores)
    const int k1 = tid % n1;
    const int j = COLZ ? tid / TP1 : (tid / n1) % J;
    const int pos = COLZ ? tid % TP1 : tid / (n1 * J);
    // stage R identity: lane lam of transform group gam
    const int gam = lane / G, lam = lane % G;

    C rring[S::RING];  // level l-1 nodes of the last s_l rows, levels Q+1..m0
    C cur[S::OUTS];
#pragma unroll
    for (int q = 0; q < S::RING; ++q) rring[q] = mk<T>(0, 0);

    __shared__ int64_t s_next;
    // stream-K: this CTA's share [lin, lin_end) of the column-block-major space in COST
    // units — each column block is its n0 - 1 warm-up rows followed by its window rows —
    // so a share that crosses into the next column block pays for that block's warm-up
    // out of its share, and every CTA costs its share plus at most one warm-up of its own
    // (kept in shared memory: the share cursor is CTA-uniform, and in registers it cost the
    // largest fp64 instantiations a spill)
    __shared__ int64_t s_lin, s_lin_end;
    if (P.streamk && tid == 0) {
        const int64_t L = P.CB * (P.p0_end - P.p0_begin + (n0 - 1));
        s_lin = (int64_t)blockIdx.x * L / gridDim.x;
        s_lin_end = (int64_t)(blockIdx.x + 1) * L / gridDim.x;
    }
    __syncthreads();
    for (int64_t tile = blockIdx.x;;) {
        int64_t cb, r0, r1;  // column block, output rows [r0, r1)
        if (P.streamk) {
            const int64_t lin = s_lin, lin_end = s_lin_end;
            if (lin >= lin_end) break;
            const int64_t U = P.p0_end - P.p0_begin + (n0 - 1);
            cb = lin / U;
            const int64_t cend = (cb + 1) * U;
            const int64_t se = lin_end < cend ? lin_end : cend;
            const int64_t a = lin - cb * U - (n0 - 1), e = se - cb * U - (n0 - 1);
            __syncthreads();  // every thread has read the cursor
            if (tid == 0) s_lin = se;
            if (e <= 0) {  // the share ends inside this block's warm-up: no rows
                __syncthreads();
                continue;
            }
            r0 = P.p0_begin + (a > 0 ? a : 0);
            r1 = P.p0_begin + e;
        } else {
            if (tile >= P.ntiles) break;
            cb = tile % P.CB;
            const int64_t rc = tile / P.CB;
            if (P.nchunks > 0) {
                r0 = P.p0_begin + P.chunk[rc];
                r1 = P.p0_begin + P.chunk[rc + 1];
            } else {
                r0 = P.p0_begin + rc * P.RCH;
                r1 = r0 + P.RCH < P.p0_end ? r0 + P.RCH : P.p0_end;
            }
        }
        const int64_t pbase = cb * TP1;
        const int64_t in_end = r1 + n0 - 1;                         // input rows [r0, in_end)
        const int nbatch = (int)((in_end - r0 + NB - 1) / NB);
        // Output addressing, kept off the per-row critical path: a running pointer to
        // the output row of tile row `rel` (advanced by one output row per stage-C row;
        // rows before the first window row are never dereferenced) and int32 bounds for
        // the rows that emit: rel in [n0 - 1, rel_hi)
        const int64_t ostride = P.P1 * (int64_t)(n0 * n1);
        C *orow = reinterpret_cast<C *>(P.out) + (pbase + pos) * (int64_t)(n0 * n1) + k1 +
                  (r0 - (n0 - 1) - P.p0_begin) * ostride;
        if constexpr (COLZ) {  // column c = (p1, k1), k0 at stride 2^col_m1; k0 = j first
            const int64_t c = pbase + pos;
            orow = reinterpret_cast<C *>(P.out) +
                   ((((c >> P.col_m1) * n0) + j) << P.col_m1) + (c & ((1LL << P.col_m1) - 1)) +
                   (r0 - (n0 - 1) - P.p0_begin) * ostride;
        }
        const int rel_hi = pbase + pos < P.P1 ? (int)(r1 - r0) + n0 - 1 : 0;

        // Input samples of this warp's stage-R tasks for one batch, prefetched one
        // batch ahead so the global-load latency hides behind stage C.
        C xs[S::TPW][V];
        auto load_batch = [&](int bb) {
            const int64_t brow = r0 + (int64_t)bb * NB;
#pragma unroll
            for (int tt = 0; tt < S::TPW; ++tt) {
                const int task = warp + tt * S::WARPS;
                const int t2 = task / S::SPLIT;
                const int rr = t2 / TPR, pg = t2 - rr * TPR;
                const int64_t row = brow + rr;
                const int64_t pcol = pbase + pg * GW + gam;
#pragma unroll
                for (int a = 0; a < V; ++a) {
                    const int64_t col = pcol + lam + G * a;
                    xs[tt][a] = ((S::TASKS % S::WARPS) == 0 || task < S::TASKS) && row < in_end &&
                                        col < P.N1
                                    ? load_raw<T>(P.x, in_dtype, row * P.ldx + col)
                                    : mk<T>(0, 0);
                }
            }
        };
        const int tsh = TMA ? tma_shift(pbase) : 0;  // staged column of window column pbase
        if constexpr (TMA) {
            if (tid == 0)
                for (int i = 0; i < S::NSTAGE - 1 && i < nbatch; ++i)
                    tma_issue(gb + i, r0 + (int64_t)i * NB, pbase);
        } else {
            load_batch(0);
        }

        for (int b = 0; b < nbatch; ++b, ++gb) {
            if constexpr (TMA) {
                if (tid == 0 && b + S::NSTAGE - 1 < nbatch)
                    tma_issue(gb + S::NSTAGE - 1, r0 + (int64_t)(b + S::NSTAGE - 1) * NB, pbase);
                mbar_wait(&mbar[gb % S::NSTAGE], (gb / S::NSTAGE) & 1);
            }
            // ---------------- stage R: row transforms of NB rows into the ring
#pragma unroll
            for (int tt = 0; tt < S::TPW; ++tt) {
                const int task = warp + tt * S::WARPS;
                if ((S::TASKS % S::WARPS) == 0 || task < S::TASKS) {
                    const int t2 = task / S::SPLIT, bsl = task - t2 * S::SPLIT;  // slot (V > 1)
                    const int rr = t2 / TPR, pg = t2 - rr * TPR;
                    const int pl = pg * GW + gam;
                    C s[V];
                    if constexpr (TMA) {
                        const unsigned char *rowp =
                            stage + (gb % S::NSTAGE) * S::STAGE_SPAN + rr * P.tma_row_bytes;
#pragma unroll
                        for (int a = 0; a < V; ++a)
                            s[a] = load_staged<T>(rowp + (tsh + pl + lam + G * a) * P.sample_bytes,
                                                  in_dtype);
                    } else {
#pragma unroll
                        for (int a = 0; a < V; ++a) s[a] = from_raw<T>(xs[tt][a], in_dtype);
                    }
                    // in-register levels (n1 > 32): classes c = lam + G*a
#pragma unroll
                    for (int L = 2; L <= V; L *= 2) {
                        C ns[V];
#pragma unroll
                        for (int a = 0; a < V / L; ++a)
#pragma unroll
                            for (int i = 0; i < L; ++i) {
                                const int ip = i % (L / 2);
                                ns[a * L + i] = bfly<EXACT>(s[a * (L / 2) + ip],
                                                            tw[i * (n1 / L) * ST1],
                                                            s[(a + V / L) * (L / 2) + ip]);
                            }
#pragma unroll
                        for (int a = 0; a < V; ++a) s[a] = ns[a];
                    }
                    // this task's slot (all V slots when the transform is not split)
                    C sv = s[0];
#pragma unroll
                    for (int a = 1; a < V; ++a)
                        if (bsl == a) sv = s[a];
                    // cross-lane levels: node (c, i) of slot be sits on lane (i/V)*(n1/L) + c
#pragma unroll
                    for (int L = 2 * V; L <= n1; L *= 2) {
                        const int sL = n1 / L;
                        const int c = lam % sL;
                        const int i = (lam / sL) * V + bsl;
                        const int ip = i % (L / 2);
                        const int srcE = gam * G + (ip / V) * (2 * sL) + c;
                        const int srcO = srcE + sL;
                        C E, O;
                        E.x = __shfl_sync(0xffffffffu, sv.x, srcE);
                        E.y = __shfl_sync(0xffffffffu, sv.y, srcE);
                        O.x = __shfl_sync(0xffffffffu, sv.x, srcO);
                        O.y = __shfl_sync(0xffffffffu, sv.y, srcO);
                        sv = bfly<EXACT>(E, tw[i * sL * ST1], O);
                    }
                    if (pl < TP1) {
                        C *dst = ring + ((b * NB + rr) & (D - 1)) * (TP1 * n1) + pl * n1 +
                                 lam * V + bsl;
                        dst[0] = sv;
                        dst[D * TP1 * n1] = sv;
                    }
                }
            }
            __syncthreads();
            if constexpr (!TMA) {
                if (b + 1 < nbatch) load_batch(b + 1);
            }
            // ---------------- stage C: column trees, NB rows, UNR rows per unrolled block
            // (UNR is a multiple of every register-ring depth, so ring slots are static)
            // this batch's first slot + D: NB divides D, so batch rows never wrap
            const C *zb = ring + (((b * NB) & (D - 1)) + D) * (TP1 * n1) + pos * n1 + k1;
#pragma unroll 1
            for (int k0r = 0; k0r < NB; k0r += S::UNR) {
                // Warm-up rows whose column-tree nodes no emitted row depends on: the
                // level-l node of tile row rel feeds emitted rows (rel >= n0 - 1) only if
                // rel >= n0 - n0/2^l, and stage C starts at level Q (rebuilt from the Z
                // ring), so rows rel < n0 - n0/J need no stage C at all — only their Z rows
                // (stage R above).  Later rows read the register ring only for such unused
                // nodes, so skipping changes no emitted value (fp64 stays bitwise).
                if (b * NB + k0r + S::UNR <= n0 - n0 / J) {
                    orow += S::UNR * ostride;
                    continue;
                }
                const C *zr = zb + k0r * (TP1 * n1);
                static_for<S::UNR>([&](auto kuc) {
                    constexpr int ku = decltype(kuc)::value;
                    const int rel = b * NB + k0r + ku;
                    C v[J];
                    static_for<J>([&](auto tc) {
                        constexpr int t = decltype(tc)::value;
                        v[t] = zr[(ku - t * (n0 / J)) * (TP1 * n1)];
                    });
                    // levels 1..Q: node j of this row's tree (the reference DAG, tree2d.py:109-112)
                    static_for<Q>([&](auto lc) {
                        constexpr int l = decltype(lc)::value + 1;
                        const C w = tw[((j & ((1 << l) - 1)) * (n0 >> l)) * ST0];
                        static_for<(1 << (Q - l))>([&](auto tc) {
                            constexpr int t = decltype(tc)::value;
                            v[t] = bfly<EXACT>(v[t + (1 << (Q - l))], w, v[t]);
                        });
                    });
                    cur[0] = v[0];
                    // levels Q+1..m0, reusing the tree s_l rows back (register ring)
                    static_for<M0 - Q>([&](auto lc) {
                        constexpr int l = decltype(lc)::value + Q + 1;
                        constexpr int sl = n0 >> l, h = 1 << (l - 1 - Q);
                        constexpr int off = (l - Q - 1) * (n0 / (2 * J)) + (ku % sl) * h;
                        static_for<h>([&](auto uc) {
                            constexpr int u = decltype(uc)::value;
                            const C E = rring[off + u];
                            const C O = cur[u];
                            const int i = j + J * u;
                            const C w0 = tw[(i * sl) * ST0];
                            // the node pair i, i + 2^(l-1): exact butterflies with their own
                            // twiddles in fp64; E + wO and 2E - (E + wO) in fp32
                            bfly_pair<EXACT>(E, w0, tw[((i + (1 << (l - 1))) * sl) * ST0], O, cur[u],
                                             cur[u + h]);
                            rring[off + u] = O;
                        });
                    });
                    // emit window row p0 = r0 + rel - (n0 - 1); the scale test is a uniform
                    // branch (predicated multiplies would cost issue slots on every row)
                    if (COLZ && rel >= n0 - 1 && rel < rel_hi) {
                        // outputs k0 = j + J u at stride J 2^col_m1: a bumped pointer
                        // (a runtime stride per u would hold OUTS 64-bit addresses)
                        const int64_t ustep = (int64_t)J << P.col_m1;
                        C *o = orow;
                        if (P.apply_scale) {
                            const T f = (T)P.scale;
                            static_for<S::OUTS>([&](auto uc) {
                                constexpr int u = decltype(uc)::value;
                                k1_store(o, cscale(cur[u], f));
                                o += ustep;
                            });
                        } else {
                            static_for<S::OUTS>([&](auto uc) {
                                constexpr int u = decltype(uc)::value;
                                k1_store(o, cur[u]);
                                o += ustep;
                            });
                        }
                    } else if (!COLZ && rel >= n0 - 1 && rel < rel_hi) {
                        if (P.apply_scale) {
                            const T f = (T)P.scale;
                            static_for<S::OUTS>([&](auto uc) {
                                constexpr int u = decltype(uc)::value;
                                k1_store(orow + (j + J * u) * n1, cscale(cur[u], f));
                            });
                        } else {
                            static_for<S::OUTS>([&](auto uc) {
                                constexpr int u = decltype(uc)::value;
                                k1_store(orow + (j + J * u) * n1, cur[u]);
                            });
                        }
                    }
                    orow += ostride;
                });
            }
            __syncthreads();
        }
        if (P.counter) {  // guided: the next tile from the shared counter (after the first wave)
            // A launch makes exactly ntiles fetches (ntiles - grid real tiles, then one
            // terminating fetch per CTA), so the fetch that returns ntiles - 1 is the last
            // one: it zeroes the counter for the next launch on this stream (the counter is
            // a per-(device, stream) slot allocated once, abi.cu k1_counter).
            if (tid == 0) {
                const unsigned long long v = atomicAdd(P.counter, 1ull);
                if (v == (unsigned long long)(P.ntiles - 1)) atomicExch(P.counter, 0ull);
                s_next = (int64_t)v + gridDim.x;
            }
            __syncthreads();
            tile = s_next;
        } else {
            tile += gridDim.x;
        }
    }
}

// Per-instantiation launcher + registry entry.
template <typename T, int M0, int M1, int Q, int TP1, bool EXACT, int MINB = 1, int NBM = 1,
          bool TMA = false, bool COLZ = false, int IND = -1>
int k1_launch(const K1Params &P, const CUtensorMap &tmap, int grid, cudaStream_t stream) {
    using S = K1Shape<M0, M1, Q, TP1, NBM>;
    constexpr size_t smem = k1_smem_bytes<T, M0, M1, Q, TP1, NBM, TMA>();
    k1_stream_kernel<T, M0, M1, Q, TP1, EXACT, MINB, NBM, TMA, COLZ, IND>
        <<<grid, S::NT, smem, stream>>>(P, tmap);
    return 0;
}

// Registry entry for an explicit shape (used by K1Inst and by the tuning harness).
// Variant index: 0 LDG input (runtime input dtype), 1 TMA input, 2 the Z-column kernel
// (COLZ), 3 LDG with float32 input as a compile-time constant (IND = 0).
template <typename T, int M0, int M1, int Q, int TP1, bool EXACT, int MINB = 1, int NBM = 1,
          bool TMA = false, bool COLZ = false, int IND = -1>
const K1Info *k1_info() {
    using S = K1Shape<M0, M1, Q, TP1, NBM>;
    static const K1Info info = {
        M0, M1, EXACT ? 1 : 0, Q, TP1, S::NT, S::NB, COLZ ? 2 : TMA ? 1 : IND == 0 ? 3 : 0,
        k1_smem_bytes<T, M0, M1, Q, TP1, NBM, TMA>(),
        (const void *)&k1_stream_kernel<T, M0, M1, Q, TP1, EXACT, MINB, NBM, TMA, COLZ, IND>,
        &k1_launch<T, M0, M1, Q, TP1, EXACT, MINB, NBM, TMA, COLZ, IND>};
    return &info;
}

// Shape per (m0, m1): J = 2^Q residue groups so that each thread emits n0/J = 4
// coefficients per row (Q = m0 - 2, at most 3: the level-Q chain costs 2^Q - 1
// butterflies per row), capped at 512 threads per window column; TP1 window columns
// per CTA so that a CTA is ~128 threads.  Shapes where the sweep over all windows
// 4..64 x 4..64 (profiles/SWEEP_r01.md) found a >3 % faster (Q, TP1) use that instead
// (fp32).  fp64-exact (DBL) butterflies cost ~2x and run without FMA: the fp64 sweep
// picked Q = 2 for m0 = 3..5 (c3 in fp64: 369 Gcoef/s at Q=2 vs 243 at Q=3; 8x8: 317
// vs 292 at Q=1).
struct K1Choice {
    int m0, m1, q, tp1, minb = 1;  // minb: __launch_bounds__ min CTAs per SM (register cap)
};
// Re-tuned after the leaner K1 epilogue: the full window sweep of profiles/sweep_r01b.jsonl
// (every (Q, TP1) around the rule, windows 4..64 x 4..64) and, for configs 2-4,
// profiles/tune_r01_f.jsonl.  With the cheaper per-row epilogue, 32-row windows prefer
// Q = 2 over 3 (32x16: 574 -> 865 Gcoef/s, 32x32: 552 -> 860, 32x8 / config 3: 808 -> 857);
// 16x16 runs with a 5-CTA register cap (config 2 0.0902 vs 0.0922 ms, config 4 level).
// 256-row windows (m0 = 8, fp32 only) take Q = 4 so their register ring stays at 32 complex.
// 64x64 (config 5) takes Q = 2 (256 threads, 244 registers, one CTA per SM like Q = 3's 512)
// since the warm-up skip: 19.60 -> 19.09 ms and 20.68 -> 20.08 in two passes
// (profiles/tune_r02_c5.jsonl; config 5 runs at the 1000 W software power cap).
constexpr K1Choice K1_TUNED_FP32[] = {
    {2, 2, 1, 8},  {2, 3, 0, 32}, {3, 2, 2, 8}, {3, 4, 1, 4}, {4, 2, 2, 16}, {4, 3, 2, 8},
    {4, 4, 2, 2, 5}, {4, 6, 1, 1}, {5, 2, 3, 8}, {5, 3, 2, 4}, {5, 4, 2, 2},  {5, 5, 2, 1},
    {5, 6, 2, 1},  {6, 2, 3, 2},  {6, 3, 3, 2}, {6, 4, 3, 1}, {6, 5, 3, 1}, {6, 6, 2, 1},
    {8, 0, 4, 8},  {8, 1, 4, 4},  {8, 2, 4, 2},  {9, 0, 5, 4},  {9, 1, 5, 2},
};
// fp64 (exact) from the fp64 window sweep (profiles/sweep64_r01c.jsonl): the rule's
// choice wherever it is within ~3 % of the best, else the best — e.g. 16x64 292 -> 336,
// 4x16 320 -> 354 Gcoef/s; 64x64 takes Q = 2 (256 threads, +2 %; like Q = 3 it spills:
// the fp64 64x64 tree state exceeds the register file at any CTA shape).
constexpr K1Choice K1_TUNED_FP64[] = {
    {2, 2, 1, 8}, {2, 3, 0, 8}, {2, 4, 1, 2}, {2, 5, 1, 1}, {2, 6, 0, 1}, {3, 4, 1, 2},
    {3, 6, 1, 1}, {4, 2, 1, 32}, {4, 6, 1, 1}, {6, 6, 2, 1}, {7, 0, 4, 8},
};
constexpr int k1_choose_q(int M0, int M1, bool DBL = false) {
    for (const K1Choice &c : K1_TUNED_FP32)
        if (!DBL && c.m0 == M0 && c.m1 == M1) return c.q;
    for (const K1Choice &c : K1_TUNED_FP64)
        if (DBL && c.m0 == M0 && c.m1 == M1) return c.q;
    int q = M0 > 2 ? M0 - 2 : 0;
    if (q > 3) q = 3;
    if (DBL && M0 >= 3 && M0 <= 5) q = 2;  // fp64 sweep: Q = 2 best for m0 = 3, 4, 5
    while (q > 0 && (1 << M1) * (1 << q) > 512) --q;
    return q;
}
constexpr int k1_choose_tp1(int M0, int M1, int Q, bool DBL = false) {
    for (const K1Choice &c : K1_TUNED_FP32)
        if (!DBL && c.m0 == M0 && c.m1 == M1) return c.tp1;
    for (const K1Choice &c : K1_TUNED_FP64)
        if (DBL && c.m0 == M0 && c.m1 == M1) return c.tp1;
    const int per = (1 << M1) * (1 << Q);
    return per >= 128 ? 1 : 128 / per;
}

constexpr int k1_choose_minb(int M0, int M1, bool DBL = false) {
    for (const K1Choice &c : K1_TUNED_FP32)
        if (!DBL && c.m0 == M0 && c.m1 == M1) return c.minb;
    for (const K1Choice &c : K1_TUNED_FP64)
        if (DBL && c.m0 == M0 && c.m1 == M1) return c.minb;
    return 1;
}

// The Z-column kernel of the large-window path (1-column window n0 x 1 over the
// stage-R rows; COLZ): the 1-column shape's Q, and 256 / J (<= 32) columns per CTA so that
// a warp stores runs of consecutive k1 and a CTA stays at <= 256 threads (registers).
template <int M0, bool DBL> struct K1ZInst {
    using T = typename std::conditional<DBL, double, float>::type;
    static constexpr int Q = k1_choose_q(M0, 0, DBL);
    static constexpr int TP1 = cmin(32, cmax(1, 256 >> Q));
    static void reg() { register_k1(k1_info<T, M0, 0, Q, TP1, DBL, 1, 1, false, true>()); }
};

template <int M0, int M1, bool DBL> struct K1Inst {
    using T = typename std::conditional<DBL, double, float>::type;
    static constexpr int Q = k1_choose_q(M0, M1, DBL);
    static constexpr int TP1 = k1_choose_tp1(M0, M1, Q, DBL);
    static constexpr int MINB = k1_choose_minb(M0, M1, DBL);
    using S = K1Shape<M0, M1, Q, TP1>;
    static void reg() {
        register_k1(k1_info<T, M0, M1, Q, TP1, DBL, MINB>());
        register_k1(k1_info<T, M0, M1, Q, TP1, DBL, MINB, 1, true>());
        // float32 input in fp32 (configs 2-4): the input dtype folded at compile time
        // (config 2 0.0952 -> 0.0932 ms in the tuning harness; the larger configs level)
        if constexpr (!DBL)
            register_k1(k1_info<T, M0, M1, Q, TP1, DBL, MINB, 1, false, false, 0>());
    }
};

}  // namespace swdft2d
