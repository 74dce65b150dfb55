// write_probe4.cu — K1's config-4 output pattern without the compute: is K1's write
// rate (6.9 TB/s) set by its store width (8-byte lanes) or by the pattern itself?
// Output [P0=4081][P1=4081][16][16] complex64; a tile = (column block of TP1 = 2 window
// columns, chunk of rows); per row a CTA writes its 2 x 256 coefficients (4 KB).
//   k1_8B   : 128 threads, thread (k1, j, pos) stores coefs (j + 4u, k1), u < 4, 8 B each
//   k1_16B  : 64 threads, each stores 16-B pairs (k1, k1 + 1) — same bytes per row
//   k1_32B  : 32 threads, 32-B stores (Blackwell st.v8.f32)
// persistent (grid = slots, tiles strided) or one tile per CTA (--oneshot rows/tile).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe4 write_probe4.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr long long P0 = 4081, P1 = 4081, W = 256;  // coefficients per window
constexpr int TP1 = 2;
constexpr long long CB = (P1 + TP1 - 1) / TP1;

template <int MODE>  // 0: 8 B, 1: 16 B, 2: 32 B
__global__ void k1pat(float2 *out, long long rch, long long ntiles) {
    const int tid = threadIdx.x;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long cb = tile % CB, rc = tile / CB;
        const long long r0 = rc * rch, r1 = r0 + rch < P0 ? r0 + rch : P0;
        for (long long r = r0; r < r1; ++r) {
            float2 *row = out + (r * P1 + cb * TP1) * W;
            if (MODE == 0) {  // 128 threads: k1 = tid % 16, j = (tid / 16) % 4, pos = tid / 64
                const int k1 = tid & 15, j = (tid >> 4) & 3, pos = tid >> 6;
                if (cb * TP1 + pos < P1)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        __stcs(row + pos * W + (j + 4 * u) * 16 + k1, make_float2((float)r, (float)u));
            } else if (MODE == 1) {  // 64 threads: k1 pair = 2 * (tid % 8)
                const int k1 = 2 * (tid & 7), j = (tid >> 3) & 3, pos = tid >> 5;
                if (cb * TP1 + pos < P1)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        __stcs(reinterpret_cast<float4 *>(row + pos * W + (j + 4 * u) * 16 + k1),
                               make_float4((float)r, (float)u, 1.f, 2.f));
            } else {  // 32 threads: k1 quad = 4 * (tid % 4)
                const int k1 = 4 * (tid & 3), j = (tid >> 2) & 3, pos = tid >> 4;
                if (cb * TP1 + pos < P1)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float *q = reinterpret_cast<float *>(row + pos * W + (j + 4 * u) * 16 + k1);
                        const float a = (float)r, b = (float)u;
                        asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(q), "f"(a), "f"(b) : "memory");
                    }
            }
        }
    }
}

// config-5 geometry: [1985][1985][64][64] complex64, one window column per CTA, 512
// threads, thread (k1 = tid % 64, j = tid / 64) stores coefs (j + 8u, k1), u < 8
__global__ void k1pat_c5(float2 *out, long long rch, long long ntiles) {
    constexpr long long Q0 = 1985, Q1 = 1985, WW = 4096;
    const int k1 = threadIdx.x & 63, j = threadIdx.x >> 6;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long cb = tile % Q1, rc = tile / Q1;
        const long long r0 = rc * rch, r1 = r0 + rch < Q0 ? r0 + rch : Q0;
        for (long long r = r0; r < r1; ++r) {
            float2 *row = out + (r * Q1 + cb) * WW;
#pragma unroll
            for (int u = 0; u < 8; ++u) __stcs(row + (j + 8 * u) * 64 + k1, make_float2((float)r, (float)u));
        }
    }
}

int main_c5(int sms) {
    const size_t bytes = 1985ull * 1985 * 4096 * 8;
    float2 *out;
    if (cudaMalloc(&out, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (bool os : {false, true})
        for (long long rch : {128LL, 1024LL, 1985LL}) {
            const long long nt = 1985LL * ((1985 + rch - 1) / rch);
            const long long grid = os ? nt : (long long)sms;
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                k1pat_c5<<<(unsigned)grid, 512>>>(out, rch, nt);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("{\"mode\": \"c5_8B\", \"oneshot\": %d, \"rch\": %lld, \"grid\": %lld, \"GBps\": %.1f, \"ms\": %.3f}\n",
                   os ? 1 : 0, rch, grid, bytes / best / 1e6, best);
            fflush(stdout);
        }
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
}

int main(int argc, char **argv) {
    if (argc > 1) {
        int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        return main_c5(sms);
    }
    const size_t bytes = (size_t)P0 * P1 * W * 8;
    float2 *out;
    if (cudaMalloc(&out, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, int mode, int threads, long long rch, bool oneshot) {
        const long long nt = CB * ((P0 + rch - 1) / rch);
        int occ = 0;
        if (mode == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1pat<0>, threads, 0);
        if (mode == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1pat<1>, threads, 0);
        if (mode == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1pat<2>, threads, 0);
        // K1 runs 4 CTAs of 128 threads per SM: cap residency the same way (16 warps/SM)
        const int warps_cap = 16, occ_cap = warps_cap * 32 / threads;
        if (occ > occ_cap) occ = occ_cap;
        long long grid = oneshot ? nt : (long long)sms * occ;
        if (grid > nt) grid = nt;
        const int smem = oneshot ? 0 : 0;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k1pat<0><<<(unsigned)grid, threads, smem>>>(out, rch, nt);
            if (mode == 1) k1pat<1><<<(unsigned)grid, threads, smem>>>(out, rch, nt);
            if (mode == 2) k1pat<2><<<(unsigned)grid, threads, smem>>>(out, rch, nt);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"mode\": \"%s\", \"oneshot\": %d, \"rch\": %lld, \"grid\": %lld, \"GBps\": %.1f, \"ms\": %.3f}\n",
               name, oneshot ? 1 : 0, rch, grid, bytes / best / 1e6, best);
        fflush(stdout);
    };
    for (bool os : {false, true})
        for (long long rch : {128LL, 1024LL, P0}) {
            run("k1_8B", 0, 128, rch, os);
            run("k1_16B", 1, 64, rch, os);
            run("k1_32B", 2, 32, rch, os);
        }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 2;
}
