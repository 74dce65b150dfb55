// write_probe3.cu — what makes a non-persistent "one-shot" store grid write HBM at
// ~7.5 TB/s when persistent grid-stride kernels stay at ~6.3 TB/s (write_probe2.cu)?
// Separates the two differences: how far apart the concurrently written regions are
// ("fronts"), and whether CTAs are persistent or short-lived.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe3 write_probe3.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st16(float4 *q, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// persistent: the buffer is F regions of n/F; every thread grid-strides over n/F and
// stores once into each region per step (F concurrent fronts, n/F apart)
template <int F>
__global__ void far_persistent(float4 *p, size_t n) {
    const size_t m = n / F, st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += st)
#pragma unroll
        for (int u = 0; u < F; ++u) st16(p + i + u * m, make_float4((float)i, 1.f, (float)u, 3.f));
}
// one-shot, F far fronts: CTA b, thread t writes element b*T+t of each region (grid = m / T)
template <int F>
__global__ void far_oneshot(float4 *p, size_t n) {
    const size_t m = n / F, i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < m)
#pragma unroll
        for (int u = 0; u < F; ++u) st16(p + i + u * m, make_float4((float)i, 1.f, (float)u, 3.f));
}
// one-shot, near: CTA b writes F consecutive blocks of T float4 (one contiguous span)
template <int F>
__global__ void near_oneshot(float4 *p, size_t n) {
    const size_t base = blockIdx.x * (size_t)blockDim.x * F;
#pragma unroll
    for (int u = 0; u < F; ++u) {
        const size_t i = base + u * blockDim.x + threadIdx.x;
        if (i < n) st16(p + i, make_float4((float)i, 1.f, (float)u, 3.f));
    }
}
// persistent, CTA-ordered like one-shot: CTA c takes "virtual CTAs" c, c+G, c+2G, ...
// and writes each one's F consecutive blocks (same addresses/order as near_oneshot)
template <int F>
__global__ void near_persistent(float4 *p, size_t n) {
    const size_t nv = n / ((size_t)blockDim.x * F);
    for (size_t v = blockIdx.x; v < nv; v += gridDim.x) {
        const size_t base = v * blockDim.x * F;
#pragma unroll
        for (int u = 0; u < F; ++u) st16(p + base + u * blockDim.x + threadIdx.x, make_float4((float)v, 1.f, (float)u, 3.f));
    }
}
// persistent, near pattern, but virtual CTA v is scrambled by an odd-multiplier bijection
// on [0, nv) (nv a power of two): consecutive steps of one CTA land at unrelated addresses
template <int F>
__global__ void near_persistent_scrambled(float4 *p, size_t n) {
    const size_t nv = n / ((size_t)blockDim.x * F);
    for (size_t v0 = blockIdx.x; v0 < nv; v0 += gridDim.x) {
        const size_t v = (v0 * 0x9E3779B1ull) & (nv - 1);
        const size_t base = v * blockDim.x * F;
#pragma unroll
        for (int u = 0; u < F; ++u) st16(p + base + u * blockDim.x + threadIdx.x, make_float4((float)v, 1.f, (float)u, 3.f));
    }
}
// persistent, each CTA owns one contiguous 1/G of the buffer (G fronts as far apart as possible)
__global__ void own_region(float4 *p, size_t n) {
    const size_t per = n / gridDim.x, b = blockIdx.x * per;
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) st16(p + b + i, make_float4((float)i, 1.f, 2.f, 3.f));
}

// "waves": grid = k x resident slots, CTA c writes virtual CTAs c, c + G, ... (near
// pattern, 4 KB blocks x 4 per virtual CTA), so k = 1 is persistent and large k one-shot
int main_waves(float4 *p, size_t n, int sms, cudaEvent_t a, cudaEvent_t b) {
    const size_t bytes = n * 16;
    for (int threads : {256, 512})
        for (int k : {1, 2, 3, 4, 6, 8, 16, 64, 256}) {
            const int slots = sms * (2048 / threads);
            const long long g = (long long)slots * k;
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                near_persistent<4><<<(unsigned)g, threads>>>(p, n);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            printf("{\"mode\": \"waves\", \"k\": %d, \"grid\": %lld, \"threads\": %d, \"GBps\": %.1f}\n", k, g, threads, bytes / best / 1e6);
            fflush(stdout);
        }
    return 0;
}

int main(int argc, char **argv) {
    size_t bytes = 16ull << 30, n = bytes / 16;
    float4 *p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char *name, long long grid, int threads, auto launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"mode\": \"%s\", \"grid\": %lld, \"threads\": %d, \"GBps\": %.1f}\n", name, grid, threads, bytes / best / 1e6);
        fflush(stdout);
    };
    if (argc > 1 && argv[1][0] == 's') {
        for (int occ : {2, 4, 8}) {
            const int g = sms * occ;
            timeit("near_persistent_F4", g, 256, [&] { near_persistent<4><<<g, 256>>>(p, n); });
            timeit("near_persistent_scrambled_F4", g, 256, [&] { near_persistent_scrambled<4><<<g, 256>>>(p, n); });
            timeit("near_persistent_scrambled_F1", g, 256, [&] { near_persistent_scrambled<1><<<g, 256>>>(p, n); });
        }
        return 0;
    }
    if (argc > 1) return main_waves(p, n, sms, a, b);
    const int T = 256;
    for (int occ : {2, 8}) {
        const int g = sms * occ;
        timeit("far_persistent_F1", g, T, [&] { far_persistent<1><<<g, T>>>(p, n); });
        timeit("far_persistent_F2", g, T, [&] { far_persistent<2><<<g, T>>>(p, n); });
        timeit("far_persistent_F4", g, T, [&] { far_persistent<4><<<g, T>>>(p, n); });
        timeit("far_persistent_F8", g, T, [&] { far_persistent<8><<<g, T>>>(p, n); });
        timeit("near_persistent_F4", g, T, [&] { near_persistent<4><<<g, T>>>(p, n); });
        timeit("near_persistent_F16", g, T, [&] { near_persistent<16><<<g, T>>>(p, n); });
        timeit("own_region", g, T, [&] { own_region<<<g, T>>>(p, n); });
    }
    timeit("far_oneshot_F1", n / T, T, [&] { far_oneshot<1><<<(unsigned)(n / T), T>>>(p, n); });
    timeit("far_oneshot_F4", n / T / 4, T, [&] { far_oneshot<4><<<(unsigned)(n / T / 4), T>>>(p, n); });
    timeit("far_oneshot_F16", n / T / 16, T, [&] { far_oneshot<16><<<(unsigned)(n / T / 16), T>>>(p, n); });
    timeit("near_oneshot_F4", n / T / 4, T, [&] { near_oneshot<4><<<(unsigned)(n / T / 4), T>>>(p, n); });
    timeit("near_oneshot_F16", n / T / 16, T, [&] { near_oneshot<16><<<(unsigned)(n / T / 16), T>>>(p, n); });
    timeit("near_oneshot_F64", n / T / 64, T, [&] { near_oneshot<64><<<(unsigned)(n / T / 64), T>>>(p, n); });
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 2;
}
