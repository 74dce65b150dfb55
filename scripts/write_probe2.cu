// write_probe2.cu — why does cudaMemsetAsync write HBM at ~7.4 TB/s when SM
// streaming-store kernels top out at ~6.6-6.9 TB/s (write_probe.cu)?  Times the
// memset next to grid-stride store kernels over block sizes, CTAs per SM, store
// widths and cache policies, so the fastest SM pattern can be copied into K1's
// epilogue.  Run the memset alone under ncu to read its launch shape / SASS:
//   ncu --set full -k regex:memset -c 1 ./write_probe2 memset
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe2 write_probe2.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

template <int POL>  // 0 default, 1 .cs, 2 L1::no_allocate, 3 .wt
__device__ __forceinline__ void st16(float4 *q, float4 v) {
    if (POL == 0) asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    else if (POL == 1) asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    else if (POL == 2) asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    else asm volatile("st.global.wt.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// grid-stride, UNROLL independent 16-B stores per thread per iteration
template <int POL, int UNROLL>
__global__ void gs(float4 *p, size_t n) {
    const size_t st = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * st < n; i += UNROLL * st) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) st16<POL>(p + i + u * st, make_float4((float)i, 1.f, (float)u, (float)threadIdx.x));
    }
    for (; i < n; i += st) st16<POL>(p + i, make_float4((float)i, 1.f, 2.f, 3.f));
}

// block-contiguous: each CTA writes a contiguous CHUNK-float4 span per step (grid walks spans)
template <int POL, int CHUNK>
__global__ void spans(float4 *p, size_t n) {
    const size_t nsp = n / CHUNK;
    for (size_t s = blockIdx.x; s < nsp; s += gridDim.x) {
        float4 *q = p + s * CHUNK;
#pragma unroll 4
        for (int i = threadIdx.x; i < CHUNK; i += blockDim.x) st16<POL>(q + i, make_float4((float)i, (float)s, 2.f, 3.f));
    }
}

int main(int argc, char **argv) {
    const bool only_memset = argc > 1 && !std::strcmp(argv[1], "memset");
    size_t bytes = 16ull << 30, n = bytes / 16;
    float4 *p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char *name, int occ, int threads, auto launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            launch(rep);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"threads\": %d, \"GBps\": %.1f}\n", name, occ, threads, bytes / best / 1e6);
        fflush(stdout);
    };
    timeit("memset", 0, 0, [&](int rep) { cudaMemsetAsync(p, rep + 1, bytes); });
    timeit("memsetD32", 0, 0, [&](int rep) { cudaMemsetAsync(p, 0x5a, bytes); });
    if (only_memset) return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
    for (int threads : {256, 512, 1024})
        for (int occ : {1, 2, 4, 8}) {
            if (threads * occ > 2048) continue;
            const int g = sms * occ;
            timeit("gs_def_u1", occ, threads, [&](int) { gs<0, 1><<<g, threads>>>(p, n); });
            timeit("gs_cs_u1", occ, threads, [&](int) { gs<1, 1><<<g, threads>>>(p, n); });
            timeit("gs_cs_u4", occ, threads, [&](int) { gs<1, 4><<<g, threads>>>(p, n); });
            timeit("gs_def_u4", occ, threads, [&](int) { gs<0, 4><<<g, threads>>>(p, n); });
            timeit("gs_na_u4", occ, threads, [&](int) { gs<2, 4><<<g, threads>>>(p, n); });
            timeit("spans8K_cs", occ, threads, [&](int) { spans<1, 512><<<g, threads>>>(p, n); });
            timeit("spans64K_cs", occ, threads, [&](int) { spans<1, 4096><<<g, threads>>>(p, n); });
            timeit("spans64K_def", occ, threads, [&](int) { spans<0, 4096><<<g, threads>>>(p, n); });
        }
    // oversubscribed grids (not persistent): many short CTAs, like memset kernels often are
    for (int threads : {256, 512}) {
        const size_t g = n / threads / 4;
        timeit("oneshot_cs_u4", -1, threads, [&](int) { gs<1, 4><<<(unsigned)g, threads>>>(p, n); });
        timeit("oneshot_def_u4", -1, threads, [&](int) { gs<0, 4><<<(unsigned)g, threads>>>(p, n); });
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 2;
}
