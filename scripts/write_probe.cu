// write_probe.cu — the B200 HBM write-only ceiling for the roofline of a
// write-bound kernel, under several access patterns:
//   gridstride  : all CTAs sweep the buffer together (st.global.cs.v4)
//   chunked     : each CTA streams its own contiguous region
//   k1pattern   : each CTA writes 32 KB blocks at a 33 MB stride (K1's C4 output pattern)
//   memset      : cudaMemsetAsync
//   gs256cs / gs256 : grid-stride 32-byte stores (st.global[.cs].v8.f32, Blackwell STG.256)
//   gs8cs       : grid-stride 8-byte streaming stores (K1's float2 store width)
//   gszero      : grid-stride 16-byte streaming stores of zeros (compressible data)
// Values are per-thread varying (not compressible) unless noted.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe write_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gridstride(float4 *p, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) __stcs(p + i, make_float4((float)i, 1.f, 2.f, (float)threadIdx.x));
}
__global__ void chunked(float4 *p, size_t n) {
    size_t per = (n + gridDim.x - 1) / gridDim.x, b = blockIdx.x * per, e = b + per < n ? b + per : n;
    for (size_t i = b + threadIdx.x; i < e; i += blockDim.x)
        __stcs(p + i, make_float4((float)i, 1.f, 2.f, (float)threadIdx.x));
}
template <bool CS>
__global__ void gridstride256(float4 *p, size_t n) {  // n float4 = n / 2 32-byte units
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n / 2; i += st) {
        float *q = reinterpret_cast<float *>(p + 2 * i);
        const float a = (float)i, b = (float)threadIdx.x;
        if (CS)
            asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" :: "l"(q), "f"(a), "f"(b) : "memory");
        else
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" :: "l"(q), "f"(a), "f"(b) : "memory");
    }
}
__global__ void gridstride8(float2 *p, size_t n) {  // n float2
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) __stcs(p + i, make_float2((float)i, (float)threadIdx.x));
}
__global__ void gridstridezero(float4 *p, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) __stcs(p + i, make_float4(0.f, 0.f, 0.f, 0.f));
}
// block of 2048 float4 (32 KB) per "row"; rows of a CTA are `stride` float4 apart
__global__ void k1pattern(float4 *p, size_t n, size_t stride, size_t nblk_per_row) {
    const size_t rows = n / stride;
    for (size_t t = blockIdx.x; t < nblk_per_row * 8; t += gridDim.x) {
        size_t cb = t % nblk_per_row, rc = t / nblk_per_row;
        for (size_t r = rc * rows / 8; r < (rc + 1) * rows / 8; ++r) {
            float4 *q = p + r * stride + cb * 2048;
            for (int i = threadIdx.x; i < 2048; i += blockDim.x)
                __stcs(q + i, make_float4((float)i, (float)r, 2.f, 3.f));
        }
    }
}

// TMA bulk store: each CTA stages CH bytes in shared memory (double-buffered) and one
// thread issues cp.async.bulk.global.shared::cta for the whole chunk.
template <int CH>
__global__ void bulkstore(float4 *p, size_t n) {
    extern __shared__ __align__(128) float4 sbuf[];  // 2 * CH bytes
    const size_t per_chunk = CH / 16, nchunks = n / per_chunk;
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        float4 *buf = sbuf + (it & 1) * per_chunk;
        if (threadIdx.x == 0)  // buffer (it & 1) was last used two chunks ago
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (int i = threadIdx.x; i < (int)per_chunk; i += blockDim.x)
            buf[i] = make_float4((float)i, (float)c, 2.f, 3.f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned sa = (unsigned)__cvta_generic_to_shared(buf);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(p + c * per_chunk), "r"(sa), "r"(CH) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    size_t bytes = 32ull << 30, n = bytes / 16;
    float4 *p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t stride = (33ull << 20) / 16, nblk = stride / 2048;
    {
        auto k = bulkstore<32768>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        auto k2 = bulkstore<16384>;
        for (int occ : {1, 2, 3}) {
            float best = 1e30f, best2 = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                k<<<sms * occ, 256, 65536>>>(p, n);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
                cudaEventRecord(a);
                k2<<<sms * occ * 2, 256, 32768>>>(p, n);
                cudaEventRecord(b); cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best2) best2 = ms;
            }
            printf("{\"mode\": \"bulkstore32K\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", occ, bytes / best / 1e6);
            printf("{\"mode\": \"bulkstore16K\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", occ * 2, bytes / best2 / 1e6);
        }
    }
    for (int mode = 0; mode < 8; ++mode)
        for (int occ : {2, 4, 8}) {
            float best = 1e30f;
            size_t written = bytes;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) gridstride<<<sms * occ, 512>>>(p, n);
                else if (mode == 1) chunked<<<sms * occ, 512>>>(p, n);
                else if (mode == 2) k1pattern<<<sms * occ, 512>>>(p, n, stride, nblk);
                else if (mode == 3) cudaMemsetAsync(p, rep + 1, bytes);
                else if (mode == 4) gridstride256<true><<<sms * occ, 512>>>(p, n);
                else if (mode == 5) gridstride256<false><<<sms * occ, 512>>>(p, n);
                else if (mode == 6) gridstride8<<<sms * occ, 512>>>(reinterpret_cast<float2 *>(p), 2 * n);
                else gridstridezero<<<sms * occ, 512>>>(p, n);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            if (mode == 2) written = (n / stride) * stride * 16;
            const char *nm[] = {"gridstride", "chunked", "k1pattern", "memset",
                                "gs256cs", "gs256", "gs8cs", "gszero"};
            printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", nm[mode], occ,
                   written / best / 1e6);
            if (mode == 3) break;
        }
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 2;
}
