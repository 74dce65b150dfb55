// Row ring of the row-push stream (SlidingRowStream2D, reference tree2d.py:205-303):
// store pushed row p0, converted to the ring's complex type, at slots p0 mod n0 and
// p0 mod n0 + n0 of a [2*n0, N1] buffer, so the n0 rows a window row needs are one
// contiguous view for K1.  One tiny grid-stride kernel per push.
#include "swdft2d_device.cuh"
#include "swdft2d_internal.h"

namespace swdft2d {

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
