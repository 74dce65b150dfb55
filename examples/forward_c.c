/*
 * forward_c.c — calling libswdft2d.so from C through the C ABI alone (include/swdft2d.h):
 * no Python, no torch.  A 64 x 48 float32 array, 8 x 4 windows, complex64 output, checked
 * against a direct double-precision DFT of a few windows.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/forward_c.c \
 *       -L paper_1707_08213_b200 -lswdft2d -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_1707_08213_b200 -o examples/forward_c && examples/forward_c
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "swdft2d.h"

#define CHECK_CUDA(e)                                                       \
    do {                                                                    \
        cudaError_t err_ = (e);                                             \
        if (err_ != cudaSuccess) {                                          \
            fprintf(stderr, "CUDA: %s (%s:%d)\n", cudaGetErrorString(err_), \
                    __FILE__, __LINE__);                                    \
            return 2;                                                       \
        }                                                                   \
    } while (0)

int main(void) {
    const int64_t N0 = 64, N1 = 48;
    const int m0 = 3, m1 = 2, n0 = 1 << m0, n1 = 1 << m1;
    int64_t P0 = 0, P1 = 0;
    if (swdft2d_abi_version() != SWDFT2D_ABI_VERSION) {
        fprintf(stderr, "ABI version mismatch\n");
        return 2;
    }
    if (swdft2d_output_shape(N0, N1, m0, m1, &P0, &P1) != SWDFT2D_OK) {
        fprintf(stderr, "%s\n", swdft2d_last_error());
        return 2;
    }
    const size_t nout = (size_t)(P0 * P1 * n0 * n1);
    float *x = (float *)malloc(sizeof(float) * N0 * N1);
    float *out = (float *)malloc(sizeof(float) * 2 * nout);
    srand(7);
    for (int64_t i = 0; i < N0 * N1; ++i) x[i] = (float)rand() / RAND_MAX - 0.5f;

    void *x_d = NULL, *out_d = NULL;
    CHECK_CUDA(cudaMalloc(&x_d, sizeof(float) * N0 * N1));
    CHECK_CUDA(cudaMalloc(&out_d, sizeof(float) * 2 * nout));
    CHECK_CUDA(cudaMemcpy(x_d, x, sizeof(float) * N0 * N1, cudaMemcpyHostToDevice));
    cudaStream_t s;
    CHECK_CUDA(cudaStreamCreate(&s));
    int rc = swdft2d_forward(x_d, SWDFT2D_IN_F32, N0, N1, N1, m0, m1, SWDFT2D_PREC_FP32, 1.0, 0, P0,
                             out_d, SWDFT2D_KERNEL_AUTO, s);
    if (rc != SWDFT2D_OK) {
        fprintf(stderr, "swdft2d_forward: %d %s\n", rc, swdft2d_last_error());
        return 1;
    }
    /* an invalid call fails with a status code and a message, not a crash */
    if (swdft2d_forward(x_d, SWDFT2D_IN_F32, N0, N1, N1, 7, m1, SWDFT2D_PREC_FP32, 1.0, 0, 1, out_d,
                        SWDFT2D_KERNEL_AUTO, s) != SWDFT2D_E_WINDOW_TOO_LARGE) {
        fprintf(stderr, "expected SWDFT2D_E_WINDOW_TOO_LARGE\n");
        return 1;
    }
    CHECK_CUDA(cudaStreamSynchronize(s));
    CHECK_CUDA(cudaMemcpy(out, out_d, sizeof(float) * 2 * nout, cudaMemcpyDeviceToHost));

    /* direct DFT of windows (p0, p1): a[k0, k1] = sum x[p0+j0, p1+j1] e^{-2 pi i (j0 k0/n0 + j1 k1/n1)} */
    const int64_t checks[4][2] = {{0, 0}, {P0 - 1, P1 - 1}, {17, 5}, {40, 30}};
    double worst = 0.0;
    for (int c = 0; c < 4; ++c) {
        const int64_t p0 = checks[c][0], p1 = checks[c][1];
        double norm = 0.0, err = 0.0;
        for (int k0 = 0; k0 < n0; ++k0)
            for (int k1 = 0; k1 < n1; ++k1) {
                double re = 0.0, im = 0.0;
                for (int j0 = 0; j0 < n0; ++j0)
                    for (int j1 = 0; j1 < n1; ++j1) {
                        const double ang = -2.0 * M_PI * ((double)j0 * k0 / n0 + (double)j1 * k1 / n1);
                        const double v = x[(p0 + j0) * N1 + p1 + j1];
                        re += v * cos(ang);
                        im += v * sin(ang);
                    }
                const size_t o = (size_t)((((p0 * P1) + p1) * n0 + k0) * n1 + k1);
                const double dr = out[2 * o] - re, di = out[2 * o + 1] - im;
                norm += re * re + im * im;
                const double e = sqrt(dr * dr + di * di);
                if (e > err) err = e;
            }
        const double rel = err / sqrt(norm);
        if (rel > worst) worst = rel;
    }
    /* the same transform host to host in one call (no CUDA calls on the caller's side):
     * malloc'd input and output, equal to the device-buffer result bit for bit */
    float *out2 = (float *)malloc(sizeof(float) * 2 * nout);
    rc = swdft2d_forward_host(x, SWDFT2D_IN_F32, N0, N1, N1, m0, m1, SWDFT2D_PREC_FP32, 1.0, 0, P0,
                              out2, (int64_t)(5 * P1 * n0 * n1 * 8), SWDFT2D_KERNEL_AUTO, NULL);
    if (rc != SWDFT2D_OK) {
        fprintf(stderr, "swdft2d_forward_host: %d %s\n", rc, swdft2d_last_error());
        return 1;
    }
    for (size_t i = 0; i < 2 * nout; ++i)
        if (out2[i] != out[i]) {
            fprintf(stderr, "forward_host differs from forward at %zu\n", i);
            return 1;
        }
    free(out2);
    printf("forward_c: %lld x %lld windows of %d x %d, max window-relative error %.3e\n",
           (long long)P0, (long long)P1, n0, n1, worst);
    cudaFree(x_d);
    cudaFree(out_d);
    cudaStreamDestroy(s);
    swdft2d_shutdown();
    free(x);
    free(out);
    return worst <= 1e-4 ? 0 : 1;
}
