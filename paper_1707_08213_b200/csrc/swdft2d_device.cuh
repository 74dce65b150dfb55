// swdft2d_device.cuh — device-side building blocks shared by the K0 and K1 kernels.
//
// The one arithmetic primitive of the reference is core.butterfly
// (/root/reference/pkg/src/swdft/core.py:223-246):
//     out = shifted + twiddle * current
//     re = fl(fl(wr*cr) - fl(wi*ci)),  im = fl(fl(wr*ci) + fl(wi*cr)),
//     out = (fl(sr + re), fl(si + im))
// Exact mode reproduces that rounding sequence with _rn intrinsics (no FMA
// contraction), which is what makes the fp64 path bitwise equal to the
// reference.  Fast (fp32) mode lets the compiler fuse into FFMAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace swdft2d {

// Compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1, so every
// register-array index inside f is a constant (keeps rings/accumulators in registers).
template <typename F, int... Is>
__device__ __forceinline__ void static_for_impl(F &&f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F> __device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}


template <typename T> struct cplx_t;
template <> struct cplx_t<float> { using type = float2; };
template <> struct cplx_t<double> { using type = double2; };
template <typename T> using cplx = typename cplx_t<T>::type;

template <typename T> __device__ __forceinline__ cplx<T> mk(T re, T im) {
    cplx<T> c;
    c.x = re;
    c.y = im;
    return c;
}

// core.butterfly, bitwise (double) — shifted + w * current.
__device__ __forceinline__ double2 bfly_exact(double2 s, double2 w, double2 c) {
    double re = __dsub_rn(__dmul_rn(w.x, c.x), __dmul_rn(w.y, c.y));
    double im = __dadd_rn(__dmul_rn(w.x, c.y), __dmul_rn(w.y, c.x));
    return make_double2(__dadd_rn(s.x, re), __dadd_rn(s.y, im));
}
// core.butterfly with the same operation order in fp32 (used when EXACT on float,
// i.e. never in product builds; kept for completeness of the template).
__device__ __forceinline__ float2 bfly_exact(float2 s, float2 w, float2 c) {
    float re = __fsub_rn(__fmul_rn(w.x, c.x), __fmul_rn(w.y, c.y));
    float im = __fadd_rn(__fmul_rn(w.x, c.y), __fmul_rn(w.y, c.x));
    return make_float2(__fadd_rn(s.x, re), __fadd_rn(s.y, im));
}

// Fast butterfly: s + w*c with FMAs.
__device__ __forceinline__ float2 bfly_fast(float2 s, float2 w, float2 c) {
    float re = fmaf(w.x, c.x, s.x);
    re = fmaf(-w.y, c.y, re);
    float im = fmaf(w.x, c.y, s.y);
    im = fmaf(w.y, c.x, im);
    return make_float2(re, im);
}
__device__ __forceinline__ double2 bfly_fast(double2 s, double2 w, double2 c) {
    double re = fma(w.x, c.x, s.x);
    re = fma(-w.y, c.y, re);
    double im = fma(w.x, c.y, s.y);
    im = fma(w.y, c.x, im);
    return make_double2(re, im);
}

__device__ __forceinline__ float fma_t(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return fma(a, b, c); }

template <bool EXACT, typename C> __device__ __forceinline__ C bfly(C s, C w, C c) {
    if constexpr (EXACT) return bfly_exact(s, w, c);
    else return bfly_fast(s, w, c);
}

// The two children of one butterfly, lo = s + w_lo c and hi = s + w_hi c, where
// w_hi = w[i + L/2] = -w_lo up to rounding.  EXACT: two reference butterflies with their own
// twiddles (the symmetry is not bitwise, App. A #3).  Fast: lo by 4 FMAs, hi = 2 s - lo by 2
// more (w_hi is not read): 6 FP instructions per pair instead of 8.
#ifndef SWDFT2D_PAIR_FMA
#define SWDFT2D_PAIR_FMA 1
#endif
template <bool EXACT, typename C>
__device__ __forceinline__ void bfly_pair(C s, C w_lo, C w_hi, C c, C &lo, C &hi) {
    if constexpr (EXACT || !SWDFT2D_PAIR_FMA) {
        lo = bfly<EXACT>(s, w_lo, c);
        hi = bfly<EXACT>(s, w_hi, c);
    } else {
        lo = bfly_fast(s, w_lo, c);
        hi.x = fma_t((decltype(s.x))2, s.x, -lo.x);
        hi.y = fma_t((decltype(s.y))2, s.y, -lo.y);
    }
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Per-component scaling, core.normalize (core.py:301): values * float64(factor).
// Multiplying each component separately is bitwise equal to numpy's complex *
// real-scalar product.
__device__ __forceinline__ float2 cscale(float2 a, float f) { return make_float2(a.x * f, a.y * f); }
__device__ __forceinline__ double2 cscale(double2 a, double f) {
    return make_double2(__dmul_rn(a.x, f), __dmul_rn(a.y, f));
}

// Load element (row, col) of x with the given element type as complex<T>.
// Real inputs get a +0.0 imaginary part, as np.asarray(x, complex128) does
// (tree2d.py:189).  in_dtype is warp-uniform, so the switch does not diverge.
template <typename T>
__device__ __forceinline__ cplx<T> load_x(const void *__restrict__ x, int in_dtype, int64_t off) {
    switch (in_dtype) {
    case 0: return mk<T>((T)__ldg((const float *)x + off), (T)0);
    case 1: return mk<T>((T)__ldg((const double *)x + off), (T)0);
    case 2: {
        float2 v = __ldg((const float2 *)x + off);
        return mk<T>((T)v.x, (T)v.y);
    }
    default: {
        double2 v = __ldg((const double2 *)x + off);
        return mk<T>((T)v.x, (T)v.y);
    }
    }
}

// Prefetch form of load_x: the loaded bits are kept as they are (packed into the
// complex<T> register pair when they fit) and converted by from_raw at use time, so a
// prefetch never waits for its load (a conversion right after the load would).
template <typename T>
__device__ __forceinline__ cplx<T> load_raw(const void *__restrict__ x, int in_dtype, int64_t off);
template <>
__device__ __forceinline__ double2 load_raw<double>(const void *__restrict__ x, int in_dtype,
                                                    int64_t off) {
    switch (in_dtype) {
    case 0: return make_double2(__hiloint2double(0, __float_as_int(__ldg((const float *)x + off))), 0.0);
    case 1: return make_double2(__ldg((const double *)x + off), 0.0);
    case 2: {
        const float2 v = __ldg((const float2 *)x + off);
        return make_double2(__hiloint2double(__float_as_int(v.y), __float_as_int(v.x)), 0.0);
    }
    default: return __ldg((const double2 *)x + off);
    }
}
template <>
__device__ __forceinline__ float2 load_raw<float>(const void *__restrict__ x, int in_dtype,
                                                  int64_t off) {
#ifdef K1_FORCE_IN_DTYPE  // tuning builds: the input dtype as a compile-time constant
    in_dtype = K1_FORCE_IN_DTYPE;
#endif
    switch (in_dtype) {
    case 0: return make_float2(__ldg((const float *)x + off), 0.f);
    case 1: {
        const double d = __ldg((const double *)x + off);
        return make_float2(__int_as_float(__double2loint(d)), __int_as_float(__double2hiint(d)));
    }
    case 2: return __ldg((const float2 *)x + off);
    default: {  // 128-bit sample does not fit the float2 pair: convert now
        const double2 v = __ldg((const double2 *)x + off);
        return make_float2((float)v.x, (float)v.y);
    }
    }
}
template <typename T> __device__ __forceinline__ cplx<T> from_raw(cplx<T> r, int in_dtype);
template <> __device__ __forceinline__ double2 from_raw<double>(double2 r, int in_dtype) {
    switch (in_dtype) {
    case 0: return make_double2((double)__int_as_float(__double2loint(r.x)), 0.0);
    case 2: return make_double2((double)__int_as_float(__double2loint(r.x)),
                                (double)__int_as_float(__double2hiint(r.x)));
    default: return r;  // f64 (imaginary part already +0.0) and c128
    }
}
template <> __device__ __forceinline__ float2 from_raw<float>(float2 r, int in_dtype) {
#ifdef K1_FORCE_IN_DTYPE
    in_dtype = K1_FORCE_IN_DTYPE;
#endif
    if (in_dtype == 1)
        return make_float2((float)__hiloint2double(__float_as_int(r.y), __float_as_int(r.x)), 0.f);
    return r;  // f32 (imaginary +0.0), c64, and c128 (converted at load)
}

// Sample of x staged in shared memory (TMA tile), element type in_dtype.
template <typename T>
__device__ __forceinline__ cplx<T> load_staged(const unsigned char *p, int in_dtype) {
    switch (in_dtype) {
    case 0: return mk<T>((T) * reinterpret_cast<const float *>(p), (T)0);
    case 1: return mk<T>((T) * reinterpret_cast<const double *>(p), (T)0);
    case 2: {
        const float2 v = *reinterpret_cast<const float2 *>(p);
        return mk<T>((T)v.x, (T)v.y);
    }
    default: {
        const double2 v = *reinterpret_cast<const double2 *>(p);
        return mk<T>((T)v.x, (T)v.y);
    }
    }
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) helpers --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 2D tensor tile global -> shared, completion counted on `bar` (transaction bytes).
__device__ __forceinline__ void tma_load_2d(void *dst, const void *tmap, uint64_t *bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// Streaming (evict-first) 8/16-byte stores for the write-once coefficient output.
__device__ __forceinline__ void st_stream(float2 *p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { __stcs(p, v); }

}  // namespace swdft2d
