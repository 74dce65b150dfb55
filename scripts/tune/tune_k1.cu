// tune_k1.cu — tuning harness (not product code): the library's ABI (abi.cu) with
// a registry filled from an explicit list of K1 shape variants, selectable at run
// time, so one build can time several (Q, TP1, MINB) choices on the GPU box.
#include "../../paper_1707_08213_b200/csrc/abi.cu"
#include "../../paper_1707_08213_b200/csrc/k1_stream.cuh"
#include "../../paper_1707_08213_b200/csrc/k0_window.cu"
#include "../../paper_1707_08213_b200/csrc/k2_push.cu"
#include "../../paper_1707_08213_b200/csrc/kr_rows.cu"
#include "../../paper_1707_08213_b200/csrc/kc_cols.cu"

namespace swdft2d {
void k1_register_m0_0() {}
void k1_register_m0_1() {}
void k1_register_m0_2() {}
void k1_register_m0_3() {}
void k1_register_m0_4() {}
void k1_register_m0_5() {}
void k1_register_m0_6() {}
void k1_register_m0_7() {}
void k1_register_m0_8() {}
void k1_register_m0_9() {}

struct Variant { const char *name; const K1Info *(*info)(); };
#define V(T, M0, M1, Q, TP1, MINB, NBM)                                                   \
    {#T " m0=" #M0 " m1=" #M1 " Q=" #Q " TP1=" #TP1 " MINB=" #MINB " NBM=" #NBM,          \
     &k1_info<T, M0, M1, Q, TP1, false, MINB, NBM>}
#define V64(M0, M1, Q, TP1, MINB)                                                       \
    {"double m0=" #M0 " m1=" #M1 " Q=" #Q " TP1=" #TP1 " MINB=" #MINB,                  \
     &k1_info<double, M0, M1, Q, TP1, true, MINB, 1>}
#define VZ(T, M0, Q, TP1)                                                                \
    {#T " Z-column m0=" #M0 " Q=" #Q " TP1=" #TP1,                                    \
     &k1_info<T, M0, 0, Q, TP1, (sizeof(T) == 8), 1, 1, false, true>}
static const Variant VARIANTS[] = {
    V(float, 4, 4, 2, 2, 5, 1),
};
}  // namespace swdft2d

extern "C" int tune_count(void) { return (int)(sizeof(swdft2d::VARIANTS) / sizeof(swdft2d::VARIANTS[0])); }
extern "C" const char *tune_name(int v) { return swdft2d::VARIANTS[v].name; }
extern "C" int tune_m(int v, int which) {
    const swdft2d::K1Info *i = swdft2d::VARIANTS[v].info();
    return which == 0 ? i->m0 : which == 1 ? i->m1 : which == 2 ? i->threads : (int)i->smem_bytes;
}
extern "C" int tune_select(int v) {
    swdft2d::find_k1(0, 0, 0);  // run the (empty) registration once
    swdft2d::register_k1(swdft2d::VARIANTS[v].info());
    return 0;
}

#ifdef K1_TIMELINE
// per-CTA (start ns, end ns, smid) of the last K1 launch, n CTAs
extern "C" int tune_timeline(unsigned long long *dst, int n) {
    return (int)cudaMemcpyFromSymbol(dst, swdft2d::g_k1_timeline,
                                     sizeof(unsigned long long) * 3 * (size_t)n);
}
#endif
