// sweep_main.cu — the library ABI with a registry filled from the generated sweep
// variants (tuning harness, not product code).
#include "../../../paper_1707_08213_b200/csrc/abi.cu"
#include "../../../paper_1707_08213_b200/csrc/k0_window.cu"
#include "../../../paper_1707_08213_b200/csrc/k2_push.cu"
#include "../../../paper_1707_08213_b200/csrc/kc_cols.cu"
#include "../../../paper_1707_08213_b200/csrc/kr_rows.cu"
#include "../tune_common.cuh"

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
extern const Variant SWEEP_2[], SWEEP_3[], SWEEP_4[], SWEEP_5[], SWEEP_6[], SWEEP_7[], SWEEP64[];
static const Variant *ALL[] = {SWEEP_2, SWEEP_3, SWEEP_4, SWEEP_5, SWEEP_6, SWEEP_7, SWEEP64};
static const Variant *nth(int v) {
    for (const Variant *a : ALL)
        for (; a->name; ++a)
            if (v-- == 0) return a;
    return nullptr;
}
}  // namespace swdft2d

extern "C" int tune_count(void) {
    int n = 0;
    while (swdft2d::nth(n)) ++n;
    return n;
}
extern "C" const char *tune_name(int v) { return swdft2d::nth(v)->name; }
extern "C" int tune_m(int v, int which) {
    const swdft2d::K1Info *i = swdft2d::nth(v)->info();
    return which == 0 ? i->m0 : which == 1 ? i->m1 : which == 2 ? i->threads :
           which == 4 ? i->prec : (int)i->smem_bytes;
}
extern "C" int tune_select(int v) {
    swdft2d::find_k1(0, 0, 0);
    swdft2d::register_k1(swdft2d::nth(v)->info());
    return 0;
}
