// k1_inst.cu — K1 instantiations for one m0 (compiled once per m0 with -DK1_M0=<m0>),
// all m1 in [0, SWDFT2D_K1_MAX_M], fp32 and fp64-exact.
#include "k1_stream.cuh"

#ifndef K1_M0
#error "compile with -DK1_M0=<m0>"
#endif

#define SWDFT2D_CAT2(a, b) a##b
#define SWDFT2D_CAT(a, b) SWDFT2D_CAT2(a, b)

namespace swdft2d {

template <int M0, int M1> static void reg_pair() {
    K1Inst<M0, M1, false>::reg();
    K1Inst<M0, M1, true>::reg();
}

void SWDFT2D_CAT(k1_register_m0_, K1_M0)() {
    reg_pair<K1_M0, 0>();
    reg_pair<K1_M0, 1>();
    reg_pair<K1_M0, 2>();
    reg_pair<K1_M0, 3>();
    reg_pair<K1_M0, 4>();
    reg_pair<K1_M0, 5>();
    reg_pair<K1_M0, 6>();
}

}  // namespace swdft2d
