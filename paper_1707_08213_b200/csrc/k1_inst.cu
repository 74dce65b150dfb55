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

#if K1_M0 == 9
// 512-row windows: fp32, n1 <= 2, Q = 5 (a 32-complex register ring again): 512x1 3.7 vs
// 2.8 TB/s on KR + KC, 512x2 3.9 vs 3.4 (profiles/sweep_m7_r01.jsonl)
void k1_register_m0_9() {
    K1ZInst<9, false>::reg();
    K1Inst<9, 0, false>::reg();
    K1Inst<9, 1, false>::reg();
}
#elif K1_M0 == 8
// 256-row windows: fp32, n1 <= 4, Q = 4 (J = 16: a 32-complex register ring, ~220-237
// registers): 256x1 4.4 vs 2.9 TB/s on KR + KC, 256x2 4.8 vs 4.1, 256x4 5.4 vs 5.1
// (profiles/sweep_m7_r01.jsonl)
void k1_register_m0_8() {
    K1ZInst<8, false>::reg();
    K1Inst<8, 0, false>::reg();
    K1Inst<8, 1, false>::reg();
    K1Inst<8, 2, false>::reg();  // (256x8 measured level with KR + KC: 5.25 vs 5.33 TB/s)
}
#elif K1_M0 == 7
// 128-row windows: fp32 n1 <= 32 (128x64 would not keep its tree state in registers at
// 512 threads); measured vs the separable KR + KC path: 128x4 6.0 vs 4.3 TB/s, 128x8 6.05
// vs 5.3, 128x16 5.9 vs 5.5, 128x32 6.3 vs 5.5 (profiles/sweep_m7_r01.jsonl)
void k1_register_m0_7() {
    // fp64 only for 128x1 (Q = 4): 3.9 vs 2.8 TB/s separable; 128x2..128x8 in fp64 were
    // slower on K1 (3.9 / 4.3 / 5.3 vs 4.2 / 5.2 / 5.7)
    K1Inst<7, 0, true>::reg();
    K1Inst<7, 0, false>::reg();
    K1ZInst<7, true>::reg();
    K1ZInst<7, false>::reg();
    K1Inst<7, 1, false>::reg();
    K1Inst<7, 2, false>::reg();
    K1Inst<7, 3, false>::reg();
    K1Inst<7, 4, false>::reg();
    K1Inst<7, 5, false>::reg();
}
#else
void SWDFT2D_CAT(k1_register_m0_, K1_M0)() {
#if K1_M0 > 0
    K1ZInst<K1_M0, false>::reg();  // the large-window path's column trees
    K1ZInst<K1_M0, true>::reg();
#endif
    reg_pair<K1_M0, 0>();
    reg_pair<K1_M0, 1>();
    reg_pair<K1_M0, 2>();
    reg_pair<K1_M0, 3>();
    reg_pair<K1_M0, 4>();
    reg_pair<K1_M0, 5>();
    reg_pair<K1_M0, 6>();
}
#endif

}  // namespace swdft2d
