// tune_common.cuh — shared declarations of the tuning harness (not product code).
#pragma once
#include "../../paper_1707_08213_b200/csrc/k1_stream.cuh"

namespace swdft2d {
struct Variant {
    const char *name;
    const K1Info *(*info)();
};
}  // namespace swdft2d

#define V(T, M0, M1, Q, TP1, MINB, NBM)                                                   \
    {#T " m0=" #M0 " m1=" #M1 " Q=" #Q " TP1=" #TP1 " MINB=" #MINB " NBM=" #NBM,          \
     &swdft2d::k1_info<T, M0, M1, Q, TP1, false, MINB, NBM>}
