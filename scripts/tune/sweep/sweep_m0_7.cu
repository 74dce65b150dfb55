// K1 variants for 128-row windows (m0 = 7, n1 <= 16), fp32 (tuning harness, not product code)
#include "../tune_common.cuh"
namespace swdft2d {
extern const Variant SWEEP_7[];
const Variant SWEEP_7[] = {
    V(float, 7, 2, 3, 4, 1, 1),
    V(float, 7, 2, 4, 2, 1, 1),
    V(float, 7, 3, 3, 1, 1, 1),
    V(float, 7, 3, 3, 2, 1, 1),
    V(float, 7, 3, 4, 1, 1, 1),
    V(float, 7, 4, 3, 1, 1, 1),
    V(float, 7, 4, 4, 1, 1, 1),
    {nullptr, nullptr},
};
}  // namespace swdft2d
