// Compiled variants of band4_kernel.cuh (split over several translation
// units so they build in parallel); dispatched by step_band4.cu.
#include "band4_kernel.cuh"

namespace ctqw {
namespace b4 {
CTQW_B4_INST(1, false, false, false, 0, 2)
CTQW_B4_INST(1, false, false, true, 0, 2)
CTQW_B4_INST(1, false, true, false, 0, 2)
CTQW_B4_INST(1, false, true, true, 0, 2)
CTQW_B4_INST(2, false, false, false, 0, 2)
CTQW_B4_INST(2, false, false, true, 0, 2)
CTQW_B4_INST(2, false, true, false, 0, 2)
CTQW_B4_INST(2, false, true, true, 0, 2)
CTQW_B4_INST(3, false, false, false, 0, 2)
CTQW_B4_INST(3, false, false, true, 0, 2)
CTQW_B4_INST(3, false, true, false, 0, 2)
CTQW_B4_INST(3, false, true, true, 0, 2)
}  // namespace b4
}  // namespace ctqw
