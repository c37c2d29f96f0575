// Compiled variants of band4_kernel.cuh (split over several translation
// units so they build in parallel); dispatched by step_band4.cu.
#include "band4_kernel.cuh"

namespace ctqw {
namespace b4 {
CTQW_B4_INST(4, false, false, false, 256, 0)
CTQW_B4_INST(4, false, false, false, 256, 2)
CTQW_B4_INST(4, false, false, false, 512, 0)
CTQW_B4_INST(4, false, false, false, 512, 2)
CTQW_B4_INST(4, false, false, false, 1024, 0)
CTQW_B4_INST(4, false, false, false, 1024, 2)
CTQW_B4_INST(4, false, false, false, 0, 2)
}  // namespace b4
}  // namespace ctqw
