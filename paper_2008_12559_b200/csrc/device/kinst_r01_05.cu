// kinst_r01_05.cu -- explicit instantiations of the kernel templates for r = 1..5
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(1, )
PFT_INSTANCES(2, )
PFT_INSTANCES(3, )
PFT_INSTANCES(4, )
PFT_INSTANCES(5, )
}  // namespace pftdev
