// kinst_r19_25.cu -- explicit instantiations of the kernel templates for r = 19..25
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(19, )
PFT_INSTANCES(20, )
PFT_INSTANCES(21, )
PFT_INSTANCES(22, )
PFT_INSTANCES(23, )
PFT_INSTANCES(24, )
PFT_INSTANCES(25, )
}  // namespace pftdev
