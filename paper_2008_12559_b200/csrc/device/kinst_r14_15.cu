// kinst_r14_15.cu -- explicit instantiations of the kernel templates for r = 14..15
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(14, )
PFT_INSTANCES(15, )
}  // namespace pftdev
