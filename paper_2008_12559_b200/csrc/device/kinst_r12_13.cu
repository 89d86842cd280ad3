// kinst_r12_13.cu -- explicit instantiations of the kernel templates for r = 12..13
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(12, )
PFT_INSTANCES(13, )
}  // namespace pftdev
