// kinst_r18_18.cu -- explicit instantiations of the kernel templates for r = 18..18
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(18, )
}  // namespace pftdev
