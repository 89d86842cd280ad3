// kinst_r16_17.cu -- explicit instantiations of the kernel templates for r = 16..17
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(16, )
PFT_INSTANCES(17, )
}  // namespace pftdev
