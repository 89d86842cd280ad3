// kinst_r06_08.cu -- explicit instantiations of the kernel templates for r = 6..8
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(6, )
PFT_INSTANCES(7, )
PFT_INSTANCES(8, )
}  // namespace pftdev
