// kinst_r09_11.cu -- explicit instantiations of the kernel templates for r = 9..11
// (one translation unit per group so the build compiles them in parallel).
#include "kernel_templates.cuh"

namespace pftdev {
PFT_INSTANCES(9, )
PFT_INSTANCES(10, )
PFT_INSTANCES(11, )
}  // namespace pftdev
