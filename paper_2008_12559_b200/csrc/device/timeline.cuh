// timeline.cuh -- optional per-CTA phase timestamps for development builds (-DPFT_TIMELINE).
// Product builds compile every PFT_STAMP* to nothing; tools/timeline.py reads the rings back
// through pft_debug_timeline / pft_debug_timeline2 from a -DPFT_TIMELINE build.
#pragma once

#ifdef PFT_TIMELINE
#include <cuda_runtime.h>
namespace pftdev {
// Development instrumentation: per-CTA %globaltimer stamps at phase boundaries, kept for the
// last 4 executes (ring indexed by the launch sequence number) so a PDL chain can be read back.
__device__ unsigned long long g_pft_timeline[4][4096][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PFT_STAMP(slot) \
    if (threadIdx.x == 0 && blockIdx.x + blockIdx.y * gridDim.x < 4096) \
        g_pft_timeline[P.tl_seq & 3][blockIdx.x + blockIdx.y * gridDim.x][slot] = gtimer();
__device__ unsigned long long g_pft_timeline2[4][4096][6];
#define PFT_STAMP2(slot) \
    if (threadIdx.x == 0 && blockIdx.x + blockIdx.y * gridDim.x < 4096) \
        g_pft_timeline2[P.tl_seq & 3][blockIdx.x + blockIdx.y * gridDim.x][slot] = gtimer();
// K2-tail worker k of signal 0 (k1_k2_tail)
#define PFT_STAMPW(k, slot) \
    if (threadIdx.x == 0 && blockIdx.y == 0 && (k) < 4096) g_pft_timeline2[P.tl_seq & 3][(k)][slot] = gtimer();
}  // namespace pftdev
#else
#define PFT_STAMP(slot)
#define PFT_STAMP2(slot)
#define PFT_STAMPW(k, slot)
#endif
