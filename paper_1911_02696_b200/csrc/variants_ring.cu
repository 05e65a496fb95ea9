// variants_ring.cu -- per-warp bulk-copy ring instantiations (SCHED 6,
// stream_ring_kernel): (nbank, depth, mode, warps per CTA, slots per warp).
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_stream.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
namespace {
using namespace dev;
#define RV(NB, L, M, NW, S)                                                       \
    {NB, L, M, NW, S, stream_ring_kernel<NB, L, M, NW, S>,                        \
     (size_t)(NW) * (S) * 32 * (size_t)((M) == 2 ? (2 << (L)) : ((NB) << (L))) * 4}
const TmaVariant kVariants[] = {
    RV(3, 5, 2, 16, 1),  // FLAG statistics default (byte frame, depth 5, 16 warps x 1 slot)
#ifdef POSPOP_TUNING  // the tuning build: measured alternatives (POSPOP_RING="warps,slots")
    RV(3, 5, 2, 12, 2), RV(3, 5, 2, 8, 3), RV(3, 4, 2, 16, 2), RV(3, 4, 2, 16, 3),
    RV(1, 7, 0, 8, 1), RV(1, 7, 0, 4, 3), RV(1, 6, 0, 16, 1), RV(1, 6, 0, 12, 2), RV(2, 6, 0, 8, 1),
#endif
};
#undef RV
}  // namespace

const TmaVariant* ring_variants(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}
}  // namespace pospop_b200
