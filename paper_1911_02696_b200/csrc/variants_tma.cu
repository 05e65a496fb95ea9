// variants_tma.cu -- TMA-staged stream kernel instantiations (SCHED 3).
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_stream.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
#ifdef POSPOP_TUNING  // tuning build only: the release library has no TMA-staged variants
namespace {
using namespace dev;
#define TV(NB, L, M, NC, ST)                                                                \
    {NB, L, M, NC, ST, stream_tma_kernel<NB, L, M, NC, ST>,                               \
     (size_t)(ST) * (NC) * 32 * (((M) == 1 ? (1 << (L)) : (M) == 2 ? (2 << (L)) : ((NB) << (L))) / 4) * 16}
const TmaVariant kVariants[] = {
    TV(1, 5, 0, 8, 6), TV(1, 6, 0, 8, 3), TV(1, 5, 0, 8, 4), TV(1, 4, 0, 8, 6), TV(1, 5, 0, 4, 6),
    TV(2, 4, 0, 8, 6), TV(2, 5, 0, 8, 3),
    TV(2, 5, 1, 8, 6), TV(2, 4, 1, 8, 6), TV(2, 6, 1, 8, 3), TV(2, 5, 1, 16, 3), TV(2, 4, 1, 16, 6),
    TV(2, 5, 1, 12, 4),
    TV(3, 5, 2, 12, 2), TV(3, 5, 2, 8, 3), TV(3, 4, 2, 15, 3), TV(3, 4, 2, 12, 4), TV(3, 4, 2, 8, 6),
};
#undef TV


}  // namespace

const TmaVariant* tma_variants(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}
#else
const TmaVariant* tma_variants(size_t* n) {
    *n = 0;
    return nullptr;
}
#endif

}  // namespace pospop_b200
