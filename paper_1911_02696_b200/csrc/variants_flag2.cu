// variants_flag2.cu -- stream_kernel instantiations for FLAG statistics, byte frame (MODE 2).
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_stream.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
namespace {
using namespace dev;
#define SV(NB, L, VB, H, B, S) {NB, L, VB, H, B, S, 0, stream_kernel<NB, L, VB, H, B, S, 0>}
#define SVF(L, VB, B, S) {2, L, VB, 0, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1>}
// FLAG variants that must fit 2 CTAs/SM (<= 128 registers); hint slot = 2 marks them.
#define SVF2(L, VB, B, S) {2, L, VB, 2, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1, 2>}
#define SVB(L, VB, B, S) {3, L, VB, 0, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2>}
#define SVB2(L, VB, B, S) {3, L, VB, 2, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2, 2>}
// The release library holds the production variants only; the tuning build
// (-DPOSPOP_TUNING) adds the alternatives (POSPOP_FLAG_VARIANT).
const StreamVariant kVariants[] = {
    // byte-frame FLAG statistics (MODE 2): defaults first
    SVB(5, 32, 0, 2),  // runtime block size (explicit grid / block; the default is the ring kernel, sched 6)
#ifdef POSPOP_TUNING  // the tuning build: measured alternatives (POSPOP_FLAG_VARIANT)
    SVB(5, 32, 512, 2),  // the LDG kernel, default until r02
    SVB(5, 32, 256, 2), SVB(4, 32, 512, 2), SVB(4, 32, 256, 2), SVB2(4, 32, 256, 2),
    SVB(4, 16, 512, 2), SVB(6, 32, 256, 2), SVB(5, 16, 512, 2), SVB2(5, 32, 256, 2),
    SVB(4, 32, 512, 4), SVB(4, 16, 512, 4), SVB(3, 32, 512, 4), SVB(4, 32, 256, 4), SVB2(3, 32, 256, 4),
    SVB(5, 32, 256, 4), SVB(5, 32, 512, 5), SVB(5, 16, 512, 5), SVB(6, 32, 256, 5),
#endif
};

#undef SV
#undef SVF
#undef SVF2
#undef SVB
#undef SVB2
#undef SVF2


}  // namespace

const StreamVariant* stream_variants_flag8(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}

}  // namespace pospop_b200
