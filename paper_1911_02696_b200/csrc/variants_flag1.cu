// variants_flag1.cu -- stream_kernel instantiations for FLAG statistics, 16-bit lanes (MODE 1).
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_stream.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
#ifdef POSPOP_TUNING  // tuning build only: the release library has no 16-bit-lane FLAG kernel
namespace {
using namespace dev;
#define SV(NB, L, VB, H, B, S) {NB, L, VB, H, B, S, 0, stream_kernel<NB, L, VB, H, B, S, 0>}
#define SVF(L, VB, B, S) {2, L, VB, 0, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1>}
// FLAG variants that must fit 2 CTAs/SM (<= 128 registers); hint slot = 2 marks them.
#define SVF2(L, VB, B, S) {2, L, VB, 2, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1, 2>}
#define SVB(L, VB, B, S) {3, L, VB, 0, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2>}
#define SVB2(L, VB, B, S) {3, L, VB, 2, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2, 2>}
// Production variants first (the defaults), then tuning variants selectable
// through POSPOP_STREAM_VARIANT="depth,vb,hint,block,sched" (POSPOP_FLAG_VARIANT
// for MODE 1).
const StreamVariant kVariants[] = {
    SVF(6, 32, 512, 2), SVF(6, 32, 0, 2),               // FLAG statistics defaults (16 warps/SM)
    SVF(6, 32, 256, 2), SVF(5, 32, 512, 2),
    SVF(5, 32, 256, 2), SVF(6, 16, 256, 2), SVF(7, 32, 256, 2),
    SVF2(5, 32, 256, 2), SVF2(5, 16, 256, 2), SVF2(4, 32, 256, 2), SVF(4, 32, 512, 2), SVF(5, 16, 512, 2),
    SVF2(6, 32, 256, 2), SVF(4, 32, 1024, 2),
};

#undef SV
#undef SVF
#undef SVF2
#undef SVB
#undef SVB2
#undef SVF2


}  // namespace

const StreamVariant* stream_variants_flag16(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}
#else
const StreamVariant* stream_variants_flag16(size_t* n) {
    *n = 0;
    return nullptr;
}
#endif

}  // namespace pospop_b200
