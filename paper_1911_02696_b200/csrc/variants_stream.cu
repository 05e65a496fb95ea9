// variants_stream.cu -- stream_kernel instantiations for counts (MODE 0).
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_stream.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
namespace {
using namespace dev;
#define SV(NB, L, VB, H, B, S) {NB, L, VB, H, B, S, 0, stream_kernel<NB, L, VB, H, B, S, 0>}
// two CTAs per SM (<= 128 registers; hint slot 2 marks them): the next launch's
// CTA can share an SM with the previous launch's tail CTA under PDL
#define SV2(NB, L, VB, B, S) {NB, L, VB, 2, B, S, 0, stream_kernel<NB, L, VB, 0, B, S, 0, 2>}
#define SVF(L, VB, B, S) {2, L, VB, 0, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1>}
// FLAG variants that must fit 2 CTAs/SM (<= 128 registers); hint slot = 2 marks them.
#define SVF2(L, VB, B, S) {2, L, VB, 2, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1, 2>}
#define SVB(L, VB, B, S) {3, L, VB, 0, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2>}
#define SVB2(L, VB, B, S) {3, L, VB, 2, B, S, 2, stream_kernel<3, L, VB, 0, B, S, 2, 2>}
// The release library holds the production variants only; the tuning build
// (-DPOSPOP_TUNING) adds the alternatives, selectable through
// POSPOP_STREAM_VARIANT="depth,vb,hint,block,sched".
const StreamVariant kVariants[] = {
    SV(1, 7, 32, 0, 256, 2), SV(2, 6, 32, 0, 256, 2),  // defaults (k <= 32 / k = 64)
    SV(1, 7, 32, 0, 0, 2), SV(2, 6, 32, 0, 0, 2),      // runtime block size (pospopcnt_async block != 0)
#ifdef POSPOP_TUNING  // the tuning build (libpospopcnt_b200_tuning.so): measured alternatives
    SV(1, 7, 32, 0, 256, 0), SV(2, 6, 32, 0, 256, 0),  // static CTA partition
    SV(1, 7, 32, 0, 0, 0), SV(2, 6, 32, 0, 0, 0),
    SV(1, 7, 32, 0, 256, 1), SV(2, 6, 32, 0, 256, 1),  // per-warp guided chunks
    SV(1, 7, 32, 0, 0, 1), SV(2, 6, 32, 0, 0, 1), SV(1, 6, 32, 0, 256, 2), SV(1, 7, 16, 0, 256, 2),
    SV2(1, 6, 32, 256, 2), SV2(1, 5, 32, 256, 2), SV2(2, 5, 32, 256, 2), SV2(1, 6, 16, 256, 2),
#endif
};

#undef SV
#undef SV2
#undef SVF
#undef SVF2
#undef SVB
#undef SVB2
#undef SVF2


}  // namespace

const StreamVariant* stream_variants_counts(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}

}  // namespace pospop_b200
