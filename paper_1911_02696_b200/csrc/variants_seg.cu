// variants_seg.cu -- segmented kernel instantiations.
// (one translation unit per registry so the instantiations compile in parallel)
#include "pospop_segmented.cuh"
#include "pospop_variants.h"

namespace pospop_b200 {
namespace {
using namespace dev;
#define SG(NB, L, VB, S) {NB, L, VB, S, segmented_kernel<NB, L, VB, S>}
#define SGP(NB, L, VB) {NB, L, VB, 2, segmented_pipe_entry<NB, L, VB>}
#define SGP2(NB, L, VB) {NB, L, VB, 3, segmented_pipe_entry<NB, L, VB, 2>}  // sched 3: pipelined, 2 CTAs/SM
#define SGP3(NB, L, VB) {NB, L, VB, 4, segmented_pipe_entry<NB, L, VB, 3>}  // sched 4: pipelined, 3 CTAs/SM
// sched 6: pipelined, bit-plane epilogue, 2 CTAs/SM; sched 7: the same at 3 CTAs/SM
#define SGPE(NB, L, VB) {NB, L, VB, 6, segmented_pipe_entry<NB, L, VB, 2, 1>}
#define SGPE3(NB, L, VB) {NB, L, VB, 7, segmented_pipe_entry<NB, L, VB, 3, 1>}
// sched 10: multi-stage cp.async ring per warp (group field = ring slots S)
#define SGC(NB, L, S) {NB, L, 16, 10, segmented_cpasync_kernel<NB, L, S>, S}
// sched 9: sched 6 with the L2::256B prefetch hint on the 16-byte loads
#define SGPEH(NB, L) {NB, L, 16, 9, segmented_pipe_entry<NB, L, 16, 2, 1, 2>}
// sched 8: adaptive (lane / grouped / pipelined chosen on the device from the mean array length)
#define SGA(NB, L) {NB, L, 16, 8, segmented_auto_kernel<NB>}
// sched 11: warp-per-array tiles, not pipelined (group field = CTAs per SM)
#define SGT(NB, L, VB, MB) {NB, L, VB, 11, segmented_tile_kernel<NB, L, VB, MB, 0>, MB}
// sched 13: sched 11 reading its first array before waiting for the previous launch
#define SGTE(NB, L, VB, MB) {NB, L, VB, 13, segmented_tile_kernel<NB, L, VB, MB, 2>, MB}
// sched 14: sched 13 with the last rounds of arrays claimed dynamically
#define SGTD(NB, L, VB, MB) {NB, L, VB, 14, segmented_tile_kernel<NB, L, VB, MB, 6>, MB}
// sched 16: even byte ranges per warp (the adaptive kernel's range mode)
#define SGR(NB, L, VB, MB) {NB, L, VB, 16, segmented_range_kernel<NB, L, VB, MB>, MB}
// sched 12: the same with one contiguous array range per CTA
#define SGTB(NB, L, VB, MB) {NB, L, VB, 12, segmented_tile_kernel<NB, L, VB, MB, 1>, MB}
// sched 5: grouped, G lanes per array, 2 CTAs/SM
#define SGG(NB, L, VB, G) {NB, L, VB, 5, segmented_group_kernel<NB, L, VB, G, 2>, G}
const SegVariant kVariants[] = {
    SGA(1, 5), SGA(2, 4),                 // the adaptive kernel (default; k <= 32 / k = 64)
    SGR(1, 7, 32, 1), SGR(2, 6, 32, 1),   // range kernel, one CTA per SM (at most one array per SM)
#ifdef POSPOP_TUNING  // the tuning build: measured alternatives (POSPOP_SEG_VARIANT)
    SGT(1, 7, 32, 1), SGT(1, 7, 16, 1), SGT(1, 6, 32, 1), SGT(1, 6, 32, 2), SGT(1, 6, 16, 2), SGT(1, 5, 32, 2),
    SGT(2, 6, 32, 1), SGT(2, 5, 32, 1), SGT(2, 5, 32, 2), SGT(2, 5, 16, 2),
    SGTE(1, 7, 32, 1), SGTE(1, 6, 32, 1), SGTE(1, 6, 32, 2), SGTE(2, 6, 32, 1),
    SGTD(1, 7, 32, 1), SGTD(1, 6, 32, 1), SGTD(1, 6, 32, 2), SGTD(2, 6, 32, 1), SGTD(2, 5, 32, 2), SGTD(2, 5, 16, 2),
    SGTD(1, 6, 16, 2), SGTD(1, 5, 16, 2), SGTD(1, 5, 32, 2),
    SGR(1, 5, 16, 2), SGR(2, 5, 16, 2), SGR(1, 5, 32, 2), SGR(1, 6, 32, 1),
    SGTB(1, 7, 32, 1), SGTB(1, 6, 32, 1), SGTB(1, 6, 32, 2), SGTB(2, 6, 32, 1), SGTB(2, 5, 32, 2), SGPEH(1, 5), SGPEH(1, 4), SGPEH(2, 4),
    SGC(1, 5, 3), SGC(1, 5, 2), SGC(1, 4, 4), SGC(2, 3, 4), SGC(2, 4, 2),
    SGPE(1, 5, 16), SGPE(1, 5, 32), SGPE(1, 4, 16), SGPE(1, 4, 32), SGPE(2, 4, 16), SGPE(2, 4, 32), SGPE(2, 3, 32),
    SGPE3(1, 4, 16), SGPE3(1, 4, 32), SGPE3(2, 3, 16),
    SGG(1, 6, 16, 8), SGG(1, 6, 16, 4), SGG(1, 5, 16, 8), SGG(1, 6, 32, 8), SGG(1, 5, 32, 8), SGG(1, 5, 16, 4),
    SGG(1, 6, 16, 16), SGG(1, 5, 32, 4),
    SGG(2, 4, 16, 8), SGG(2, 4, 32, 8), SGG(2, 4, 16, 4),
    SG(1, 5, 16, 0), SG(2, 5, 16, 1),  // defaults (k <= 32 / k = 64)
    SG(1, 5, 16, 1), SG(2, 5, 16, 0), SG(1, 4, 16, 0), SG(1, 4, 16, 1), SG(1, 5, 32, 0), SG(1, 5, 32, 1),
    SG(2, 4, 16, 0), SG(2, 4, 16, 1), SG(2, 4, 32, 1),
    SGP(1, 5, 16), SGP(1, 4, 16), SGP(1, 4, 32), SGP(1, 5, 32), SGP(2, 4, 16), SGP(2, 3, 32), SGP(2, 4, 32),
    SGP2(2, 4, 16), SGP2(2, 3, 32), SGP2(2, 3, 16), SGP2(1, 5, 16), SGP2(1, 5, 32),
    SGP3(1, 4, 16), SGP3(1, 4, 32), SGP3(1, 5, 16), SGP3(2, 3, 16), SGP3(2, 3, 32),
#endif
};
#undef SGP2
#undef SGP3
#undef SGG
#undef SGT
#undef SGTB
#undef SGTE
#undef SGTD
#undef SGR
#undef SGA
#undef SGPE
#undef SGPE3
#undef SGPEH
#undef SGC
#undef SG
#undef SGP


}  // namespace

#ifdef POSPOP_TUNING
// Diagnostics entry of the tuning build (not in the public header): the
// per-warp trace buffer of the segmented tile mode (NULL = off).  Defined in
// this translation unit because the segmented kernels live in its module.
extern "C" int pospop_tuning_seg_trace(void* d_buf) {
    unsigned long long* p = static_cast<unsigned long long*>(d_buf);
    return (int)cudaMemcpyToSymbol(dev::g_seg_trace, &p, sizeof p);
}
#endif

const SegVariant* seg_variants(size_t* n) {
    *n = sizeof(kVariants) / sizeof(kVariants[0]);
    return kVariants;
}

}  // namespace pospop_b200
