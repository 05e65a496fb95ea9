// pospop_variants.h -- registries of the tuned kernel instantiations.
// Each registry lives in its own translation unit (variants_*.cu) so the
// instantiations compile in parallel; pospop_kernels.cu picks from them.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "pospop_stream.cuh"

namespace pospop_b200 {

using StreamKernel = void (*)(const dev::StreamArgs);

// stream_kernel<NBANK, L, VB, HINT, BLOCK, SCHED, MODE, MINB>; hint slot 2 marks
// MINB = 2 instantiations of the FLAG modes.
struct StreamVariant {
    int nbank, depth, vb, hint, block, sched, mode;
    StreamKernel fn;
};

// TMA-staged variants (SCHED 3): (nbank, depth, mode, consumer warps, ring stages).
struct TmaVariant {
    int nbank, depth, mode, nc, stages;
    StreamKernel fn;
    size_t smem;  // dynamic shared memory: stages x stage bytes
};

using SegKernel = void (*)(const uint8_t*, const unsigned long long*, unsigned long long, int, uint32_t,
                           unsigned long long*, unsigned long long*, unsigned int*, unsigned);

struct SegVariant {
    int nbank, depth, vb, sched;
    SegKernel fn;
    int group = 0;  // sched 5: lanes per array
};

const StreamVariant* stream_variants_counts(size_t* n);  // MODE 0      (variants_stream.cu)
const StreamVariant* stream_variants_flag16(size_t* n);  // MODE 1      (variants_flag1.cu)
const StreamVariant* stream_variants_flag8(size_t* n);   // MODE 2      (variants_flag2.cu)
const TmaVariant* tma_variants(size_t* n);                // SCHED 3     (variants_tma.cu)
const TmaVariant* ring_variants(size_t* n);               // SCHED 6     (variants_ring.cu; nc = warps per CTA)
const SegVariant* seg_variants(size_t* n);                // segmented   (variants_seg.cu)

}  // namespace pospop_b200
