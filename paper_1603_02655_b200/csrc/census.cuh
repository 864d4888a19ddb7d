#pragma once
#include "tc_internal.cuh"

namespace tc {

// Work lists of the degree-binned scheduler (a2), device pointers.
struct BinLists {
    const BinItem2 *t = nullptr;   // thread bin: one thread per dyad
    const BinItem2 *w = nullptr;   // warp bin: one warp per dyad
    const BinItem4 *b = nullptr;   // block bin: one block per <= kBlockSpan diagonals
    uint64_t count[kNumBins] = {0, 0, 0};
};

// a3 + a4: launches the bin kernels; ADDS classes 2..16 into d_counts[1..15]
tc_status launch_bins(const tc_graph *g, const BinLists &bl, cudaStream_t s, uint64_t *d_counts,
                      tc_profile *prof, uint64_t *launches);

}  // namespace tc
