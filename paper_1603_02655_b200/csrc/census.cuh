#pragma once
#include "tc_internal.cuh"

namespace tc {

// Work lists of the degree-binned scheduler (a2), all device memory.  The
// item counts stay on the device (the kernels read them), so planning and
// the census need no host round trip.
struct BinLists {
    const BinItemT *t = nullptr;            // thread bin: tile-local lists sorted by length
    const uint32_t *t_count = nullptr;      // device: thread-bin items per tile
    uint64_t ntiles = 0;                    // tiles of kPlanTile canonical dyads
    const BinItemW *w = nullptr;            // warp bin: <= kWarpChunk diagonals per item
    const unsigned long long *w_count = nullptr;   // device: number of warp-bin items
    unsigned long long *cursor = nullptr;   // device, zeroed: thread-bin unit dispatch cursor
    unsigned long long *wcursor = nullptr;  // device, zeroed: warp-bin item dispatch cursor
    const uint32_t *du = nullptr, *de = nullptr, *dpb = nullptr;   // dyad arrays of the range
    const uint64_t *tagpre = nullptr;       // tag prefix counts (skewed-pair items) or null
};

constexpr int kCensusThreads = 256;
constexpr int kPlanThreads = 256;
constexpr int kPlanItems = 16;
constexpr int kPlanTile = kPlanThreads * kPlanItems;   // canonical dyads per plan tile
static_assert(kPlanTile == kPlanTileItems, "plan tile size");


// a3 + a4: launches the bin kernels; ADDS classes 2..16 into d_counts[1..15]
// (mode64: TriadCodes 1..63 into d_counts[1..63])
tc_status launch_bins(const tc_graph *g, const BinLists &bl, cudaStream_t s, uint64_t *d_counts,
                      cudaEvent_t *ev /* 4 events or null */, uint64_t *launches, int mode64);

}  // namespace tc
