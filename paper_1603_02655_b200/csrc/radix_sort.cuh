#pragma once
#include "tc_internal.cuh"

namespace tc {

struct RadixPass {
    int shift;   // lowest bit of the digit
    int bits;    // digit width, 1..8
};

// Stable LSD sort of keys[0..n) by the digits in `passes` (least significant
// first).  tmp must hold n keys; *sorted receives keys or tmp.
tc_status radix_sort_u64(Mem &mem, uint64_t *keys, uint64_t *tmp, size_t n,
                         const RadixPass *passes, int npasses, cudaStream_t s,
                         uint64_t *launches, uint64_t **sorted);

// passes covering bits [lo, lo + width) with digits of at most 8 bits
int radix_passes_for(int lo, int width, RadixPass *out);

}  // namespace tc
