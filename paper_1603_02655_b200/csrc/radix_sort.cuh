#pragma once
#include "tc_internal.cuh"

namespace tc {

struct RadixPass {
    int shift;   // lowest bit of the digit
    int bits;    // digit width, 1..8
};

// Arc list the first pass reads instead of keys (csr_build.cu): nv = vertex
// count; scratch[0] = min index of an out-of-range arc (init ~0), scratch[1]
// += arcs dropped (self-loops + out of range).
struct ArcSource {
    const uint32_t *src, *dst;
    uint64_t nv;
    unsigned long long *scratch;
};

// Stable LSD sort of keys[0..n) by the digits in `passes` (least significant
// first).  tmp must hold n keys; *sorted receives keys or tmp.  With `arcs`,
// the keys of pass 0 are the canonical arc keys computed on the fly (keys'
// contents are ignored; npasses >= 1).  With `dn`, the key count is *dn
// (device memory, read by the kernels; n is then its host-side upper bound
// and sizes the launches), so the caller needs no host round trip.
tc_status radix_sort_u64(Mem &mem, uint64_t *keys, uint64_t *tmp, size_t n,
                         const RadixPass *passes, int npasses, cudaStream_t s,
                         uint64_t *launches, uint64_t **sorted,
                         const ArcSource *arcs = nullptr, const uint32_t *dn = nullptr);

// passes covering bits [lo, lo + width) with digits of at most 8 bits
int radix_passes_for(int lo, int width, RadixPass *out);

}  // namespace tc
