/*
 * tests/native/tri_count.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Undirected triangle count of a sanitised digraph (arcs -> unordered
 * pairs, loops dropped, duplicates merged), for the triangle rows of the
 * linear census identities: sum over classes with
 * three connected pairs = T, with two = sum_u C(d_u,2) - 3T, and
 * 012 + 102 = D n - sum d^2 + 3T.  Independent of both census
 * implementations: the classic forward algorithm (orient every edge from
 * the lower to the higher (degree, id) rank; every triangle is found once,
 * at its lowest-ranked vertex, by marking that vertex's out-neighbours).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* Returns T, or UINT64_MAX on allocation failure. */
uint64_t tri_count(uint64_t n, const uint32_t *src, const uint32_t *dst, uint64_t m)
{
    uint64_t *pk = (uint64_t *)malloc((m ? m : 1) * sizeof(uint64_t));
    if (!pk) return UINT64_MAX;
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; i++) {
        uint64_t a = src[i], b = dst[i];
        if (a == b) continue;
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        pk[k++] = (lo << 32) | hi;
    }
    qsort(pk, k, sizeof(uint64_t), cmp_u64);
    uint64_t D = 0;
    for (uint64_t i = 0; i < k; i++)
        if (i == 0 || pk[i] != pk[i - 1]) pk[D++] = pk[i];
    uint64_t *deg = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
    uint64_t *off = (uint64_t *)calloc(n + 2, sizeof(uint64_t));
    uint32_t *col = (uint32_t *)malloc((D ? D : 1) * sizeof(uint32_t));
    uint64_t *mark = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!deg || !off || !col || !mark) {
        free(pk); free(deg); free(off); free(col); free(mark);
        return UINT64_MAX;
    }
    for (uint64_t i = 0; i < D; i++) {
        deg[pk[i] >> 32]++;
        deg[pk[i] & 0xffffffffu]++;
    }
    /* x precedes y in rank if (deg, id) is smaller */
#define RANK_LT(x, y) (deg[x] < deg[y] || (deg[x] == deg[y] && (x) < (y)))
    for (uint64_t i = 0; i < D; i++) {
        uint64_t a = pk[i] >> 32, b = pk[i] & 0xffffffffu;
        off[(RANK_LT(a, b) ? a : b) + 1]++;
    }
    for (uint64_t v = 0; v < n; v++) off[v + 1] += off[v];
    uint64_t *pos = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    if (!pos) {
        free(pk); free(deg); free(off); free(col); free(mark);
        return UINT64_MAX;
    }
    memcpy(pos, off, (n + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < D; i++) {
        uint64_t a = pk[i] >> 32, b = pk[i] & 0xffffffffu;
        if (RANK_LT(a, b)) col[pos[a]++] = (uint32_t)b;
        else col[pos[b]++] = (uint32_t)a;
    }
#undef RANK_LT
    for (uint64_t v = 0; v < n; v++) mark[v] = UINT64_MAX;
    uint64_t T = 0;
    for (uint64_t u = 0; u < n; u++) {
        for (uint64_t i = off[u]; i < off[u + 1]; i++) mark[col[i]] = u;
        for (uint64_t i = off[u]; i < off[u + 1]; i++) {
            uint64_t v = col[i];
            for (uint64_t j = off[v]; j < off[v + 1]; j++)
                if (mark[col[j]] == u) T++;
        }
    }
    free(pk); free(deg); free(off); free(col); free(mark); free(pos);
    return T;
}
