// Host-side reverse Cuthill-McKee (reference: pkg/src/mpkrylov/reorder.py:22-63),
// native so that reordering the paper's SuiteSparse-size matrices (10^6-10^7
// vertices) is a C++ BFS, not a per-vertex Python loop.
//
// Semantics (identical permutation to the reference): the input is the
// symmetrized off-diagonal pattern (row-sorted CSR); components are rooted
// at the unvisited vertex of smallest (degree, index); BFS appends each
// vertex's unvisited neighbours ordered by (degree, index); every
// component's segment is reversed; components keep their discovery order.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

extern "C" int mpk_rcm_host(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *perm) {
    if (n < 0 || (n > 0 && (!indptr || !perm))) return -1;
    std::vector<int64_t> deg(n);
    for (int64_t v = 0; v < n; ++v) deg[v] = indptr[v + 1] - indptr[v];
    std::vector<int64_t> sweep(n);
    std::iota(sweep.begin(), sweep.end(), 0);
    std::stable_sort(sweep.begin(), sweep.end(), [&](int64_t a, int64_t b) { return deg[a] < deg[b]; });
    std::vector<char> seen(n, 0);
    std::vector<int64_t> nb;
    int64_t pos = 0, at = 0;
    while (pos < n) {
        while (seen[sweep[at]]) ++at;
        const int64_t comp = pos;
        const int64_t root = sweep[at];
        seen[root] = 1;
        perm[pos++] = root;
        for (int64_t head = comp; head < pos; ++head) {
            const int64_t u = perm[head];
            nb.clear();
            for (int64_t p = indptr[u]; p < indptr[u + 1]; ++p)
                if (!seen[indices[p]]) nb.push_back(indices[p]);
            // (degree, index): the adjacency is index-sorted, so a stable
            // sort by degree keeps index order within equal degrees
            std::stable_sort(nb.begin(), nb.end(), [&](int64_t a, int64_t b) { return deg[a] < deg[b]; });
            for (int64_t v : nb) {
                seen[v] = 1;
                perm[pos++] = v;
            }
        }
        std::reverse(perm + comp, perm + pos);
    }
    return 0;
}
