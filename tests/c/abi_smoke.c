/* Plain-C client of libriki.so through include/riki.h only (no Python, no torch): loads the
 * 5-node worked example of SPEC S:365/S:548 (tests/golden/five_node.json; one
 * RPG with S^c = 2, S^m = 2, S^r = 2.0, directed edges {k1->v, k2->v, m->k1}), sets exact
 * activation levels, runs
 * one search and one batch, and prints the results.  Exit code 0 iff they match. */
#include <stdio.h>
#include <string.h>

#include "riki.h"

#define CHECK(x)                                                                   \
    do {                                                                           \
        riki_status s_ = (x);                                                      \
        if (s_ != RIKI_OK) {                                                       \
            fprintf(stderr, "%s failed: %d %s\n", #x, (int)s_, riki_last_error()); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(void) {
    /* tests/golden/five_node.json: nodes 0 = k1, 1 = v, 2 = k2, 3 = m, 4 = x; undirected
     * edges k1-v, v-k2, m-k1 (a = 1) and x-k2 (a = 7), each as two directed edges 2i, 2i+1 */
    const uint32_t und[4][3] = {{0, 1, 1}, {1, 2, 1}, {3, 0, 1}, {4, 2, 7}};
    uint32_t src[8], dst[8];
    uint8_t act[8];
    for (int i = 0; i < 4; i++) {
        src[2 * i] = und[i][0]; dst[2 * i] = und[i][1];
        src[2 * i + 1] = und[i][1]; dst[2 * i + 1] = und[i][0];
        act[2 * i] = act[2 * i + 1] = (uint8_t)und[i][2];
    }
    const uint64_t tptr[4] = {0, 1, 2, 3};
    const uint32_t post[3] = {0, 2, 3}; /* term 0 = k1, term 1 = k2, term 2 = m */
    riki_graph *g = NULL;
    CHECK(riki_load_graph(0, 5, 8, src, dst, NULL, 3, tptr, post, &g));
    CHECK(riki_set_activation_levels(g, act));
    const uint32_t central[2] = {0, 1}, marginal[1] = {2};
    riki_results *r = NULL;
    CHECK(riki_rpq_search(g, central, 2, marginal, 1, 1, 20, NULL, NULL, &r));
    int ok = riki_results_count(r) == 1;
    if (ok) {
        riki_rpg x;
        CHECK(riki_results_get(r, 0, &x));
        printf("rpg central=%u sc=%u sm=%u score=%.3f nodes=%u edges=", x.central_node, x.sc, x.sm, x.score,
               x.n_nodes);
        uint32_t want = 0;
        for (uint32_t i = 0; i < x.n_edges; i++) {
            uint64_t e = x.edge_ids[i];
            printf("%u->%u ", src[e], dst[e]);
            if ((src[e] == 0 && dst[e] == 1) || (src[e] == 2 && dst[e] == 1) || (src[e] == 3 && dst[e] == 0)) want++;
        }
        printf("\n");
        ok = x.central_node == 1 && x.sc == 2 && x.sm == 2 && x.score == 2.0 && x.n_edges == 3 && want == 3;
    }
    riki_results_free(r);
    /* the same query as a 2-query batch: both answers identical */
    const uint64_t cptr[3] = {0, 2, 4}, mptr[3] = {0, 1, 2};
    const uint32_t cterms[4] = {0, 1, 0, 1}, mterms[2] = {2, 2};
    riki_results *rb[2] = {NULL, NULL};
    CHECK(riki_rpq_search_batch(g, 2, cptr, cterms, mptr, mterms, 1, 20, NULL, rb));
    for (int q = 0; q < 2; q++) {
        riki_rpg x;
        ok = ok && riki_results_count(rb[q]) == 1 && riki_results_get(rb[q], 0, &x) == RIKI_OK && x.central_node == 1 &&
             x.score == 2.0;
        riki_results_free(rb[q]);
    }
    /* error path: an empty central set */
    riki_results *re = NULL;
    ok = ok && riki_rpq_search(g, central, 0, marginal, 1, 1, 20, NULL, NULL, &re) == RIKI_EEMPTY_CENTRAL;
    riki_free_graph(g);
    printf("%s\n", ok ? "ABI_SMOKE_OK" : "ABI_SMOKE_FAIL");
    return ok ? 0 : 1;
}
