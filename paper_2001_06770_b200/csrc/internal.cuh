// internal.cuh -- libriki.so internal structures shared by graph.cu, engine.cu, api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/riki.h"
#include "common.cuh"

struct Workspace;  // engine.cu

// Vertex-partitioned mode (dist.cu).  Rank r owns the internal-id range
// [bounds[r], bounds[r+1]) and relaxes only the in-edges of its own nodes (pull, owner
// computes); the nodes it reached at level l+1 go into its slice of a bit-plane buffer that
// one in-place all-gather per level makes identical on every rank, after which every rank
// applies all slices to its replicated H.  `simulated`: nranks partitions driven by ONE
// process on one device (every partition's pull runs here, the all-gather is the identity
// because all slices already live in the same buffer) -- the single-GPU test of the
// partitioned arithmetic.
struct DistState {
    int nranks = 1, rank = 0, mode = 0;  // mode 0 replicated (no data-path collective), 1 vertex-partitioned
    bool simulated = false;
    void *comm = nullptr;                // ncclComm_t (real mode)
    std::vector<uint32_t> bounds;        // nranks + 1 internal-id bounds; each a multiple of 32 or V
    uint32_t *d_bounds = nullptr;
    uint32_t wc = 0;                     // u32 words per rank, per slot and bit plane
    uint32_t *d_x = nullptr;             // exchange buffer [rank][pull slot][plane][wc]
    size_t x_words = 0;
    uint64_t exchanges = 0, exchanged_bytes = 0;
    // push mode (default): bit-plane slices every rank ORs into over peer memory (dist.cu)
    bool push = true;
    size_t slice_words = 0;        // words per slice: slots * 8 planes * wc
    uint32_t *d_slices = nullptr;  // simulated: [nranks][slice_words]; real: own slices [3][slice_words]
    uint32_t *d_gather = nullptr;  // real: all-gathered slices [nranks][chunk]
    uint32_t **d_xs = nullptr;     // device pointer table: [3][nranks] slice of each owner per level mod 3
    std::vector<void *> peer_bases;  // real: peers' d_slices opened through CUDA IPC (index = rank)
    uint64_t t = 0;                // level counter of the push exchange (slices rotate mod 3)
    size_t used[3] = {0, 0, 0};    // words written into own slice t mod 3
    int *d_one = nullptr;          // barrier operand
};

// Device view of the resident graph (P:339 CSR).  Out-rows are sorted by activation
// ascending (then by edge id), so the Alg. 1 gate a <= l reads a row prefix.  In-rows
// (Alg. 2 line 5, N_i) are sorted the same way and carry the forward edge's activation
// and the caller's edge id.
// Gate offset table: for out-rows longer than 8 edges (activation-sorted), entry k is the index
// of the first edge with activation > k, k < AOFF_LEVELS: the expansion's gate ranges a <= l and
// a == l are two loads from one 64-byte line instead of two binary searches.
#define AOFF_LEVELS 16

struct GraphDev {
    uint32_t V;
    uint64_t E;
    const uint32_t *row, *col;  // out-CSR
    const uint8_t *act;
    const uint4 *desc;          // per node: {row start, degree, packed activations of rows <= 8 edges
                                //            | index into aoff for longer rows}
    const uint32_t *aoff;       // per row of > 8 edges: AOFF_LEVELS gate offsets (first edge with a > k)
    const uint32_t *irow, *isrc, *ieid;  // in-CSR
    const uint8_t *iact;
    const uint4 *idesc;         // in-rows: same layout as desc
    const uint32_t *iaoff;      // in-rows of > 8 edges: gate offsets
    const uint32_t *src, *dst;  // caller's edge list by edge id
    const uint64_t *tptr;       // inverted index (internal ids)
    const uint32_t *post;
    const uint32_t *perm, *iperm;  // caller id -> internal id (degree-descending), and back
    const unsigned long long *wfix;  // fine weight of each caller edge id as round(w * 2^32) (tie-break R29), or null
    uint32_t Vh;                   // internal ids [0, Vh) have in-degree > 32 (pull: warp per node)
};

struct riki_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint32_t V = 0;
    uint64_t E = 0;
    uint32_t n_terms = 0;
    uint32_t *d_src = nullptr, *d_dst = nullptr, *d_cls = nullptr;
    uint8_t *d_act_e = nullptr;  // activation by caller edge id
    bool has_act = false;
    uint32_t *d_row = nullptr, *d_col = nullptr;
    uint8_t *d_act = nullptr;
    uint4 *d_desc = nullptr;
    uint32_t *d_aoff = nullptr;  // AOFF_LEVELS entries per out-row of more than 8 edges
    uint32_t n_aoff = 0;         // number of such rows
    uint4 *d_idesc = nullptr;    // in-CSR descriptors and gate offsets (recovery, pull)
    uint32_t *d_iaoff = nullptr;
    uint32_t n_iaoff = 0;
    uint32_t *d_irow = nullptr, *d_isrc = nullptr, *d_ieid = nullptr;
    uint8_t *d_iact = nullptr;
    uint64_t *d_tptr = nullptr;
    uint32_t *d_post = nullptr;
    uint32_t *d_perm = nullptr, *d_iperm = nullptr;
    unsigned long long *d_wfix = nullptr;  // set with the fine weights (set_edge/node/label_weights)
    uint32_t Vh = 0;
    std::vector<uint64_t> h_tptr;
    uint64_t graph_bytes = 0;
    Workspace *ws = nullptr;
    bool profiling = false, debug = false, pull_on = false, joint_on = false;
    uint32_t batch_slots = 0;
    riki_stats stats{};
    DistState *dist = nullptr;  // set by riki_dist_init
    std::vector<riki_results *> dev_stash;
    uint32_t *d_qmap = nullptr;  // device batch: query order of the row-width groups
    uint32_t qmap_cap = 0;
    uint64_t arena_limit = 0;  // riki_set_arena_limit (tests): 0 = the 32-bit offset limit
    uint32_t slots_cap = 0;    // chunk size learnt from an arena-limited full-width batch (0 = none)
    uint64_t slots_cap_key = 0;  // ... and the batch shape it applies to (depth, row widths, k)
    // Serialises every call on this handle (riki_rpq_search*, fetch, hitting levels, weights,
    // dist): the workspace, its cached CUDA graphs and the device-batch stash are per handle,
    // so concurrent callers on one graph run one after the other (include/riki.h, Threading).
    mutable std::recursive_mutex mu;
    bool vp() const { return dist && dist->mode == 1; }

    GraphDev dev() const {
        GraphDev g;
        memset(&g, 0, sizeof(g));  // padding too: the struct is part of CUDA-graph cache keys
        g.V = V; g.E = E;
        g.row = d_row; g.col = d_col; g.act = d_act; g.desc = d_desc; g.aoff = d_aoff; g.idesc = d_idesc; g.iaoff = d_iaoff;
        g.irow = d_irow; g.isrc = d_isrc; g.ieid = d_ieid; g.iact = d_iact;
        g.src = d_src; g.dst = d_dst; g.tptr = d_tptr; g.post = d_post; g.perm = d_perm; g.iperm = d_iperm; g.Vh = Vh;
        g.wfix = d_wfix;
        return g;
    }
};

// graph.cu
void graph_load(riki_graph *g, uint32_t n_nodes, uint64_t n_edges, const uint32_t *src, const uint32_t *dst,
                const uint32_t *cls, uint32_t n_terms, const uint64_t *tptr, const uint32_t *post, bool device_inputs);
void graph_free(riki_graph *g);
void graph_set_edge_weights(riki_graph *g, const double *w01, double alpha, double avg);
void graph_set_node_weights(riki_graph *g, const double *w01, double alpha, double avg);
void graph_set_label_weights(riki_graph *g, double alpha, double avg);
void graph_set_act(riki_graph *g, const uint8_t *a);
void graph_get_act(const riki_graph *g, uint8_t *a);
void graph_debug_ln_table(int device, uint64_t n0, uint64_t count, double *out_host);

// engine.cu
struct QueryIn {
    uint32_t nc, nm;
    uint32_t c[RIKI_MAX_TERMS], m[RIKI_MAX_TERMS];
};
struct HostRPG {
    uint32_t central_node, sc, sm;
    double score;
    uint8_t ptc;
    std::vector<uint32_t> nodes, vc;
    std::vector<uint64_t> edges;
    uint8_t cdist[RIKI_MAX_TERMS], mdist[RIKI_MAX_TERMS];
};
struct riki_results {
    uint32_t nc = 0, nm = 0;
    std::vector<HostRPG> rpgs;
    riki_query_stats stats{};
    std::vector<uint64_t> cand;  // (sc << 32 | v), debug only
};
void engine_search(riki_graph *g, const std::vector<QueryIn> &qs, uint32_t k, uint32_t depth, const riki_params &p,
                   cudaStream_t stream, std::vector<riki_results *> *out);
void engine_search_device(riki_graph *g, uint32_t nq, const uint64_t *d_cptr, const uint32_t *d_cterms,
                          const uint64_t *d_mptr, const uint32_t *d_mterms, uint32_t k, uint32_t depth,
                          const riki_params &p);
void engine_fetch(riki_graph *g, uint32_t nq, std::vector<riki_results *> *out);
void engine_hitting_levels(riki_graph *g, const uint32_t *terms, uint32_t T, uint32_t depth, int block_mode,
                           uint8_t *H_out, uint8_t *block_out, uint64_t *relax_out, int32_t *L_out);
void engine_free(riki_graph *g);

// hops.cu
void graph_sample_hops(riki_graph *g, uint32_t n_pairs, const uint32_t *src, const uint32_t *dst, uint32_t max_hops,
                       uint32_t *dist_out);

// dist.cu
void dist_unique_id(void *out128);
void dist_init(riki_graph *g, int nranks, int rank, const void *uid, int mode);
void dist_partition(const uint32_t *irow, uint32_t V, uint32_t nranks, uint32_t *bounds);
uint32_t *dist_exchange_buffer(riki_graph *g, size_t chunk_words);  // [nranks][chunk_words], zeroed by the caller
void dist_allgather(riki_graph *g, uint32_t *x, size_t chunk_words, cudaStream_t s);
void dist_free(riki_graph *g);
// vertex-partitioned push (dist.cu): slices sized for `slots` pull positions; per level t the
// table of owners' slices to OR into, then the exchange that makes every rank's planes visible
void dist_push_setup(riki_graph *g, uint32_t slots);
uint32_t *const *dist_push_targets(riki_graph *g);
const uint32_t *dist_push_exchange(riki_graph *g, size_t chunk_words, cudaStream_t s, size_t *stride);
uint64_t engine_workspace_bytes(const riki_graph *g);
