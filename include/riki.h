/*
 * riki.h -- C-ABI of libriki.so, the B200 (sm_100a) hot path of RIKI radial-pattern
 * keyword search (Yang & Tung, "Efficient Radial Pattern Keyword Search on Knowledge
 * Graphs in Parallel", arXiv 2001.06770).  "P:n" cites PAPER.md line n; "R<n>" the
 * readings listed in DESIGN.md §3.
 *
 * Conventions (all entry points)
 *   - Return riki_status: 0 = RIKI_OK, < 0 = error.  Never throw, never abort; a
 *     thread-local message is available from riki_last_error().
 *   - Node ids are dense uint32 in [0, n_nodes); edge ids are the caller's indices into
 *     the directed edge list given to riki_load_graph (multi-edges stay distinct, R24).
 *   - "host" pointers are ordinary CPU memory, "device" pointers are CUDA global memory
 *     on the graph's device.  Inputs are only read; the library copies what it keeps.
 *   - There is no CPU fallback: every step of the search runs in CUDA kernels; without a
 *     usable sm_100 device the calls return RIKI_ECUDA.
 *   - Infinity for a hitting level is 0xFF; finite levels are <= depth <= 254 (R8).
 *   - Threading: every call on a graph handle holds that handle's lock, so one handle
 *     serves concurrent callers (threads) safely -- their searches run one after the other
 *     on the handle's device workspace (the GPU is saturated by one lock-step batch; use one
 *     handle per device and batch the queries).  Different handles are independent.
 *     riki_set_*_weights may be called between searches; it too takes the lock.
 *   - Result order (Def. RPKSP, Eq. 6): ascending (S^r, S^c, v) with v the
 *     caller's central node id (R23).  This departs from SPEC.md's RankedResult order
 *     (S^r, edge-weight sum, v) in two ways, both documented readings: S^c is the secondary
 *     key (central focus first: of two RPGs with equal S^r the one whose CG is tighter wins,
 *     e.g. S^c = 2 / S^m = 4 before S^c = 4 / S^m = 2 at gamma = 0.5), and the paper's
 *     weight-sum re-ranking is opt-in (tie_break = 1: (S^r, S^c, W, v)).
 */
#ifndef RIKI_H
#define RIKI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RIKI_OK = 0,
    RIKI_EINVAL = -1,          /* bad argument (null pointer, id out of range, k == 0, ...)     */
    RIKI_ENOMEM = -2,          /* device or host allocation failed / workspace overflow          */
    RIKI_ECUDA = -3,           /* CUDA runtime error (message has the CUDA error string)         */
    RIKI_EEMPTY_CENTRAL = -4,  /* C = empty set; Def. RPQ requires C != empty            */
    RIKI_EUNRESOLVED = -5,     /* a query term has an empty posting list (message names it)      */
    RIKI_ENOWEIGHTS = -6,      /* search before activation levels were set                       */
    RIKI_EDEPTH = -7,          /* depth > 254                                                    */
    RIKI_ENCCL = -8,           /* NCCL could not be loaded or a collective failed (riki_dist_*)  */
    RIKI_ENOSYS = -9           /* not implemented in this build                                  */
} riki_status;

#define RIKI_MAX_TERMS 8       /* keywords per phase (central or marginal), T <= 8              */
#define RIKI_MAX_DEPTH 254

typedef struct riki_graph riki_graph;     /* opaque, device-resident, owned by the library */
typedef struct riki_results riki_results; /* opaque, host-resident, owned by the library   */

/* ---------------------------------------------------------------------------------------
 * Graph residency (CSR "pre-stored in the main memory of ... a GPU").
 * The caller's edge list is directed and ALREADY bidirected: one reverse edge per original
 * triple.  label_class[e] identifies the edge's label class (label, inverse flag;
 * R3) and is used only by riki_set_label_weights.  term_ptr/postings is the keyword ->
 * node inverted index (replaces MongoDB; R28): the posting list of term t is
 * postings[term_ptr[t] .. term_ptr[t+1]), sorted ascending, unique.  All inputs are host
 * pointers and are copied; the caller keeps ownership.  n_edges must be < 2^32.
 * Errors: RIKI_EINVAL (null/out of range ids, unsorted postings), RIKI_ENOMEM, RIKI_ECUDA.
 * ------------------------------------------------------------------------------------- */
riki_status riki_load_graph(int device, uint32_t n_nodes, uint64_t n_edges,
                            const uint32_t *src, const uint32_t *dst, const uint32_t *label_class,
                            uint32_t n_terms, const uint64_t *term_ptr, const uint32_t *postings,
                            riki_graph **out);
/* Same, with every array a DEVICE pointer on `device` (e.g. torch tensors): the inputs are
 * validated on the device and copied device-to-device (the CSR build reorders them anyway),
 * so the caller may free them after the call.  term_ptr is also read back to the host
 * (n_terms + 1 words).  Errors as riki_load_graph (without the offending index). */
riki_status riki_load_graph_device(int device, uint32_t n_nodes, uint64_t n_edges,
                                   const uint32_t *src, const uint32_t *dst, const uint32_t *label_class,
                                   uint32_t n_terms, const uint64_t *term_ptr, const uint32_t *postings,
                                   riki_graph **out);
void riki_free_graph(riki_graph *g);

/* ---------------------------------------------------------------------------------------
 * Edge activation levels a_e.  Each setter computes a_e on the device and
 * re-sorts every CSR row by activation (rows are stored activation-ascending so that the
 * gate a_e <= l of Alg. 1 line 9 reads only a row prefix).  Not on the query path.
 *
 * riki_set_edge_weights: w01[n_edges] (host, fine weights already rescaled to [0,1],
 *   P:194) -> a_e = Rounding(A - A(alpha-w)/alpha) if w <= alpha else
 *   Rounding(A + A(w-alpha)/(1-alpha)) (Eq. 1-3, half-up rounding R1, fp64 in exactly that
 *   operation order R5).  0 < alpha < 1, avg_hops > 0 (the raw average A, R4).
 * riki_set_node_weights: w01[n_nodes] (host); node-weighted special case
 *   a(f->n) = coarsen(w[n]) (north star "set_node_weights"; P:196 contrasts node weighting).
 * riki_set_label_weights: computes the fine weights on the device from label classes,
 *   w_ij = ln(#out-edges of v_i in class(e) + #in-edges of v_j in class(e)) (both
 *   counts include e, R3), min-max rescaled (all 0 if max == min, R2), then Eq. 1-3.
 * riki_set_activation_levels: a[n_edges] (host) given directly (exact control, tests).
 * riki_get_activation_levels: copies a_e (by caller edge id) to host a[n_edges].
 * Errors: RIKI_EINVAL (alpha/avg out of range, null), RIKI_ENOMEM, RIKI_ECUDA.
 * ------------------------------------------------------------------------------------- */
riki_status riki_set_edge_weights(riki_graph *g, const double *w01, double alpha, double avg_hops);
riki_status riki_set_node_weights(riki_graph *g, const double *w01, double alpha, double avg_hops);
riki_status riki_set_label_weights(riki_graph *g, double alpha, double avg_hops);
riki_status riki_set_activation_levels(riki_graph *g, const uint8_t *a);
riki_status riki_get_activation_levels(const riki_graph *g, uint8_t *a);

/* Debug / verification boundary for the coarsening's only transcendental step (R2):
 * out[i] = the device's ln(n0 + i) exactly as the fine-weight kernel computes ln(cA + cB),
 * for i < count (host out[count]; n0 >= 1).  A test compares it bit for bit with the
 * oracle's libm log over the whole integer domain label counts can take.  Errors:
 * RIKI_EINVAL, RIKI_ECUDA. */
riki_status riki_debug_ln_table(int device, uint64_t n0, uint64_t count, double *out);

/* ---------------------------------------------------------------------------------------
 * Search parameters (defaults in brackets; riki_params_default fills them).
 *   gamma      Eq. 6 weight [0.5, R22]
 *   beam_w     beam width w of the first level [0 -> w = k]
 *   beam_mode  0 = keep every CG identified by the terminating level (ties, R13) [0];
 *              1 = truncate the candidate CGs to the first w by (S^c, v)
 *   tie_break  0 = (S^r, S^c, v) ascending (R23) [0]; 1 = (S^r, S^c, W, v), W = sum of the
 *              fine weights of the result's distinct edges as round(w * 2^32) (P:293 re-ranking,
 *              R29; needs set_edge/node/label_weights, else RIKI_ENOWEIGHTS); with beam_mode 1
 *              the beam keeps the w smallest (S^c, W(CG), v)
 *   ptc_mode   0 = filter PTC failures, RPG-wide endpoint-inclusive (R19') [0];
 *              1 = keep failures, flagged ptc = 0; 2 = filter, PTC evaluated on G^m only;
 *              3 = filter, SPEC's exclusive form (V_C-resident marginal nodes never qualify)
 *   early_term 0 = exact bound (R21) [0]; 1 = the paper's literal inequality (Theorem
 *              earlyTermination P:375-378): it reduces to S^c(kth) <= min S^c(unattached) and
 *              is exact for gamma < 1, but at gamma = 1 it can stop before an equal-score CG
 *              with a smaller id attaches (tests/golden/early_term_literal_gamma1.json);
 *              2 = none (exhaustive)
 * ------------------------------------------------------------------------------------- */
typedef struct {
    double gamma;
    uint32_t beam_w;
    int beam_mode;
    int tie_break;
    int ptc_mode;
    int early_term;
} riki_params;
void riki_params_default(riki_params *p);

/* ---------------------------------------------------------------------------------------
 * Radial Pattern Query search (Def. RPQ, Def. RPKSP).
 * central[n_central] / marginal[n_marginal] are TERM ids (host).  1 <= n_central <= 8,
 * 0 <= n_marginal <= 8 (M = empty returns the top-k CGs).  k >= 1 results;
 * depth = maximum Glevel D (<= 254; paper default 20).  Runs, on the device:
 * central run (seed, level loop of enqueue / identification / Alg. 1 expansion with CF
 * blocking, termination at >= w CGs) -> candidate CGs -> Alg. 2 recovery of each CG ->
 * marginal run (fresh H, stop rule for |M| >= 2, attach, RPG recovery + PTC, exact early
 * termination) -> top-k by (S^r, S^c, v).  p == NULL uses defaults.  cuda_stream == NULL
 * uses the library's stream; otherwise a cudaStream_t on the graph's device: every kernel
 * launch and copy of the search is issued on that stream, after the caller's earlier work
 * on it; the call returns once the results are on the host (the stream is synchronised).
 * *out receives a host result set (count may be 0: success with no result).
 * Errors: RIKI_EEMPTY_CENTRAL, RIKI_EUNRESOLVED, RIKI_ENOWEIGHTS, RIKI_EDEPTH, RIKI_EINVAL,
 *         RIKI_ENOMEM (workspace overflow, message says which), RIKI_ECUDA.
 * ------------------------------------------------------------------------------------- */
riki_status riki_rpq_search(riki_graph *g, const uint32_t *central, uint32_t n_central,
                            const uint32_t *marginal, uint32_t n_marginal, uint32_t k, uint32_t depth,
                            const riki_params *p, void *cuda_stream, riki_results **out);

/* Batch of independent queries (host arrays): query q has central terms
 * c_terms[c_ptr[q] .. c_ptr[q+1]) and marginal terms m_terms[m_ptr[q] .. m_ptr[q+1]).
 * Queries run concurrently on the device in level-synchronous lock-step.  out[q] receives
 * query q's results (n_queries handles).  On error no handle is returned. */
riki_status riki_rpq_search_batch(riki_graph *g, uint32_t n_queries,
                                  const uint64_t *c_ptr, const uint32_t *c_terms,
                                  const uint64_t *m_ptr, const uint32_t *m_terms,
                                  uint32_t k, uint32_t depth, const riki_params *p,
                                  riki_results **out);

/* Device-resident batch (benchmark / pipeline path): identical computation, but the query
 * arrays are DEVICE pointers and results stay on the device (no D2H); results are
 * retrievable afterwards with riki_batch_fetch (which performs the D2H).  Returns after
 * the work has been enqueued and completed on the library stream.  A batch whose recovery
 * arena (32-bit word offsets) would exceed 2^32 words runs in chunks of fewer queries, and
 * then each chunk's results are copied to the host before the next chunk runs. */
riki_status riki_rpq_search_batch_device(riki_graph *g, uint32_t n_queries,
                                         const uint64_t *d_c_ptr, const uint32_t *d_c_terms,
                                         const uint64_t *d_m_ptr, const uint32_t *d_m_terms,
                                         uint32_t k, uint32_t depth, const riki_params *p);
riki_status riki_batch_fetch(riki_graph *g, uint32_t n_queries, riki_results **out);

/* One result RPG (CG when M = empty).  Pointers stay valid until riki_results_free. */
typedef struct {
    uint32_t central_node;     /* v~ (Def. CG)                                       */
    uint32_t sc, sm;           /* S^c (Eq. 4) and S^m (Eq. 5); sm = 0 when M = empty        */
    double score;              /* S^r (Eq. 6); = S^c when M = empty                          */
    uint8_t ptc;               /* 1 = PTC holds (always 1 unless ptc_mode = 1)               */
    uint32_t n_nodes; const uint32_t *nodes;     /* sorted node ids of G^r                   */
    uint32_t n_edges; const uint64_t *edge_ids;  /* sorted caller edge ids, CG u G^m         */
    uint32_t n_vc; const uint32_t *vc;           /* sorted V_C                       */
    const uint8_t *cdist;      /* [n_central] h_c[v~][j] = D(c_j, v~)                      */
    const uint8_t *mdist;      /* [n_marginal] D(m_i, V_C) (Def. distKeyword2NodeSet)       */
} riki_rpg;

uint32_t riki_results_count(const riki_results *r);
riki_status riki_results_get(const riki_results *r, uint32_t i, riki_rpg *out);
/* per-query statistics: terminating levels of the two runs (-1 = not run), number of
 * candidate CGs, attached candidates, PTC rejects, (edge, keyword) relaxations per run */
typedef struct {
    int32_t L_central, L_marginal;
    uint32_t n_candidates, n_attached, n_ptc_fail;
    uint64_t relax_central, relax_marginal;
} riki_query_stats;
riki_status riki_results_stats(const riki_results *r, riki_query_stats *out);
/* candidate CGs in (S^c, v) order (only when riki_set_debug(g, 1) was on for the search) */
uint32_t riki_results_ncand(const riki_results *r);
riki_status riki_results_cand(const riki_results *r, uint32_t i, uint32_t *v, uint32_t *sc);
void riki_results_free(riki_results *r);

/* Bulk export of n result sets (e.g. a batch) into flat caller buffers, avoiding one call
 * per RPG.  riki_results_export_sizes gives the totals; riki_results_export then fills
 *   rpg_count[n]        RPGs per result set
 *   hdr[8 * n_rpg]      per RPG: central_node, sc, sm, ptc, n_nodes, n_edges, n_vc, 0
 *   score[n_rpg]        S^r
 *   nodes[n_nodes], edges[n_edges], vc[n_vc]   concatenated sorted lists, in RPG order
 *   cdist[8 * n_rpg], mdist[8 * n_rpg]         distances (RIKI_MAX_TERMS slots per RPG)
 *   stats[n]            per-query statistics (may be NULL)
 * All buffers are host memory owned by the caller. */
typedef struct {
    uint64_t n_rpg, n_nodes, n_edges, n_vc;
} riki_export_sizes;
riki_status riki_results_export_sizes(riki_results *const *rs, uint32_t n, riki_export_sizes *out);
riki_status riki_results_export(riki_results *const *rs, uint32_t n, uint32_t *rpg_count, uint32_t *hdr, double *score,
                                uint32_t *nodes, uint64_t *edges, uint32_t *vc, uint8_t *cdist, uint8_t *mdist,
                                riki_query_stats *stats);

/* ---------------------------------------------------------------------------------------
 * Debug / parity boundary (minimum slice): one exploration run with no termination other
 * than depth or an empty frontier.  terms[n_terms] term ids (1..8); block_mode 0 = none,
 * 1 = central CF (node identified when reached by all terms),
 * 2 = marginal stop rule (only when n_terms >= 2, R11).  H_out (host, V*n_terms
 * bytes, node-major) receives h; block_out (host, V bytes) the level at which the node was
 * blocked (0xFF if never; closed form R10).  relax_out (may be NULL) the relaxation count.
 * ------------------------------------------------------------------------------------- */
riki_status riki_hitting_levels(riki_graph *g, const uint32_t *terms, uint32_t n_terms, uint32_t depth,
                                int block_mode, uint8_t *H_out, uint8_t *block_out, uint64_t *relax_out,
                                int32_t *L_end_out);

/* ---------------------------------------------------------------------------------------
 * Instrumentation: when enabled, every expansion launch is bracketed by CUDA events on the
 * launching stream and its algorithmic bytes accumulated.
 * ------------------------------------------------------------------------------------- */
typedef struct {
    uint64_t expand_launches;      /* expansion kernel launches (light + heavy)            */
    double expand_ms;              /* summed CUDA-event time of those launches             */
    uint64_t expand_bytes;         /* algorithmic bytes of those launches                  */
    uint64_t relaxations;          /* (edge, keyword) relaxations                          */
    uint64_t kernel_launches;      /* all library kernel launches                          */
    uint64_t queries;              /* queries completed                                    */
    double section_ms[4];          /* host wall time: central run, CG recovery, marginal run, finalize
                                      (exact only with profiling on, which syncs at section ends) */
    uint64_t levels;               /* lock-step level iterations (one host sync each)       */
    uint64_t retries;              /* batches re-run after a workspace capacity overflow    */
    uint64_t reallocs;             /* workspace (re)allocations                             */
    /* expansion work counted on the device (every batch, profiling or not), the units of the
       SURVEY §8(d) algorithmic-byte model of the expansion kernel: */
    uint64_t exp_items;            /* frontier items (f, l) consumed, incl. duplicates/blocked */
    uint64_t exp_items_work;       /* items with a non-empty due edge range: distinct (f, L) */
    uint64_t exp_edges;            /* edge reads = distinct (e, L) pairs P_e                */
    uint64_t exp_new_cells;        /* H cells written (inf -> l+1)                          */
    uint64_t exp_enqueued;         /* next-frontier queue entries written                   */
    uint64_t exp_atomics;          /* relaxation atomics issued (rows read with a selected
                                      inf cell): the random-access roofline's second term;
                                      counted only with profiling on (riki_set_profiling)   */
} riki_stats;
riki_status riki_set_profiling(riki_graph *g, int on);
riki_status riki_get_stats(const riki_graph *g, riki_stats *out);
riki_status riki_reset_stats(riki_graph *g);
riki_status riki_set_debug(riki_graph *g, int on);
/* Expansion direction: 0 = push (Alg. 1 order; default), 1 = direction-optimising (bottom-up
 * pull for frontiers large against the unvisited remainder, Beamer's rule; identical results,
 * faster only when most gated/unblocked nodes end up reached). */
riki_status riki_set_direction(riki_graph *g, int mode);
/* Joint multi-query traversal: for batches of >= 32 queries whose H rows are
 * <= 4 bytes (<= 4 keywords per run), every frontier node and due edge is visited once per
 * level for the whole batch, reading all queries' rows of a node with one coalesced access
 * (node-major H).  Identical results.  on = 1 enables it (default 0). */
riki_status riki_set_joint(riki_graph *g, int on);
/* Batch slots (queries in flight per launch); 0 = automatic from free device memory. */
riki_status riki_set_batch_slots(riki_graph *g, uint32_t slots);
/* Abar estimation: "We sample ten thousand pairs of nodes for
 * estimation of Abar", the average shortest hops that Eq. 1-3 scale around.
 * src/dst: n_pairs node ids (caller ids, host arrays); the caller draws the pairs.  d(s, t)
 * = fewest edges of a directed path s -> t in the caller's edge list (bidirected: the
 * undirected distance), found by batched level-synchronous BFS on the device, at most
 * max_hops levels (>= 1).  Outputs (each may be NULL): mean and sample standard deviation
 * (n - 1) over the n_reached pairs with a path (NaN when n_reached < 1 / < 2), computed from
 * exact integer moments (R30); dist_out[n_pairs] the distances (0xFFFFFFFF = no path within
 * max_hops).  Needs no activation levels.  Errors: RIKI_EINVAL (ids, max_hops), RIKI_ENOMEM. */
riki_status riki_sample_avg_hops(riki_graph *g, uint32_t n_pairs, const uint32_t *src, const uint32_t *dst,
                                 uint32_t max_hops, double *mean, double *stddev, uint64_t *n_reached,
                                 uint32_t *dist_out);
/* Recovery-arena limit in 32-bit words (0 = default: the 2^32 addressable by its offsets).
 * A batch whose recovered subgraphs and memoised predecessor lists (Alg. 2) need more runs
 * in chunks of fewer queries; a device batch that ran in chunks has its results collected
 * to the host per chunk (riki_batch_fetch returns them as usual).  Tests use small limits. */
riki_status riki_set_arena_limit(riki_graph *g, uint64_t words);
/* device memory footprint of the resident graph and of the search workspace (bytes) */
riki_status riki_memory_footprint(const riki_graph *g, uint64_t *graph_bytes, uint64_t *workspace_bytes);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU.  One process per GPU, each with its own graph
 * handle (graph replicated: riki_load_graph on every rank).
 *
 * mode 0, replicated: queries are independent units (Def. RPQ); each rank runs
 *   its shard of a batch and no collective touches the data path (results are gathered by
 *   the caller).  riki_dist_init with mode 0 only records nranks/rank.
 * mode 1, vertex-partitioned: rank r owns the contiguous internal-node range
 *   [bounds[r], bounds[r+1]) (balanced by in-degree + 1, riki_dist_partition) and performs
 *   the level-l relaxations INTO its nodes bottom-up over their in-edges (a node takes
 *   h = l+1 in column j iff some in-edge (f -> n) has a <= l, h_fj <= l and f not blocked
 *   at l; the same H as Alg. 1's push, by Def. expansionBehavior).
 *   The reached cells of level l+1 travel as bit planes (one bit per node and keyword), one
 *   in-place ncclAllGather per level on the search stream (NCCL has no bitwise-OR
 *   reduction); every rank then applies all slices, so H, blocks, candidates, termination
 *   and results are identical on every rank without further collectives.  Every rank must
 *   issue the same searches in the same order (collective semantics).
 *
 * riki_dist_unique_id: out128 (host, 128 bytes) receives a fresh NCCL unique id (call on
 *   one rank, broadcast it, e.g. with torch.distributed).  RIKI_ENCCL if NCCL is missing.
 * riki_dist_init: nranks in [1, 1024], rank in [0, nranks), nccl_unique_id = the 128-byte
 *   id (host) or NULL.  With mode 1 and NULL id and nranks > 1, the nranks partitions are
 *   SIMULATED inside this process on its one device (every partition's pull runs here and
 *   the exchange is the identity): the single-GPU test of the partitioned arithmetic.  A
 *   graph's previous distributed state is released first.  Disables the joint traversal.
 *   Errors: RIKI_EINVAL (ranges, mode), RIKI_ENCCL, RIKI_ENOMEM.
 * riki_dist_partition: HOST-only helper (no device needed): bounds[nranks + 1] for an
 *   in-CSR row pointer irow[V + 1] (internal ids); bounds[0] = 0, bounds[nranks] = V, every
 *   bound a multiple of 32 or V, non-decreasing (ranges may be empty).
 * riki_dist_info: nranks, rank, mode, bounds (may be NULL; nranks + 1 entries, internal
 *   ids), exchanges and exchanged bytes so far (may be NULL).
 * ------------------------------------------------------------------------------------- */
riki_status riki_dist_unique_id(void *out128);
riki_status riki_dist_init(riki_graph *g, int nranks, int rank, const void *nccl_unique_id, int mode);
riki_status riki_dist_partition(const uint32_t *irow, uint32_t n_nodes, uint32_t nranks, uint32_t *bounds);
riki_status riki_dist_info(const riki_graph *g, int *nranks, int *rank, int *mode, uint32_t *bounds,
                           uint64_t *exchanges, uint64_t *exchanged_bytes);

const char *riki_last_error(void);
const char *riki_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RIKI_H */
