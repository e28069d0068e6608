// api.cu -- the C-ABI entry points of libriki.so (include/riki.h): argument checks,
// exception-to-status translation, thread-local error text and host result objects.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.cuh"

namespace {
thread_local std::string g_err;

template <class F> riki_status guard(F &&f) {
    try {
        f();
        g_err.clear();
        return RIKI_OK;
    } catch (const RikiError &e) {
        g_err = e.msg;
        return (riki_status)e.code;
    } catch (const std::bad_alloc &) {
        g_err = "host allocation failed";
        return RIKI_ENOMEM;
    } catch (const std::exception &e) {
        g_err = e.what();
        return RIKI_EINVAL;
    } catch (...) {
        g_err = "unknown error";
        return RIKI_EINVAL;
    }
}

// Every call on a graph handle holds its lock (include/riki.h, Threading): concurrent
// searches on one handle run one after the other on its workspace.
#define HANDLE_LOCK(g) std::lock_guard<std::recursive_mutex> handle_lock_((g)->mu)

void need(bool c, const char *msg) {
    if (!c) RIKI_THROW(RIKI_EINVAL, msg);
}

void check_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        RIKI_THROW(RIKI_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    }
    if (device < 0 || device >= n) RIKI_THROW(RIKI_EINVAL, "device index out of range");
    cudaDeviceProp p;
    CUDA_TRY(cudaGetDeviceProperties(&p, device));
    if (p.major != 10) RIKI_THROW(RIKI_ECUDA, "libriki.so is built for sm_100a (B200); found sm_" +
                                                  std::to_string(p.major) + std::to_string(p.minor));
}

QueryIn make_query(const uint32_t *c, uint32_t nc, const uint32_t *m, uint32_t nm) {
    QueryIn q{};
    if (nc == 0) RIKI_THROW(RIKI_EEMPTY_CENTRAL, "C must be non-empty (Def. RPQ, P:105)");
    if (nc > RIKI_MAX_TERMS || nm > RIKI_MAX_TERMS) RIKI_THROW(RIKI_EINVAL, "at most 8 terms per keyword class");
    need(c != nullptr, "null central term array");
    need(nm == 0 || m != nullptr, "null marginal term array");
    q.nc = nc;
    q.nm = nm;
    for (uint32_t j = 0; j < nc; j++) q.c[j] = c[j];
    for (uint32_t j = 0; j < nm; j++) q.m[j] = m[j];
    return q;
}
}  // namespace

extern "C" {

const char *riki_last_error(void) { return g_err.c_str(); }
const char *riki_version(void) { return "riki-b200 0.1 (sm_100a)"; }

void riki_params_default(riki_params *p) {
    if (!p) return;
    p->gamma = 0.5;
    p->beam_w = 0;
    p->beam_mode = 0;
    p->tie_break = 0;
    p->ptc_mode = 0;
    p->early_term = 0;
}

static riki_status load_graph(int device, uint32_t n_nodes, uint64_t n_edges, const uint32_t *src, const uint32_t *dst,
                              const uint32_t *label_class, uint32_t n_terms, const uint64_t *term_ptr,
                              const uint32_t *postings, riki_graph **out, bool device_inputs) {
    return guard([&] {
        need(out != nullptr, "null out");
        *out = nullptr;
        check_device(device);
        riki_graph *g = new riki_graph();
        g->device = device;
        try {
            graph_load(g, n_nodes, n_edges, src, dst, label_class, n_terms, term_ptr, postings, device_inputs);
        } catch (...) {
            graph_free(g);
            delete g;
            throw;
        }
        *out = g;
    });
}

riki_status riki_load_graph(int device, uint32_t n_nodes, uint64_t n_edges, const uint32_t *src, const uint32_t *dst,
                            const uint32_t *label_class, uint32_t n_terms, const uint64_t *term_ptr,
                            const uint32_t *postings, riki_graph **out) {
    return load_graph(device, n_nodes, n_edges, src, dst, label_class, n_terms, term_ptr, postings, out, false);
}

riki_status riki_load_graph_device(int device, uint32_t n_nodes, uint64_t n_edges, const uint32_t *src,
                                   const uint32_t *dst, const uint32_t *label_class, uint32_t n_terms,
                                   const uint64_t *term_ptr, const uint32_t *postings, riki_graph **out) {
    return load_graph(device, n_nodes, n_edges, src, dst, label_class, n_terms, term_ptr, postings, out, true);
}

void riki_free_graph(riki_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    engine_free(g);
    dist_free(g);
    graph_free(g);
    delete g;
}

riki_status riki_set_edge_weights(riki_graph *g, const double *w01, double alpha, double avg_hops) {
    return guard([&] { need(g, "null graph"); CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g); graph_set_edge_weights(g, w01, alpha, avg_hops); });
}
riki_status riki_set_node_weights(riki_graph *g, const double *w01, double alpha, double avg_hops) {
    return guard([&] { need(g, "null graph"); CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g); graph_set_node_weights(g, w01, alpha, avg_hops); });
}
riki_status riki_set_label_weights(riki_graph *g, double alpha, double avg_hops) {
    return guard([&] { need(g, "null graph"); CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g); graph_set_label_weights(g, alpha, avg_hops); });
}
riki_status riki_set_activation_levels(riki_graph *g, const uint8_t *a) {
    return guard([&] { need(g, "null graph"); CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g); graph_set_act(g, a); });
}
riki_status riki_get_activation_levels(const riki_graph *g, uint8_t *a) {
    return guard([&] { need(g && a, "null argument"); CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g); graph_get_act(g, a); });
}

riki_status riki_rpq_search(riki_graph *g, const uint32_t *central, uint32_t n_central, const uint32_t *marginal,
                            uint32_t n_marginal, uint32_t k, uint32_t depth, const riki_params *p, void *cuda_stream,
                            riki_results **out) {
    return guard([&] {
        need(g && out, "null argument");
        *out = nullptr;
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        riki_params prm;
        riki_params_default(&prm);
        if (p) prm = *p;
        std::vector<QueryIn> qs{make_query(central, n_central, marginal, n_marginal)};
        std::vector<riki_results *> res;
        engine_search(g, qs, k, depth, prm, (cudaStream_t)cuda_stream, &res);
        *out = res[0];
    });
}

riki_status riki_rpq_search_batch(riki_graph *g, uint32_t n_queries, const uint64_t *c_ptr, const uint32_t *c_terms,
                                  const uint64_t *m_ptr, const uint32_t *m_terms, uint32_t k, uint32_t depth,
                                  const riki_params *p, riki_results **out) {
    return guard([&] {
        need(g && out, "null argument");
        need(n_queries == 0 || (c_ptr && m_ptr), "null pointer arrays");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        riki_params prm;
        riki_params_default(&prm);
        if (p) prm = *p;
        std::vector<QueryIn> qs(n_queries);
        for (uint32_t q = 0; q < n_queries; q++) {
            need(c_ptr[q + 1] >= c_ptr[q] && m_ptr[q + 1] >= m_ptr[q], "pointer arrays not monotone");
            qs[q] = make_query(c_terms + c_ptr[q], (uint32_t)(c_ptr[q + 1] - c_ptr[q]),
                               m_terms ? m_terms + m_ptr[q] : nullptr, (uint32_t)(m_ptr[q + 1] - m_ptr[q]));
        }
        std::vector<riki_results *> res;
        engine_search(g, qs, k, depth, prm, nullptr, &res);
        for (uint32_t q = 0; q < n_queries; q++) out[q] = res[q];
    });
}

riki_status riki_rpq_search_batch_device(riki_graph *g, uint32_t n_queries, const uint64_t *d_c_ptr,
                                         const uint32_t *d_c_terms, const uint64_t *d_m_ptr,
                                         const uint32_t *d_m_terms, uint32_t k, uint32_t depth, const riki_params *p) {
    return guard([&] {
        need(g, "null graph");
        need(n_queries > 0 && d_c_ptr && d_m_ptr && d_c_terms, "null device arrays");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        riki_params prm;
        riki_params_default(&prm);
        if (p) prm = *p;
        engine_search_device(g, n_queries, d_c_ptr, d_c_terms, d_m_ptr, d_m_terms, k, depth, prm);
    });
}

riki_status riki_batch_fetch(riki_graph *g, uint32_t n_queries, riki_results **out) {
    return guard([&] {
        need(g && out, "null argument");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        std::vector<riki_results *> res;
        engine_fetch(g, n_queries, &res);
        for (uint32_t q = 0; q < n_queries; q++) out[q] = res[q];
    });
}

uint32_t riki_results_count(const riki_results *r) { return r ? (uint32_t)r->rpgs.size() : 0; }

riki_status riki_results_get(const riki_results *r, uint32_t i, riki_rpg *o) {
    return guard([&] {
        need(r && o, "null argument");
        need(i < r->rpgs.size(), "result index out of range");
        const HostRPG &p = r->rpgs[i];
        o->central_node = p.central_node;
        o->sc = p.sc;
        o->sm = p.sm;
        o->score = p.score;
        o->ptc = p.ptc;
        o->n_nodes = (uint32_t)p.nodes.size();
        o->nodes = p.nodes.data();
        o->n_edges = (uint32_t)p.edges.size();
        o->edge_ids = p.edges.data();
        o->n_vc = (uint32_t)p.vc.size();
        o->vc = p.vc.data();
        o->cdist = p.cdist;
        o->mdist = p.mdist;
    });
}

riki_status riki_results_stats(const riki_results *r, riki_query_stats *o) {
    return guard([&] {
        need(r && o, "null argument");
        *o = r->stats;
    });
}

uint32_t riki_results_ncand(const riki_results *r) { return r ? (uint32_t)r->cand.size() : 0; }
riki_status riki_results_cand(const riki_results *r, uint32_t i, uint32_t *v, uint32_t *sc) {
    return guard([&] {
        need(r && v && sc, "null argument");
        need(i < r->cand.size(), "candidate index out of range");
        *v = (uint32_t)r->cand[i];
        *sc = (uint32_t)(r->cand[i] >> 32);
    });
}
void riki_results_free(riki_results *r) { delete r; }

riki_status riki_results_export_sizes(riki_results *const *rs, uint32_t n, riki_export_sizes *out) {
    return guard([&] {
        need(out && (n == 0 || rs), "null argument");
        riki_export_sizes z{0, 0, 0, 0};
        for (uint32_t i = 0; i < n; i++) {
            need(rs[i] != nullptr, "null result handle");
            for (const HostRPG &p : rs[i]->rpgs) {
                z.n_rpg++;
                z.n_nodes += p.nodes.size();
                z.n_edges += p.edges.size();
                z.n_vc += p.vc.size();
            }
        }
        *out = z;
    });
}

riki_status riki_results_export(riki_results *const *rs, uint32_t n, uint32_t *rpg_count, uint32_t *hdr, double *score,
                                uint32_t *nodes, uint64_t *edges, uint32_t *vc, uint8_t *cdist, uint8_t *mdist,
                                riki_query_stats *stats) {
    return guard([&] {
        need(n == 0 || (rs && rpg_count && hdr && score && cdist && mdist), "null argument");
        uint64_t r = 0, on = 0, oe = 0, ov = 0;
        for (uint32_t i = 0; i < n; i++) {
            need(rs[i] != nullptr, "null result handle");
            rpg_count[i] = (uint32_t)rs[i]->rpgs.size();
            if (stats) stats[i] = rs[i]->stats;
            for (const HostRPG &p : rs[i]->rpgs) {
                uint32_t *h = hdr + 8 * r;
                h[0] = p.central_node; h[1] = p.sc; h[2] = p.sm; h[3] = p.ptc;
                h[4] = (uint32_t)p.nodes.size(); h[5] = (uint32_t)p.edges.size(); h[6] = (uint32_t)p.vc.size(); h[7] = 0;
                score[r] = p.score;
                memcpy(cdist + 8 * r, p.cdist, RIKI_MAX_TERMS);
                memcpy(mdist + 8 * r, p.mdist, RIKI_MAX_TERMS);
                if (nodes && !p.nodes.empty()) memcpy(nodes + on, p.nodes.data(), p.nodes.size() * 4);
                if (edges && !p.edges.empty()) memcpy(edges + oe, p.edges.data(), p.edges.size() * 8);
                if (vc && !p.vc.empty()) memcpy(vc + ov, p.vc.data(), p.vc.size() * 4);
                on += p.nodes.size(); oe += p.edges.size(); ov += p.vc.size();
                r++;
            }
        }
    });
}

riki_status riki_hitting_levels(riki_graph *g, const uint32_t *terms, uint32_t n_terms, uint32_t depth, int block_mode,
                                uint8_t *H_out, uint8_t *block_out, uint64_t *relax_out, int32_t *L_end_out) {
    return guard([&] {
        need(g && terms, "null argument");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        engine_hitting_levels(g, terms, n_terms, depth, block_mode, H_out, block_out, relax_out, L_end_out);
    });
}

riki_status riki_debug_ln_table(int device, uint64_t n0, uint64_t count, double *out) {
    return guard([&] {
        need(out != nullptr || count == 0, "null output");
        need(n0 >= 1, "ln is taken of counts >= 1");
        check_device(device);
        graph_debug_ln_table(device, n0, count, out);
    });
}

riki_status riki_set_profiling(riki_graph *g, int on) {
    return guard([&] { need(g, "null graph"); HANDLE_LOCK(g); g->profiling = on != 0; });
}
riki_status riki_get_stats(const riki_graph *g, riki_stats *o) {
    return guard([&] { need(g && o, "null argument"); HANDLE_LOCK(g); *o = g->stats; });
}
riki_status riki_reset_stats(riki_graph *g) {
    return guard([&] { need(g, "null graph"); HANDLE_LOCK(g); g->stats = riki_stats{}; });
}
riki_status riki_set_debug(riki_graph *g, int on) {
    return guard([&] { need(g, "null graph"); HANDLE_LOCK(g); g->debug = on != 0; });
}
riki_status riki_set_direction(riki_graph *g, int mode) {
    return guard([&] {
        need(g, "null graph");
        HANDLE_LOCK(g);
        need(mode == 0 || mode == 1, "direction mode must be 0 or 1");
        g->pull_on = mode == 1;
    });
}
riki_status riki_set_joint(riki_graph *g, int on) {
    return guard([&] {
        need(g, "null graph");
        HANDLE_LOCK(g);
        need(!(on && g->vp()), "joint traversal is not available in vertex-partitioned mode");
        g->joint_on = on != 0;
    });
}

riki_status riki_sample_avg_hops(riki_graph *g, uint32_t n_pairs, const uint32_t *src, const uint32_t *dst,
                                 uint32_t max_hops, double *mean, double *stddev, uint64_t *n_reached,
                                 uint32_t *dist_out) {
    return guard([&] {
        need(g, "null graph");
        need(n_pairs == 0 || (src && dst), "null pair arrays");
        need(max_hops >= 1, "max_hops must be >= 1");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        std::vector<uint32_t> dist(n_pairs);
        graph_sample_hops(g, n_pairs, src, dst, max_hops, dist.data());
        // exact integer moments, then one division each (order independent; R30)
        uint64_t n = 0, s1 = 0;
        unsigned __int128 s2 = 0;
        for (uint32_t i = 0; i < n_pairs; i++) {
            if (dist[i] == 0xFFFFFFFFu) continue;
            n++;
            s1 += dist[i];
            s2 += (unsigned __int128)dist[i] * dist[i];
        }
        if (mean) *mean = n ? (double)s1 / (double)n : NAN;
        if (stddev) {
            if (n >= 2) {
                const unsigned __int128 num = (unsigned __int128)n * s2 - (unsigned __int128)s1 * s1;
                *stddev = sqrt((double)num / ((double)n * (double)(n - 1)));
            } else {
                *stddev = NAN;
            }
        }
        if (n_reached) *n_reached = n;
        if (dist_out && n_pairs) memcpy(dist_out, dist.data(), (size_t)n_pairs * 4);
    });
}

riki_status riki_set_arena_limit(riki_graph *g, uint64_t words) {
    return guard([&] {
        need(g, "null graph");
        HANDLE_LOCK(g);
        need(words == 0 || words >= 4096, "arena limit must be 0 or >= 4096 words");
        g->arena_limit = words;
        g->slots_cap = 0;
    });
}

riki_status riki_dist_unique_id(void *out128) {
    return guard([&] {
        need(out128 != nullptr, "null output");
        dist_unique_id(out128);
    });
}
riki_status riki_dist_init(riki_graph *g, int nranks, int rank, const void *uid, int mode) {
    return guard([&] {
        need(g, "null graph");
        CUDA_TRY(cudaSetDevice(g->device)); HANDLE_LOCK(g);
        dist_init(g, nranks, rank, uid, mode);
    });
}
riki_status riki_dist_partition(const uint32_t *irow, uint32_t n_nodes, uint32_t nranks, uint32_t *bounds) {
    return guard([&] {
        need(irow && bounds, "null argument");
        need(nranks >= 1 && nranks <= 1024, "nranks must be in [1, 1024]");
        for (uint32_t v = 0; v < n_nodes; v++) need(irow[v] <= irow[v + 1], "row pointer must be non-decreasing");
        dist_partition(irow, n_nodes, nranks, bounds);
    });
}
riki_status riki_dist_info(const riki_graph *g, int *nranks, int *rank, int *mode, uint32_t *bounds, uint64_t *exchanges,
                           uint64_t *bytes) {
    return guard([&] {
        need(g, "null graph");
        const DistState *d = g->dist;
        if (nranks) *nranks = d ? d->nranks : 1;
        if (rank) *rank = d ? d->rank : 0;
        if (mode) *mode = d ? d->mode : 0;
        if (bounds) {
            if (d && !d->bounds.empty()) std::copy(d->bounds.begin(), d->bounds.end(), bounds);
            else { bounds[0] = 0; bounds[1] = g->V; }
        }
        if (exchanges) *exchanges = d ? d->exchanges : 0;
        if (bytes) *bytes = d ? d->exchanged_bytes : 0;
    });
}
riki_status riki_set_batch_slots(riki_graph *g, uint32_t slots) {
    return guard([&] {
        need(g, "null graph");
        HANDLE_LOCK(g);
        need(slots <= 1024, "at most 1024 slots");
        g->batch_slots = slots;
        g->slots_cap = 0;
    });
}
riki_status riki_memory_footprint(const riki_graph *g, uint64_t *gb, uint64_t *wb) {
    return guard([&] {
        need(g, "null graph");
        if (gb) *gb = g->graph_bytes;
        if (wb) *wb = engine_workspace_bytes(g);
    });
}

}  // extern "C"
