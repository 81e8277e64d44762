// extern "C" boundary (include/vlq_gpu.h).  No exception crosses it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <random>
#include <string>

#include "../../include/vlq_gpu.h"
#include "engine.h"
#include "group.h"

// One engine per index.  Every call on an engine takes its mutex, so calls
// from several host threads are serialised here: the reference's search is
// const and may be called concurrently with the GIL released
// (proj/python/bindings.cpp:99-126, :107), while this engine's staging and
// workspace buffers are per-engine state.
struct vlq_engine {
    vlq::Engine* impl;
    std::mutex mu;
};

// A multi-GPU group (group.cu); calls serialised by its own mutex.
struct vlq_group {
    vlq::Group* impl;
    std::mutex mu;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* msg) {
    g_last_error = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return VLQ_OK;
    } catch (const vlq::CudaError& e) {
        return fail(VLQ_ERR_CUDA, e.what());
    } catch (const std::bad_alloc&) {
        return fail(VLQ_ERR_INVALID, "out of host memory");
    } catch (const std::exception& e) {
        const char* w = e.what();
        const bool io = std::strstr(w, "cannot open") || std::strstr(w, "truncated") || std::strstr(w, "bad magic") ||
                        std::strstr(w, "unsupported version") || std::strstr(w, "invalid header") ||
                        std::strstr(w, "write failed");
        return fail(io ? VLQ_ERR_IO : VLQ_ERR_INVALID, w);
    } catch (...) {
        return fail(VLQ_ERR_INVALID, "unknown error");
    }
}

}  // namespace

extern "C" {

const char* vlq_last_error(void) { return g_last_error.c_str(); }

int vlq_engine_create(const vlq_config* cfg, vlq_engine** out) {
    if (!out) return fail(VLQ_ERR_INVALID, "vlq_engine_create: out is NULL");
    *out = nullptr;
    return guarded([&] {
        vlq::EngineConfig c;
        if (cfg) {
            c.device = cfg->device;
            c.shard_rank = cfg->shard_rank;
            c.shard_count = cfg->shard_count ? cfg->shard_count : 1;
            if (cfg->workspace_bytes) c.workspace_bytes = cfg->workspace_bytes;
            if (cfg->max_tile) c.max_tile = cfg->max_tile;
            c.force_exact = cfg->force_exact;
        }
        auto* e = new vlq_engine{nullptr};
        try {
            e->impl = new vlq::Engine(c);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

void vlq_engine_destroy(vlq_engine* e) {
    if (!e) return;
    {
        std::lock_guard<std::mutex> lk(e->mu);  // waits for a call still running on another thread
        delete e->impl;
        e->impl = nullptr;
    }
    delete e;
}

#define ENGINE_OR_FAIL(e)                                                        \
    if (!(e) || !(e)->impl) return fail(VLQ_ERR_INVALID, "engine handle is NULL"); \
    std::lock_guard<std::mutex> engine_lock_((e)->mu)

int vlq_engine_load_vlq1(vlq_engine* e, const char* path) {
    ENGINE_OR_FAIL(e);
    if (!path) return fail(VLQ_ERR_INVALID, "path is NULL");
    return guarded([&] { e->impl->load_vlq1(path); });
}

int vlq_engine_save_vlq1(vlq_engine* e, const char* path, int store_t3) {
    ENGINE_OR_FAIL(e);
    if (!path) return fail(VLQ_ERR_INVALID, "path is NULL");
    return guarded([&] { e->impl->save_vlq1(path, store_t3 != 0); });
}

int vlq_engine_set_model(vlq_engine* e, uint32_t dim, uint32_t k, uint32_t n, uint32_t m, int clamp_lambda,
                         float lambda_lo, float lambda_hi, const float* centroids, const uint32_t* neighbor_ids,
                         const float* edge_sq_len, const float* pq_sub_centroids, const float* t3_or_null) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (dim == 0 || k == 0 || n == 0 || n >= k || m == 0 || dim % m != 0)
            throw std::runtime_error("set_model: invalid model header");
        if (!centroids || !neighbor_ids || !edge_sq_len || !pq_sub_centroids)
            throw std::runtime_error("set_model: NULL array");
        vlq::HostModel hm;
        hm.dim = dim;
        hm.k = k;
        hm.n = n;
        hm.m = m;
        hm.clamp = clamp_lambda != 0;
        hm.lo = lambda_lo;
        hm.hi = lambda_hi;
        hm.centroids.assign(centroids, centroids + (size_t)k * dim);
        hm.nbr.assign(neighbor_ids, neighbor_ids + (size_t)k * n);
        hm.elen.assign(edge_sq_len, edge_sq_len + (size_t)k * n);
        hm.pq.assign(pq_sub_centroids, pq_sub_centroids + (size_t)m * 256 * (dim / m));
        if (t3_or_null) hm.t3.assign(t3_or_null, t3_or_null + (size_t)k * m * 256);
        e->impl->set_model(hm);
    });
}

int vlq_engine_train(vlq_engine* e, const float* train, uint64_t nt, uint32_t dim, uint32_t k, uint32_t n, uint32_t m,
                     uint32_t iters, uint64_t seed, int clamp_lambda) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (nt && !train) throw std::runtime_error("train: NULL array");
        vlq::HostModel hm =
            vlq::train_model_device(e->impl->device(), train, nt, dim, k, n, m, iters, seed, clamp_lambda != 0);
        e->impl->set_model(hm);
    });
}

int vlq_train_kmeans(int device, const float* x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed,
                     const float* init_or_null, float* out_centroids) {
    return guarded([&] {
        if ((n && !x) || !out_centroids) throw std::runtime_error("train_kmeans: NULL array");
        vlq::train_kmeans_host(device, x, n, dim, k, iters, seed, init_or_null, out_centroids);
    });
}

int vlq_engine_add(vlq_engine* e, const float* base, uint64_t n, uint32_t dim) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("add: no model loaded");
        if (e->impl->ntotal() != 0) throw std::runtime_error("index already holds a base set");
        if (dim != e->impl->dim()) throw std::runtime_error("build_index: dimension mismatch");
        if (n && !base) throw std::runtime_error("add: base is NULL");
        e->impl->add_host(base, n);
    });
}

int vlq_engine_add_vecs(vlq_engine* e, const char* path, uint64_t chunk_rows) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!path) throw std::runtime_error("add_vecs: path is NULL");
        e->impl->add_vecs(path, chunk_rows);
    });
}

int vlq_engine_search(vlq_engine* e, const float* queries, uint64_t nq, uint32_t dim, uint32_t w1, float alpha,
                      uint32_t k, int64_t* out_ids, float* out_dists, uint64_t* out_scanned) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("search: no model loaded");
        if (dim != e->impl->dim()) throw std::runtime_error("search_batch: dimension mismatch");
        if (nq && (!queries || (k && (!out_ids || !out_dists)))) throw std::runtime_error("search: NULL buffer");
        e->impl->search_host(queries, nq, w1, alpha, k, out_ids, out_dists, out_scanned);
    });
}

int vlq_engine_search_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                             uint32_t k, int64_t* d_ids, float* d_dists, uint64_t* d_scanned, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->search_device(d_queries, nq, w1, alpha, k, d_ids, d_dists, d_scanned,
                               stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_search_coarse_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, uint32_t* d_top,
                                    void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->search_coarse_device(d_queries, nq, w1, d_top, stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_search_fine_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                  uint32_t k, const uint32_t* d_top, int64_t* d_ids, float* d_dists,
                                  uint64_t* d_scanned, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->search_fine_device(d_queries, nq, w1, alpha, k, d_top, d_ids, d_dists, d_scanned,
                                    stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_search_select_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                    uint32_t* d_sel, float* d_ab, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->search_select_device(d_queries, nq, w1, alpha, d_sel, d_ab,
                                      stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_search_fine_sel_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                      uint32_t k, const uint32_t* d_sel, const float* d_ab, int64_t* d_ids,
                                      float* d_dists, uint64_t* d_scanned, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->search_fine_sel_device(d_queries, nq, w1, alpha, k, d_sel, d_ab, d_ids, d_dists, d_scanned,
                                        stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_set_tuning(vlq_engine* e, const char* key, int64_t value) {
    ENGINE_OR_FAIL(e);
    if (!key) return fail(VLQ_ERR_INVALID, "set_tuning: key is NULL");
    return guarded([&] { e->impl->set_tuning(key, value); });
}

// ---- IVFADC comparison baseline (proj/src/ivf_baseline.cpp) ----------------
int vlq_engine_ivf_build(vlq_engine* e, const float* base, uint64_t n, uint32_t dim) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("build_ivf_baseline: no model loaded");
        if (dim != e->impl->dim()) throw std::runtime_error("build_ivf_baseline: dimension mismatch");
        if (n && !base) throw std::runtime_error("build_ivf_baseline: base is NULL");
        e->impl->ivf_build_host(base, n);
    });
}

int vlq_engine_ivf_build_synthetic(vlq_engine* e, uint64_t n, uint32_t clusters, float spread, uint64_t seed) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("build_ivf_baseline: no model loaded");
        if (clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        if (!(spread > 0)) throw std::runtime_error("gen_synthetic: spread must be positive");
        const uint32_t dim = e->impl->dim();
        const uint64_t chunk = std::max<uint64_t>(1, (512ull << 20) / (4ull * dim));
        e->impl->ivf_build_stream(n, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
            vlq::launch_synth(first, count, dim, clusters, spread, seed, dst, st);
        });
    });
}

int vlq_engine_ivf_search(vlq_engine* e, const float* queries, uint64_t nq, uint32_t dim, uint32_t w, uint32_t k,
                          int64_t* out_ids, float* out_dists, uint64_t* out_scanned) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (dim != e->impl->dim()) throw std::runtime_error("search_ivf_baseline: dimension mismatch");
        if (nq && (!queries || (k && (!out_ids || !out_dists)))) throw std::runtime_error("search: NULL buffer");
        e->impl->ivf_search_host(queries, nq, w, k, out_ids, out_dists, out_scanned);
    });
}

int vlq_engine_ivf_search_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w, uint32_t k,
                                 int64_t* d_ids, float* d_dists, uint64_t* d_scanned, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        e->impl->ivf_search_device(d_queries, nq, w, k, d_ids, d_dists, d_scanned,
                                   stream ? (cudaStream_t)stream : e->impl->stream());
    });
}

int vlq_engine_ivf_get_lists(vlq_engine* e, uint64_t* count, uint64_t* list_off, uint32_t* ids, uint8_t* codes) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (count) *count = e->impl->ivf_built() ? e->impl->ivf_count() : 0;
        if (list_off || ids || codes) e->impl->ivf_get_lists(list_off, ids, codes);
    });
}

int vlq_engine_sync(vlq_engine* e, void* stream) {
    ENGINE_OR_FAIL(e);
    return guarded([&] { e->impl->check_device_errors(stream ? (cudaStream_t)stream : e->impl->stream()); });
}

int vlq_engine_add_synthetic(vlq_engine* e, uint64_t n, uint32_t clusters, float spread, uint64_t seed) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("add: no model loaded");
        if (e->impl->ntotal() != 0) throw std::runtime_error("index already holds a base set");
        if (clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        if (!(spread > 0)) throw std::runtime_error("gen_synthetic: spread must be positive");
        const uint32_t dim = e->impl->dim();
        const uint64_t chunk = std::max<uint64_t>(1, (512ull << 20) / (4ull * dim));
        e->impl->add_stream(n, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
            vlq::launch_synth(first, count, dim, clusters, spread, seed, dst, st);
        });
    });
}

int vlq_gen_synthetic_device(int device, uint64_t first, uint64_t count, uint32_t dim, uint32_t clusters, float spread,
                             uint64_t seed, float* d_out, void* stream) {
    return guarded([&] {
        if (dim == 0 || clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        if (!(spread > 0)) throw std::runtime_error("gen_synthetic: spread must be positive");
        vlq::DeviceGuard g(device);
        vlq::launch_synth(first, count, dim, clusters, spread, seed, d_out, (cudaStream_t)stream);
    });
}

int vlq_brute_force_gt_synthetic(int device, uint64_t nb, uint32_t dim, uint32_t clusters, float spread, uint64_t seed,
                                 const float* queries, uint64_t nq, uint32_t k, uint32_t* out) {
    return guarded([&] {
        if (dim == 0 || clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        vlq::Engine::brute_force_gt_source(
            device,
            [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
                vlq::launch_synth(first, count, dim, clusters, spread, seed, dst, st);
            },
            nb, queries, nq, dim, k, out);
    });
}

int vlq_engine_set_profiling(vlq_engine* e, int on) {
    ENGINE_OR_FAIL(e);
    return guarded([&] { e->impl->set_profiling(on != 0); });
}

int vlq_engine_get_stats(vlq_engine* e, vlq_stats* out) {
    ENGINE_OR_FAIL(e);
    if (!out) return fail(VLQ_ERR_INVALID, "stats: out is NULL");
    return guarded([&] {  // folding in the profile syncs on CUDA events and may throw
        const vlq::EngineStats& s = e->impl->stats();
        out->launches = s.launches;
        out->tiles = s.tiles;
        out->flagged = s.flagged;
        out->tc_fallbacks = s.tc_refine_fallbacks;
        for (int p = 0; p < 8; p++) out->phase_ms[p] = s.phase_ms[p];
    });
}

int vlq_engine_reset_stats(vlq_engine* e) {
    ENGINE_OR_FAIL(e);
    return guarded([&] { e->impl->reset_stats(); });
}

int vlq_engine_info(vlq_engine* e, vlq_info* out) {
    ENGINE_OR_FAIL(e);
    if (!out) return fail(VLQ_ERR_INVALID, "info: out is NULL");
    out->dim = e->impl->dim();
    out->k = e->impl->k();
    out->n = e->impl->n();
    out->m = e->impl->m();
    out->clamp_lambda = e->impl->clamp() ? 1 : 0;
    out->lambda_lo = e->impl->lo();
    out->lambda_hi = e->impl->hi();
    out->ntotal = e->impl->ntotal();
    out->local_entries = e->impl->local_entries();
    return VLQ_OK;
}

int vlq_engine_get_model(vlq_engine* e, float* centroids, uint32_t* neighbor_ids, float* edge_sq_len, float* pq) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (!e->impl->has_model()) throw std::runtime_error("get_model: no model loaded");
        const vlq::HostModel& m = e->impl->model();
        if (centroids) std::memcpy(centroids, m.centroids.data(), m.centroids.size() * 4);
        if (neighbor_ids) std::memcpy(neighbor_ids, m.nbr.data(), m.nbr.size() * 4);
        if (edge_sq_len) std::memcpy(edge_sq_len, m.elen.data(), m.elen.size() * 4);
        if (pq) std::memcpy(pq, m.pq.data(), m.pq.size() * 4);
    });
}

int vlq_engine_get_lists(vlq_engine* e, uint64_t* list_off, uint32_t* ids, uint8_t* codes, uint8_t* lambdas) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        vlq::HostLists L;
        e->impl->get_lists(L, !ids && !codes && !lambdas);
        if (list_off) std::memcpy(list_off, L.off.data(), L.off.size() * 8);
        if (ids) std::memcpy(ids, L.ids.data(), L.ids.size() * 4);
        if (codes) std::memcpy(codes, L.codes.data(), L.codes.size());
        if (lambdas) std::memcpy(lambdas, L.lambdas.data(), L.lambdas.size());
    });
}

int vlq_engine_get_cells(vlq_engine* e, const uint32_t* cells, uint32_t ncells, uint64_t* counts, uint32_t* ids,
                         uint8_t* codes, uint8_t* lambdas) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (ncells && !cells) throw std::runtime_error("get_cells: cells is NULL");
        e->impl->get_cells(cells, ncells, counts, ids, codes, lambdas);
    });
}

int vlq_engine_encode(vlq_engine* e, const float* x, uint64_t n, uint32_t* cells, float* lambdas, uint8_t* codes,
                      uint8_t* lambda_bytes) {
    ENGINE_OR_FAIL(e);
    return guarded([&] {
        if (n == 0) return;
        e->impl->encode_host(x, n, cells, lambdas, codes, lambda_bytes);
    });
}

int vlq_merge_topk_device(int device, const int64_t* d_in_ids, const float* d_in_dists, uint32_t nparts, uint64_t nq,
                          uint32_t k, int64_t* d_out_ids, float* d_out_dists, void* stream) {
    return guarded([&] {
        if (nparts == 0 || nparts * (uint64_t)k > 8192) throw std::runtime_error("merge_topk: nparts*k must be in [1, 8192]");
        vlq::DeviceGuard g(device);
        vlq::launch_merge_topk(d_in_ids, d_in_dists, nparts, nq, k, d_out_ids, d_out_dists, (cudaStream_t)stream);
    });
}

int vlq_brute_force_gt(int device, const float* base, uint64_t nb, const float* queries, uint64_t nq, uint32_t dim,
                       uint32_t k, uint32_t* out) {
    return guarded([&] {
        if (dim == 0) throw std::runtime_error("brute_force_gt: dimension mismatch");
        vlq::Engine::brute_force_gt(device, base, nb, queries, nq, dim, k, out);
    });
}

// gen_synthetic (proj/src/dataset.cpp:13-44).  The stream is defined by
// std::mt19937_64 and libstdc++'s uniform_real / normal / uniform_int
// distributions, so this host generator reproduces the reference's data
// bit-for-bit when built with the same standard library.
int vlq_gen_synthetic(uint64_t count, uint32_t dim, uint32_t clusters, float spread, uint64_t seed, float* out) {
    return guarded([&] {
        if (dim == 0 || clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        if (!(spread > 0)) throw std::runtime_error("gen_synthetic: spread must be positive");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<float> unif(0.0f, 1.0f);
        std::vector<float> centers((size_t)clusters * dim);
        for (float& v : centers) v = unif(rng);
        std::normal_distribution<float> gauss(0.0f, spread);
        std::uniform_int_distribution<uint32_t> pick(0, clusters - 1);
        for (uint64_t i = 0; i < count; i++) {
            const uint32_t c = pick(rng);
            const float* ctr = centers.data() + (size_t)c * dim;
            float* row = out + i * dim;
            for (uint32_t j = 0; j < dim; j++) row[j] = ctr[j] + gauss(rng);
        }
    });
}

uint32_t vlq_w2(uint32_t w1, float alpha, uint32_t n) { return vlq::w2_of(w1, alpha, n); }

uint32_t vlq_shard_of_cell(uint32_t cell, uint32_t shards) { return shards ? vlq::shard_of_cell(cell, shards) : 0u; }

int vlq_code_banks(const uint32_t* cooc, uint32_t m, uint8_t* perm) {
    if (!cooc || !perm) return fail(VLQ_ERR_INVALID, "code_banks: NULL argument");
    return guarded([&] {
        for (uint32_t p = 0; p < m; p++) vlq::choose_code_banks_1(cooc + (size_t)p * 65536, perm + (size_t)p * 256);
    });
}


// ---- multi-GPU group --------------------------------------------------------

int vlq_group_create(const int* devices, uint32_t ndevices, uint32_t shards, const vlq_config* cfg, vlq_group** out) {
    if (!out) return fail(VLQ_ERR_INVALID, "vlq_group_create: out is NULL");
    *out = nullptr;
    return guarded([&] {
        if (!devices || ndevices == 0) throw std::runtime_error("vlq_group_create: no devices");
        vlq::EngineConfig c;
        if (cfg) {
            if (cfg->workspace_bytes) c.workspace_bytes = cfg->workspace_bytes;
            if (cfg->max_tile) c.max_tile = cfg->max_tile;
            c.force_exact = cfg->force_exact;
        }
        std::vector<int> devs(devices, devices + ndevices);
        auto* g = new vlq_group{nullptr};
        try {
            g->impl = new vlq::Group(devs, shards, c);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

void vlq_group_destroy(vlq_group* g) {
    if (!g) return;
    try {
        delete g->impl;
    } catch (...) {
    }
    delete g;
}

#define GROUP_OR_FAIL(g)                                                        \
    if (!(g) || !(g)->impl) return fail(VLQ_ERR_INVALID, "group handle is NULL"); \
    std::lock_guard<std::mutex> lock_((g)->mu)

int vlq_group_load_vlq1(vlq_group* g, const char* path) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (!path) throw std::runtime_error("load: path is NULL");
        g->impl->load_vlq1(path);
    });
}

int vlq_group_set_model(vlq_group* g, uint32_t dim, uint32_t k, uint32_t n, uint32_t m, int clamp_lambda,
                        float lambda_lo, float lambda_hi, const float* centroids, const uint32_t* neighbor_ids,
                        const float* edge_sq_len, const float* pq_sub_centroids, const float* t3_or_null) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (dim == 0 || k == 0 || n == 0 || n >= k || m == 0 || dim % m != 0)
            throw std::runtime_error("set_model: invalid model header");
        if (!centroids || !neighbor_ids || !edge_sq_len || !pq_sub_centroids)
            throw std::runtime_error("set_model: NULL array");
        vlq::HostModel hm;
        hm.dim = dim;
        hm.k = k;
        hm.n = n;
        hm.m = m;
        hm.clamp = clamp_lambda != 0;
        hm.lo = lambda_lo;
        hm.hi = lambda_hi;
        hm.centroids.assign(centroids, centroids + (size_t)k * dim);
        hm.nbr.assign(neighbor_ids, neighbor_ids + (size_t)k * n);
        hm.elen.assign(edge_sq_len, edge_sq_len + (size_t)k * n);
        hm.pq.assign(pq_sub_centroids, pq_sub_centroids + (size_t)m * 256 * (dim / m));
        if (t3_or_null) hm.t3.assign(t3_or_null, t3_or_null + (size_t)k * m * 256);
        g->impl->set_model(hm);
    });
}

int vlq_group_add(vlq_group* g, const float* base, uint64_t n, uint32_t dim) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        vlq::Engine& e0 = g->impl->engine(0);
        if (!e0.has_model()) throw std::runtime_error("add: no model loaded");
        if (dim != e0.dim()) throw std::runtime_error("build_index: dimension mismatch");
        if (e0.ntotal() != 0) throw std::runtime_error("index already holds a base set");
        if (n == 0) throw std::runtime_error("build_index: empty base set");
        if (!base) throw std::runtime_error("add: base is NULL");
        g->impl->add_host(base, n);
    });
}

int vlq_group_add_synthetic(vlq_group* g, uint64_t n, uint32_t clusters, float spread, uint64_t seed) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        vlq::Engine& e0 = g->impl->engine(0);
        if (!e0.has_model()) throw std::runtime_error("add: no model loaded");
        if (e0.ntotal() != 0) throw std::runtime_error("index already holds a base set");
        if (clusters == 0) throw std::runtime_error("gen_synthetic: dim and clusters must be positive");
        if (!(spread > 0)) throw std::runtime_error("gen_synthetic: spread must be positive");
        const uint32_t dim = e0.dim();
        const uint64_t chunk = std::max<uint64_t>(1, (512ull << 20) / (4ull * dim));
        g->impl->add_stream(n, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
            vlq::launch_synth(first, count, dim, clusters, spread, seed, dst, st);
        });
    });
}

int vlq_group_search(vlq_group* g, const float* queries, uint64_t nq, uint32_t dim, uint32_t w1, float alpha,
                     uint32_t k, int64_t* out_ids, float* out_dists, uint64_t* out_scanned) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (nq && (!queries || !out_ids || !out_dists)) throw std::runtime_error("search: NULL buffer");
        g->impl->search_host(queries, nq, dim, w1, alpha, k, out_ids, out_dists, out_scanned);
    });
}

int vlq_group_set_queries(vlq_group* g, const float* queries, uint64_t nq, uint32_t dim) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (nq && !queries) throw std::runtime_error("set_queries: NULL buffer");
        g->impl->upload_queries(queries, nq, dim);
    });
}

int vlq_group_search_resident(vlq_group* g, uint32_t w1, float alpha, uint32_t k, float* out_ms) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        const float ms = g->impl->search_resident(w1, alpha, k);
        if (out_ms) *out_ms = ms;
    });
}

int vlq_group_results(vlq_group* g, int64_t* out_ids, float* out_dists, uint64_t* out_scanned) {
    GROUP_OR_FAIL(g);
    return guarded([&] { g->impl->results(out_ids, out_dists, out_scanned); });
}

int vlq_group_info(vlq_group* g, uint32_t member, vlq_info* out) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (!out) throw std::runtime_error("info: out is NULL");
        if (member >= g->impl->size()) throw std::runtime_error("info: member out of range");
        vlq::Engine& e = g->impl->engine(member);
        out->dim = e.dim();
        out->k = e.k();
        out->n = e.n();
        out->m = e.m();
        out->clamp_lambda = e.clamp() ? 1 : 0;
        out->lambda_lo = e.lo();
        out->lambda_hi = e.hi();
        out->ntotal = e.ntotal();
        out->local_entries = e.local_entries();
    });
}

int vlq_group_set_profiling(vlq_group* g, int on) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        for (uint32_t i = 0; i < g->impl->size(); i++) g->impl->engine(i).set_profiling(on != 0);
    });
}

int vlq_group_get_stats(vlq_group* g, uint32_t member, vlq_stats* out, int reset) {
    GROUP_OR_FAIL(g);
    return guarded([&] {
        if (!out) throw std::runtime_error("stats: out is NULL");
        if (member >= g->impl->size()) throw std::runtime_error("stats: member out of range");
        vlq::Engine& e = g->impl->engine(member);
        const vlq::EngineStats& s = e.stats();
        out->launches = s.launches;
        out->tiles = s.tiles;
        out->flagged = s.flagged;
        out->tc_fallbacks = s.tc_refine_fallbacks;
        for (int p = 0; p < 8; p++) out->phase_ms[p] = s.phase_ms[p];
        if (reset) e.reset_stats();
    });
}

uint32_t vlq_group_size(vlq_group* g) { return (g && g->impl) ? g->impl->size() : 0u; }

}  // extern "C"
