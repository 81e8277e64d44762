/*
 * vlq_gpu.h -- C ABI of the B200-native VLQ-ADC engine (libvlqgpu.so).
 *
 * This is the drop-in boundary for the reference's index API.  Every entry
 * point below replaces one call site of the reference C++ library
 * (/root/reference/proj) that its pybind11 binding
 * (proj/python/bindings.cpp) wraps; the citation on each declaration names
 * the interface it stands in for.  INTEGRATION.md shows the bindings a
 * maintainer adds (ctypes, pybind11, cgo-style C).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Host pointers are owned by the caller;
 *    the engine owns all device memory.  "_device" variants take device
 *    pointers and a cudaStream_t passed as void*.
 *  - Every call returns 0 on success or a negative status; it never throws
 *    across the ABI.  vlq_last_error() returns the thread-local message,
 *    which uses the reference's own text where one exists (e.g.
 *    "first_level_scan: need 0 < w1 <= k", "deserialize_index: bad magic
 *    in <path>", "index already holds a base set").
 *  - One engine per index (or per shard of an index).  Calls on one engine
 *    are serialised internally by a per-engine mutex, so any number of host
 *    threads may call vlq_engine_search on the same engine concurrently (the
 *    reference's search is const and runs with the GIL released,
 *    proj/python/bindings.cpp:99-126); each call sees the engine as left by
 *    the previous one.  The "_device" variants only enqueue work: the mutex
 *    orders the enqueues, and the caller orders its own streams.
 *    vlq_engine_destroy waits for a call in flight on another thread.
 *  - There is no CPU fallback: without a CUDA device vlq_engine_create fails.
 */
#ifndef VLQ_GPU_H
#define VLQ_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLQ_OK 0
#define VLQ_ERR_INVALID -1   /* bad argument / reference-level runtime_error */
#define VLQ_ERR_CUDA -2      /* CUDA runtime error */
#define VLQ_ERR_IO -3        /* file error (open / truncated / bad magic) */

typedef struct vlq_engine vlq_engine;
typedef struct vlq_group vlq_group;

typedef struct {
    int device;                /* CUDA ordinal */
    int shard_rank;            /* posting lists c with ((c * 0x9E3779B97F4A7C15) >> 40) % shard_count
                                  == shard_rank live here (64-bit product) */
    int shard_count;           /* 1 = whole index on this device */
    uint64_t workspace_bytes;  /* per-query-tile scratch budget (0 = 4 GiB) */
    uint32_t max_tile;         /* max queries per tile (0 = 16384) */
    int force_exact;           /* 1 = exact reference-order scan for every query */
} vlq_config;

typedef struct {
    uint32_t dim, k, n, m;
    int clamp_lambda;
    float lambda_lo, lambda_hi;
    uint64_t ntotal;         /* base_count (all shards) */
    uint64_t local_entries;  /* posting entries held by this engine */
} vlq_info;

typedef struct {
    uint64_t launches;      /* engine kernels launched by search calls */
    uint64_t tiles;         /* query tiles processed */
    uint64_t flagged;       /* queries whose certificate failed -> exact scan (profiling on) */
    uint64_t tc_fallbacks;  /* tensor-core coarse rows / add points that needed the exact full scan */
    double phase_ms[8];     /* CUDA-event ms per phase (profiling on): coarse, first-level,
                               second-level, term5, scan, rescore, fallback, output */
} vlq_stats;

/* Thread-local message of the last failing call on this thread. */
const char* vlq_last_error(void);

/* Engine lifetime.  Replaces constructing vlq::InvertedIndex
 * (proj/include/vlq/index.hpp:38-72) / PyIndex (bindings.cpp:41-42). */
int vlq_engine_create(const vlq_config* cfg, vlq_engine** out);
void vlq_engine_destroy(vlq_engine* e);

/* Index.load: deserialize_index (proj/src/index_io.cpp:100-159, VLQ1). */
int vlq_engine_load_vlq1(vlq_engine* e, const char* path);

/* Index.save: serialize_index (proj/src/index_io.cpp:63-98). */
int vlq_engine_save_vlq1(vlq_engine* e, const char* path, int store_t3);

/* Installs trained quantizers (the model half of Index.train,
 * bindings.cpp:44-81; make_model in proj/tools/vlq_cli.cpp:19-34).  t3 may be
 * NULL (computed exactly as compute_t3, proj/src/index.cpp:54-74). */
int vlq_engine_set_model(vlq_engine* e, uint32_t dim, uint32_t k, uint32_t n, uint32_t m, int clamp_lambda,
                         float lambda_lo, float lambda_hi, const float* centroids, const uint32_t* neighbor_ids,
                         const float* edge_sq_len, const float* pq_sub_centroids, const float* t3_or_null);

/* Index.train (bindings.cpp:44-81) on the device: k-means codebook
 * (vlq_train_kmeans), exact n-NN centroid graph, anchor displacements,
 * per-subspace PQ k-means; installs the model into `e` (an index with zero
 * points). */
int vlq_engine_train(vlq_engine* e, const float* train, uint64_t nt, uint32_t dim, uint32_t k, uint32_t n, uint32_t m,
                     uint32_t iters, uint64_t seed, int clamp_lambda);

/* train_kmeans (proj/include/vlq/kmeans.hpp, proj/src/kmeans.cpp:104-185) on
 * the device: k-means++ seeding (D^2 sampling, kmeans.cpp:54-102), Lloyd
 * iterations with exact strict-'<' assignment and in-order double centroid
 * sums, the reference's empty-cluster repair (kmeans.cpp:157-181).  x is
 * n*dim host floats, out_centroids k*dim.  With init_or_null (k*dim host
 * floats) the seeding is skipped and the result equals the reference's
 * Lloyd loop from those centroids bit for bit; the seeding's random stream
 * is the engine's own (a counter-based hash, not mt19937_64). */
int vlq_train_kmeans(int device, const float* x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed,
                     const float* init_or_null, float* out_centroids);

/* Index.add: build_index (proj/src/index.cpp:134-203) + once-only rule and
 * observe_lambda_range for unclamped models (bindings.cpp:83-97). */
int vlq_engine_add(vlq_engine* e, const float* base, uint64_t n, uint32_t dim);

/* Index.add of a vector file without loading it into host memory: the
 * reference's read_vecs (vecs_io.cpp:29-86: .bvecs -> bytes, .ivecs -> int32,
 * otherwise float32; every record's dimension checked; same error texts)
 * followed by build_index, streamed through double-buffered pinned staging
 * (chunk_rows rows per chunk, 0 = 128 MiB of floats).  Ids are the record
 * numbers.  Equivalent to vlq_engine_add(read_vecs(path)). */
int vlq_engine_add_vecs(vlq_engine* e, const char* path, uint64_t chunk_rows);

/* Index.search: search_batch (proj/src/search.cpp:169-191) with the
 * binding's padding (bindings.cpp:111-125): out_ids/out_dists are nq*k,
 * rows ascending by (dist, id), unfilled slots -1/+inf.  out_scanned
 * (nullable) receives the per-query scanned-candidate count
 * (SearchStats::scanned_candidates, search.cpp:163-165). */
int vlq_engine_search(vlq_engine* e, const float* queries, uint64_t nq, uint32_t dim, uint32_t w1, float alpha,
                      uint32_t k, int64_t* out_ids, float* out_dists, uint64_t* out_scanned);

/* Same with device-resident queries/outputs, asynchronous on `stream`
 * (cudaStream_t).  Call vlq_engine_sync to surface deferred errors. */
int vlq_engine_search_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                             uint32_t k, int64_t* d_ids, float* d_dists, uint64_t* d_scanned, void* stream);
int vlq_engine_sync(vlq_engine* e, void* stream);

/* Index.search split at the first-level boundary, for the query-split
 * multi-GPU path (each rank runs the coarse stage on a slice of the batch,
 * the slices are all-gathered, every rank runs the fine stage on its shard):
 *  - coarse: first_level_scan (proj/src/search.cpp:11-36) -> d_top[nq*w1],
 *    the exact top-w1 region ids of each query in (dist, id) order;
 *  - fine: second_level_rank .. select_topk (search.cpp:38-167) from d_top.
 * coarse followed by fine on the same engine equals vlq_engine_search_device. */
int vlq_engine_search_coarse_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, uint32_t* d_top,
                                    void* stream);
int vlq_engine_search_fine_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                  uint32_t k, const uint32_t* d_top, int64_t* d_ids, float* d_dists,
                                  uint64_t* d_scanned, void* stream);

/* Index.search split after second_level_rank, for the select-split multi-GPU
 * path (each rank runs the coarse stage AND the cell selection for a slice of
 * the batch; the selections are all-gathered; every rank runs the scan stage
 * on its shard):
 *  - select: first_level_scan + second_level_rank (search.cpp:11-78) ->
 *    d_sel[nq*w2] selected cell ids (i*n + j, the reference's order) and
 *    d_ab[nq*w2*2] their exact (a, b) = (|y - c_i|^2, |y - c_nbr|^2);
 *  - fine_sel: query_term5 .. select_topk (search.cpp:80-167) on this shard
 *    from a gathered selection (w2 = the same alpha-derived count).
 * select followed by fine_sel on the same engine equals vlq_engine_search_device. */
int vlq_engine_search_select_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                    uint32_t* d_sel, float* d_ab, void* stream);
int vlq_engine_search_fine_sel_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w1, float alpha,
                                      uint32_t k, const uint32_t* d_sel, const float* d_ab, int64_t* d_ids,
                                      float* d_dists, uint64_t* d_scanned, void* stream);
/* w2 = max(1, floor(alpha * w1 * n)) clamped to w1 * n (search.hpp:16-20): the
 * row length of the select-split buffers. */
uint32_t vlq_w2(uint32_t w1, float alpha, uint32_t n);
/* The multi-GPU owner of posting list `cell` among `shards` engines
 * (vlq_config.shard_rank / shard_count): ((cell * 0x9E3779B97F4A7C15) mod 2^64
 * >> 40) mod shards.  Host-only, no device needed. */
uint32_t vlq_shard_of_cell(uint32_t cell, uint32_t shards);
/* The fast scan's bank-aware code relabeling (built at add / load; no reference
 * counterpart, results do not depend on it): from m sub-spaces' 256 x 256
 * co-occurrence counts of code values in 32-entry warp blocks (upper triangle,
 * diagonal = occurrences), perm[p * 256 + c] = the value code c of sub-space p
 * takes in the scan copy; values v with equal v mod 32 share a shared-memory
 * bank, 8 per bank.  Host-only, no device needed. */
int vlq_code_banks(const uint32_t* cooc, uint32_t m, uint8_t* perm);

/* Streamed Index.add of the engine's counter-based synthetic generator
 * (the reference's Gaussian-mixture law, dataset.cpp:13-44): rows are
 * generated on the device chunk by chunk, so 1e8-1e9-point bases never touch
 * host memory.  Same once-only / error semantics as vlq_engine_add. */
int vlq_engine_add_synthetic(vlq_engine* e, uint64_t n, uint32_t clusters, float spread, uint64_t seed);

/* Rows [first, first+count) of that generator into device memory. */
int vlq_gen_synthetic_device(int device, uint64_t first, uint64_t count, uint32_t dim, uint32_t clusters, float spread,
                             uint64_t seed, float* d_out, void* stream);

/* Exact brute-force k-NN of host queries against rows [0, nb) of the device
 * generator (ground truth at scale). */
int vlq_brute_force_gt_synthetic(int device, uint64_t nb, uint32_t dim, uint32_t clusters, float spread, uint64_t seed,
                                 const float* queries, uint64_t nq, uint32_t k, uint32_t* out);

/* IVFADC comparison baseline (proj/include/vlq/ivf_baseline.hpp), built
 * with this engine's codebook and PQ as eval.cpp:182 does:
 *  - build: build_ivf_baseline (proj/src/ivf_baseline.cpp:11-51) -- exact
 *    assign_nearest, residual x - c, pq_encode, ordered appends; a host base
 *    array or the device synthetic generator;
 *  - search: search_ivf_baseline (ivf_baseline.cpp:53-126) -- exact top-w
 *    regions, per-region residual LUT, exact (dist, id) top-k, -1/+inf
 *    padded; out_scanned = SearchStats::scanned_candidates per query;
 *  - get_lists: count of points and the region-major lists
 *    (list_off[k+1], ids[count], codes[count*m]); any pointer may be NULL. */
int vlq_engine_ivf_build(vlq_engine* e, const float* base, uint64_t n, uint32_t dim);
int vlq_engine_ivf_build_synthetic(vlq_engine* e, uint64_t n, uint32_t clusters, float spread, uint64_t seed);
int vlq_engine_ivf_search(vlq_engine* e, const float* queries, uint64_t nq, uint32_t dim, uint32_t w, uint32_t k,
                          int64_t* out_ids, float* out_dists, uint64_t* out_scanned);
int vlq_engine_ivf_search_device(vlq_engine* e, const float* d_queries, uint64_t nq, uint32_t w, uint32_t k,
                                 int64_t* d_ids, float* d_dists, uint64_t* d_scanned, void* stream);
int vlq_engine_ivf_get_lists(vlq_engine* e, uint64_t* count, uint64_t* list_off, uint32_t* ids, uint8_t* codes);

/* Study knobs, not part of the reference surface: "scan_variant" (0 = v6
 * packed-fp32 fast scan, 2/3/4 = v5 LUT layouts, 1 = generic scan, 5-8 = v7
 * bulk-async staged entry ring, 9 = v6 with the u8-quantized LUT),
 * "scan_slots" (entry slots per lane: 4/6/8; +100 = 4 CTAs/SM),
 * "scan_prefetch" (L2 prefetch distance in chunks), "scan_packed" (packed
 * e-term|lambda stream), "scan_keep_min" (lower bound on the fast-scan
 * survivors k'), "scan_cap" (candidate buffer keys per CTA), "tc_persist",
 * "tc_pass1_single", "tc_search_min_k", "force_exact".  Results are identical
 * for every setting. */
int vlq_engine_set_tuning(vlq_engine* e, const char* key, int64_t value);

/* Per-phase CUDA-event timing (recorded on the search stream) and counters. */
int vlq_engine_set_profiling(vlq_engine* e, int on);
int vlq_engine_get_stats(vlq_engine* e, vlq_stats* out);
int vlq_engine_reset_stats(vlq_engine* e);

/* Index.k / n / m / dim / ntotal (bindings.cpp:222-232). */
int vlq_engine_info(vlq_engine* e, vlq_info* out);

/* Copies the trained quantizers back to the host (any pointer may be NULL):
 * centroids[k*dim], neighbor_ids[k*n], edge_sq_len[k*n], pq[m*256*(dim/m)]. */
int vlq_engine_get_model(vlq_engine* e, float* centroids, uint32_t* neighbor_ids, float* edge_sq_len, float* pq);

/* Copies the (this shard's) posting lists back to the host:
 * list_off[k*n+1], ids[local_entries], codes[local_entries*m], lambdas[...]; with
 * ids, codes and lambdas all NULL only the offsets are copied. */
int vlq_engine_get_lists(vlq_engine* e, uint64_t* list_off, uint32_t* ids, uint8_t* codes, uint8_t* lambdas);

/* The posting lists of the given cells only (index.hpp:26-34 PostingList),
 * concatenated in request order: counts[i] = length of list cells[i]; ids,
 * codes (x m) and lambdas hold sum(counts) entries.  ids, codes and lambdas
 * may all be NULL (counts only).  For sampled checks of 1e9-entry indexes
 * without copying the whole index to the host. */
int vlq_engine_get_cells(vlq_engine* e, const uint32_t* cells, uint32_t ncells, uint64_t* counts, uint32_t* ids,
                         uint8_t* codes, uint8_t* lambdas);

/* Per-point add-path outputs without mutating the index: assign_point +
 * assign_edge + residual + pq_encode + quantize_lambda (index.cpp:86-106,
 * 167-188).  Any output pointer may be NULL. */
int vlq_engine_encode(vlq_engine* e, const float* x, uint64_t n, uint32_t* cells, float* lambdas, uint8_t* codes,
                      uint8_t* lambda_bytes);

/* Merges nparts per-shard top-k result blocks [nparts][nq][k] (device
 * pointers) into the global (dist, id) top-k (the paper's multi-GPU join,
 * PAPER.md:498-499).  Every row must be ascending by (dist, id) with -1/+inf
 * padding at the end -- as every search output is -- and an id may appear in
 * one part only (each base point lives in one shard). */
int vlq_merge_topk_device(int device, const int64_t* d_in_ids, const float* d_in_dists, uint32_t nparts, uint64_t nq,
                          uint32_t k, int64_t* d_out_ids, float* d_out_dists, void* stream);

/* brute_force_gt (proj/src/dataset.cpp:46-92): exact k-NN ids, ties by id. */
int vlq_brute_force_gt(int device, const float* base, uint64_t nb, const float* queries, uint64_t nq, uint32_t dim,
                       uint32_t k, uint32_t* out);

/* gen_synthetic (proj/src/dataset.cpp:13-44): identical stream. */
int vlq_gen_synthetic(uint64_t count, uint32_t dim, uint32_t clusters, float spread, uint64_t seed, float* out);

/* ---- Multi-GPU group: one process, one engine per device ------------------
 * The paper's multi-GPU search (split the index into b parts, search locally,
 * join: PAPER.md:498-499) behind one handle: engine g on
 * devices[g] holds the posting lists c with vlq_shard_of_cell(c, n) == g; the
 * coarse quantizer is replicated.  Per batch: query-split selection (device g
 * runs first_level_scan + second_level_rank, search.cpp:11-78, for its slice
 * of the batch), every device scans its shard for the whole batch reading the
 * selections from their owners over NVLink peer memory, and device g merges
 * its slice of the per-shard top-k by (dist, id) from every device's block
 * (peer loads) -- results equal the single-engine search_batch bit for bit.
 * Needs peer access between every pair of distinct devices; a device may be
 * listed more than once.  Calls on one group are serialised internally. */
/* shards (S) must divide ndevices (G): G / S replicas of an S-way list
 * sharding, each replica searching its own 1/(G/S) of every batch (0: S = G,
 * pure list sharding).  Replicas cut the per-GPU work that does not shrink
 * with the shard (per-query tables, re-score, selection hand-off). */
int vlq_group_create(const int* devices, uint32_t ndevices, uint32_t shards, const vlq_config* cfg_or_null,
                     vlq_group** out);
void vlq_group_destroy(vlq_group* g);
uint32_t vlq_group_size(vlq_group* g);
/* Index.load / the model half of Index.train / Index.add for every member */
int vlq_group_load_vlq1(vlq_group* g, const char* path);
int vlq_group_set_model(vlq_group* g, uint32_t dim, uint32_t k, uint32_t n, uint32_t m, int clamp_lambda,
                        float lambda_lo, float lambda_hi, const float* centroids, const uint32_t* neighbor_ids,
                        const float* edge_sq_len, const float* pq_sub_centroids, const float* t3_or_null);
int vlq_group_add(vlq_group* g, const float* base, uint64_t n, uint32_t dim);
int vlq_group_add_synthetic(vlq_group* g, uint64_t n, uint32_t clusters, float spread, uint64_t seed);
/* Index.search (search_batch, proj/src/search.cpp:169-191) over the group:
 * host queries in, merged host results out (vlq_engine_search conventions;
 * out_scanned = the sum over the shards, i.e. the reference's count). */
int vlq_group_search(vlq_group* g, const float* queries, uint64_t nq, uint32_t dim, uint32_t w1, float alpha,
                     uint32_t k, int64_t* out_ids, float* out_dists, uint64_t* out_scanned);
/* Device-resident batch: copy the queries to every device once, run timed
 * searches (out_ms = device time of the batch, max over the devices), read
 * the last result. */
int vlq_group_set_queries(vlq_group* g, const float* queries, uint64_t nq, uint32_t dim);
int vlq_group_search_resident(vlq_group* g, uint32_t w1, float alpha, uint32_t k, float* out_ms);
int vlq_group_results(vlq_group* g, int64_t* out_ids, float* out_dists, uint64_t* out_scanned);
/* Per-phase CUDA-event profile of member `member` (vlq_engine_get_stats
 * conventions; reset != 0 clears it afterwards). */
int vlq_group_set_profiling(vlq_group* g, int on);
int vlq_group_get_stats(vlq_group* g, uint32_t member, vlq_stats* out, int reset);
/* The info record of member `member` (local_entries: its shard). */
int vlq_group_info(vlq_group* g, uint32_t member, vlq_info* out);

#ifdef __cplusplus
}
#endif

#endif /* VLQ_GPU_H */
