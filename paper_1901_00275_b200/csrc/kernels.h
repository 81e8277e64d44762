// Kernel argument structs and launcher declarations shared by the engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace vlq {

// grid of the kernels launched over a device-side query list (certificate
// failures, overflow rows): a small grid strides over the list, so an empty
// list costs one short launch instead of one block per query of the tile
constexpr uint32_t VLQ_LIST_GRID = 592;
inline unsigned list_grid(uint64_t nblocks, bool is_list) {
    return (unsigned)(is_list && nblocks > VLQ_LIST_GRID ? VLQ_LIST_GRID : nblocks);
}

struct QueryMeta {
    unsigned long long scanned;  // reference-semantics scanned candidates (search.cpp:163-165)
    float dmax;                  // bound on |term1| over the query's selected cells
    float s5max;                 // bound on |sum5|
    uint32_t flag;               // 1: certificate failed -> exact fallback
    float qerr;                  // extra bound on |fast - exact| (0: every scan LUT is exact fp32)
};

// Device views used by the search kernels (all pointers device-resident).
struct SearchArgs {
    // index (replicated coarse structures + this shard's posting lists)
    uint32_t dim, k, n, m;
    float lo, hi, lam_absmax, emax;
    float lam_delta, lam0;  // fast-path dequantization: lam ~= lam0 + b * lam_delta
    const float* centroids;
    const uint32_t* nbr;
    const float* elen;
    const float* pq;
    const float* t2;
    const float* t3;
    const uint64_t* list_off;
    const uint8_t* codes;
    const uint8_t* lambdas;
    const uint32_t* ids;
    const float* eterm;
    // per-tile workspace
    float* ws;        // [T, k] exact centroid distances
    uint32_t* top;    // [T, w1]
    float* dbuf;      // [T, w1*n]
    uint32_t* sel;    // [T, w2] selected cell ids (ascending)
    float* t5;        // [T, m, 256]
    uint64_t* cand;   // [T, keep] fast-scan survivors (key = dist | pos)
    QueryMeta* meta;  // [T]
    unsigned int* error_flag;
    const float* Y;  // non-null: ws holds approximate (tensor-core) rows; second level
                     // recomputes neighbour distances exactly from the query vectors
    // v6 scan input stream: e-term with its low 8 mantissa bits replaced by the
    // entry's lambda byte (one 4-byte load per entry instead of 4 + 1);
    // e_pack_err bounds the e-term change (2^-15 Emax), added to the
    // certificate when the packed stream was scanned
    const uint32_t* eterm_lam;
    float e_pack_err;
    // scan order (engine.cu build_scan_order): within each list the entries
    // sorted by their leading code bytes, so a warp's lanes share LUT words more
    // often; eterm_lam is then in this order too, scodes / sids are the codes and
    // ids in it (null: the canonical id order)
    const uint8_t* scodes;
    const uint32_t* sids;
    // scodes' byte values are relabeled per sub-space (engine.cu
    // choose_code_banks): code_perm [m][256] maps a code to its scodes value
    // (the scan stores LUT[p][perm[p][c]] = term5[p][c]), code_inv back
    const uint8_t* code_perm;
    const uint8_t* code_inv;
    uint32_t scan_cap;  // fast-scan candidate buffer (keys per CTA); 0 = default
    uint32_t round_cap = 0;  // fast scan: most chunks per warp between block barriers (0 = 32)
    bool sel_agg;       // fast-scan flush: warp-aggregated (match_any) histogram atomics
    bool flush_exact;   // fast-scan intermediate flushes: exact k' selection (else one-pass approximate)
    // retry pass (certificate failures): the kernel's block b handles query
    // qlist[b] (blocks >= *qcount exit) and its cand row is b, not q
    const uint32_t* qlist;
    const unsigned int* qcount;
    bool qorder = false;  // qlist is a full permutation of the tile (one block per entry, no striding)
};

// Add-path device views.
struct AddArgs {
    uint32_t dim, k, n, m;
    int clamp;
    float lo, hi;
    const float* centroids;
    const uint32_t* nbr;
    const float* elen;
    const float* pq;
    const float* t2;
    const float* t3;
    unsigned int* error_flag;
};

void launch_sqdist_matrix(const float* Y, uint64_t ny, const float* C, uint64_t nc, uint32_t dim, float* out,
                          uint64_t ldo, cudaStream_t st);
void launch_first_level(const float* ws, uint64_t nq, uint32_t k, uint32_t w1, uint32_t* top, cudaStream_t st);
void launch_second_level(const SearchArgs& a, uint64_t nq, uint32_t w1, uint32_t w2, cudaStream_t st);
// select-split multi-GPU schedule: publish / apply a query's selected cells
// with their (a, b) = (ws[i], ws[nbr]) pairs ([nq, w2] u32 / [nq, w2, 2] f32)
void launch_pack_selection(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t* sel_out, float* ab,
                           cudaStream_t st);
void launch_apply_selection(const SearchArgs& a, uint64_t nq, uint32_t w2, const uint32_t* sel_in, const float* ab,
                            cudaStream_t st);

// Multi-GPU group (group.cu): per-device buffers addressed directly by the
// kernels over NVLink peer memory (P2P loads), at most VLQ_MAX_PARTS devices.
constexpr uint32_t VLQ_MAX_PARTS = 16;
// the batch's selection in parts: query q's row is row q % per of part q / per
struct SelParts {
    const uint32_t* sel[VLQ_MAX_PARTS];  // [per, w2] cells
    const float* ab[VLQ_MAX_PARTS];      // [per, w2, 2] exact (a, b)
    uint32_t nparts;
    uint64_t per;
};
// per-shard top-k blocks: row r of part g at ids[g] + r * topk
struct TopkParts {
    const int64_t* ids[VLQ_MAX_PARTS];
    const float* d[VLQ_MAX_PARTS];
    uint32_t nparts;
};
// k_apply_selection reading each query's row from its part (q = q0 + block)
void launch_apply_selection_parts(const SearchArgs& a, uint64_t nq, uint32_t w2, const SelParts& p, uint64_t q0,
                                  cudaStream_t st);
// (dist, id) merge of rows [row0, row0 + nrows) of every part into out[0 .. nrows)
void launch_merge_topk_parts(const TopkParts& p, uint64_t row0, uint64_t nrows, uint32_t topk, int64_t* out_ids,
                             float* out_d, cudaStream_t st);
// pqT: the PQ codebook transposed to [p][t][j] (j = codeword, fastest)
// cert_slack: added to the re-score certificate's error bound (0 in production;
// tests widen it to force the retry and exact-fallback paths)
void launch_term5(float cert_slack, const float* Y, const float* pqT, uint32_t dim, uint32_t m, float* t5, QueryMeta* meta,
                  uint64_t nq, cudaStream_t st);
size_t scan_smem_bytes(uint32_t m, uint32_t nwarps, uint32_t buf);
void launch_scan(const SearchArgs& a, uint64_t nblocks, uint32_t w2, uint32_t keep, uint32_t buf, uint32_t nwarps,
                 bool fast, const uint32_t* qlist, const unsigned int* qcount, cudaStream_t st);
// eterm_lam[e] = (bits(eterm[e]) & ~0xff) | lambdas[e]
void launch_pack_eterm_lam(const float* eterm, const uint8_t* lambdas, uint64_t n, uint32_t* out, cudaStream_t st);
bool launch_scan_fast(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int slots, cudaStream_t st);
void launch_rescore(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, uint32_t topk, int64_t* out_ids,
                    float* out_d, cudaStream_t st);
void launch_emit_exact(const SearchArgs& a, const uint32_t* qlist, const unsigned int* qcount, uint64_t nblocks,
                       uint32_t keep, uint32_t topk, int64_t* out_ids, float* out_d, cudaStream_t st);
// select_topk for k > 1024 (large_k.cu): exact keys of every scanned entry,
// sorted per query in groups of at most budget_keys keys; h_scanned = the
// per-query scanned counts (host)
void launch_topk_large(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t topk, const uint64_t* h_scanned,
                       uint64_t budget_keys, int64_t* out_ids, float* out_d, cudaStream_t st);
void launch_merge_topk(const int64_t* in_ids, const float* in_d, uint32_t nparts, uint64_t nq, uint32_t topk,
                       int64_t* out_ids, float* out_d, cudaStream_t st);

// add path
void launch_tables(const float* centroids, uint32_t k, uint32_t dim, const float* pq, uint32_t m, float* t2,
                   float* t3, cudaStream_t st);
void launch_assign_nearest(const AddArgs& a, const float* X, uint64_t nx, uint32_t* best, cudaStream_t st);
void launch_encode(const AddArgs& a, const float* X, uint64_t nx, const uint32_t* best, int clamp_for_edges,
                   uint32_t* cell_out, float* lam_out, uint8_t* codes_out, uint8_t* lamb_out, float* eterm_out,
                   unsigned int* emax_bits, cudaStream_t st, float* resid_out = nullptr);
void launch_minmax(const float* v, uint64_t n, float* out2, cudaStream_t st);
void launch_gather_entries(const uint32_t* order, uint64_t n, uint32_t m, uint64_t first_id,
                           const uint8_t* codes_pt, const uint8_t* lamb_pt, const float* eterm_pt,
                           uint32_t* ids, uint8_t* codes, uint8_t* lambdas, float* eterm, cudaStream_t st);
// scan order of the posting entries (engine.cu): order[] = the canonical
// positions sorted by (cell, leading code bytes)
void launch_code_cooc(const uint64_t* list_off, uint32_t ncell, uint32_t stride, const uint8_t* codes, uint32_t m,
                      unsigned int* cooc, cudaStream_t st);
void launch_relabel_codes(uint8_t* codes, uint64_t n, uint32_t m, const uint8_t* perm, cudaStream_t st);
void launch_scan_order_keys(const uint64_t* list_off, uint32_t ncell, const uint8_t* codes, uint32_t m, uint64_t n,
                            uint64_t* keys, uint32_t* vals, cudaStream_t st);
void launch_gather_scan_order(const uint32_t* order, uint64_t n, uint32_t m, const uint8_t* codes, const uint32_t* ids,
                              const uint32_t* eterm_lam, uint8_t* scodes, uint32_t* sids, uint32_t* seterm_lam,
                              cudaStream_t st);
void launch_histogram(const uint32_t* cells, uint64_t n, unsigned long long* counts, cudaStream_t st);

}  // namespace vlq

namespace vlq {
void launch_compact_flags(const QueryMeta* meta, uint64_t nq, uint32_t* qlist, unsigned int* count, cudaStream_t st);
// longest-first order of a tile's queries for the fast scan (count := nq)
void launch_lpt_order(const QueryMeta* meta, uint64_t nq, uint32_t* order, unsigned int* count, cudaStream_t st);
void launch_copy_scanned(const QueryMeta* meta, uint64_t nq, uint64_t* out, cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st);
void launch_synth(uint64_t first, uint64_t count, uint32_t dim, uint32_t clusters, float spread, uint64_t seed,
                  float* out, cudaStream_t st);
void launch_eterm_lists(const AddArgs& a, const uint64_t* list_off, uint32_t ncell, const uint8_t* codes,
                        const uint8_t* lambdas, uint64_t nent, float* eterm, unsigned int* emax_bits, cudaStream_t st);
void launch_gt_merge(const float* dist, uint64_t ldd, uint64_t nq, uint32_t k, uint32_t npos,
                     const uint32_t* sel_pos, uint64_t base_id, uint64_t* running, cudaStream_t st);
void launch_select_rows(const float* vals, uint64_t ld, uint64_t nrows, uint32_t len, uint32_t L, uint32_t* out,
                        cudaStream_t st);
}  // namespace vlq

namespace vlq {
// tensor-core coarse stage (coarse_tc.cu)
bool coarse_tc_supported(uint32_t dim);
// chunk-select coarse stage (select_fused.cu)
void launch_chunk_select(const float* tmin, uint64_t nq, uint32_t nchunk, uint32_t L, const float* Y, uint32_t dim,
                         float cmax, uint32_t capc, uint32_t* clist, uint32_t* ccnt, float* T, cudaStream_t st,
                         const float* mu = nullptr);
// split form of the fused kernel (select_fused.cu): row kernels + light
// per-query selection kernels; ldn = select_need_capacity(n, w1)
uint32_t select_need_capacity(uint32_t n, uint32_t w1);
uint32_t select_chunk_keys();  // exactly evaluated chunk centroids per query (row stride of the values)
bool select_split_supported(uint32_t k, uint32_t n, uint32_t w1, uint32_t w2, uint32_t dim, uint32_t capc);
void launch_rows(const float* C, const float* Y, uint32_t k, uint32_t dim, int chunks, const uint32_t* list,
                 const uint32_t* cnt, uint32_t ld, uint32_t capc, float* out, uint32_t ldo, uint64_t nq,
                 cudaStream_t st);
void launch_top_need(const SearchArgs& a, uint64_t nblocks, const float* Y, uint32_t w1, uint32_t w2,
                     const uint32_t* clist, const uint32_t* ccnt, uint32_t capc, const float* T, float cmax,
                     const uint32_t* qlist, const unsigned int* qcount, uint32_t* flagged, unsigned int* nflag,
                     const float* vals, uint32_t* nid, uint32_t* nneed, uint32_t ldn, cudaStream_t st,
                     const float* mu = nullptr);
void launch_second_sel(const SearchArgs& a, uint64_t nq, uint32_t w1, uint32_t w2, const uint32_t* nid,
                       const float* nval, const uint32_t* nneed, uint32_t ldn, uint32_t* sel_out, float* ab_out,
                       cudaStream_t st);
bool coarse_tc_split_supported(uint32_t dim);
void launch_relayout_centroids(const float* C, uint32_t k, uint32_t dim, float* out, float* out_lo, float* norm_out,
                               cudaStream_t st, int rna = 0, const float* mu = nullptr);
void launch_relayout_khalf(const float* C, uint32_t k, uint32_t dim, float* out_hi, float* out_lo, cudaStream_t st);
void launch_coarse_tc(int mode, const float* X, uint64_t nx, uint32_t dim, const float* cent_tc, const float* cent_lo,
                      const float* cnorm, uint32_t k, float* out_row, uint64_t ldo, uint32_t* top_idx, float* top_d,
                      cudaStream_t st, const float* tau = nullptr, uint32_t* cnt = nullptr, uint32_t cap = 0,
                      const float* Xtc = nullptr, const float* Xlo_tc = nullptr);
void launch_tau_rows(const float* tmin, uint64_t nq, uint32_t nchunk, uint32_t L, uint32_t* scratch, float* tau,
                     cudaStream_t st, const float* Y = nullptr, uint32_t dim = 0, float cmax = 0.0f,
                     int pass2_split = 1);
void launch_refine_list(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, const uint32_t* cand,
                        const uint32_t* cnt, uint32_t cap, const float* tau, uint32_t w1, float cmax, int split,
                        uint32_t* top, uint32_t* flagged, unsigned int* nflag, cudaStream_t st);
void launch_refine_argmin(const float* X, uint64_t nx, uint32_t dim, const float* C, const uint32_t* top_idx,
                          const float* top_d, float cmax, uint32_t* best, uint32_t* flagged, unsigned int* nflag,
                          cudaStream_t st);
void launch_gather_rows_list(const float* X, uint32_t dim, const uint32_t* rows, uint32_t nr, float* out,
                             cudaStream_t st);
void launch_scatter_u32(const uint32_t* vals, const uint32_t* rows, uint32_t nr, uint32_t* out, cudaStream_t st);
void launch_refine_first(const float* Y, uint64_t nq, uint32_t dim, const float* C, float* ws, uint32_t k,
                         const uint32_t* cand, uint32_t L, uint32_t w1, float cmax, uint32_t* top, uint32_t* flagged,
                         unsigned int* nflag, int split, cudaStream_t st);
void launch_exact_rows(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, float* ws,
                       const uint32_t* qlist, const unsigned int* count, cudaStream_t st);
void launch_exact_needed(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, uint32_t n,
                         const uint32_t* nbr, float* ws, const uint32_t* top, uint32_t w1, cudaStream_t st);
size_t exact_needed_smem(uint32_t k, uint32_t n, uint32_t w1, uint32_t dim);
void launch_first_level_list(const float* ws, uint64_t nq, uint32_t k, uint32_t w1, uint32_t* top,
                             const uint32_t* qlist, const unsigned int* count, cudaStream_t st);
}  // namespace vlq
