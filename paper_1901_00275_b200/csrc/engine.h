// VLQ-ADC engine: one index (or one shard of it) resident on one B200.
//
// Host-side mirror of the reference InvertedIndex (proj/include/vlq/index.hpp:
// 38-72) with the posting lists flattened into device SoA arrays:
//   codes[N*m] u8 | lambdas[N] u8 | ids[N] u32 | eterm[N] f32 | list_off[K*n+1] u64
// (cell = i*n + j, lists concatenated in cell order, ids ascending per list),
// plus replicated coarse structures (codebook, graph, PQ, t2, t3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "kernels.h"

namespace vlq {

// Shard of posting list (cell) c among `shards` (multi-GPU ownership; the
// Python tests restate it as ((c * 0x9E3779B97F4A7C15) mod 2^64) >> 40, mod shards).
__host__ __device__ inline uint32_t shard_of_cell(uint32_t cell, uint32_t shards) {
    return (uint32_t)((((uint64_t)cell * 0x9E3779B97F4A7C15ull) >> 40) % shards);
}

// One sub-space's bank-aware code relabeling (engine.cu): cooc = 256 x 256
// co-occurrence counts (upper triangle + diagonal), perm[c] = c's new value;
// value v's LUT word sits in bank v mod 32, 8 values per bank.
void choose_code_banks_1(const unsigned int* cooc, uint8_t* perm);

// Touch every 4 KB page of a host output buffer (parallel), so its first-touch
// page faults can overlap with device work (engine.cu).
void par_prefault(void* dst, size_t bytes);

struct EngineConfig {
    int device = 0;
    int shard_rank = 0;    // this engine holds the posting lists c with shard_of_cell(c) == shard_rank
    int shard_count = 1;
    uint64_t workspace_bytes = 4ull << 30;  // per-query-tile scratch budget
    uint32_t max_tile = 16384;
    int force_exact = 0;   // 1: skip the fast scan, run the exact scan for every query
    int scan_variant = 0;  // 0 default (fused fast scan + exact re-score), 1 generic warp-buffer scan
    int scan_slots = 0;    // entry-slots per lane per chunk of the fast scan (4 / 6 / 8; +100 = 4 CTAs/SM;
                           // 306 = 6 slots in 6-warp CTAs, 4 per SM);
                           // 0 = auto: 306, or 104 on shards of >= 4 (1/4 or less of the
                           // entries per query: measured 3% faster at 8 shards, neutral unsharded)
    float cert_slack = 0.0f;  // test knob (cert_slack_milli): widens the re-score certificate -> retry / exact paths
    int scan_sel_agg = 0;        // study knob: warp-aggregated histogram atomics in the flush select
    int scan_flush_exact = 0;    // study knob: exact (multi-pass) intermediate flushes in the fast scan
    uint32_t scan_cap = 0;       // study knob: fast-scan candidate buffer per CTA (0 = 2048 keys)
    int scan_reorder = 1;        // the fast scan reads the within-list reordered copy (build_scan_order)
    int scan_reorder_build = 1;  // build that copy at add / load (env VLQ_SCAN_REORDER=0 skips it)
    int scan_relabel = 1;        // relabel the copy's code bytes so co-occurring values use distinct LUT banks
                                 // (at add / load; env VLQ_SCAN_RELABEL=0 skips it)
    int scan_lpt = 1;            // fast scan + re-score visit a tile's queries longest first (by scanned count)
    uint32_t scan_round_cap = 0; // study knob: most chunks per warp between the fast scan's block barriers (0 = 32)
    int scan_retry = 1;          // certificate failures: fast scan again with 4x k' before the exact scan
    int scan_adapt_keep = 1;     // raise k' (x2, up to x4) after a batch whose certificate failed for > 2% of queries
    uint32_t scan_keep_min = 0;  // study knob: lower bound on k' (fast-scan survivors)
    int scan_packed = 1;   // v6 scan reads the packed e-term | lambda-byte stream (one load per entry)
    int use_tc = 1;         // tensor-core (tcgen05 TF32) coarse stage + add assignment when supported
    uint32_t tc_min_k = 1024;         // add-path assignment on tensor cores for K >= this (env VLQ_TC_MIN_K)
    uint32_t tc_search_min_k = 16384; // search coarse stage on tensor cores for K >= this (env VLQ_TC_SEARCH_MIN_K)
    int tc_store_rows = 0;  // 1: materialise approximate rows + radix select instead of the two-pass filter
    int tc_persist = 1;     // search coarse kernels as a persistent grid (one CTA per SM)
    int tc_pass1_single = 1;  // two-pass coarse filter: first pass in 1xTF32 (tau raised by its error bound)
    int tc_pass2_single = 0;  // ... and the filter pass in 1xTF32 too (tau raised by both bounds; more candidates)
    int tc_chunk_select = 1;  // chunk-select coarse stage (one 1xTF32 pass of 8-centroid chunk minima, exact
                              // evaluation of the selected chunks, fused first + second level; select_fused.cu)
    uint32_t tc_chunk_cap = 256;  // selected chunks per query before the exact full-row fallback (study knob)
    int tc_center = 1;  // chunk-select pass on centered operands (queries and centroids minus the centroid mean):
                        // a smaller TF32 bound, fewer chunks evaluated exactly
};

// Trained quantizers (a VLQ1 "model": an index with zero points).
struct HostModel {
    uint32_t dim = 0, k = 0, n = 0, m = 0;
    bool clamp = true;
    float lo = 0.0f, hi = 1.0f;
    std::vector<float> centroids;  // k*dim
    std::vector<uint32_t> nbr;     // k*n
    std::vector<float> elen;       // k*n
    std::vector<float> pq;         // m*256*(dim/m)
    std::vector<float> t3;         // k*m*256 or empty (computed)
};

struct HostLists {
    std::vector<uint64_t> off;  // k*n+1
    std::vector<uint32_t> ids;
    std::vector<uint8_t> codes;
    std::vector<uint8_t> lambdas;
    uint64_t base_count = 0;
};

// sets the current device for a scope, restoring the caller's on exit
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CUDA_CHECK(cudaGetDevice(&prev));
        if (prev != dev) CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// grow-only pinned host buffer (staging for the host-pointer API)
struct PinnedBuf {
    unsigned char* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() { reset(); }
    void reset() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t bytes) {
        if (bytes <= n && p) return;
        reset();
        CUDA_CHECK(cudaMallocHost(&p, bytes));
        n = bytes;
    }
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count <= n && p) return;
        reset();
        if (count == 0) return;
        // 64 bytes of slack: the staged scan's bulk copies round their sizes up
        // to 16 bytes and may read up to 15 bytes past the last entry
        CUDA_CHECK(cudaMalloc(&p, count * sizeof(T) + 64));
        n = count;
    }
    T* get() const { return p; }
};

enum Phase { PH_COARSE = 0, PH_FIRST, PH_SECOND, PH_TERM5, PH_SCAN, PH_RESCORE, PH_FALLBACK, PH_OUT, PH_COUNT };

struct EngineStats {
    uint64_t launches = 0;      // kernels launched by search calls
    uint64_t tc_refine_fallbacks = 0;  // coarse/assignment rows that needed the exact full scan
    uint64_t tiles = 0;
    uint64_t flagged = 0;       // queries that took the exact fallback
    double phase_ms[PH_COUNT] = {0};  // CUDA-event time per phase (profiling on)
};

class Engine {
public:
    explicit Engine(const EngineConfig& cfg);
    ~Engine();

    // model / index management
    void set_model(const HostModel& m);
    void load_vlq1(const std::string& path);
    void save_vlq1(const std::string& path, bool store_t3);
    bool has_model() const { return model_ok_; }
    uint32_t dim() const { return dim_; }
    uint32_t k() const { return k_; }
    uint32_t n() const { return n_; }
    uint32_t m() const { return m_; }
    uint64_t ntotal() const { return base_count_; }
    uint64_t local_entries() const { return nent_; }
    bool clamp() const { return clamp_; }
    float lo() const { return lo_; }
    float hi() const { return hi_; }
    // shard owning posting list (cell) c: a multiplicative hash of the cell id,
    // so the n lists of a region -- and the lists of the hub regions almost
    // every query visits -- spread over all ranks (region-granular i % G left
    // a 14% scanned-bytes imbalance at C4, 8 shards)
    int owner(uint32_t cell) const { return (int)shard_of_cell(cell, (uint32_t)cfg_.shard_count); }

    // add (Index.add, proj/python/bindings.cpp:83-97)
    void add_host(const float* base, uint64_t nb);
    // streamed add of a .fvecs / .bvecs / .ivecs file (the reference CLI's
    // `build` input, read_vecs vecs_io.cpp:29-86 semantics and error texts)
    // through double-buffered pinned staging: the base never has to fit in
    // host memory
    void add_vecs(const std::string& path, uint64_t chunk_rows = 0);
    // streamed add: the source writes points [first, first+count) to a device buffer
    using ChunkSource = std::function<void(uint64_t first, uint64_t count, float* dst, cudaStream_t st)>;
    void add_stream(uint64_t nb, uint64_t chunk, const ChunkSource& src);

    // search (Index.search, bindings.cpp:99-126): device pointers, async on `st`
    void search_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* d_ids,
                       float* d_dists, uint64_t* d_scanned, cudaStream_t st);
    // Staged search for the query-split multi-GPU path:
    //   coarse: first_level_scan only (search.cpp:11-36) -> exact top-w1 region
    //           ids per query, d_top [nq, w1] in (dist, id) order;
    //   fine:   everything after it (search.cpp:38-167) from a given d_top, on
    //           this engine's shard.  coarse + fine == search_device.
    void search_coarse_device(const float* d_q, uint64_t nq, uint32_t w1, uint32_t* d_top, cudaStream_t st);
    void search_fine_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                            const uint32_t* d_top, int64_t* d_ids, float* d_dists, uint64_t* d_scanned,
                            cudaStream_t st);
    // Select-split schedule (dist.py): select = first_level_scan + second_level_rank
    // for a query slice, publishing the selected cells [nq, w2] and their
    // (a, b) pairs [nq, w2, 2]; fine_sel = everything after second_level_rank
    // from a gathered selection, on this engine's shard.  select + fine_sel ==
    // search_device.
    void search_select_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t* d_sel, float* d_ab,
                              cudaStream_t st);
    void search_fine_sel_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                                const uint32_t* d_sel, const float* d_ab, int64_t* d_ids, float* d_dists,
                                uint64_t* d_scanned, cudaStream_t st);
    // fine_sel from a selection split in parts over several GPUs (group.cu): query q's
    // cells / (a, b) are row q % per of part q / per, read over NVLink peer memory
    void search_fine_sel_parts(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                               const SelParts& parts, int64_t* d_ids, float* d_dists, uint64_t* d_scanned,
                               cudaStream_t st);
    void search_host(const float* q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* ids,
                     float* dists, uint64_t* scanned);
    void check_device_errors(cudaStream_t st);

    // per-point add-path outputs for parity tests (no index mutation)
    void encode_host(const float* x, uint64_t nx, uint32_t* cells, float* lambdas, uint8_t* codes,
                     uint8_t* lam_bytes);
    void get_lists(HostLists& out, bool offsets_only = false);
    // the posting lists of the given cells only, concatenated in request order
    // (counts[i] = length of cells[i]); ids/codes/lambdas may be null (counts only)
    void get_cells(const uint32_t* cells, uint32_t ncells, uint64_t* counts, uint32_t* ids, uint8_t* codes,
                   uint8_t* lambdas);
    void get_tables(std::vector<float>& t2, std::vector<float>& t3);

    cudaStream_t stream() const { return stream_; }
    int device() const { return cfg_.device; }
    const HostModel& model() const { return model_; }

    // exact brute-force k-NN (dataset.cpp:46-92) on the device
    static void brute_force_gt(int device, const float* base, uint64_t nb, const float* queries, uint64_t nq,
                               uint32_t dim, uint32_t k, uint32_t* out);
    using BaseSource = std::function<void(uint64_t first, uint64_t count, float* dst, cudaStream_t st)>;
    static void brute_force_gt_source(int device, const BaseSource& src, uint64_t nb, const float* queries,
                                      uint64_t nq, uint32_t dim, uint32_t k, uint32_t* out);

    // IVFADC comparison baseline (proj/src/ivf_baseline.cpp, ivf.cu) with this
    // engine's codebook and PQ: build_ivf_baseline / search_ivf_baseline
    void ivf_build_host(const float* base, uint64_t nb);
    void ivf_build_stream(uint64_t nb, uint64_t chunk, const ChunkSource& src);
    void ivf_search_device(const float* d_q, uint64_t nq, uint32_t w, uint32_t topk, int64_t* d_ids, float* d_dists,
                           uint64_t* d_scanned, cudaStream_t st);
    void ivf_search_host(const float* q, uint64_t nq, uint32_t w, uint32_t topk, int64_t* ids, float* dists,
                         uint64_t* scanned);
    void ivf_get_lists(uint64_t* off, uint32_t* ids, uint8_t* codes);
    bool ivf_built() const { return ivf_ok_; }
    uint64_t ivf_count() const { return ivf_n_; }

    void set_profiling(bool on);
    // study knobs (scan_variant, scan_slots, use_tc_search): take effect on the next search
    void set_tuning(const std::string& key, int64_t value);
    uint32_t scan_keep(uint32_t topk) const;
    const EngineStats& stats();  // folds in the pending per-tile profile (syncs on its events)
    void reset_stats();

private:
    void upload_model();
    void upload_lists(const HostLists& L);
    void compute_eterm();
    void pack_eterm_lam();
    void build_scan_order();
    void choose_code_banks();
    AddArgs add_args() const;
    SearchArgs search_args() const;
    enum Stage { STAGE_ALL = 0, STAGE_COARSE = 1, STAGE_FINE = 2, STAGE_SELECT = 3, STAGE_FINE_SEL = 4 };
    // stage inputs / outputs of the multi-GPU schedules (batch-level pointers)
    struct StageIO {
        const uint32_t* top_in = nullptr;  // STAGE_FINE: [nq, w1]
        uint32_t* top_out = nullptr;       // STAGE_COARSE
        const uint32_t* sel_in = nullptr;  // STAGE_FINE_SEL: [nq, w2] cells
        const float* ab_in = nullptr;      //                 [nq, w2, 2]
        uint32_t* sel_out = nullptr;       // STAGE_SELECT
        float* ab_out = nullptr;
        const SelParts* parts = nullptr;   // STAGE_FINE_SEL from a selection in parts (multi-GPU group)
        uint64_t q0 = 0;                   //   batch row of this tile's first query
        StageIO at(uint64_t t0, uint32_t w1, uint32_t w2) const;
    };
    void search_staged(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* d_ids,
                       float* d_dists, uint64_t* d_scanned, const StageIO& io, Stage stage, cudaStream_t st);
    // returns whether the tensor-core path ran; *fused: the chunk-select path
    // also ran second_level_rank (sel_, ws_ a/b entries, meta_ written; and
    // the select-split hand-off into sel_out / ab_out when given)
    bool coarse_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint64_t& launches, cudaStream_t st,
                     bool* fused, uint32_t* sel_out = nullptr, float* ab_out = nullptr);
    bool fine_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint32_t topk, int64_t* d_ids,
                   float* d_dists, uint64_t* d_scanned, uint64_t& launches, cudaStream_t st,
                   const StageIO* sel = nullptr, bool second_done = false);
    void search_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint32_t topk, int64_t* d_ids,
                     float* d_dists, uint64_t* d_scanned, const StageIO& io, Stage stage, cudaStream_t st);

    // first member, so destroyed last: puts the caller's CUDA device back
    // after ~Engine and every member buffer has released its memory
    struct DeviceRestore {
        int prev = -1;
        ~DeviceRestore() {
            if (prev >= 0) cudaSetDevice(prev);
        }
    } restore_;
    EngineConfig cfg_;
    cudaStream_t stream_ = nullptr;
    bool profiling_ = false;
    struct ProfSlot {
        cudaEvent_t ev[PH_COUNT + 1] = {};
        cudaEvent_t done = nullptr;
        unsigned int* counts = nullptr;  // pinned [2]: fast-scan flagged, tc refine fallbacks
        bool fast = false, tc = false;
    };
    std::vector<ProfSlot> prof_;  // one per tile searched since the last collect_profile()
    size_t prof_used_ = 0;
    void mark_phase(int ph, cudaStream_t st);
    void grow_profile(size_t slots);
    void collect_profile();
    EngineStats stats_;
    void assign_chunk(const float* X, uint64_t nx, uint32_t* best, cudaStream_t st);
    DevBuf<uint32_t> tc_idx_, tc_flag_, tc_best_;
    DevBuf<float> tc_d_, tc_rows_;
    static constexpr uint32_t kListCap = 1024;  // per-query candidate list of the two-pass coarse filter
    DevBuf<float> tmin_, tau_, ld_;
    DevBuf<float> xtc_, xlo_;  // query rows in the UMMA layout (persistent coarse kernels)
    DevBuf<float> xtc1_;       // unsplit copy for the 1xTF32 first pass
    DevBuf<uint32_t> lcnt_, lidx_;
    DevBuf<float> tmin8_, tch_;          // chunk-select path: 8-centroid chunk minima, threshold T per query
    DevBuf<uint32_t> clist_, ccnt_;      // selected chunks per query
    DevBuf<float> svals_, snval_;        // split form: chunk-centroid / needed-id exact distances
    DevBuf<uint32_t> snid_, snneed_;     // split form: needed ids per query (ascending) and their count
    bool model_ok_ = false;
    uint32_t dim_ = 0, k_ = 0, n_ = 0, m_ = 0;
    bool clamp_ = true;
    float lo_ = 0.0f, hi_ = 1.0f;
    uint64_t base_count_ = 0;  // global N (all shards)
    uint64_t nent_ = 0;        // entries held by this shard
    float emax_ = 0.0f;
    HostModel model_;

    DevBuf<float> centroids_, elen_, pq_, pqT_, t2_, t3_;  // pqT_: [p][t][j] copy for term5
    DevBuf<float> cent_tc_, cnorm_tc_;  // UMMA-layout centroids + norms (tensor-core path)
    DevBuf<float> cent_hi_, cent_lo_;   // 3xTF32 split halves (search coarse stage)
    bool tc_ = false, tc_split_ = false;
    float cmax_ = 0.0f;  // max centroid norm (certificate bound)
    DevBuf<float> mu_, cent_tcc_, cnorm_tcc_;  // centroid mean; centered TF32 copy + norms (chunk-select pass)
    float cmaxc_ = 0.0f;                       // max centered centroid norm
    DevBuf<uint32_t> nbr_;
    DevBuf<uint64_t> list_off_;
    DevBuf<uint8_t> codes_, lambdas_;
    DevBuf<uint32_t> ids_;
    DevBuf<float> eterm_;
    DevBuf<uint32_t> eterm_lam_;  // packed e-term | lambda byte (v6 scan stream)
    DevBuf<uint8_t> scodes_;      // the fast scan's reordered copy: codes, ids, packed stream
    DevBuf<uint32_t> sids_, seterm_lam_;
    DevBuf<uint8_t> code_perm_, code_inv_;  // [m][256] relabeling of scodes_ (choose_code_banks), empty: none
    DevBuf<unsigned int> err_;  // [0] error flag, [1] emax bits, [2] flagged count, [3..4] minmax

    // IVFADC baseline lists (region-major; ids ascending within a list)
    DevBuf<uint64_t> ivf_off_;
    DevBuf<uint32_t> ivf_ids_;
    DevBuf<uint8_t> ivf_codes_;
    uint64_t ivf_n_ = 0;
    bool ivf_ok_ = false;

    // host-pointer search staging (search_host)
    DevBuf<float> sq_, sd_;
    DevBuf<int64_t> si_;
    DevBuf<uint64_t> ss_;
    PinnedBuf pin_;
    std::thread flusher_;  // background cache flush of the host-search output staging
    // adaptive k': the previous fine stage's certificate-failure count lands
    // here asynchronously (read one call later; a stale value only delays
    // the adaptation), and k' doubles while more than 2% of a batch fails
    PinnedBuf flag_seen_;
    uint64_t flag_seen_nq_ = 0;
    uint32_t keep_boost_ = 1;

    // search workspace
    DevBuf<float> ws_, dbuf_, t5_;
    DevBuf<uint32_t> top_, sel_, qlist_, cand_top_;
    DevBuf<uint64_t> cand_, cand2_;  // fast-scan survivors (k') / of the retry pass (4 k')
    DevBuf<uint32_t> qlist2_;
    DevBuf<uint32_t> lpt_;           // longest-first query order of the fast scan
    DevBuf<unsigned int> lpt_cnt_;
    DevBuf<unsigned int> cnt2_;
    DevBuf<QueryMeta> meta_;
};

uint32_t w2_of(uint32_t w1, float alpha, uint32_t n);

// Index.train on the device (train.cu); t3 is left empty (computed on upload).
void train_kmeans_host(int device, const float* X, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters,
                       uint64_t seed, const float* init, float* out);
HostModel train_model_device(int device, const float* train, uint64_t nt, uint32_t dim, uint32_t k, uint32_t n,
                             uint32_t m, uint32_t iters, uint64_t seed, bool clamp);

}  // namespace vlq
