// Engine orchestration: model upload, batched add/encode with stable
// bucketing, tiled batched search, VLQ1 load/save.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.h"

namespace vlq {

namespace {

uint32_t next_pow2(uint32_t v) {
    uint32_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <typename T>
void h2d(DevBuf<T>& dst, const std::vector<T>& src, cudaStream_t st) {
    dst.alloc(std::max<size_t>(src.size(), 1));
    if (!src.empty()) CUDA_CHECK(cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

__global__ void k_mask_cells(uint32_t* cells, uint64_t n, uint32_t shards, uint32_t rank, uint32_t sentinel) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (shard_of_cell(cells[i], shards) != rank) cells[i] = sentinel;
}

}  // namespace

// QueryParams::w2 (proj/include/vlq/search.hpp:16-20)
uint32_t w2_of(uint32_t w1, float alpha, uint32_t n) {
    uint32_t full = w1 * n;
    uint32_t w = (uint32_t)((double)alpha * full);
    return w == 0 ? 1 : (w > full ? full : w);
}

Engine::Engine(const EngineConfig& cfg) : cfg_(cfg) {
    if (const char* v = std::getenv("VLQ_SCAN_VARIANT")) cfg_.scan_variant = std::atoi(v);
    if (const char* v = std::getenv("VLQ_SCAN_U")) cfg_.scan_slots = std::atoi(v);
    if (const char* v = std::getenv("VLQ_SCAN_REORDER")) cfg_.scan_reorder = cfg_.scan_reorder_build = std::atoi(v);
    if (const char* v = std::getenv("VLQ_SCAN_RELABEL")) cfg_.scan_relabel = std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC")) cfg_.use_tc = std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC_MIN_K")) cfg_.tc_min_k = cfg_.tc_search_min_k = (uint32_t)std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC_SEARCH_MIN_K")) cfg_.tc_search_min_k = (uint32_t)std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC_STORE_ROWS")) cfg_.tc_store_rows = std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC_PERSIST")) cfg_.tc_persist = std::atoi(v);
    if (const char* v = std::getenv("VLQ_TC_CHUNK_SELECT")) cfg_.tc_chunk_select = std::atoi(v);
    if (cfg_.shard_count < 1 || cfg_.shard_rank < 0 || cfg_.shard_rank >= cfg_.shard_count)
        throw std::runtime_error("engine: invalid shard configuration");
    int ndev = 0;
    CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (cfg_.device < 0 || cfg_.device >= ndev) throw std::runtime_error("engine: invalid CUDA device");
    DeviceGuard g(cfg_.device);
    CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    err_.alloc(8);
    CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 8 * sizeof(unsigned int), stream_));
}

Engine::~Engine() {
    if (flusher_.joinable()) flusher_.join();
    for (auto& sl : prof_) {
        for (auto& e : sl.ev)
            if (e) cudaEventDestroy(e);
        if (sl.done) cudaEventDestroy(sl.done);
        if (sl.counts) cudaFreeHost(sl.counts);
    }
    // the device buffers (members) are freed after this body on the engine's
    // device; restore_ (declared first, destroyed last) then restores the
    // caller's device
    if (cudaGetDevice(&restore_.prev) != cudaSuccess) restore_.prev = -1;
    cudaSetDevice(cfg_.device);
    if (stream_) {
        cudaStreamSynchronize(stream_);
        cudaStreamDestroy(stream_);
    }
}

AddArgs Engine::add_args() const {
    AddArgs a{};
    a.dim = dim_;
    a.k = k_;
    a.n = n_;
    a.m = m_;
    a.clamp = clamp_;
    a.lo = lo_;
    a.hi = hi_;
    a.centroids = centroids_.p;
    a.nbr = nbr_.p;
    a.elen = elen_.p;
    a.pq = pq_.p;
    a.t2 = t2_.p;
    a.t3 = t3_.p;
    a.error_flag = err_.p;
    return a;
}

SearchArgs Engine::search_args() const {
    SearchArgs a{};
    a.dim = dim_;
    a.k = k_;
    a.n = n_;
    a.m = m_;
    a.lo = lo_;
    a.hi = hi_;
    a.lam_absmax = std::max(std::max(std::fabs(lo_), std::fabs(hi_)), 0.0f);
    a.emax = emax_;
    a.lam_delta = (hi_ - lo_) * (1.0f / 256.0f);
    a.lam0 = lo_ + 0.5f * a.lam_delta;
    a.centroids = centroids_.p;
    a.nbr = nbr_.p;
    a.elen = elen_.p;
    a.pq = pq_.p;
    a.t2 = t2_.p;
    a.t3 = t3_.p;
    a.list_off = list_off_.p;
    a.codes = codes_.p;
    a.lambdas = lambdas_.p;
    a.ids = ids_.p;
    a.eterm = eterm_.p;
    a.ws = ws_.p;
    a.top = top_.p;
    a.dbuf = dbuf_.p;
    a.sel = sel_.p;
    a.t5 = t5_.p;
    a.cand = cand_.p;
    a.meta = meta_.p;
    a.error_flag = err_.p;
    return a;
}

void Engine::set_model(const HostModel& m) {
    if (m.dim == 0 || m.k == 0 || m.n == 0 || m.n >= m.k || m.m == 0 || m.dim % m.m != 0)
        throw std::runtime_error("set_model: invalid model header");
    if (m.centroids.size() != (size_t)m.k * m.dim || m.nbr.size() != (size_t)m.k * m.n ||
        m.elen.size() != (size_t)m.k * m.n || m.pq.size() != (size_t)m.m * VLQ_KSUB * (m.dim / m.m) ||
        (!m.t3.empty() && m.t3.size() != (size_t)m.k * m.m * VLQ_KSUB))
        throw std::runtime_error("set_model: array sizes do not match the header");
    for (uint32_t v : m.nbr)
        if (v >= m.k) throw std::runtime_error("set_model: neighbour id out of range");
    model_ = m;
    dim_ = m.dim;
    k_ = m.k;
    n_ = m.n;
    m_ = m.m;
    clamp_ = m.clamp;
    lo_ = m.lo;
    hi_ = m.hi;
    base_count_ = 0;
    nent_ = 0;
    emax_ = 0.0f;
    upload_model();
    HostLists empty;
    empty.off.assign((size_t)k_ * n_ + 1, 0);
    upload_lists(empty);
    model_ok_ = true;
}

void Engine::upload_model() {
    DeviceGuard g(cfg_.device);
    h2d(centroids_, model_.centroids, stream_);
    h2d(nbr_, model_.nbr, stream_);
    h2d(elen_, model_.elen, stream_);
    h2d(pq_, model_.pq, stream_);
    {  // [p][j][t] -> [p][t][j]: coalesced term5 loads
        const uint32_t dsub = dim_ / m_;
        std::vector<float> pqT(model_.pq.size());
        for (uint32_t p = 0; p < m_; p++)
            for (uint32_t j = 0; j < VLQ_KSUB; j++)
                for (uint32_t t = 0; t < dsub; t++)
                    pqT[((size_t)p * dsub + t) * VLQ_KSUB + j] = model_.pq[((size_t)p * VLQ_KSUB + j) * dsub + t];
        h2d(pqT_, pqT, stream_);
        CUDA_CHECK(cudaStreamSynchronize(stream_));  // pqT (host) is freed at scope exit
    }
    t2_.alloc((size_t)m_ * VLQ_KSUB);
    t3_.alloc(std::max<size_t>((size_t)k_ * m_ * VLQ_KSUB, 1));
    // t2 (pq.cpp:11-18, recomputed on load: index_io.cpp:140) and t3
    // (compute_t3, index.cpp:54-74) in the reference's exact order
    launch_tables(centroids_.p, k_, dim_, pq_.p, m_, t2_.p, t3_.p, stream_);
    if (!model_.t3.empty())
        CUDA_CHECK(cudaMemcpyAsync(t3_.p, model_.t3.data(), model_.t3.size() * 4, cudaMemcpyHostToDevice, stream_));
    // tensor-core coarse stage: centroids re-laid out for tcgen05 (UMMA
    // K-major interleaved tiles of 128) + exact norms
    tc_ = cfg_.use_tc && coarse_tc_supported(dim_) && k_ >= cfg_.tc_min_k;
    if (tc_) {
        const uint32_t ntiles = (k_ + 127) / 128;
        cent_tc_.alloc((size_t)ntiles * 128 * dim_);
        cnorm_tc_.alloc((size_t)ntiles * 128);
        // TF32-rounded (RNA) centroids: exact MMA operands (the chunk-select bound
        // relies on it; the add path's truncation bound covers them as well)
        launch_relayout_centroids(centroids_.p, k_, dim_, cent_tc_.p, nullptr, cnorm_tc_.p, stream_, /*rna=*/1);
        // 3xTF32 split copy for the search coarse stage (hi/lo halves)
        tc_split_ = coarse_tc_split_supported(dim_);
        if (tc_split_) {
            cent_hi_.alloc((size_t)ntiles * 128 * dim_);
            cent_lo_.alloc((size_t)ntiles * 128 * dim_);
            launch_relayout_khalf(centroids_.p, k_, dim_, cent_hi_.p, cent_lo_.p, stream_);
        }
        double mx = 0.0;
        for (uint32_t i = 0; i < k_; i++) {
            double s = 0.0;
            for (uint32_t d = 0; d < dim_; d++) s += (double)model_.centroids[(size_t)i * dim_ + d] * model_.centroids[(size_t)i * dim_ + d];
            mx = std::max(mx, s);
        }
        cmax_ = (float)(std::sqrt(mx) * (1.0 + 1e-6)) + 1e-30f;
        // centered copy for the chunk-select pass: mu = the centroid mean,
        // c' = fl(c - mu) (the kernels subtract in fp32 the same way)
        std::vector<double> acc(dim_, 0.0);
        for (uint32_t i = 0; i < k_; i++)
            for (uint32_t d = 0; d < dim_; d++) acc[d] += model_.centroids[(size_t)i * dim_ + d];
        std::vector<float> mu(dim_);
        for (uint32_t d = 0; d < dim_; d++) mu[d] = (float)(acc[d] / k_);
        double mxc = 0.0;
        for (uint32_t i = 0; i < k_; i++) {
            double s = 0.0;
            for (uint32_t d = 0; d < dim_; d++) {
                const float c = model_.centroids[(size_t)i * dim_ + d] - mu[d];
                s += (double)c * c;
            }
            mxc = std::max(mxc, s);
        }
        cmaxc_ = (float)(std::sqrt(mxc) * (1.0 + 1e-6)) + 1e-30f;
        mu_.alloc(dim_);
        CUDA_CHECK(cudaMemcpyAsync(mu_.p, mu.data(), (size_t)dim_ * 4, cudaMemcpyHostToDevice, stream_));
        cent_tcc_.alloc((size_t)ntiles * 128 * dim_);
        cnorm_tcc_.alloc((size_t)ntiles * 128);
        launch_relayout_centroids(centroids_.p, k_, dim_, cent_tcc_.p, nullptr, cnorm_tcc_.p, stream_, /*rna=*/1,
                                  mu_.p);
        CUDA_CHECK(cudaStreamSynchronize(stream_));  // mu (host) is freed at scope exit
    }
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// Exact nearest centroid (assign_point, index.cpp:86-106) for a chunk: the
// tensor-core GEMM proposes 4 candidates per point, k_refine_argmin settles
// them exactly when the TF32 bound proves the set complete, and the rest go
// through the exact CUDA-core full scan.
void Engine::assign_chunk(const float* X, uint64_t nx, uint32_t* best, cudaStream_t st) {
    AddArgs a = add_args();
    if (!tc_) {
        launch_assign_nearest(a, X, nx, best, st);
        return;
    }
    tc_idx_.alloc(nx * 4);
    tc_d_.alloc(nx * 4);
    tc_flag_.alloc(nx);
    launch_coarse_tc(0, X, nx, dim_, cent_tc_.p, nullptr, cnorm_tc_.p, k_, nullptr, 0, tc_idx_.p, tc_d_.p, st);
    CUDA_CHECK(cudaMemsetAsync(err_.p + 5, 0, 4, st));
    launch_refine_argmin(X, nx, dim_, centroids_.p, tc_idx_.p, tc_d_.p, cmax_, best, tc_flag_.p, err_.p + 5, st);
    unsigned int nflag = 0;
    CUDA_CHECK(cudaMemcpyAsync(&nflag, err_.p + 5, 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (nflag) {
        stats_.tc_refine_fallbacks += nflag;
        tc_rows_.alloc((size_t)nflag * dim_);
        tc_best_.alloc(nflag);
        launch_gather_rows_list(X, dim_, tc_flag_.p, nflag, tc_rows_.p, st);
        launch_assign_nearest(a, tc_rows_.p, nflag, tc_best_.p, st);
        launch_scatter_u32(tc_best_.p, tc_flag_.p, nflag, best, st);
    }
}

void Engine::upload_lists(const HostLists& L) {
    DeviceGuard g(cfg_.device);
    h2d(list_off_, L.off, stream_);
    h2d(ids_, L.ids, stream_);
    h2d(codes_, L.codes, stream_);
    h2d(lambdas_, L.lambdas, stream_);
    nent_ = L.ids.size();
    eterm_.alloc(std::max<uint64_t>(nent_, 1));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::compute_eterm() {
    DeviceGuard g(cfg_.device);
    CUDA_CHECK(cudaMemsetAsync(err_.p + 1, 0, sizeof(unsigned int), stream_));
    launch_eterm_lists(add_args(), list_off_.p, k_ * n_, codes_.p, lambdas_.p, nent_, eterm_.p, err_.p + 1, stream_);
    unsigned int bits = 0;
    CUDA_CHECK(cudaMemcpyAsync(&bits, err_.p + 1, 4, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    std::memcpy(&emax_, &bits, 4);
    pack_eterm_lam();
}

void Engine::pack_eterm_lam() {
    DeviceGuard g(cfg_.device);
    eterm_lam_.alloc(std::max<uint64_t>(nent_, 1));
    launch_pack_eterm_lam(eterm_.p, lambdas_.p, nent_, eterm_lam_.p, stream_);
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    try {
        build_scan_order();
    } catch (const CudaError&) {
        // the reordered copy is an optimisation (24 B per entry of temporary
        // and 20 B of permanent device memory): without room for it the fast
        // scan reads the canonical arrays
        scodes_.reset();
        sids_.reset();
        seterm_lam_.reset();
        code_perm_.reset();
        code_inv_.reset();
        (void)cudaGetLastError();
        CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
}

// The fast scan's copy of the entries: inside every list, sorted by the first
// code bytes (the scan's tie-break is the entry position, the re-score reads
// the id from sids_, and the result is the exact (dist, id) top-k either way).
// Neighbouring lanes then share LUT words more often: at C4 the simulated
// shared-memory wavefronts per LUT lookup drop from 1.93 to 1.81
// (profiles/r2_bank_sim_c4.txt).  Canonical (id-order) arrays stay for the
// exact paths, the re-score of non-reordered data, save and get_lists.
void Engine::build_scan_order() {
    scodes_.reset();
    sids_.reset();
    seterm_lam_.reset();
    code_perm_.reset();
    code_inv_.reset();
    const uint64_t ncell = (uint64_t)k_ * n_;
    if (!cfg_.scan_reorder_build || nent_ == 0 || !(m_ == 16 || m_ == 8 || m_ == 4) || ncell >= (1ull << 24) ||
        nent_ >= (1ull << 31))
        return;
    DeviceGuard g(cfg_.device);
    DevBuf<uint64_t> k0, k1;
    DevBuf<uint32_t> v0, v1;
    k0.alloc(nent_);
    k1.alloc(nent_);
    v0.alloc(nent_);
    v1.alloc(nent_);
    launch_scan_order_keys(list_off_.p, (uint32_t)ncell, codes_.p, m_, nent_, k0.p, v0.p, stream_);
    int cell_bits = 1;
    while ((1ull << cell_bits) < ncell) cell_bits++;
    cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p);
    cub::DoubleBuffer<uint32_t> vb(v0.p, v1.p);
    size_t tb = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)nent_, 0, 40 + cell_bits, stream_));
    DevBuf<unsigned char> temp;
    temp.alloc(std::max<size_t>(tb, 1));
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp.p, tb, kb, vb, (int)nent_, 0, 40 + cell_bits, stream_));
    scodes_.alloc(nent_ * m_);
    sids_.alloc(nent_);
    seterm_lam_.alloc(nent_);
    launch_gather_scan_order(vb.Current(), nent_, m_, codes_.p, ids_.p, eterm_lam_.p, scodes_.p, sids_.p,
                             seterm_lam_.p, stream_);
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    if (cfg_.scan_relabel) choose_code_banks();
}

// One sub-space's 256 code values onto the 32 shared-memory banks, 8 values
// per bank, so that values which occur together in a warp block rarely share
// a bank.  W[a][b] = the blocks holding both a and b (sampled).  Greedy in
// descending frequency (each value to the open bank with the least
// co-occurrence weight), then pairwise swaps while one lowers the total.
// Slot = bank + 32 * (rank inside the bank), so the LUT word of a relabeled
// value v sits in bank v mod 32.
void choose_code_banks_1(const unsigned int* cooc, uint8_t* perm) {
    constexpr int V = 256, B = 32, PER = V / B;
    std::vector<double> W((size_t)V * V, 0.0), cost((size_t)V * B, 0.0);
    std::vector<double> f(V);
    for (int a = 0; a < V; a++) {
        f[a] = cooc[a * V + a];
        for (int b = a + 1; b < V; b++) W[(size_t)a * V + b] = W[(size_t)b * V + a] = cooc[a * V + b];
    }
    std::vector<int> order(V), bank(V, -1), size(B, 0);
    for (int i = 0; i < V; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return f[x] > f[y]; });
    for (int c : order) {
        int best = -1;
        for (int b = 0; b < B; b++)
            if (size[b] < PER && (best < 0 || cost[(size_t)c * B + b] < cost[(size_t)c * B + best])) best = b;
        bank[c] = best;
        size[best]++;
        for (int x = 0; x < V; x++) cost[(size_t)x * B + best] += W[(size_t)x * V + c];
    }
    for (int pass = 0; pass < 16; pass++) {
        bool improved = false;
        for (int a = 0; a < V; a++)
            for (int b = a + 1; b < V; b++) {
                const int ba = bank[a], bb = bank[b];
                if (ba == bb) continue;
                const double wab = W[(size_t)a * V + b];
                const double d = (cost[(size_t)a * B + bb] - wab) - cost[(size_t)a * B + ba] +
                                 (cost[(size_t)b * B + ba] - wab) - cost[(size_t)b * B + bb];
                if (d < -1e-9) {
                    for (int x = 0; x < V; x++) {
                        cost[(size_t)x * B + ba] += W[(size_t)x * V + b] - W[(size_t)x * V + a];
                        cost[(size_t)x * B + bb] += W[(size_t)x * V + a] - W[(size_t)x * V + b];
                    }
                    bank[a] = bb;
                    bank[b] = ba;
                    improved = true;
                }
            }
        if (!improved) break;
    }
    int cnt[B] = {0};
    for (int c = 0; c < V; c++) perm[c] = (uint8_t)(bank[c] + B * cnt[bank[c]]++);
}

// The fast scan's LUT lookups are random 8-bit indices: a warp's lookup costs
// one shared-memory wavefront per distinct LUT word in its most-hit bank.
// Relabeling the copy's code bytes per sub-space (the scan writes the LUT at
// the relabeled positions, the re-score maps back through code_inv) spreads
// the values that co-occur in a warp block over different banks; the order of
// the copy, the LUT values and every sum are unchanged, so results are too.
// Statistics from a sample of ~32M entries (every stride-th list).
void Engine::choose_code_banks() {
    if (!scodes_.p || m_ > 16 || nent_ == 0) return;
    DeviceGuard g(cfg_.device);
    const uint64_t ncell = (uint64_t)k_ * n_;
    const uint32_t stride = (uint32_t)std::max<uint64_t>(1, nent_ >> 25);
    DevBuf<unsigned int> cooc;
    cooc.alloc((uint64_t)m_ * 65536);
    CUDA_CHECK(cudaMemsetAsync(cooc.p, 0, (size_t)m_ * 65536 * 4, stream_));
    launch_code_cooc(list_off_.p, (uint32_t)ncell, stride, scodes_.p, m_, cooc.p, stream_);
    std::vector<unsigned int> h((size_t)m_ * 65536);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), cooc.p, h.size() * 4, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    std::vector<uint8_t> perm((size_t)m_ * 256), inv((size_t)m_ * 256);
    std::vector<std::thread> th;
    for (uint32_t p = 0; p < m_; p++)
        th.emplace_back([&, p] { choose_code_banks_1(h.data() + (size_t)p * 65536, perm.data() + (size_t)p * 256); });
    for (auto& t : th) t.join();
    for (uint32_t p = 0; p < m_; p++)
        for (uint32_t c = 0; c < 256; c++) inv[p * 256 + perm[p * 256 + c]] = (uint8_t)c;
    code_perm_.alloc(perm.size());
    code_inv_.alloc(inv.size());
    CUDA_CHECK(cudaMemcpyAsync(code_perm_.p, perm.data(), perm.size(), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaMemcpyAsync(code_inv_.p, inv.data(), inv.size(), cudaMemcpyHostToDevice, stream_));
    launch_relabel_codes(scodes_.p, nent_, m_, code_perm_.p, stream_);
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::check_device_errors(cudaStream_t st) {
    unsigned int flag = 0;
    CUDA_CHECK(cudaMemcpyAsync(&flag, err_.p, 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (flag) {
        CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 4, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        throw std::runtime_error("line_lambda: degenerate edge (c == 0)");
    }
}

// ---------------------------------------------------------------------------
// add: build_index (index.cpp:134-203) on the device
// ---------------------------------------------------------------------------
void Engine::add_host(const float* base, uint64_t nb) {
    if (!model_ok_) throw std::runtime_error("add: no model loaded");
    if (base_count_ != 0) throw std::runtime_error("index already holds a base set");
    if (nb == 0) throw std::runtime_error("build_index: empty base set");
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(nb, (256ull << 20) / (4ull * dim_)));
    add_stream(nb, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
        CUDA_CHECK(cudaMemcpyAsync(dst, base + first * dim_, count * dim_ * 4, cudaMemcpyHostToDevice, st));
    });
}

void Engine::add_vecs(const std::string& path, uint64_t chunk_rows) {
    if (!model_ok_) throw std::runtime_error("add: no model loaded");
    if (base_count_ != 0) throw std::runtime_error("index already holds a base set");
    auto ends_with = [&](const char* suf) {  // vecs_kind_from_path (vecs_io.cpp:11-23)
        const size_t n = std::strlen(suf);
        return path.size() >= n && path.compare(path.size() - n, n, suf) == 0;
    };
    const int kind = ends_with(".bvecs") ? 1 : (ends_with(".ivecs") ? 2 : 0);  // 0 f32, 1 u8, 2 i32
    const uint64_t vsz = kind == 1 ? 1 : 4;
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("read_vecs: cannot open " + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    int32_t d0 = 0;
    const size_t got = std::fread(&d0, 1, 4, f);
    if (got == 0) throw std::runtime_error("read_vecs: no records in " + path);
    if (got != 4) throw std::runtime_error("read_vecs: truncated record header in " + path);
    if (d0 <= 0) throw std::runtime_error("read_vecs: non-positive dimension in " + path);
    if (std::fseek(f, 0, SEEK_END) != 0) throw std::runtime_error("read_vecs: cannot seek " + path);
    const uint64_t fsize = (uint64_t)std::ftell(f);
    const uint64_t rowb = 4 + (uint64_t)d0 * vsz;
    const uint64_t nb = fsize / rowb;
    if (nb * rowb != fsize) {  // the reference reads record by record and fails on the partial last one
        const uint64_t tail = fsize - nb * rowb;
        throw std::runtime_error(tail < 4 ? "read_vecs: truncated record header in " + path
                                          : "read_vecs: truncated record payload in " + path);
    }
    if ((uint32_t)d0 != dim_) throw std::runtime_error("build_index: dimension mismatch");
    const uint64_t chunk = chunk_rows ? chunk_rows : std::max<uint64_t>(1, (128ull << 20) / (4ull * dim_));
    const uint64_t crows = std::min(chunk, nb);
    PinnedBuf raw, fl[2];
    raw.alloc(crows * rowb);
    fl[0].alloc(crows * dim_ * 4);
    fl[1].alloc(crows * dim_ * 4);
    cudaEvent_t ev[2];
    CUDA_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } evg{ev};
    bool used[2] = {false, false};
    int cur = 0;
    add_stream(nb, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
        if (std::fseek(f, (long)(first * rowb), SEEK_SET) != 0 || std::fread(raw.p, 1, count * rowb, f) != count * rowb)
            throw std::runtime_error("read_vecs: truncated record payload in " + path);
        if (used[cur]) CUDA_CHECK(cudaEventSynchronize(ev[cur]));  // the H2D that last read this buffer
        float* out = reinterpret_cast<float*>(fl[cur].p);
        for (uint64_t r = 0; r < count; r++) {
            const unsigned char* rec = raw.p + r * rowb;
            int32_t d;
            std::memcpy(&d, rec, 4);
            if (d <= 0) throw std::runtime_error("read_vecs: non-positive dimension in " + path);
            if ((uint32_t)d != dim_) throw std::runtime_error("read_vecs: mismatched record dimension in " + path);
            float* o = out + r * dim_;
            if (kind == 0) {
                std::memcpy(o, rec + 4, 4ull * dim_);
            } else if (kind == 1) {
                for (uint32_t t = 0; t < dim_; t++) o[t] = (float)rec[4 + t];
            } else {
                for (uint32_t t = 0; t < dim_; t++) {
                    int32_t v;
                    std::memcpy(&v, rec + 4 + 4ull * t, 4);
                    o[t] = (float)v;
                }
            }
            for (uint32_t t = 0; t < dim_; t++)
                if (!std::isfinite(o[t])) throw std::runtime_error("VectorSet: non-finite value");
        }
        CUDA_CHECK(cudaMemcpyAsync(dst, out, count * dim_ * 4, cudaMemcpyHostToDevice, st));
        CUDA_CHECK(cudaEventRecord(ev[cur], st));
        used[cur] = true;
        cur ^= 1;
    });
}

void Engine::add_stream(uint64_t nb, uint64_t chunk, const ChunkSource& src) {
    if (!model_ok_) throw std::runtime_error("add: no model loaded");
    if (base_count_ != 0) throw std::runtime_error("index already holds a base set");
    if (nb == 0) throw std::runtime_error("build_index: empty base set");
    if (nb > 0xffffffffull) throw std::runtime_error("add: more than 2^32-1 points (VLQ1 ids are u32)");
    DeviceGuard g(cfg_.device);
    cudaStream_t st = stream_;
    // the reference assigns the index only after build_index succeeds
    // (bindings.cpp:89-96): a failed add must leave the lambda range of an
    // unclamped model unchanged
    struct RangeRollback {
        Engine* e;
        float lo, hi;
        bool armed = true;
        ~RangeRollback() {
            if (!armed) return;
            e->lo_ = e->model_.lo = lo;
            e->hi_ = e->model_.hi = hi;
        }
    } rollback{this, lo_, hi_};
    chunk = std::max<uint64_t>(1, std::min(chunk, nb));
    DevBuf<float> X;
    DevBuf<uint32_t> best;
    DevBuf<float> lam;
    X.alloc(chunk * dim_);
    best.alloc(chunk);
    lam.alloc(chunk);
    CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 8 * sizeof(unsigned int), st));
    // observe_lambda_range (index.cpp:110-132) for unclamped models
    if (!clamp_) {
        unsigned int init[2] = {0xffffffffu, 0u};
        CUDA_CHECK(cudaMemcpyAsync(err_.p + 3, init, 8, cudaMemcpyHostToDevice, st));
        AddArgs a = add_args();
        for (uint64_t f = 0; f < nb; f += chunk) {
            uint64_t c = std::min(chunk, nb - f);
            src(f, c, X.p, st);
            assign_chunk(X.p, c, best.p, st);
            launch_encode(a, X.p, c, best.p, 0, nullptr, lam.p, nullptr, nullptr, nullptr, nullptr, st);
            launch_minmax(lam.p, c, reinterpret_cast<float*>(err_.p + 3), st);
        }
        unsigned int mm[2];
        CUDA_CHECK(cudaMemcpyAsync(mm, err_.p + 3, 8, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        auto unord = [](unsigned int u) {
            u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
            float f;
            std::memcpy(&f, &u, 4);
            return f;
        };
        float lo = unord(mm[0]), hi = unord(mm[1]);
        if (!(lo < hi)) hi = lo + 1.0f;
        lo_ = lo;
        hi_ = hi;
        model_.lo = lo;
        model_.hi = hi;
    }
    // encode pass: point-order outputs
    DevBuf<uint32_t> cells;
    DevBuf<uint8_t> codes_pt, lamb_pt;
    DevBuf<float> eterm_pt;
    cells.alloc(nb);
    codes_pt.alloc(nb * m_);
    lamb_pt.alloc(nb);
    eterm_pt.alloc(nb);
    {
        AddArgs a = add_args();
        for (uint64_t f = 0; f < nb; f += chunk) {
            uint64_t c = std::min(chunk, nb - f);
            src(f, c, X.p, st);
            assign_chunk(X.p, c, best.p, st);
            launch_encode(a, X.p, c, best.p, clamp_ ? 1 : 0, cells.p + f, nullptr, codes_pt.p + f * m_, lamb_pt.p + f,
                          eterm_pt.p + f, err_.p + 1, st);
        }
    }
    X.reset();
    best.reset();
    lam.reset();
    // stable bucketing by cell (index.cpp:189-200): ids ascend within a list
    const uint32_t ncell = k_ * n_;
    const uint32_t sentinel = ncell;
    if (cfg_.shard_count > 1) {
        k_mask_cells<<<1184, 256, 0, st>>>(cells.p, nb, (uint32_t)cfg_.shard_count, (uint32_t)cfg_.shard_rank,
                                           sentinel);
        CUDA_LAUNCH_CHECK();
    }
    int end_bit = 1;
    while ((1ull << end_bit) <= (uint64_t)sentinel) end_bit++;
    DevBuf<uint32_t> cells_sorted, iota, order;
    cells_sorted.alloc(nb);
    iota.alloc(nb);
    order.alloc(nb);
    launch_iota(iota.p, nb, st);
    size_t temp_bytes = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, cells.p, cells_sorted.p, iota.p, order.p, nb, 0,
                                               end_bit, st));
    {
        DevBuf<unsigned char> temp;
        temp.alloc(temp_bytes);
        CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, cells.p, cells_sorted.p, iota.p, order.p, nb, 0,
                                                   end_bit, st));
    }
    iota.reset();
    DevBuf<unsigned long long> counts;
    counts.alloc((size_t)ncell + 2);
    CUDA_CHECK(cudaMemsetAsync(counts.p, 0, ((size_t)ncell + 2) * 8, st));
    launch_histogram(cells_sorted.p, nb, counts.p, st);
    list_off_.alloc((size_t)ncell + 1);
    temp_bytes = 0;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts.p, reinterpret_cast<unsigned long long*>(list_off_.p),
                                             (int)(ncell + 1), st));
    {
        DevBuf<unsigned char> temp;
        temp.alloc(temp_bytes);
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp.p, temp_bytes, counts.p,
                                                 reinterpret_cast<unsigned long long*>(list_off_.p), (int)(ncell + 1), st));
    }
    uint64_t nloc = 0;
    CUDA_CHECK(cudaMemcpyAsync(&nloc, list_off_.p + ncell, 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    cells.reset();
    cells_sorted.reset();
    counts.reset();
    ids_.reset();
    codes_.reset();
    lambdas_.reset();
    eterm_.reset();
    ids_.alloc(std::max<uint64_t>(nloc, 1));
    codes_.alloc(std::max<uint64_t>(nloc * m_, 1));
    lambdas_.alloc(std::max<uint64_t>(nloc, 1));
    eterm_.alloc(std::max<uint64_t>(nloc, 1));
    launch_gather_entries(order.p, nloc, m_, 0, codes_pt.p, lamb_pt.p, eterm_pt.p, ids_.p, codes_.p, lambdas_.p,
                          eterm_.p, st);
    unsigned int flags[2];
    CUDA_CHECK(cudaMemcpyAsync(flags, err_.p, 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (flags[0]) {
        CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 4, st));
        HostLists empty;
        empty.off.assign((size_t)ncell + 1, 0);
        upload_lists(empty);
        throw std::runtime_error("line_lambda: degenerate edge (c == 0)");
    }
    std::memcpy(&emax_, &flags[1], 4);
    nent_ = nloc;
    pack_eterm_lam();
    base_count_ = nb;
    rollback.armed = false;
}

void Engine::encode_host(const float* x, uint64_t nx, uint32_t* cells, float* lambdas, uint8_t* codes,
                         uint8_t* lam_bytes) {
    if (!model_ok_) throw std::runtime_error("encode: no model loaded");
    DeviceGuard g(cfg_.device);
    cudaStream_t st = stream_;
    DevBuf<float> X, lam, et;
    DevBuf<uint32_t> best, cl;
    DevBuf<uint8_t> cd, lb;
    X.alloc(std::max<uint64_t>(nx * dim_, 1));
    lam.alloc(std::max<uint64_t>(nx, 1));
    et.alloc(std::max<uint64_t>(nx, 1));
    best.alloc(std::max<uint64_t>(nx, 1));
    cl.alloc(std::max<uint64_t>(nx, 1));
    cd.alloc(std::max<uint64_t>(nx * m_, 1));
    lb.alloc(std::max<uint64_t>(nx, 1));
    CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 8 * sizeof(unsigned int), st));
    CUDA_CHECK(cudaMemcpyAsync(X.p, x, nx * dim_ * 4, cudaMemcpyHostToDevice, st));
    AddArgs a = add_args();
    assign_chunk(X.p, nx, best.p, st);
    launch_encode(a, X.p, nx, best.p, clamp_ ? 1 : 0, cl.p, lam.p, cd.p, lb.p, et.p, err_.p + 1, st);
    if (cells) CUDA_CHECK(cudaMemcpyAsync(cells, cl.p, nx * 4, cudaMemcpyDeviceToHost, st));
    if (lambdas) CUDA_CHECK(cudaMemcpyAsync(lambdas, lam.p, nx * 4, cudaMemcpyDeviceToHost, st));
    if (codes) CUDA_CHECK(cudaMemcpyAsync(codes, cd.p, nx * m_, cudaMemcpyDeviceToHost, st));
    if (lam_bytes) CUDA_CHECK(cudaMemcpyAsync(lam_bytes, lb.p, nx, cudaMemcpyDeviceToHost, st));
    check_device_errors(st);
}

void Engine::get_lists(HostLists& out, bool offsets_only) {
    DeviceGuard g(cfg_.device);
    out.off.resize((size_t)k_ * n_ + 1);
    out.base_count = base_count_;
    CUDA_CHECK(cudaMemcpyAsync(out.off.data(), list_off_.p, out.off.size() * 8, cudaMemcpyDeviceToHost, stream_));
    if (!offsets_only) {
        out.ids.resize(nent_);
        out.codes.resize(nent_ * m_);
        out.lambdas.resize(nent_);
    }
    if (nent_ && !offsets_only) {
        CUDA_CHECK(cudaMemcpyAsync(out.ids.data(), ids_.p, nent_ * 4, cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaMemcpyAsync(out.codes.data(), codes_.p, nent_ * m_, cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaMemcpyAsync(out.lambdas.data(), lambdas_.p, nent_, cudaMemcpyDeviceToHost, stream_));
    }
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// one CTA per requested cell: copy its entries to their slot of the
// request-ordered output (sampled add replay of 1e9-entry indexes without
// copying the whole index to the host)
__global__ void k_gather_cells(const uint32_t* __restrict__ cells, const uint64_t* __restrict__ dst_off,
                               const uint64_t* __restrict__ list_off, const uint32_t* __restrict__ ids,
                               const uint8_t* __restrict__ codes, const uint8_t* __restrict__ lambdas, uint32_t m,
                               uint32_t* __restrict__ o_ids, uint8_t* __restrict__ o_codes,
                               uint8_t* __restrict__ o_lam) {
    const uint32_t c = cells[blockIdx.x];
    const uint64_t src = list_off[c], len = list_off[c + 1] - src, dst = dst_off[blockIdx.x];
    for (uint64_t e = threadIdx.x; e < len; e += blockDim.x) {
        o_ids[dst + e] = ids[src + e];
        o_lam[dst + e] = lambdas[src + e];
    }
    for (uint64_t b = threadIdx.x; b < len * m; b += blockDim.x) o_codes[dst * m + b] = codes[src * m + b];
}

void Engine::get_cells(const uint32_t* cells, uint32_t ncells, uint64_t* counts, uint32_t* ids, uint8_t* codes,
                       uint8_t* lambdas) {
    DeviceGuard g(cfg_.device);
    const uint64_t ncell_total = (uint64_t)k_ * n_;
    for (uint32_t i = 0; i < ncells; ++i)
        if (cells[i] >= ncell_total) throw std::runtime_error("get_cells: cell id out of range");
    std::vector<uint64_t> off(ncell_total + 1);
    CUDA_CHECK(cudaMemcpyAsync(off.data(), list_off_.p, off.size() * 8, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    std::vector<uint64_t> dst(ncells + 1, 0);
    for (uint32_t i = 0; i < ncells; ++i) {
        const uint64_t len = off[cells[i] + 1] - off[cells[i]];
        if (counts) counts[i] = len;
        dst[i + 1] = dst[i] + len;
    }
    const uint64_t total = dst[ncells];
    if ((!ids && !codes && !lambdas) || total == 0 || ncells == 0) return;
    DevBuf<uint32_t> d_cells, o_ids;
    DevBuf<uint64_t> d_dst;
    DevBuf<uint8_t> o_codes, o_lam;
    d_cells.alloc(ncells);
    d_dst.alloc(ncells + 1);
    o_ids.alloc(total);
    o_codes.alloc(total * m_);
    o_lam.alloc(total);
    CUDA_CHECK(cudaMemcpyAsync(d_cells.p, cells, ncells * 4ull, cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaMemcpyAsync(d_dst.p, dst.data(), (ncells + 1) * 8ull, cudaMemcpyHostToDevice, stream_));
    k_gather_cells<<<ncells, 256, 0, stream_>>>(d_cells.p, d_dst.p, list_off_.p, ids_.p, codes_.p, lambdas_.p, m_,
                                                 o_ids.p, o_codes.p, o_lam.p);
    CUDA_CHECK(cudaGetLastError());
    if (ids) CUDA_CHECK(cudaMemcpyAsync(ids, o_ids.p, total * 4, cudaMemcpyDeviceToHost, stream_));
    if (codes) CUDA_CHECK(cudaMemcpyAsync(codes, o_codes.p, total * m_, cudaMemcpyDeviceToHost, stream_));
    if (lambdas) CUDA_CHECK(cudaMemcpyAsync(lambdas, o_lam.p, total, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::get_tables(std::vector<float>& t2, std::vector<float>& t3) {
    DeviceGuard g(cfg_.device);
    t2.resize((size_t)m_ * VLQ_KSUB);
    t3.resize((size_t)k_ * m_ * VLQ_KSUB);
    CUDA_CHECK(cudaMemcpyAsync(t2.data(), t2_.p, t2.size() * 4, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaMemcpyAsync(t3.data(), t3_.p, t3.size() * 4, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// ---------------------------------------------------------------------------
// search: search_batch (search.cpp:169-191), tiled over queries
// ---------------------------------------------------------------------------
Engine::StageIO Engine::StageIO::at(uint64_t t0, uint32_t w1, uint32_t w2) const {
    StageIO o;
    o.top_in = top_in ? top_in + t0 * w1 : nullptr;
    o.top_out = top_out ? top_out + t0 * w1 : nullptr;
    o.sel_in = sel_in ? sel_in + t0 * w2 : nullptr;
    o.ab_in = ab_in ? ab_in + t0 * w2 * 2 : nullptr;
    o.sel_out = sel_out ? sel_out + t0 * w2 : nullptr;
    o.ab_out = ab_out ? ab_out + t0 * w2 * 2 : nullptr;
    o.parts = parts;
    o.q0 = q0 + t0;
    return o;
}

void Engine::search_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* d_ids,
                           float* d_dists, uint64_t* d_scanned, cudaStream_t st) {
    search_staged(d_q, nq, w1, alpha, topk, d_ids, d_dists, d_scanned, StageIO{}, STAGE_ALL, st);
}

void Engine::search_coarse_device(const float* d_q, uint64_t nq, uint32_t w1, uint32_t* d_top, cudaStream_t st) {
    if (!d_top) throw std::runtime_error("search_coarse: top output is NULL");
    StageIO io;
    io.top_out = d_top;
    search_staged(d_q, nq, w1, 0.0f, 1, nullptr, nullptr, nullptr, io, STAGE_COARSE, st);
}

void Engine::search_fine_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                                const uint32_t* d_top, int64_t* d_ids, float* d_dists, uint64_t* d_scanned,
                                cudaStream_t st) {
    if (!d_top) throw std::runtime_error("search_fine: top input is NULL");
    StageIO io;
    io.top_in = d_top;
    search_staged(d_q, nq, w1, alpha, topk, d_ids, d_dists, d_scanned, io, STAGE_FINE, st);
}
void Engine::search_select_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t* d_sel,
                                  float* d_ab, cudaStream_t st) {
    if (!d_sel || !d_ab) throw std::runtime_error("search_select: selection output is NULL");
    StageIO io;
    io.sel_out = d_sel;
    io.ab_out = d_ab;
    search_staged(d_q, nq, w1, alpha, 1, nullptr, nullptr, nullptr, io, STAGE_SELECT, st);
}
void Engine::search_fine_sel_device(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                                    const uint32_t* d_sel, const float* d_ab, int64_t* d_ids, float* d_dists,
                                    uint64_t* d_scanned, cudaStream_t st) {
    if (!d_sel || !d_ab) throw std::runtime_error("search_fine_sel: selection input is NULL");
    StageIO io;
    io.sel_in = d_sel;
    io.ab_in = d_ab;
    search_staged(d_q, nq, w1, alpha, topk, d_ids, d_dists, d_scanned, io, STAGE_FINE_SEL, st);
}

void Engine::search_fine_sel_parts(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk,
                                   const SelParts& parts, int64_t* d_ids, float* d_dists, uint64_t* d_scanned,
                                   cudaStream_t st) {
    if (parts.nparts == 0 || parts.nparts > VLQ_MAX_PARTS) throw std::runtime_error("search_fine_sel: bad parts");
    StageIO io;
    io.parts = &parts;
    search_staged(d_q, nq, w1, alpha, topk, d_ids, d_dists, d_scanned, io, STAGE_FINE_SEL, st);
}

void Engine::search_staged(const float* d_q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* d_ids,
                           float* d_dists, uint64_t* d_scanned, const StageIO& io, Stage stage, cudaStream_t st) {
    if (!model_ok_) throw std::runtime_error("search: no model loaded");
    if (w1 == 0 || w1 > k_) throw std::runtime_error("first_level_scan: need 0 < w1 <= k");
    if (nq == 0) return;
    DeviceGuard g(cfg_.device);
    const uint32_t w2 = w2_of(w1, alpha, n_);
    if (cfg_.scan_adapt_keep) {
        if (!flag_seen_.p) {
            flag_seen_.alloc(64);
            std::memset(flag_seen_.p, 0, 64);
        }
        const uint32_t f = *reinterpret_cast<volatile uint32_t*>(flag_seen_.p);
        if (flag_seen_nq_ && (uint64_t)f * 50 > flag_seen_nq_ && keep_boost_ < 4) keep_boost_ *= 2;
    }
    const uint32_t keep = scan_keep(topk);
    const uint64_t per_q = 4ull * k_ + 8ull * w1 + 128 + 4ull * w1 * n_ + 4ull * w2 + 4ull * VLQ_KSUB * m_ + 8ull * keep +
                           sizeof(QueryMeta) + 4;
    uint64_t tile = std::max<uint64_t>(1, cfg_.workspace_bytes / per_q);
    tile = std::min<uint64_t>(tile, cfg_.max_tile);
    tile = std::min<uint64_t>(tile, nq);
    ws_.alloc(tile * k_);
    top_.alloc(tile * w1);
    cand_top_.alloc(tile * (uint64_t)std::min<uint32_t>(k_, w1 + std::max<uint32_t>(32, w1 / 2)));
    if (tc_) {
        const uint32_t tn = tc_split_ ? 64 : 128;
        tmin_.alloc(tile * (uint64_t)(((k_ + tn - 1) / tn) * (tn / 32)));
        tau_.alloc(tile);
        lcnt_.alloc(tile);
        lidx_.alloc(tile * (uint64_t)kListCap);
        ld_.alloc(tile * (uint64_t)kListCap);
        if (cfg_.tc_chunk_select) {
            tmin8_.alloc(tile * (uint64_t)(((k_ + 127) / 128) * 16));
            tch_.alloc(tile);
            ccnt_.alloc(tile);
            clist_.alloc(tile * (uint64_t)cfg_.tc_chunk_cap);
        }
    }
    dbuf_.alloc(tile * (uint64_t)w1 * n_);
    sel_.alloc(tile * w2);
    t5_.alloc(tile * VLQ_KSUB * m_);
    cand_.alloc(tile * keep);
    if (cfg_.scan_retry) cand2_.alloc(tile * (uint64_t)std::min<uint32_t>(512, 4 * keep));
    qlist2_.alloc(tile);
    cnt2_.alloc(1);
    meta_.alloc(tile);
    qlist_.alloc(tile);
    lpt_.alloc(tile);
    lpt_cnt_.alloc(1);
    for (uint64_t t0 = 0; t0 < nq; t0 += tile) {
        const uint64_t nt = std::min(tile, nq - t0);
        search_tile(d_q + t0 * dim_, nt, w1, w2, topk, d_ids ? d_ids + t0 * topk : nullptr,
                    d_dists ? d_dists + t0 * topk : nullptr, d_scanned ? d_scanned + t0 : nullptr,
                    io.at(t0, w1, w2), stage, st);
    }
}

void Engine::search_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint32_t topk, int64_t* d_ids,
                         float* d_dists, uint64_t* d_scanned, const StageIO& io, Stage stage, cudaStream_t st) {
    auto mark = [&](int ph) { mark_phase(ph, st); };
    uint64_t launches = 0;
    bool tc = false, fast = false, fused = false;
    mark(PH_COARSE);
    if (stage == STAGE_FINE) {
        // top-w1 from another rank's coarse stage: exact distances of the
        // regions and neighbours the later stages read (as the TC path does)
        CUDA_CHECK(cudaMemcpyAsync(top_.p, io.top_in, nt * w1 * 4, cudaMemcpyDeviceToDevice, st));
        mark(PH_FIRST);
        if (exact_needed_smem(k_, n_, w1, dim_) <= 200 * 1024)
            launch_exact_needed(d_q, nt, dim_, centroids_.p, k_, n_, nbr_.p, ws_.p, top_.p, w1, st);
        else
            launch_sqdist_matrix(d_q, nt, centroids_.p, k_, dim_, ws_.p, k_, st);
        launches += 1;
    } else if (stage == STAGE_FINE_SEL) {
        mark(PH_FIRST);  // the selection (and its coarse values) comes from another rank
    } else {
        tc = coarse_tile(d_q, nt, w1, w2, launches, st, &fused, stage == STAGE_SELECT ? io.sel_out : nullptr,
                         stage == STAGE_SELECT ? io.ab_out : nullptr);
    }
    if (stage == STAGE_COARSE) {
        CUDA_CHECK(cudaMemcpyAsync(io.top_out, top_.p, nt * w1 * 4, cudaMemcpyDeviceToDevice, st));
        for (int p = PH_SECOND; p <= PH_COUNT; p++) mark(p);
    } else if (stage == STAGE_SELECT) {
        SearchArgs a = search_args();
        mark(PH_SECOND);
        if (!fused) {
            launch_second_level(a, nt, w1, w2, st);
            launch_pack_selection(a, nt, w2, io.sel_out, io.ab_out, st);
            launches += 2;
        }
        for (int p = PH_TERM5; p <= PH_COUNT; p++) mark(p);
    } else {
        fast = fine_tile(d_q, nt, w1, w2, topk, d_ids, d_dists, d_scanned, launches, st,
                         stage == STAGE_FINE_SEL ? &io : nullptr, fused);
    }
    stats_.launches += launches;
    stats_.tiles += 1;
    if (profiling_) {
        // counters travel with the events; everything is read lazily in
        // collect_profile(), so profiling never blocks the host mid-batch
        ProfSlot& sl = prof_[prof_used_];
        sl.fast = fast;
        sl.tc = tc;
        unsigned int* hv = sl.counts;
        if (fast) CUDA_CHECK(cudaMemcpyAsync(hv, err_.p + 2, 4, cudaMemcpyDeviceToHost, st));
        if (tc) CUDA_CHECK(cudaMemcpyAsync(hv + 1, err_.p + 6, 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaEventRecord(sl.done, st));
        prof_used_++;
    }
}

// first_level_scan (search.cpp:11-36): exact top-w1 regions into top_ (and,
// on the tensor-core path, exact ws_ entries for them and their neighbours).
// Returns whether the tensor-core path ran.
bool Engine::coarse_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint64_t& launches, cudaStream_t st,
                         bool* fused, uint32_t* sel_out, float* ab_out) {
    auto mark = [&](int ph) { mark_phase(ph, st); };
    *fused = false;
    // chunk-select path (select_fused.cu): one 1xTF32 pass of 8-centroid chunk
    // minima, the chunks within the TF32 bound of the w1-th smallest, exact
    // evaluation + first and second level fused per query
    if (w2 > 0 && tc_ && cfg_.tc_chunk_select && k_ >= cfg_.tc_search_min_k && k_ <= 262144 && w1 < k_ &&
        (k_ + 7) / 8 >= 2 * w1 &&
        select_split_supported(k_, n_, w1, w2, dim_, cfg_.tc_chunk_cap) && tmin8_.p) {
        const uint32_t nchunk8 = ((k_ + 127) / 128) * 16;
        const float* x1 = nullptr;
        // centered operands (queries relaid out here, so the persistent form only)
        const bool cen = cfg_.tc_center && cfg_.tc_persist && cent_tcc_.p;
        const float* mu = cen ? mu_.p : nullptr;
        const float cmx = cen ? cmaxc_ : cmax_;
        if (cfg_.tc_persist) {
            const uint64_t rows = ((nt + 127) / 128) * 128;
            if (!xtc1_.p || xtc1_.n < rows * dim_) xtc1_.alloc(rows * dim_);
            launch_relayout_centroids(d_q, (uint32_t)nt, dim_, xtc1_.p, nullptr, nullptr, st, /*rna=*/1, mu);
            x1 = xtc1_.p;
            launches += 1;
        }
        launch_coarse_tc(4, d_q, nt, dim_, cen ? cent_tcc_.p : cent_tc_.p, nullptr, cen ? cnorm_tcc_.p : cnorm_tc_.p,
                         k_, tmin8_.p, nchunk8, nullptr, nullptr, st, nullptr, nullptr, 0, x1, nullptr);
        mark(PH_FIRST);  // the coarse phase is the tensor-core GEMM alone (its roofline in bench.py)
        launch_chunk_select(tmin8_.p, nt, nchunk8, w1, d_q, dim_, cmx, cfg_.tc_chunk_cap, clist_.p, ccnt_.p,
                            tch_.p, st, mu);
        SearchArgs a = search_args();
        CUDA_CHECK(cudaMemsetAsync(err_.p + 6, 0, 4, st));
        // row kernels at full occupancy + light per-query selections (select_fused.cu)
        const uint32_t ldn = select_need_capacity(n_, w1), nk = select_chunk_keys();
        svals_.alloc((uint64_t)nt * nk);
        snid_.alloc((uint64_t)nt * ldn);
        snval_.alloc((uint64_t)nt * ldn);
        snneed_.alloc(nt);
        launch_rows(centroids_.p, d_q, k_, dim_, 1, clist_.p, ccnt_.p, cfg_.tc_chunk_cap, cfg_.tc_chunk_cap,
                    svals_.p, nk, nt, st);
        launch_top_need(a, nt, d_q, w1, w2, clist_.p, ccnt_.p, cfg_.tc_chunk_cap, tch_.p, cmx, nullptr, nullptr,
                        qlist_.p, err_.p + 6, svals_.p, snid_.p, snneed_.p, ldn, st, mu);
        // certificate failures / chunk-list overflows: exact full rows, exact
        // top-w1, then the needed ids from that top-w1
        launch_exact_rows(d_q, nt, dim_, centroids_.p, k_, ws_.p, qlist_.p, err_.p + 6, st);
        launch_first_level_list(ws_.p, nt, k_, w1, top_.p, qlist_.p, err_.p + 6, st);
        launch_top_need(a, nt, d_q, w1, w2, nullptr, nullptr, 0, nullptr, cmax_, qlist_.p, err_.p + 6, nullptr,
                        nullptr, svals_.p, snid_.p, snneed_.p, ldn, st);
        launch_rows(centroids_.p, d_q, k_, dim_, 0, snid_.p, snneed_.p, ldn, 0, snval_.p, ldn, nt, st);
        launch_second_sel(a, nt, w1, w2, snid_.p, snval_.p, snneed_.p, ldn, sel_out, ab_out, st);
        launches += 8;
        *fused = true;
        return true;
    }
    const uint32_t L = std::min<uint32_t>(k_, w1 + std::max<uint32_t>(32, w1 / 2));
    const bool tc = tc_ && k_ >= cfg_.tc_search_min_k && L <= 2048 && w1 < k_ &&
                    exact_needed_smem(k_, n_, w1, dim_) <= 200 * 1024;
    const float* c_hi = tc_split_ ? cent_hi_.p : cent_tc_.p;
    const float* c_lo = tc_split_ ? cent_lo_.p : nullptr;
    const uint32_t tn = tc_split_ ? 64 : 128;
    const uint32_t nchunk = ((k_ + tn - 1) / tn) * (tn / 32);
    const bool two_pass = tc && nchunk >= 2 * L && !cfg_.tc_store_rows;
    // persistent coarse kernels (all SMs busy at any batch size): the query
    // rows re-laid out once per tile in the UMMA layout (hi / lo halves)
    const float* xtc = nullptr;
    const float* xlo = nullptr;
    if (tc && cfg_.tc_persist) {
        const uint64_t rows = ((nt + 127) / 128) * 128;
        xtc_.alloc(rows * dim_);
        if (tc_split_) xlo_.alloc(rows * dim_);
        launch_relayout_centroids(d_q, (uint32_t)nt, dim_, xtc_.p, tc_split_ ? xlo_.p : nullptr, nullptr, st);
        xtc = xtc_.p;
        xlo = tc_split_ ? xlo_.p : nullptr;
        launches += 1;
    }
    // filter pass in 1xTF32 as well (study knob): tau raised by two 1x bounds
    const bool p2single = two_pass && tc_split_ && cfg_.tc_pass1_single && cfg_.tc_pass2_single;
    if (two_pass) {
        // pass 1: chunk minima -> tau (upper bound of the L-th smallest);
        // pass 2: recompute, keep only approx <= tau (no K-wide row in HBM)
        const float* x1 = nullptr;
        if (tc_split_ && cfg_.tc_pass1_single) {
            // pass 1 in 1xTF32 on 128-centroid tiles (a third of the MMAs; same
            // 32-column chunks), tau raised by its error bound
            if (!xtc1_.p || xtc1_.n < ((nt + 127) / 128) * 128 * dim_) {
                xtc1_.alloc(((nt + 127) / 128) * 128 * dim_);
            }
            if (cfg_.tc_persist) {
                launch_relayout_centroids(d_q, (uint32_t)nt, dim_, xtc1_.p, nullptr, nullptr, st);
                x1 = xtc1_.p;
            }
            launch_coarse_tc(2, d_q, nt, dim_, cent_tc_.p, nullptr, cnorm_tc_.p, k_, tmin_.p, nchunk, nullptr, nullptr,
                             st, nullptr, nullptr, 0, x1, nullptr);
            launch_tau_rows(tmin_.p, nt, nchunk, L, cand_top_.p, tau_.p, st, d_q, dim_, cmax_, p2single ? 0 : 1);
        } else {
            launch_coarse_tc(2, d_q, nt, dim_, c_hi, c_lo, cnorm_tc_.p, k_, tmin_.p, nchunk, nullptr, nullptr, st,
                             nullptr, nullptr, 0, xtc, xlo);
            launch_tau_rows(tmin_.p, nt, nchunk, L, cand_top_.p, tau_.p, st);
        }
        CUDA_CHECK(cudaMemsetAsync(lcnt_.p, 0, nt * 4, st));
        if (p2single)
            launch_coarse_tc(3, d_q, nt, dim_, cent_tc_.p, nullptr, cnorm_tc_.p, k_, nullptr, 0, lidx_.p, ld_.p, st,
                             tau_.p, lcnt_.p, kListCap, x1, nullptr);
        else
            launch_coarse_tc(3, d_q, nt, dim_, c_hi, c_lo, cnorm_tc_.p, k_, nullptr, 0, lidx_.p, ld_.p, st, tau_.p,
                             lcnt_.p, kListCap, xtc, xlo);
        launches += 3;
    } else if (tc) {
        // approximate rows on the tensor cores, then top-L on them
        launch_coarse_tc(1, d_q, nt, dim_, c_hi, c_lo, cnorm_tc_.p, k_, ws_.p, k_, nullptr, nullptr, st, nullptr,
                         nullptr, 0, xtc, xlo);
        launches += 1;
    } else {
        launch_sqdist_matrix(d_q, nt, centroids_.p, k_, dim_, ws_.p, k_, st);
        launches += 1;
    }
    mark(PH_FIRST);
    if (tc) {
        CUDA_CHECK(cudaMemsetAsync(err_.p + 6, 0, 4, st));
        if (two_pass) {
            launch_refine_list(d_q, nt, dim_, centroids_.p, k_, lidx_.p, lcnt_.p, kListCap, tau_.p, w1, cmax_,
                               (tc_split_ && !p2single) ? 1 : 0, top_.p, qlist_.p, err_.p + 6, st);
        } else {
            launch_first_level(ws_.p, nt, k_, L, cand_top_.p, st);
            launch_refine_first(d_q, nt, dim_, centroids_.p, ws_.p, k_, cand_top_.p, L, w1, cmax_, top_.p, qlist_.p,
                                err_.p + 6, tc_split_ ? 1 : 0, st);
        }
        launch_exact_rows(d_q, nt, dim_, centroids_.p, k_, ws_.p, qlist_.p, err_.p + 6, st);
        launch_first_level_list(ws_.p, nt, k_, w1, top_.p, qlist_.p, err_.p + 6, st);
        launch_exact_needed(d_q, nt, dim_, centroids_.p, k_, n_, nbr_.p, ws_.p, top_.p, w1, st);
        launches += 5;
    } else {
        launch_first_level(ws_.p, nt, k_, w1, top_.p, st);
        launches += 1;
    }
    return tc;
}

// second_level_rank -> query_term5 -> fused scan + top-k' -> exact re-score
// (search.cpp:38-167) from top_ / ws_.  Returns whether the fast scan ran.
bool Engine::fine_tile(const float* d_q, uint64_t nt, uint32_t w1, uint32_t w2, uint32_t topk, int64_t* d_ids,
                       float* d_dists, uint64_t* d_scanned, uint64_t& launches, cudaStream_t st,
                       const StageIO* sel, bool second_done) {
    auto mark = [&](int ph) { mark_phase(ph, st); };
    SearchArgs a = search_args();
    mark(PH_SECOND);
    if (sel && sel->parts) launch_apply_selection_parts(a, nt, w2, *sel->parts, sel->q0, st);
    else if (sel) launch_apply_selection(a, nt, w2, sel->sel_in, sel->ab_in, st);
    else if (!second_done) launch_second_level(a, nt, w1, w2, st);
    mark(PH_TERM5);
    launch_term5(cfg_.cert_slack, d_q, pqT_.p, dim_, m_, t5_.p, meta_.p, nt, st);
    launches += 2;
    const uint32_t keep_x = next_pow2(std::max<uint32_t>(32, topk));
    const uint32_t buf_x = 2 * keep_x;
    const uint32_t warps_x = std::min<uint32_t>(8, std::max<uint32_t>(1, 8192 / buf_x));
    const bool fast = !cfg_.force_exact && topk > 0 && topk <= 768;
    if (fast) {
        const uint32_t keep = scan_keep(topk);
        mark(PH_SCAN);
        if (cfg_.scan_packed && cfg_.scan_variant == 0 && eterm_lam_.p && (m_ == 16 || m_ == 8 || m_ == 4)) {
            a.eterm_lam = eterm_lam_.p;
            if (cfg_.scan_reorder && scodes_.p) {  // the reordered copy (build_scan_order)
                a.eterm_lam = seterm_lam_.p;
                a.scodes = scodes_.p;
                a.sids = sids_.p;
                a.code_perm = code_perm_.p;
                a.code_inv = code_inv_.p;
            }
            a.e_pack_err = std::ldexp(emax_, -15) * 1.0001f;  // |e - e'| <= 2^-15 |e|
        }
        a.scan_cap = cfg_.scan_cap;
        a.round_cap = cfg_.scan_round_cap;
        a.sel_agg = cfg_.scan_sel_agg != 0;
        a.flush_exact = cfg_.scan_flush_exact != 0;
        const int slots = cfg_.scan_slots ? cfg_.scan_slots : (cfg_.shard_count >= 4 ? 104 : 306);
        // fast_kind: the fused fast scan ran (the only kernel with the retry indirection)
        const bool fast_kind = cfg_.scan_variant == 0 && (m_ == 16 || m_ == 8 || m_ == 4) && w2 <= 4096 &&
                               keep <= 512;
        // the fast scan (and its re-score) visit the queries longest first
        SearchArgs sa = a;
        if (fast_kind && cfg_.scan_lpt && nt > 1) {
            launch_lpt_order(meta_.p, nt, lpt_.p, lpt_cnt_.p, st);
            sa.qlist = lpt_.p;
            sa.qcount = lpt_cnt_.p;
            sa.qorder = true;
            launches += 1;
        }
        if (!fast_kind || !launch_scan_fast(sa, nt, w2, keep, slots, st)) {
            // the generic scan keys canonical positions: re-score from the canonical arrays
            a.scodes = nullptr;
            a.sids = nullptr;
            a.code_perm = a.code_inv = nullptr;
            if (a.eterm_lam) a.eterm_lam = eterm_lam_.p;
            sa = a;
            launch_scan(a, nt, w2, keep, 2 * keep, 8, true, nullptr, nullptr, st);
        }
        mark(PH_RESCORE);
        launch_rescore(sa, nt, w2, keep, topk, d_ids, d_dists, st);
        mark(PH_FALLBACK);
        CUDA_CHECK(cudaMemsetAsync(err_.p + 2, 0, 4, st));
        launch_compact_flags(meta_.p, nt, qlist_.p, err_.p + 2, st);
        if (cfg_.scan_adapt_keep && flag_seen_.p) {
            CUDA_CHECK(cudaMemcpyAsync(flag_seen_.p, err_.p + 2, 4, cudaMemcpyDeviceToHost, st));
            flag_seen_nq_ = nt;
        }
        const uint32_t keep2 = std::min<uint32_t>(512, 4 * keep);
        if (cfg_.scan_retry && keep2 > keep && fast_kind) {
            // certificate failures (near-ties at the k'-th fast distance): the
            // fast scan again with 4x the survivors, for the listed queries only
            // (blocks past the device-side count exit at once), then re-score;
            // what still fails takes the exact scan
            SearchArgs r = a;
            r.cand = cand2_.p;
            r.qlist = qlist_.p;
            r.qcount = err_.p + 2;
            // few queries: the 8-warp CTAs finish each one sooner
            launch_scan_fast(r, nt, w2, keep2, slots == 306 ? 6 : slots, st);
            launch_rescore(r, nt, w2, keep2, topk, d_ids, d_dists, st);
            CUDA_CHECK(cudaMemsetAsync(cnt2_.p, 0, 4, st));
            launch_compact_flags(meta_.p, nt, qlist2_.p, cnt2_.p, st);
            launch_scan(a, nt, w2, keep_x, buf_x, warps_x, false, qlist2_.p, cnt2_.p, st);
            launch_emit_exact(a, qlist2_.p, cnt2_.p, nt, keep_x, topk, d_ids, d_dists, st);
            launches += 7;
        } else {
            launch_scan(a, nt, w2, keep_x, buf_x, warps_x, false, qlist_.p, err_.p + 2, st);
            launch_emit_exact(a, qlist_.p, err_.p + 2, nt, keep_x, topk, d_ids, d_dists, st);
            launches += 5;
        }
    } else {
        mark(PH_SCAN);
        mark(PH_RESCORE);
        mark(PH_FALLBACK);
        if (topk > 1024) {
            // k beyond the exact scan's block buffers: every scanned entry's exact
            // key, sorted per query (large_k.cu); the scanned counts size the groups
            std::vector<uint64_t> h_sc(nt);
            DevBuf<uint64_t> d_sc;
            d_sc.alloc(nt);
            launch_copy_scanned(meta_.p, nt, d_sc.p, st);
            CUDA_CHECK(cudaMemcpyAsync(h_sc.data(), d_sc.p, nt * 8, cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaStreamSynchronize(st));
            launch_topk_large(a, nt, w2, topk, h_sc.data(), 64ull << 20, d_ids, d_dists, st);
            launches += 4;
        } else if (topk > 0) {
            launch_scan(a, nt, w2, keep_x, buf_x, warps_x, false, nullptr, nullptr, st);
            launch_emit_exact(a, nullptr, nullptr, nt, keep_x, topk, d_ids, d_dists, st);
            launches += 2;
        }
    }
    mark(PH_OUT);
    if (d_scanned) {
        launch_copy_scanned(meta_.p, nt, d_scanned, st);
        launches += 1;
    }
    mark(PH_COUNT);
    return fast;
}

// fast-scan survivors per query (k'): the smallest power of two >= k + max(16, k/4),
// at least scan_keep_min (a study knob), at most 512 (the fast scan's limit)
uint32_t Engine::scan_keep(uint32_t topk) const {
    uint32_t keep = next_pow2(std::max<uint32_t>(32, topk + std::max<uint32_t>(16, topk / 4)));
    if (keep_boost_ > 1 && keep < 512) keep = std::min<uint32_t>(512, keep * keep_boost_);
    if (cfg_.scan_keep_min > keep) keep = std::min<uint32_t>(512, next_pow2(cfg_.scan_keep_min));
    return keep;
}

void Engine::set_tuning(const std::string& key, int64_t value) {
    if (key == "scan_variant") cfg_.scan_variant = (int)value;
    else if (key == "scan_slots") cfg_.scan_slots = (int)value;
    else if (key == "scan_reorder") cfg_.scan_reorder = (int)value;
    else if (key == "scan_relabel") {  // rebuilds the scan copy with / without the relabeling
        cfg_.scan_relabel = (int)value;
        if (scodes_.p) build_scan_order();
    }
    else if (key == "scan_lpt") cfg_.scan_lpt = (int)value;
    else if (key == "scan_round_cap") cfg_.scan_round_cap = (uint32_t)value;
    else if (key == "cert_slack_milli") cfg_.cert_slack = (float)value * 1e-3f;
    else if (key == "tc_search_min_k") cfg_.tc_search_min_k = (uint32_t)value;
    else if (key == "force_exact") cfg_.force_exact = (int)value;
    else if (key == "tc_persist") cfg_.tc_persist = (int)value;
    else if (key == "tc_pass1_single") cfg_.tc_pass1_single = (int)value;
    else if (key == "tc_pass2_single") cfg_.tc_pass2_single = (int)value;
    else if (key == "tc_chunk_select") cfg_.tc_chunk_select = (int)value;
    else if (key == "tc_chunk_cap") cfg_.tc_chunk_cap = (uint32_t)value;
    else if (key == "tc_center") cfg_.tc_center = (int)value;
    else if (key == "scan_packed") cfg_.scan_packed = (int)value;
    else if (key == "scan_keep_min") cfg_.scan_keep_min = (uint32_t)value;
    else if (key == "scan_cap") cfg_.scan_cap = (uint32_t)value;
    else if (key == "scan_retry") cfg_.scan_retry = (int)value;
    else if (key == "scan_adapt_keep") {
        cfg_.scan_adapt_keep = (int)value;
        keep_boost_ = 1;
        flag_seen_nq_ = 0;
    }
    else if (key == "scan_sel_agg") cfg_.scan_sel_agg = (int)value;
    else if (key == "scan_flush_exact") cfg_.scan_flush_exact = (int)value;
    else throw std::runtime_error("set_tuning: unknown key " + key);
}

// Per-tile phase events (profiling on): a pool of event sets, one per tile
// searched since the last collection; no host synchronisation until
// collect_profile().
void Engine::grow_profile(size_t slots) {
    while (prof_.size() < slots) {
        prof_.emplace_back();
        ProfSlot& sl = prof_.back();
        for (auto& e : sl.ev) CUDA_CHECK(cudaEventCreate(&e));
        CUDA_CHECK(cudaEventCreate(&sl.done));
        CUDA_CHECK(cudaMallocHost(&sl.counts, 2 * sizeof(unsigned int)));
    }
}

void Engine::mark_phase(int ph, cudaStream_t st) {
    if (!profiling_) return;
    if (prof_used_ == prof_.size()) grow_profile(2 * prof_.size() + 16);  // slots are pre-made by set_profiling
    CUDA_CHECK(cudaEventRecord(prof_[prof_used_].ev[ph], st));
}

void Engine::collect_profile() {
    if (prof_used_ == 0) return;
    DeviceGuard g(cfg_.device);
    for (size_t i = 0; i < prof_used_; i++) {
        ProfSlot& sl = prof_[i];
        CUDA_CHECK(cudaEventSynchronize(sl.done));
        for (int p = 0; p < PH_COUNT; p++) {
            float ms = 0.0f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, sl.ev[p], sl.ev[p + 1]));
            stats_.phase_ms[p] += ms;
        }
        const unsigned int* hv = sl.counts;
        if (sl.fast) stats_.flagged += hv[0];
        if (sl.tc) stats_.tc_refine_fallbacks += hv[1];
    }
    prof_used_ = 0;
}

const EngineStats& Engine::stats() {
    collect_profile();
    return stats_;
}

void Engine::reset_stats() {
    collect_profile();
    stats_ = EngineStats();
}

void Engine::set_profiling(bool on) {
    DeviceGuard g(cfg_.device);
    if (!on) collect_profile();
    // event sets and pinned counters are created here, never inside a timed
    // batch (cudaMallocHost synchronises the device)
    if (on) grow_profile(64);
    profiling_ = on;
}

// host copy between the caller's (pageable) arrays and the pinned staging:
// split over a small persistent worker pool above 1 MiB -- a single thread is
// bound by the first-touch page faults of freshly allocated numpy outputs
// (~1 ms for the 12 MB of a 10k x 100 result), and spawning threads per call
// costs about as much as it saves
namespace {
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    unsigned workers() const { return (unsigned)th_.size(); }
    // runs fn(0..n-1): parts 1..n-1 on the workers, part 0 on the caller
    void run(unsigned n, const std::function<void(unsigned)>& fn) {
        std::unique_lock<std::mutex> lk(call_mu_);  // one batch at a time
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            next_ = 1;
            total_ = n;
            pending_ = n - 1;
            gen_++;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            gen_++;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned i = 0; i + 1 < std::min(8u, hw); i++) th_.emplace_back([this] { loop(); });
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> g(mu_);
        for (;;) {
            cv_.wait(g, [&] { return stop_ || (gen_ != seen && next_ < total_); });
            if (stop_) return;
            seen = gen_;
            while (next_ < total_) {
                const unsigned part = next_++;
                const std::function<void(unsigned)>* fn = fn_;
                g.unlock();
                (*fn)(part);
                g.lock();
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(unsigned)>* fn_ = nullptr;
    unsigned next_ = 0, total_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
}  // namespace

// every float of [p, p + n) finite (VectorSet::validate, vecset.cpp:14-18):
// an exponent-field test the compiler vectorises
static bool all_finite(const float* p, size_t n) {
    uint32_t bad = 0;
    for (size_t i = 0; i < n; i++) {
        uint32_t u;
        std::memcpy(&u, p + i, 4);
        bad |= (uint32_t)((u & 0x7f800000u) == 0x7f800000u);
    }
    return bad == 0;
}

// Evicts [p, p + n) from every CPU cache.  Pinned staging lines left dirty
// or shared in several cores' caches by the worker threads make the next DMA
// snoop them: measured on the GPU box (scripts/cuda/copy_probe.cu), a 3.84 MB
// H2D fell from 45 to 6.4 GB/s and a 12 MB D2H from 55 to 15 GB/s after an
// 8-thread copy, and recovered fully with this flush.
#if defined(__x86_64__)
__attribute__((target("clflushopt"))) static void flush_lines_opt(const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    for (size_t i = 0; i < n; i += 64) _mm_clflushopt(const_cast<char*>(c + i));
    _mm_sfence();
}
static void flush_lines(const void* p, size_t n) {
    static const bool opt = __builtin_cpu_supports("clflushopt");
    if (opt) {
        flush_lines_opt(p, n);
        return;
    }
    const char* c = static_cast<const char*>(p);
    for (size_t i = 0; i < n; i += 64) _mm_clflush(c + i);
    _mm_mfence();
}
#else
static void flush_lines(const void*, size_t) {}
#endif

enum class Pinned { Dst, Src, NoFlush };  // the side of a staging copy to flush (the pinned DMA buffer)

// copies `bytes` and, when check_f32, returns whether every copied float is
// finite (checked on the cache-hot destination); the pinned side's lines are
// flushed afterwards by the thread that touched them
static bool par_memcpy(void* dst, const void* src, size_t bytes, Pinned pinned, bool check_f32 = false) {
    const size_t kMin = 1u << 20;
    CopyPool& pool = CopyPool::get();
    const unsigned nt = (unsigned)std::min<size_t>(pool.workers() + 1, bytes / kMin);
    if (nt <= 1) {  // one thread's cache: the DMA snoops it cheaply (measured), no flush
        std::memcpy(dst, src, bytes);
        return !check_f32 || all_finite(static_cast<const float*>(dst), bytes / 4);
    }
    const size_t per = ((bytes + nt - 1) / nt + 4095) & ~(size_t)4095;
    std::atomic<bool> ok{true};
    pool.run(nt, [&](unsigned t) {
        if (t * per < bytes) {
            const size_t nb = std::min(per, bytes - t * per);
            char* d = static_cast<char*>(dst) + t * per;
            const char* sp = static_cast<const char*>(src) + t * per;
            std::memcpy(d, sp, nb);
            if (check_f32 && !all_finite(reinterpret_cast<const float*>(d), nb / 4)) ok = false;
            if (pinned != Pinned::NoFlush)
                flush_lines(pinned == Pinned::Dst ? static_cast<const void*>(d) : static_cast<const void*>(sp), nb);
        }
    });
    return ok;
}

// Touch every page of a (typically freshly allocated) host output buffer so
// its page faults -- the kernel zeroing ~3000 pages for 12 MB of results --
// happen while the GPU is still searching, not inside the final copy.
void par_prefault(void* dst, size_t bytes) {
    if (!dst || bytes == 0) return;
    const size_t kMin = 1u << 20;
    CopyPool& pool = CopyPool::get();
    const unsigned nt = (unsigned)std::max<size_t>(1, std::min<size_t>(pool.workers() + 1, bytes / kMin));
    const size_t per = ((bytes + nt - 1) / nt + 4095) & ~(size_t)4095;
    auto touch = [&](unsigned t) {
        volatile char* d = static_cast<volatile char*>(dst);
        for (size_t o = t * per; o < std::min(bytes, (size_t)(t + 1) * per); o += 4096) d[o] = 0;
    };
    if (nt <= 1) touch(0);
    else pool.run(nt, touch);
}

void Engine::search_host(const float* q, uint64_t nq, uint32_t w1, float alpha, uint32_t topk, int64_t* ids,
                         float* dists, uint64_t* scanned) {
    if (!model_ok_) throw std::runtime_error("search: no model loaded");
    if (nq == 0) return;  // search_batch runs no query, so first_level_scan never checks w1 (search.cpp:169-191)
    DeviceGuard g(cfg_.device);
    cudaStream_t st = stream_;
    static const bool timing = std::getenv("VLQ_HOST_TIMING") != nullptr;  // diagnostics: phase wall times
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t0 = now();
    // grow-only device buffers and pinned host staging: no per-call
    // cudaMalloc/cudaFree (cudaFree synchronises the device) and full-speed
    // DMA instead of pageable copies
    const size_t qb = nq * dim_ * 4, ib = nq * topk * 8, db = nq * topk * 4, sb = nq * 8;
    sq_.alloc(nq * dim_);
    si_.alloc(std::max<uint64_t>(nq * topk, 1));
    sd_.alloc(std::max<uint64_t>(nq * topk, 1));
    ss_.alloc(nq);
    if (qb + ib + db + sb > pin_.n && flusher_.joinable()) flusher_.join();  // never free a buffer being flushed
    pin_.alloc(qb + ib + db + sb);
    unsigned char* pq = pin_.p;
    unsigned char* pi = pq + qb;
    unsigned char* pd = pi + ib;
    unsigned char* ps = pd + db;
    // the query copy validates it too (to_vecset's VectorSet::validate,
    // bindings.cpp:23-31): the Python mirror skips its own numpy pass
    if (!par_memcpy(pq, q, qb, Pinned::Dst, /*check_f32=*/true))
        throw std::runtime_error("VectorSet: non-finite value");
    if (w1 == 0 || w1 > k_) throw std::runtime_error("first_level_scan: need 0 < w1 <= k");
    const auto t1 = now();
    cudaEvent_t tev[4] = {};
    if (timing)
        for (auto& e : tev) CUDA_CHECK(cudaEventCreate(&e));
    if (timing) CUDA_CHECK(cudaEventRecord(tev[0], st));
    CUDA_CHECK(cudaMemsetAsync(err_.p, 0, 4, st));
    CUDA_CHECK(cudaMemcpyAsync(sq_.p, pq, qb, cudaMemcpyHostToDevice, st));
    if (timing) CUDA_CHECK(cudaEventRecord(tev[1], st));
    search_device(sq_.p, nq, w1, alpha, topk, si_.p, sd_.p, ss_.p, st);
    if (timing) CUDA_CHECK(cudaEventRecord(tev[2], st));
    if (topk) {  // overlapped with the search
        par_prefault(ids, ib);
        par_prefault(dists, db);
    }
    if (scanned) par_prefault(scanned, sb);
    // the previous call's output lines must be out of the CPU caches before
    // this call's D2H lands on them (flushed in the background meanwhile)
    if (flusher_.joinable()) flusher_.join();
    const auto t2 = now();
    if (topk) {
        CUDA_CHECK(cudaMemcpyAsync(pi, si_.p, ib, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(pd, sd_.p, db, cudaMemcpyDeviceToHost, st));
    }
    if (scanned) CUDA_CHECK(cudaMemcpyAsync(ps, ss_.p, sb, cudaMemcpyDeviceToHost, st));
    if (timing) CUDA_CHECK(cudaEventRecord(tev[3], st));
    check_device_errors(st);
    const auto t3 = now();
    if (topk) {
        par_memcpy(ids, pi, ib, Pinned::NoFlush);
        par_memcpy(dists, pd, db, Pinned::NoFlush);
    }
    if (scanned) par_memcpy(scanned, ps, sb, Pinned::NoFlush);
    // evict the output staging lines the copy threads just read, off the
    // caller's critical path (joined before the next D2H into them)
    flusher_ = std::thread([pi, n = ib + db + sb] { flush_lines(pi, n); });
    if (timing) {
        float g[3];
        for (int e = 0; e < 3; e++) CUDA_CHECK(cudaEventElapsedTime(&g[e], tev[e], tev[e + 1]));
        for (auto& e : tev) cudaEventDestroy(e);
        std::fprintf(stderr,
                     "[search_host] stage+check %.3f ms, enqueue %.3f ms, wait %.3f ms, copy-out %.3f ms | "
                     "GPU: h2d %.3f, search %.3f, d2h %.3f ms\n",
                     ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, now()), g[0], g[1], g[2]);
    }
}

// ---------------------------------------------------------------------------
// brute_force_gt (proj/src/dataset.cpp:46-92) on the device
// ---------------------------------------------------------------------------
void Engine::brute_force_gt(int device, const float* base, uint64_t nb, const float* queries, uint64_t nq,
                            uint32_t dim, uint32_t k, uint32_t* out) {
    brute_force_gt_source(
        device,
        [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
            CUDA_CHECK(cudaMemcpyAsync(dst, base + first * dim, count * dim * 4, cudaMemcpyHostToDevice, st));
        },
        nb, queries, nq, dim, k, out);
}

void Engine::brute_force_gt_source(int device, const BaseSource& src, uint64_t nb, const float* queries, uint64_t nq,
                                   uint32_t dim, uint32_t k, uint32_t* out) {
    if ((uint64_t)k > nb) throw std::runtime_error("brute_force_gt: k exceeds base count");
    if (nq == 0 || k == 0) return;
    if (k > 4096) throw std::runtime_error("brute_force_gt: k > 4096 is not supported by the GPU engine");
    DeviceGuard g(device);
    cudaStream_t st;
    CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const uint64_t C = std::min<uint64_t>(nb, 65536);
    const uint64_t T = std::min<uint64_t>(nq, std::max<uint64_t>(1, (2ull << 30) / (4 * C)));
    DevBuf<float> B, Q, dist;
    DevBuf<uint32_t> sel;
    DevBuf<uint64_t> running;
    B.alloc(C * dim);
    Q.alloc(nq * dim);
    dist.alloc(T * C);
    sel.alloc(T * (uint64_t)k);
    running.alloc(nq * (uint64_t)k);
    CUDA_CHECK(cudaMemcpyAsync(Q.p, queries, nq * dim * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemsetAsync(running.p, 0xff, nq * (uint64_t)k * 8, st));
    for (uint64_t c0 = 0; c0 < nb; c0 += C) {
        const uint64_t cn = std::min(C, nb - c0);
        src(c0, cn, B.p, st);
        for (uint64_t q0 = 0; q0 < nq; q0 += T) {
            const uint64_t tn = std::min(T, nq - q0);
            launch_sqdist_matrix(Q.p + q0 * dim, tn, B.p, cn, dim, dist.p, cn, st);
            const uint32_t L = (uint32_t)std::min<uint64_t>(k, cn);
            launch_select_rows(dist.p, cn, tn, (uint32_t)cn, L, sel.p, st);
            launch_gt_merge(dist.p, cn, tn, k, (uint32_t)cn, sel.p, c0, running.p + q0 * k, st);
        }
    }
    std::vector<uint64_t> keys(nq * (uint64_t)k);
    CUDA_CHECK(cudaMemcpyAsync(keys.data(), running.p, keys.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    CUDA_CHECK(cudaStreamDestroy(st));
    for (size_t i = 0; i < keys.size(); i++) out[i] = (uint32_t)keys[i];
}

// ---------------------------------------------------------------------------
// VLQ1 file (proj/src/index_io.cpp:63-159)
// ---------------------------------------------------------------------------
namespace {

constexpr char kMagic[4] = {'V', 'L', 'Q', '1'};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kFlagClamped = 1u << 0;
constexpr uint32_t kFlagT3 = 1u << 1;

struct Reader {
    std::ifstream in;
    std::string path;
    explicit Reader(const std::string& p) : in(p, std::ios::binary), path(p) {
        if (!in) throw std::runtime_error("deserialize_index: cannot open " + p);
    }
    void bytes(void* p, size_t n) {
        in.read(reinterpret_cast<char*>(p), (std::streamsize)n);
        if ((size_t)in.gcount() != n) throw std::runtime_error("deserialize_index: truncated file " + path);
    }
    uint32_t u32() {
        uint32_t v;
        bytes(&v, 4);
        return v;
    }
    float f32() {
        float v;
        bytes(&v, 4);
        return v;
    }
};

struct Writer {
    std::ofstream out;
    explicit Writer(const std::string& path) : out(path, std::ios::binary | std::ios::trunc) {
        if (!out) throw std::runtime_error("serialize_index: cannot open " + path);
    }
    void bytes(const void* p, size_t n) { out.write(reinterpret_cast<const char*>(p), (std::streamsize)n); }
    void u32(uint32_t v) { bytes(&v, 4); }
    void f32(float v) { bytes(&v, 4); }
};

}  // namespace

void Engine::load_vlq1(const std::string& path) {
    Reader r(path);
    char magic[4];
    r.bytes(magic, 4);
    if (std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error("deserialize_index: bad magic in " + path);
    if (r.u32() != kVersion) throw std::runtime_error("deserialize_index: unsupported version in " + path);
    const uint32_t flags = r.u32();
    HostModel m;
    m.dim = r.u32();
    m.k = r.u32();
    m.n = r.u32();
    m.m = r.u32();
    const uint32_t base_count = r.u32();
    if (m.dim == 0 || m.k == 0 || m.n == 0 || m.n >= m.k || m.m == 0 || m.dim % m.m != 0)
        throw std::runtime_error("deserialize_index: invalid header in " + path);
    m.clamp = (flags & kFlagClamped) != 0;
    m.lo = r.f32();
    m.hi = r.f32();
    m.centroids.resize((size_t)m.k * m.dim);
    r.bytes(m.centroids.data(), m.centroids.size() * 4);
    m.nbr.resize((size_t)m.k * m.n);
    r.bytes(m.nbr.data(), m.nbr.size() * 4);
    m.elen.resize((size_t)m.k * m.n);
    r.bytes(m.elen.data(), m.elen.size() * 4);
    m.pq.resize((size_t)m.m * VLQ_KSUB * (m.dim / m.m));
    r.bytes(m.pq.data(), m.pq.size() * 4);
    if (flags & kFlagT3) {
        m.t3.resize((size_t)m.k * m.m * VLQ_KSUB);
        r.bytes(m.t3.data(), m.t3.size() * 4);
    }
    const size_t ncell = (size_t)m.k * m.n;
    HostLists L;
    L.off.assign(ncell + 1, 0);
    std::vector<uint8_t> seen(base_count, 0);
    bool bad_partition = false;
    uint64_t total = 0;
    std::vector<uint32_t> ids;
    std::vector<uint8_t> codes;
    for (size_t c = 0; c < ncell; c++) {
        const uint32_t len = r.u32();
        ids.resize(len);
        r.bytes(ids.data(), (size_t)len * 4);
        codes.resize((size_t)len * m.m + len);
        r.bytes(codes.data(), codes.size());
        for (uint32_t id : ids) {  // validate() partition check (index.cpp:23-52)
            if (id >= base_count || seen[id]) bad_partition = true;
            else seen[id] = 1;
        }
        total += len;
        const bool own = owner((uint32_t)c) == cfg_.shard_rank;
        if (own) {
            L.ids.insert(L.ids.end(), ids.begin(), ids.end());
            L.codes.insert(L.codes.end(), codes.begin(), codes.begin() + (size_t)len * m.m);
            L.lambdas.insert(L.lambdas.end(), codes.begin() + (size_t)len * m.m, codes.end());
        }
        L.off[c + 1] = L.ids.size();
    }
    // validate() order (index.cpp:23-52): lambda range, partition, total
    if (!(m.lo < m.hi)) throw std::runtime_error("InvertedIndex: bad lambda range");
    if (bad_partition) throw std::runtime_error("InvertedIndex: ids do not partition the base set");
    if (total != base_count) throw std::runtime_error("InvertedIndex: list lengths do not sum to N");
    set_model(m);
    upload_lists(L);
    base_count_ = base_count;
    compute_eterm();
}

void Engine::save_vlq1(const std::string& path, bool store_t3) {
    if (!model_ok_) throw std::runtime_error("save: no model loaded");
    if (cfg_.shard_count != 1) throw std::runtime_error("save: a sharded engine cannot write a complete VLQ1 index");
    HostLists L;
    get_lists(L, /*offsets_only=*/true);  // the lists themselves are streamed below
    std::vector<float> t2, t3;
    if (store_t3) get_tables(t2, t3);
    Writer w(path);
    w.bytes(kMagic, 4);
    w.u32(kVersion);
    w.u32((clamp_ ? kFlagClamped : 0) | (store_t3 ? kFlagT3 : 0));
    w.u32(dim_);
    w.u32(k_);
    w.u32(n_);
    w.u32(m_);
    w.u32((uint32_t)base_count_);
    w.f32(lo_);
    w.f32(hi_);
    w.bytes(model_.centroids.data(), model_.centroids.size() * 4);
    w.bytes(model_.nbr.data(), model_.nbr.size() * 4);
    w.bytes(model_.elen.data(), model_.elen.size() * 4);
    w.bytes(model_.pq.data(), model_.pq.size() * 4);
    if (store_t3) w.bytes(t3.data(), t3.size() * 4);
    // posting lists (index_io.cpp:63-98 record order), streamed: batches of
    // whole cells (<= 8M entries unless one cell is larger) are copied to
    // double-buffered pinned memory while the previous batch is written, so
    // a 1B-entry index never needs a host copy of its ~21 GB of lists
    const size_t ncell = (size_t)k_ * n_;
    const uint64_t kBatch = 8ull << 20;
    std::vector<std::pair<size_t, size_t>> batches;
    uint64_t maxb = 1;
    for (size_t c0 = 0; c0 < ncell;) {
        size_t c1 = c0 + 1;
        while (c1 < ncell && L.off[c1 + 1] - L.off[c0] <= kBatch) c1++;
        batches.emplace_back(c0, c1);
        maxb = std::max<uint64_t>(maxb, L.off[c1] - L.off[c0]);
        c0 = c1;
    }
    DeviceGuard g(cfg_.device);
    PinnedBuf pb[2];
    cudaEvent_t ev[2];
    for (int b = 0; b < 2; b++) {
        pb[b].alloc(maxb * (4 + m_ + 1));
        CUDA_CHECK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } evg{ev};
    auto fetch = [&](size_t bi) {  // D2H of batch bi into buffer bi % 2
        const uint64_t e0 = L.off[batches[bi].first], ne = L.off[batches[bi].second] - e0;
        unsigned char* p = pb[bi & 1].p;
        if (ne) {
            CUDA_CHECK(cudaMemcpyAsync(p, ids_.p + e0, ne * 4, cudaMemcpyDeviceToHost, stream_));
            CUDA_CHECK(cudaMemcpyAsync(p + ne * 4, codes_.p + e0 * m_, ne * m_, cudaMemcpyDeviceToHost, stream_));
            CUDA_CHECK(cudaMemcpyAsync(p + ne * (4 + m_), lambdas_.p + e0, ne, cudaMemcpyDeviceToHost, stream_));
        }
        CUDA_CHECK(cudaEventRecord(ev[bi & 1], stream_));
    };
    if (!batches.empty()) fetch(0);
    for (size_t bi = 0; bi < batches.size(); bi++) {
        if (bi + 1 < batches.size()) fetch(bi + 1);  // its buffer's previous batch (bi - 1) is fully written
        CUDA_CHECK(cudaEventSynchronize(ev[bi & 1]));
        const uint64_t e0 = L.off[batches[bi].first], ne = L.off[batches[bi].second] - e0;
        const unsigned char* p = pb[bi & 1].p;
        for (size_t c = batches[bi].first; c < batches[bi].second; c++) {
            const uint64_t b0 = L.off[c] - e0, len = L.off[c + 1] - L.off[c];
            w.u32((uint32_t)len);
            w.bytes(p + b0 * 4, len * 4);
            w.bytes(p + ne * 4 + b0 * m_, len * m_);
            w.bytes(p + ne * (4 + m_) + b0, len);
        }
    }
    if (!w.out) throw std::runtime_error("serialize_index: write failed for " + path);
}

}  // namespace vlq
