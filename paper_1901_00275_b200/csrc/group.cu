// Multi-GPU search group: one process drives G GPUs of one box (SURVEY.md
// §2.3, §8e; the paper's "split the index into b parts, search locally,
// join").
//
// Engine g (device dev[g]) holds the posting lists c with
// shard_of_cell(c, G) == g; the coarse quantizer, graph, PQ and t3 are
// replicated.  Per batch, on per-device streams, with cross-device event
// waits (no host round trip):
//
//   1. select   device g runs first_level_scan + second_level_rank for its
//               query slice [g per, (g + 1) per): the selected cells and their
//               exact (a, b) pairs stay in ITS memory;
//   2. fine     every device runs apply-selection + term5 + the fused scan +
//               the exact re-score for the whole batch on its shard; the
//               apply kernel reads query q's selection row directly from the
//               device that selected it (k_apply_selection over NVLink peer
//               memory: the all-gather is fused into the consumer);
//   3. merge    device g merges the G per-shard exact top-k rows of ITS query
//               slice, reading the other devices' blocks over NVLink
//               (k_merge_sorted with peer pointers: gather + merge in one
//               kernel), and returns that slice to the host.
//
// Every shard returns its exact local top-k under the reference's (dist, id)
// order, so the merged rows equal the single-engine result bit for bit.  The
// collectives are P2P loads by the consuming kernels (cudaDeviceEnablePeerAccess
// between every pair of devices; NVSwitch gives every pair full bandwidth), so
// the step needs no NCCL call and no PyTorch.  A group may list the same device
// several times (parity tests on one GPU): peer pointers are then plain local
// pointers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "group.h"

namespace vlq {

namespace {
uint64_t slice_per(uint64_t nq, uint32_t G) { return (nq + G - 1) / G; }
}  // namespace

namespace {
// fn(lo, hi) over [0, n) on up to 8 host threads (host staging copies)
template <typename F>
void par_for(uint64_t n, F&& fn) {
    const uint64_t T = std::min<uint64_t>(8, std::max<uint64_t>(1, n >> 18));
    if (T <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < T; t++) th.emplace_back([&, t] { fn(n * t / T, n * (t + 1) / T); });
    for (auto& x : th) x.join();
}
}  // namespace


Group::Group(const std::vector<int>& devices, uint32_t shards, const EngineConfig& base) : dev_(devices) {
    const uint32_t G = (uint32_t)dev_.size();
    if (G == 0 || G > VLQ_MAX_PARTS) throw std::runtime_error("group: need 1..16 devices");
    shards_ = shards ? shards : G;
    if (G % shards_ != 0) throw std::runtime_error("group: shards must divide the number of devices");
    int ndev = 0;
    CUDA_CHECK(cudaGetDeviceCount(&ndev));
    for (int d : dev_)
        if (d < 0 || d >= ndev) throw std::runtime_error("group: device index out of range");
    // NVLink peer access between every pair of distinct devices (the fused
    // exchange kernels load peer memory directly)
    for (uint32_t a = 0; a < G; a++)
        for (uint32_t b = 0; b < G; b++) {
            if (dev_[a] == dev_[b]) continue;
            int ok = 0;
            CUDA_CHECK(cudaDeviceCanAccessPeer(&ok, dev_[a], dev_[b]));
            if (!ok) throw std::runtime_error("group: devices " + std::to_string(dev_[a]) + " and " +
                                              std::to_string(dev_[b]) + " have no peer access");
            DeviceGuard g(dev_[a]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(dev_[b], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else CUDA_CHECK(e);
        }
    for (uint32_t g = 0; g < G; g++) per_.emplace_back();
    for (uint32_t g = 0; g < G; g++) {
        EngineConfig c = base;
        c.device = dev_[g];
        c.shard_rank = (int)(g % shards_);
        c.shard_count = (int)shards_;
        eng_.emplace_back(new Engine(c));
        DeviceGuard dg(dev_[g]);
        PerDevice& p = per_[g];
        CUDA_CHECK(cudaStreamCreateWithFlags(&p.st, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&p.ev_sel, &p.ev_fine, &p.ev_done})
            CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreate(&p.ev_t0));
        CUDA_CHECK(cudaEventCreate(&p.ev_t1));
    }
}

Group::~Group() {
    for (uint32_t g = 0; g < per_.size(); g++) {
        DeviceGuard dg(dev_[g]);
        PerDevice& p = per_[g];
        if (p.st) cudaStreamSynchronize(p.st);
        for (cudaEvent_t e : {p.ev_sel, p.ev_fine, p.ev_done, p.ev_t0, p.ev_t1})
            if (e) cudaEventDestroy(e);
        p.q.reset();
        p.sel.reset();
        p.ab.reset();
        p.lids.reset();
        p.ld.reset();
        p.lsc.reset();
        p.oids.reset();
        p.od.reset();
        if (p.st) cudaStreamDestroy(p.st);
    }
    if (pin_) cudaFreeHost(pin_);
    if (out_pin_) cudaFreeHost(out_pin_);
    eng_.clear();
}

void Group::for_each_device(const std::function<void(uint32_t)>& fn) {
    // one host thread per engine (set-up work: loads, adds); errors re-thrown
    const uint32_t G = size();
    std::vector<std::string> err(G);
    std::vector<std::thread> th;
    for (uint32_t g = 0; g < G; g++)
        th.emplace_back([&, g] {
            try {
                fn(g);
            } catch (const std::exception& e) {
                err[g] = e.what();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (!e.empty()) throw std::runtime_error(e);
}

void Group::load_vlq1(const std::string& path) {
    for_each_device([&](uint32_t g) { eng_[g]->load_vlq1(path); });
}

void Group::set_model(const HostModel& m) {
    for_each_device([&](uint32_t g) { eng_[g]->set_model(m); });
}

void Group::add_host(const float* base, uint64_t nb) {
    for_each_device([&](uint32_t g) { eng_[g]->add_host(base, nb); });
}

void Group::add_stream(uint64_t nb, uint64_t chunk, const Engine::ChunkSource& src) {
    for_each_device([&](uint32_t g) { eng_[g]->add_stream(nb, chunk, src); });
}

void Group::sub_batch(uint64_t nq, uint32_t r, uint64_t& r0, uint64_t& r1) const {
    const uint64_t nqr = slice_per(nq, replicas());
    r0 = std::min(nq, r * nqr);
    r1 = std::min(nq, r0 + nqr);
}

void Group::reserve(uint64_t nq, uint32_t w2, uint32_t k) {
    const uint32_t G = size();
    const uint64_t nqr = slice_per(nq, replicas());
    const uint64_t per = slice_per(nqr, shards_);
    const uint32_t dim = eng_[0]->dim();
    for (uint32_t g = 0; g < G; g++) {
        DeviceGuard dg(dev_[g]);
        PerDevice& p = per_[g];
        p.q.alloc(std::max<uint64_t>(1, nq * dim));
        p.sel.alloc(std::max<uint64_t>(1, per * w2));
        p.ab.alloc(std::max<uint64_t>(1, per * w2 * 2));
        p.lids.alloc(std::max<uint64_t>(1, nqr * k));
        p.ld.alloc(std::max<uint64_t>(1, nqr * k));
        p.lsc.alloc(std::max<uint64_t>(1, nqr));
        p.oids.alloc(std::max<uint64_t>(1, per * k));
        p.od.alloc(std::max<uint64_t>(1, per * k));
    }
}

void Group::upload_queries(const float* q, uint64_t nq, uint32_t dim, bool validate) {
    if (dim != eng_[0]->dim()) throw std::runtime_error("search_batch: dimension mismatch");
    const uint64_t bytes = nq * dim * 4;
    if (pin_bytes_ < bytes) {
        if (pin_) CUDA_CHECK(cudaFreeHost(pin_));
        pin_ = nullptr;
        CUDA_CHECK(cudaHostAlloc(&pin_, bytes, cudaHostAllocPortable));  // pinned for every device's DMA
        pin_bytes_ = bytes;
    }
    // staged copy (and VectorSet::validate, vecset.cpp:14-18) on host threads
    std::atomic<bool> finite{true};
    float* dst = static_cast<float*>(pin_);
    par_for(nq * dim, [&](uint64_t a, uint64_t b) {
        std::memcpy(dst + a, q + a, (b - a) * 4);
        if (validate)
            for (uint64_t i = a; i < b; i++)
                if (!std::isfinite(dst[i])) finite = false;
    });
    if (!finite) throw std::runtime_error("VectorSet: non-finite value");
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        per_[g].q.alloc(std::max<uint64_t>(1, nq * dim));
        CUDA_CHECK(cudaMemcpyAsync(per_[g].q.p, pin_, bytes, cudaMemcpyHostToDevice, per_[g].st));
    }
    nq_q_ = nq;
}

void Group::enqueue_search(uint64_t nq, uint32_t w1, float alpha, uint32_t k) {
    const uint32_t S = shards_, R = replicas();
    const uint32_t dim = eng_[0]->dim();
    for (uint32_t r = 0; r < R; r++) {  // replicas work on disjoint query sub-batches, independently
        uint64_t r0, r1;
        sub_batch(nq, r, r0, r1);
        const uint64_t nqr = r1 - r0, per = slice_per(nqr, S);
        auto mem = [&](uint32_t s) { return r * S + s; };
        // 1. query-split selection inside the replica
        for (uint32_t s = 0; s < S; s++) {
            PerDevice& p = per_[mem(s)];
            DeviceGuard dg(dev_[mem(s)]);
            const uint64_t lo = std::min(nqr, s * per), hi = std::min(nqr, lo + per);
            if (hi > lo)
                eng_[mem(s)]->search_select_device(p.q.p + (r0 + lo) * dim, hi - lo, w1, alpha, p.sel.p, p.ab.p,
                                                   p.st);
            CUDA_CHECK(cudaEventRecord(p.ev_sel, p.st));
        }
        // 2. sharded fine stage, the selection read from its owners over NVLink
        SelParts sp{};
        for (uint32_t s = 0; s < S; s++) {
            sp.sel[s] = per_[mem(s)].sel.p;
            sp.ab[s] = per_[mem(s)].ab.p;
        }
        sp.nparts = S;
        sp.per = per;
        for (uint32_t s = 0; s < S; s++) {
            PerDevice& p = per_[mem(s)];
            DeviceGuard dg(dev_[mem(s)]);
            for (uint32_t h = 0; h < S; h++)
                if (h != s) CUDA_CHECK(cudaStreamWaitEvent(p.st, per_[mem(h)].ev_sel, 0));
            if (nqr > 0)
                eng_[mem(s)]->search_fine_sel_parts(p.q.p + r0 * dim, nqr, w1, alpha, k, sp, p.lids.p, p.ld.p,
                                                    p.lsc.p, p.st);
            CUDA_CHECK(cudaEventRecord(p.ev_fine, p.st));
        }
        // 3. each device merges its query slice from every shard's block (peer loads)
        TopkParts tp{};
        for (uint32_t s = 0; s < S; s++) {
            tp.ids[s] = per_[mem(s)].lids.p;
            tp.d[s] = per_[mem(s)].ld.p;
        }
        tp.nparts = S;
        for (uint32_t s = 0; s < S; s++) {
            PerDevice& p = per_[mem(s)];
            DeviceGuard dg(dev_[mem(s)]);
            for (uint32_t h = 0; h < S; h++)
                if (h != s) CUDA_CHECK(cudaStreamWaitEvent(p.st, per_[mem(h)].ev_fine, 0));
            const uint64_t lo = std::min(nqr, s * per), hi = std::min(nqr, lo + per);
            launch_merge_topk_parts(tp, lo, hi - lo, k, p.oids.p, p.od.p, p.st);
            CUDA_CHECK(cudaEventRecord(p.ev_done, p.st));
        }
        // no device may reuse its selection / result buffers (next batch) before
        // every peer of its replica finished reading them
        for (uint32_t s = 0; s < S; s++) {
            DeviceGuard dg(dev_[mem(s)]);
            for (uint32_t h = 0; h < S; h++)
                if (h != s) CUDA_CHECK(cudaStreamWaitEvent(per_[mem(s)].st, per_[mem(h)].ev_done, 0));
        }
    }
}

void Group::check_errors() {
    for (uint32_t g = 0; g < size(); g++) eng_[g]->check_device_errors(per_[g].st);
}

float Group::search_resident(uint32_t w1, float alpha, uint32_t k) {
    const uint64_t nq = nq_q_;
    if (nq == 0) return 0.0f;
    if (w1 == 0 || w1 > eng_[0]->k()) throw std::runtime_error("first_level_scan: need 0 < w1 <= k");
    reserve(nq, w2_of(w1, alpha, eng_[0]->n()), k);
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        CUDA_CHECK(cudaStreamSynchronize(per_[g].st));
    }
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        CUDA_CHECK(cudaEventRecord(per_[g].ev_t0, per_[g].st));
    }
    enqueue_search(nq, w1, alpha, k);
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        CUDA_CHECK(cudaEventRecord(per_[g].ev_t1, per_[g].st));
    }
    float ms = 0.0f;
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        CUDA_CHECK(cudaEventSynchronize(per_[g].ev_t1));
        float t = 0.0f;
        CUDA_CHECK(cudaEventElapsedTime(&t, per_[g].ev_t0, per_[g].ev_t1));
        ms = std::max(ms, t);  // the job's time: max over the devices
    }
    check_errors();
    last_k_ = k;
    return ms;
}

void Group::results(int64_t* ids, float* dists, uint64_t* scanned) {
    const uint64_t nq = nq_q_;
    const uint32_t S = shards_, k = last_k_;
    // every device's merged slice (and scanned counts) into pinned staging at
    // once, then one parallel copy into the caller's buffers
    const uint64_t ib = nq * k * 8, db = nq * k * 4;
    const uint64_t nqr_max = slice_per(nq, replicas());
    const uint64_t sb = scanned ? (uint64_t)size() * nqr_max * 8 : 0;
    if (out_pin_bytes_ < ib + db + sb) {
        if (out_pin_) CUDA_CHECK(cudaFreeHost(out_pin_));
        out_pin_ = nullptr;
        CUDA_CHECK(cudaHostAlloc(&out_pin_, ib + db + sb, cudaHostAllocPortable));
        out_pin_bytes_ = ib + db + sb;
    }
    int64_t* pi = reinterpret_cast<int64_t*>(out_pin_);
    float* pd = reinterpret_cast<float*>(static_cast<unsigned char*>(out_pin_) + ib);
    uint64_t* ps = reinterpret_cast<uint64_t*>(static_cast<unsigned char*>(out_pin_) + ib + db);
    for (uint32_t g = 0; g < size(); g++) {
        const uint32_t r = g / S, s = g % S;
        uint64_t r0, r1;
        sub_batch(nq, r, r0, r1);
        const uint64_t nqr = r1 - r0, per = slice_per(nqr, S);
        DeviceGuard dg(dev_[g]);
        PerDevice& p = per_[g];
        const uint64_t lo = std::min(nqr, s * per), hi = std::min(nqr, lo + per);
        if (hi > lo) {
            CUDA_CHECK(cudaMemcpyAsync(pi + (r0 + lo) * k, p.oids.p, (hi - lo) * k * 8, cudaMemcpyDeviceToHost, p.st));
            CUDA_CHECK(cudaMemcpyAsync(pd + (r0 + lo) * k, p.od.p, (hi - lo) * k * 4, cudaMemcpyDeviceToHost, p.st));
        }
        if (scanned && nqr > 0)
            CUDA_CHECK(cudaMemcpyAsync(ps + (uint64_t)g * nqr_max, p.lsc.p, nqr * 8, cudaMemcpyDeviceToHost, p.st));
    }
    for (uint32_t g = 0; g < size(); g++) {
        DeviceGuard dg(dev_[g]);
        CUDA_CHECK(cudaStreamSynchronize(per_[g].st));
    }
    par_for(nq, [&](uint64_t a, uint64_t b) {
        if (ids) std::memcpy(ids + a * k, pi + a * k, (b - a) * k * 8);
        if (dists) std::memcpy(dists + a * k, pd + a * k, (b - a) * k * 4);
    });
    if (scanned) {  // reference-semantics scanned count = the sum over the replica's shards
        for (uint32_t r = 0; r < replicas(); r++) {
            uint64_t r0, r1;
            sub_batch(nq, r, r0, r1);
            for (uint64_t q = r0; q < r1; q++) {
                uint64_t t = 0;
                for (uint32_t s = 0; s < S; s++) t += ps[(uint64_t)(r * S + s) * nqr_max + (q - r0)];
                scanned[q] = t;
            }
        }
    }
}

void Group::search_host(const float* q, uint64_t nq, uint32_t dim, uint32_t w1, float alpha, uint32_t k,
                        int64_t* ids, float* dists, uint64_t* scanned) {
    if (dim != eng_[0]->dim()) throw std::runtime_error("search_batch: dimension mismatch");
    if (w1 == 0 || w1 > eng_[0]->k()) throw std::runtime_error("first_level_scan: need 0 < w1 <= k");
    if (nq == 0) return;
    upload_queries(q, nq, dim, /*validate=*/true);
    reserve(nq, w2_of(w1, alpha, eng_[0]->n()), k);
    enqueue_search(nq, w1, alpha, k);
    par_prefault(ids, nq * k * 8);  // the output pages fault in while the GPUs search
    par_prefault(dists, nq * k * 4);
    if (scanned) par_prefault(scanned, nq * 8);
    check_errors();
    last_k_ = k;
    results(ids, dists, scanned);
}

uint64_t Group::local_entries(uint32_t g) const { return eng_[g]->local_entries(); }

}  // namespace vlq
