// Multi-GPU search group (group.cu): one process, G engines on G devices,
// list-sharded index, query-split selection, fused P2P exchange + merge.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "engine.h"

namespace vlq {

class Group {
public:
    // shards S divides G = devices.size(): G / S replicas of an S-way list
    // sharding; member g is shard g % S of replica g / S (0: S = G)
    Group(const std::vector<int>& devices, uint32_t shards, const EngineConfig& base);
    ~Group();
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;

    uint32_t size() const { return (uint32_t)eng_.size(); }
    uint32_t shards() const { return shards_; }
    uint32_t replicas() const { return size() / shards_; }
    Engine& engine(uint32_t g) { return *eng_[g]; }
    int device(uint32_t g) const { return dev_[g]; }
    uint64_t local_entries(uint32_t g) const;

    // set-up, one host thread per engine
    void load_vlq1(const std::string& path);
    void set_model(const HostModel& m);
    void add_host(const float* base, uint64_t nb);
    void add_stream(uint64_t nb, uint64_t chunk, const Engine::ChunkSource& src);

    // Index.search over the group: host queries in, merged host results out
    void search_host(const float* q, uint64_t nq, uint32_t dim, uint32_t w1, float alpha, uint32_t k, int64_t* ids,
                     float* dists, uint64_t* scanned);
    // device-resident batch (bench): upload once, then timed searches
    // (device ms, max over the devices), then results()
    void upload_queries(const float* q, uint64_t nq, uint32_t dim, bool validate = true);
    float search_resident(uint32_t w1, float alpha, uint32_t k);
    void results(int64_t* ids, float* dists, uint64_t* scanned);

private:
    struct PerDevice {
        cudaStream_t st = nullptr;
        cudaEvent_t ev_sel = nullptr, ev_fine = nullptr, ev_done = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
        DevBuf<float> q;         // the whole batch [nq, dim]
        DevBuf<uint32_t> sel;    // this device's query slice: selected cells [per, w2]
        DevBuf<float> ab;        //                             exact (a, b) [per, w2, 2]
        DevBuf<int64_t> lids;    // this shard's exact top-k, its replica's sub-batch [nq_r, k]
        DevBuf<float> ld;
        DevBuf<uint64_t> lsc;    // this shard's scanned counts [nq_r]
        DevBuf<int64_t> oids;    // merged top-k of this device's query slice [per, k]
        DevBuf<float> od;
    };
    void for_each_device(const std::function<void(uint32_t)>& fn);
    void reserve(uint64_t nq, uint32_t w2, uint32_t k);
    void enqueue_search(uint64_t nq, uint32_t w1, float alpha, uint32_t k);
    void check_errors();

    // replica r's query sub-batch [r0, r1) of an nq batch; shard slices inside it
    void sub_batch(uint64_t nq, uint32_t r, uint64_t& r0, uint64_t& r1) const;
    std::vector<int> dev_;
    uint32_t shards_ = 1;
    std::vector<std::unique_ptr<Engine>> eng_;
    std::deque<PerDevice> per_;  // deque: PerDevice (DevBuf) is neither copyable nor movable
    void* pin_ = nullptr;  // query staging
    uint64_t pin_bytes_ = 0;
    void* out_pin_ = nullptr;  // result staging
    uint64_t out_pin_bytes_ = 0;
    uint64_t nq_q_ = 0;
    uint32_t last_k_ = 0;
};

}  // namespace vlq
