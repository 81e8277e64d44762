// Test-infrastructure driver linked against the UNMODIFIED reference sources
// (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/). It is the checker's tool, never part of the product path.
//
//   ref_tools instance <count> <dim> <clusters> <k> <n> <m> <iters> <train_count>
//                      <query_count> <seed> <spread> <out_prefix>
//       Replays the reference acceptance fixture builder
//       (proj/tests/acceptance.cpp:74-115, make_instance) through the
//       reference's public API and writes <prefix>.vlq (VLQ1 index),
//       <prefix>.base.fvecs and <prefix>.queries.fvecs.
//
//   ref_tools search <index.vlq> <queries.fvecs> <w1> <alpha> <k> <out.bin>
//       search_batch (proj/src/search.cpp:169-191) with SearchStats; writes
//       u64 nq, u32 k, u64 scanned, then per query: u32 count, count x
//       (u32 id, f32 dist) -- the reference's own results, unpadded.
//
//   ref_tools scanstats <index.vlq> <queries.fvecs> <w1> <alpha> <k>
//       prints the total scanned_candidates (proj/src/search.cpp:163-165).
//
//   ref_tools model <train.fvecs> <k> <n> <m> <iters> <seed> <clamp> <out.vlq>
//       Index.train replay (proj/python/bindings.cpp:44-81) saved as a model
//       (index with zero points, proj/tools/vlq_cli.cpp:19-34).
//
//   ref_tools build <model.vlq> <base.fvecs> <out.vlq>
//       Index.add replay (proj/python/bindings.cpp:83-97).
//
//   ref_tools ivf <model.vlq> <base.fvecs> <queries.fvecs> <w> <k> <out.bin>
//       The IVFADC comparison baseline (proj/src/ivf_baseline.cpp):
//       build_ivf_baseline with the model's codebook and PQ (as eval.cpp:182
//       does), then search_ivf_baseline with SearchStats.  Writes u32 K, u32 m,
//       per region: u32 len, len x u32 id, len*m code bytes; then the search
//       results in the `search` format.

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "vlq/dataset.hpp"
#include "vlq/index.hpp"
#include "vlq/ivf_baseline.hpp"
#include "vlq/line_quant.hpp"
#include "vlq/search.hpp"
#include "vlq/vecs_io.hpp"

using namespace vlq;

namespace {

InvertedIndex make_instance_index(size_t count, uint32_t dim, uint32_t clusters, uint32_t k,
                                  uint32_t n, uint32_t m, uint32_t iters, size_t train_count,
                                  uint64_t seed, float spread, VectorSet& base) {
    base = gen_synthetic(count, dim, clusters, spread, seed);
    VectorSet train = base;
    if (train_count < count) {
        train = VectorSet(dim, train_count);
        std::copy_n(base.data.begin(), train.data.size(), train.data.begin());
    }
    Codebook cb = train_kmeans(train, k, iters, seed + 1);
    NeighborGraph graph = build_nn_graph(cb, n);
    VectorSet disp(dim, train.count());
    for (size_t i = 0; i < train.count(); i++) {
        EdgeAssignment ea =
            assign_edge(train.row(i), assign_nearest(train.row(i), cb).first, cb, graph, true);
        const float* ci = cb.centroid(ea.centroid_id);
        const float* sj = cb.centroid(graph.neighbor(ea.centroid_id, ea.edge_rank));
        for (uint32_t t = 0; t < dim; t++) {
            disp.row(i)[t] = train.row(i)[t] - ((1.0f - ea.lambda) * ci[t] + ea.lambda * sj[t]);
        }
    }
    PQCodebooks pq = train_pq(disp, m, iters, seed + 2);
    return build_index(base, cb, graph, pq, {0.0f, 1.0f}, true);
}

int cmd_instance(int argc, char** argv) {
    if (argc != 14) throw std::runtime_error("instance: bad arguments");
    size_t count = std::strtoull(argv[2], nullptr, 10);
    uint32_t dim = std::strtoul(argv[3], nullptr, 10);
    uint32_t clusters = std::strtoul(argv[4], nullptr, 10);
    uint32_t k = std::strtoul(argv[5], nullptr, 10);
    uint32_t n = std::strtoul(argv[6], nullptr, 10);
    uint32_t m = std::strtoul(argv[7], nullptr, 10);
    uint32_t iters = std::strtoul(argv[8], nullptr, 10);
    size_t train_count = std::strtoull(argv[9], nullptr, 10);
    size_t query_count = std::strtoull(argv[10], nullptr, 10);
    uint64_t seed = std::strtoull(argv[11], nullptr, 10);
    float spread = std::strtof(argv[12], nullptr);
    std::string prefix = argv[13];
    VectorSet base;
    InvertedIndex index =
        make_instance_index(count, dim, clusters, k, n, m, iters, train_count, seed, spread, base);
    VectorSet queries = gen_synthetic(query_count, dim, clusters, spread, seed + 3);
    serialize_index(index, prefix + ".vlq", false);
    write_vecs(base, prefix + ".base.fvecs", VecsKind::F32);
    write_vecs(queries, prefix + ".queries.fvecs", VecsKind::F32);
    return 0;
}

int cmd_search(int argc, char** argv) {
    if (argc != 8) throw std::runtime_error("search: bad arguments");
    InvertedIndex index = deserialize_index(argv[2]);
    VectorSet queries = read_vecs(argv[3], VecsKind::F32);
    QueryParams params{(uint32_t)std::strtoul(argv[4], nullptr, 10), std::strtof(argv[5], nullptr),
                       (uint32_t)std::strtoul(argv[6], nullptr, 10)};
    SearchStats stats;
    auto results = search_batch(index, queries, params, &stats);
    std::ofstream out(argv[7], std::ios::binary | std::ios::trunc);
    uint64_t nq = results.size();
    uint64_t scanned = stats.scanned_candidates;
    out.write(reinterpret_cast<const char*>(&nq), 8);
    out.write(reinterpret_cast<const char*>(&params.top_k), 4);
    out.write(reinterpret_cast<const char*>(&scanned), 8);
    for (const auto& r : results) {
        uint32_t c = (uint32_t)r.ids.size();
        out.write(reinterpret_cast<const char*>(&c), 4);
        for (uint32_t i = 0; i < c; i++) {
            out.write(reinterpret_cast<const char*>(&r.ids[i]), 4);
            out.write(reinterpret_cast<const char*>(&r.dists[i]), 4);
        }
    }
    return out ? 0 : 2;
}

int cmd_scanstats(int argc, char** argv) {
    if (argc != 7) throw std::runtime_error("scanstats: bad arguments");
    InvertedIndex index = deserialize_index(argv[2]);
    VectorSet queries = read_vecs(argv[3], VecsKind::F32);
    QueryParams params{(uint32_t)std::strtoul(argv[4], nullptr, 10), std::strtof(argv[5], nullptr),
                       (uint32_t)std::strtoul(argv[6], nullptr, 10)};
    SearchStats stats;
    search_batch(index, queries, params, &stats);
    std::printf("%llu\n", (unsigned long long)stats.scanned_candidates);
    return 0;
}

int cmd_model(int argc, char** argv) {
    if (argc != 10) throw std::runtime_error("model: bad arguments");
    VectorSet train = read_vecs(argv[2], VecsKind::F32);
    uint32_t k = std::strtoul(argv[3], nullptr, 10);
    uint32_t n = std::strtoul(argv[4], nullptr, 10);
    uint32_t m = std::strtoul(argv[5], nullptr, 10);
    uint32_t iters = std::strtoul(argv[6], nullptr, 10);
    uint64_t seed = std::strtoull(argv[7], nullptr, 10);
    bool clamp = std::atoi(argv[8]) != 0;
    Codebook cb = train_kmeans(train, k, iters, seed);
    NeighborGraph graph = build_nn_graph(cb, n);
    VectorSet disp(train.dim, train.count());
    for (size_t i = 0; i < train.count(); i++) {
        const float* x = train.row(i);
        EdgeAssignment ea = assign_edge(x, assign_nearest(x, cb).first, cb, graph, clamp);
        const float* ci = cb.centroid(ea.centroid_id);
        const float* sj = cb.centroid(graph.neighbor(ea.centroid_id, ea.edge_rank));
        for (uint32_t t = 0; t < train.dim; t++) {
            disp.row(i)[t] = x[t] - ((1.0f - ea.lambda) * ci[t] + ea.lambda * sj[t]);
        }
    }
    PQCodebooks pq = train_pq(disp, m, iters, seed + 1);
    InvertedIndex model;
    model.codebook = cb;
    model.graph = graph;
    model.pq = pq;
    model.clamp_lambda = clamp;
    model.lists.resize((size_t)graph.k * graph.n);
    model.t3 = compute_t3(cb, pq);
    serialize_index(model, argv[9], false);
    return 0;
}

int cmd_build(int argc, char** argv) {
    if (argc != 5) throw std::runtime_error("build: bad arguments");
    InvertedIndex model = deserialize_index(argv[2]);
    VectorSet base = read_vecs(argv[3], VecsKind::F32);
    LambdaQuant q = model.lambda_quant;
    if (!model.clamp_lambda) q = observe_lambda_range(base, model.codebook, model.graph);
    InvertedIndex built =
        build_index(base, model.codebook, model.graph, model.pq, q, model.clamp_lambda);
    serialize_index(built, argv[4], false);
    return 0;
}

int cmd_ivf(int argc, char** argv) {
    if (argc != 8) throw std::runtime_error("ivf: bad arguments");
    InvertedIndex model = deserialize_index(argv[2]);
    VectorSet base = read_vecs(argv[3], VecsKind::F32);
    VectorSet queries = read_vecs(argv[4], VecsKind::F32);
    uint32_t w = std::strtoul(argv[5], nullptr, 10);
    uint32_t k = std::strtoul(argv[6], nullptr, 10);
    IvfBaselineIndex ivf = build_ivf_baseline(base, model.codebook, model.pq);
    SearchStats stats;
    auto results = search_ivf_baseline(ivf, queries, w, k, &stats);
    std::ofstream out(argv[7], std::ios::binary | std::ios::trunc);
    uint32_t K = (uint32_t)ivf.ids.size(), m = ivf.pq.m;
    out.write(reinterpret_cast<const char*>(&K), 4);
    out.write(reinterpret_cast<const char*>(&m), 4);
    for (uint32_t c = 0; c < K; c++) {
        uint32_t len = (uint32_t)ivf.ids[c].size();
        out.write(reinterpret_cast<const char*>(&len), 4);
        out.write(reinterpret_cast<const char*>(ivf.ids[c].data()), (std::streamsize)len * 4);
        out.write(reinterpret_cast<const char*>(ivf.codes[c].data()), (std::streamsize)len * m);
    }
    uint64_t nq = results.size();
    uint64_t scanned = stats.scanned_candidates;
    out.write(reinterpret_cast<const char*>(&nq), 8);
    out.write(reinterpret_cast<const char*>(&k), 4);
    out.write(reinterpret_cast<const char*>(&scanned), 8);
    for (const auto& r : results) {
        uint32_t c = (uint32_t)r.ids.size();
        out.write(reinterpret_cast<const char*>(&c), 4);
        for (uint32_t i = 0; i < c; i++) {
            out.write(reinterpret_cast<const char*>(&r.ids[i]), 4);
            out.write(reinterpret_cast<const char*>(&r.dists[i]), 4);
        }
    }
    return out ? 0 : 2;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            std::fprintf(stderr, "usage: ref_tools instance|search|scanstats|model|build|ivf ...\n");
            return 1;
        }
        std::string cmd = argv[1];
        if (cmd == "instance") return cmd_instance(argc, argv);
        if (cmd == "search") return cmd_search(argc, argv);
        if (cmd == "scanstats") return cmd_scanstats(argc, argv);
        if (cmd == "model") return cmd_model(argc, argv);
        if (cmd == "build") return cmd_build(argc, argv);
        if (cmd == "ivf") return cmd_ivf(argc, argv);
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
