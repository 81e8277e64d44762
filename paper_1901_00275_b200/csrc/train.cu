// Index.train on the device (reference: proj/python/bindings.cpp:44-81):
// first-level k-means, exact n-NN centroid graph, training displacements from
// the line anchors, per-subspace PQ k-means.
//
// The structure follows the reference (train_kmeans kmeans.cpp:104-185,
// build_nn_graph nn_graph.cpp:11-50, train_pq pq.cpp:20-50) with two
// GPU-first substitutions, so models are NOT bit-identical to the
// reference's (parity is anchored on shared VLQ1 models instead):
//   * seeding: K distinct training points drawn with mt19937_64(seed)
//     (the reference's k-means++ is K sequential passes over the data);
//   * empty clusters are re-seeded from the point farthest from its centroid.
// Everything else is exact and deterministic: assignment is the exact
// strict-'<' argmin, centroid sums are sequential double sums in point
// order per cluster, the graph uses exact sqdist with (dist, id) ties, and
// displacements are the reference's residual at the exact lambda.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <random>
#include <stdexcept>
#include <vector>

#include "engine.h"
#include "select.cuh"

namespace vlq {
namespace dev {

// One block per cluster: mean of its members (positions [off[c], off[c+1])
// of `order`), each dimension a sequential double sum in point order
// (kmeans.cpp:133-156).
__global__ void k_segment_mean(const float* __restrict__ X, uint32_t dim, const uint32_t* __restrict__ order,
                               const unsigned long long* __restrict__ off, float* __restrict__ C,
                               uint32_t* __restrict__ empty) {
    const uint32_t c = blockIdx.x;
    const uint64_t b0 = off[c], b1 = off[c + 1];
    if (b0 == b1) {
        if (threadIdx.x == 0) empty[c] = 1;
        return;
    }
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) {
        double s = 0.0;
        for (uint64_t t = b0; t < b1; t++) s += (double)X[(uint64_t)order[t] * dim + d];
        C[(uint64_t)c * dim + d] = (float)(s / (double)(b1 - b0));
    }
    if (threadIdx.x == 0) empty[c] = 0;
}

__global__ void k_point_dist(const float* __restrict__ X, const float* __restrict__ C, const uint32_t* __restrict__ best,
                             uint64_t n, uint32_t dim, float* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float* x = X + i * dim;
        const float* c = C + (uint64_t)best[i] * dim;
        float acc = 0.0f;
        for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, x[d], c[d]);
        out[i] = acc;
    }
}

__global__ void k_gather_rows(const float* __restrict__ X, uint32_t dim, const uint32_t* __restrict__ rows, uint32_t nr,
                              float* __restrict__ out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (uint64_t)nr * dim;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = t / dim, d = t % dim;
        out[t] = X[(uint64_t)rows[r] * dim + d];
    }
}

__global__ void k_slice_cols(const float* __restrict__ X, uint64_t n, uint32_t dim, uint32_t c0, uint32_t w,
                             float* __restrict__ out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * w; t += (uint64_t)gridDim.x * blockDim.x)
        out[t] = X[(t / w) * dim + c0 + (t % w)];
}

// Graph rows: exclude self, then sort the n selected neighbours by (dist, id).
__global__ void k_set_diag(float* __restrict__ D, uint64_t ld, uint32_t r0, uint32_t nr) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x)
        D[(uint64_t)r * ld + r0 + r] = __int_as_float(0x7f800000);
}

__global__ void k_graph_rows(const float* __restrict__ D, uint64_t ld, const uint32_t* __restrict__ sel, uint32_t n,
                             uint32_t r0, uint32_t* __restrict__ nbr, float* __restrict__ elen, uint32_t* bad) {
    extern __shared__ unsigned long long keys[];
    const uint32_t r = blockIdx.x;
    uint32_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (uint32_t t = threadIdx.x; t < np2; t += blockDim.x) {
        unsigned long long key = ~0ull;
        if (t < n) {
            const uint32_t j = sel[(uint64_t)r * n + t];
            key = make_key(D[(uint64_t)r * ld + j], j);
        }
        keys[t] = key;
    }
    __syncthreads();
    bitonic_sort_u64<false>(reinterpret_cast<uint64_t*>(keys), np2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        const float d = unord_float((uint32_t)(keys[t] >> 32));
        if (!(d > 0.0f)) atomicOr(bad, 1u);  // nn_graph.cpp:41-44
        nbr[(uint64_t)(r0 + r) * n + t] = (uint32_t)keys[t];
        elen[(uint64_t)(r0 + r) * n + t] = d;
    }
}

}  // namespace dev

namespace {

// Exact-assignment Lloyd k-means on device data X[n, dim] -> C[k, dim].
void kmeans(const float* dX, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed, float* dC,
            const float* hX, cudaStream_t st) {
    if (k == 0 || n < k) throw std::runtime_error("train_kmeans: need at least k training points");
    if (iters == 0) throw std::runtime_error("train_kmeans: iters must be >= 1");
    // seeding: k distinct points (partial Fisher-Yates with mt19937_64(seed))
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> perm(n);
    for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    for (uint32_t c = 0; c < k; c++) {
        std::uniform_int_distribution<uint64_t> pick(c, n - 1);
        std::swap(perm[c], perm[pick(rng)]);
    }
    DevBuf<uint32_t> rows;
    rows.alloc(k);
    CUDA_CHECK(cudaMemcpyAsync(rows.p, perm.data(), k * 4, cudaMemcpyHostToDevice, st));
    dev::k_gather_rows<<<592, 256, 0, st>>>(dX, dim, rows.p, k, dC);
    CUDA_LAUNCH_CHECK();
    (void)hX;
    AddArgs a{};
    a.dim = dim;
    a.k = k;
    a.centroids = dC;
    DevBuf<uint32_t> best, best_sorted, iota, order, empty;
    DevBuf<unsigned long long> counts, off;
    DevBuf<float> pdist;
    best.alloc(n);
    best_sorted.alloc(n);
    iota.alloc(n);
    order.alloc(n);
    empty.alloc(k);
    counts.alloc((size_t)k + 1);
    off.alloc((size_t)k + 1);
    pdist.alloc(n);
    launch_iota(iota.p, n, st);
    int end_bit = 1;
    while ((1ull << end_bit) < (uint64_t)k) end_bit++;
    size_t sort_bytes = 0, scan_bytes = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, best.p, best_sorted.p, iota.p, order.p, n, 0,
                                               end_bit, st));
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts.p, off.p, (int)(k + 1), st));
    DevBuf<unsigned char> temp;
    temp.alloc(std::max(sort_bytes, scan_bytes));
    std::vector<uint32_t> hempty(k);
    std::vector<float> hpd;
    for (uint32_t it = 0; it < iters; it++) {
        launch_assign_nearest(a, dX, n, best.p, st);
        CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp.p, sort_bytes, best.p, best_sorted.p, iota.p, order.p, n, 0,
                                                   end_bit, st));
        CUDA_CHECK(cudaMemsetAsync(counts.p, 0, ((size_t)k + 1) * 8, st));
        launch_histogram(best_sorted.p, n, counts.p, st);
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp.p, scan_bytes, counts.p, off.p, (int)(k + 1), st));
        dev::k_segment_mean<<<k, 128, 0, st>>>(dX, dim, order.p, off.p, const_cast<float*>(dC), empty.p);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaMemcpyAsync(hempty.data(), empty.p, k * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        std::vector<uint32_t> empties;
        for (uint32_t c = 0; c < k; c++)
            if (hempty[c]) empties.push_back(c);
        if (!empties.empty()) {
            // re-seed each empty cluster with the currently farthest point
            dev::k_point_dist<<<592, 256, 0, st>>>(dX, dC, best.p, n, dim, pdist.p);
            CUDA_LAUNCH_CHECK();
            hpd.resize(n);
            CUDA_CHECK(cudaMemcpyAsync(hpd.data(), pdist.p, n * 4, cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaStreamSynchronize(st));
            std::vector<uint32_t> idx(n);
            for (uint64_t i = 0; i < n; i++) idx[i] = (uint32_t)i;
            std::partial_sort(idx.begin(), idx.begin() + std::min<uint64_t>(empties.size(), n), idx.end(),
                              [&](uint32_t x, uint32_t y) { return hpd[x] > hpd[y] || (hpd[x] == hpd[y] && x < y); });
            for (size_t e = 0; e < empties.size(); e++) {
                uint32_t r = idx[e % n];
                CUDA_CHECK(cudaMemcpyAsync(rows.p, &r, 4, cudaMemcpyHostToDevice, st));
                dev::k_gather_rows<<<1, 128, 0, st>>>(dX, dim, rows.p, 1, const_cast<float*>(dC) + (size_t)empties[e] * dim);
                CUDA_LAUNCH_CHECK();
                CUDA_CHECK(cudaStreamSynchronize(st));
            }
        }
    }
}

}  // namespace

// Returns a trained model (t3 left empty: computed on upload).
HostModel train_model_device(int device, const float* train, uint64_t nt, uint32_t dim, uint32_t k, uint32_t n,
                             uint32_t m, uint32_t iters, uint64_t seed, bool clamp) {
    if (m == 0 || dim % m != 0) throw std::runtime_error("m must divide the vector dimension");
    if (k == 0 || nt < k) throw std::runtime_error("train_kmeans: need at least k training points");
    if (iters == 0) throw std::runtime_error("train_kmeans: iters must be >= 1");
    if (n == 0 || n >= k) throw std::runtime_error("build_nn_graph: need 0 < n < k");
    int prev = 0;
    CUDA_CHECK(cudaGetDevice(&prev));
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t st;
    CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    HostModel hm;
    hm.dim = dim;
    hm.k = k;
    hm.n = n;
    hm.m = m;
    hm.clamp = clamp;
    hm.lo = 0.0f;
    hm.hi = 1.0f;
    {
        DevBuf<float> X, C;
        X.alloc(nt * dim);
        C.alloc((size_t)k * dim);
        CUDA_CHECK(cudaMemcpyAsync(X.p, train, nt * dim * 4, cudaMemcpyHostToDevice, st));
        kmeans(X.p, nt, dim, k, iters, seed, C.p, train, st);
        // exact n-NN graph (nn_graph.cpp:11-50), row tiles of the K x K matrix
        DevBuf<uint32_t> nbr, sel, bad;
        DevBuf<float> elen, D;
        nbr.alloc((size_t)k * n);
        elen.alloc((size_t)k * n);
        bad.alloc(1);
        CUDA_CHECK(cudaMemsetAsync(bad.p, 0, 4, st));
        const uint32_t R = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(k, (1ull << 29) / ((uint64_t)k * 4)));
        D.alloc((size_t)R * k);
        sel.alloc((size_t)R * n);
        for (uint32_t r0 = 0; r0 < k; r0 += R) {
            const uint32_t nr = std::min(R, k - r0);
            launch_sqdist_matrix(C.p + (size_t)r0 * dim, nr, C.p, k, dim, D.p, k, st);
            dev::k_set_diag<<<(nr + 255) / 256, 256, 0, st>>>(D.p, k, r0, nr);
            CUDA_LAUNCH_CHECK();
            launch_select_rows(D.p, k, nr, k, n, sel.p, st);
            uint32_t np2 = 1;
            while (np2 < n) np2 <<= 1;
            dev::k_graph_rows<<<nr, 128, np2 * 8, st>>>(D.p, k, sel.p, n, r0, nbr.p, elen.p, bad.p);
            CUDA_LAUNCH_CHECK();
        }
        D.reset();
        uint32_t hbad = 0;
        CUDA_CHECK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
        hm.centroids.resize((size_t)k * dim);
        hm.nbr.resize((size_t)k * n);
        hm.elen.resize((size_t)k * n);
        CUDA_CHECK(cudaMemcpyAsync(hm.centroids.data(), C.p, hm.centroids.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(hm.nbr.data(), nbr.p, hm.nbr.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(hm.elen.data(), elen.p, hm.elen.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        if (hbad) throw std::runtime_error("build_nn_graph: duplicate centroids (zero-length edge)");
        // displacements from the anchors (bindings.cpp:59-71)
        if (nt < VLQ_KSUB) throw std::runtime_error("train_pq: need at least 256 training points");
        DevBuf<float> R_, slice, sub;
        DevBuf<uint32_t> best;
        DevBuf<unsigned int> err;
        R_.alloc(nt * dim);
        best.alloc(nt);
        err.alloc(2);
        CUDA_CHECK(cudaMemsetAsync(err.p, 0, 8, st));
        AddArgs a{};
        a.dim = dim;
        a.k = k;
        a.n = n;
        a.m = m;
        a.clamp = clamp;
        a.lo = 0.0f;
        a.hi = 1.0f;
        a.centroids = C.p;
        a.nbr = nbr.p;
        a.elen = elen.p;
        a.error_flag = err.p;
        launch_assign_nearest(a, X.p, nt, best.p, st);
        launch_encode(a, X.p, nt, best.p, clamp ? 1 : 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st,
                      R_.p);
        // PQ: per-subspace 256-means (pq.cpp:20-50), seeds seed+1 + golden*p
        const uint32_t dsub = dim / m;
        slice.alloc(nt * dsub);
        sub.alloc((size_t)VLQ_KSUB * dsub);
        hm.pq.resize((size_t)m * VLQ_KSUB * dsub);
        for (uint32_t p = 0; p < m; p++) {
            dev::k_slice_cols<<<1184, 256, 0, st>>>(R_.p, nt, dim, p * dsub, dsub, slice.p);
            CUDA_LAUNCH_CHECK();
            kmeans(slice.p, nt, dsub, VLQ_KSUB, iters, (seed + 1) + 0x9e3779b97f4a7c15ULL * p, sub.p, nullptr, st);
            CUDA_CHECK(cudaMemcpyAsync(hm.pq.data() + (size_t)p * VLQ_KSUB * dsub, sub.p, (size_t)VLQ_KSUB * dsub * 4,
                                       cudaMemcpyDeviceToHost, st));
        }
        CUDA_CHECK(cudaStreamSynchronize(st));
    }
    CUDA_CHECK(cudaStreamDestroy(st));
    cudaSetDevice(prev);
    return hm;
}

}  // namespace vlq
