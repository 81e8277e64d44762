// Index.train on the device (reference: proj/python/bindings.cpp:44-81):
// first-level k-means, exact n-NN centroid graph, training displacements from
// the line anchors, per-subspace PQ k-means.
//
// train_kmeans follows the reference (kmeans.cpp:104-185) step for step:
//   * k-means++ seeding (seed_centroids, kmeans.cpp:54-102): the first centre
//     uniform, every further centre drawn with probability proportional to
//     min_d, the exact (reference-order) squared distance to the nearest
//     centre chosen so far; "all points covered" -> uniform;
//   * Lloyd iterations: exact strict-'<' argmin assignment, centroid sums
//     as sequential double sums in point order per cluster, mean = (float)
//     (sum / count) for non-empty clusters;
//   * the reference's empty-cluster repair (kmeans.cpp:157-181): each empty
//     cluster, in id order, takes the farthest member of the cluster with
//     the largest accumulated error, updating the errors as it goes.
// The one difference is the random stream: D^2 draws use a counter-based
// hash instead of mt19937_64, and K sequential passes over the training set
// become K/R rounds (see seed_pp), so codebooks are equal to the
// reference's in distribution, not bit for bit (parity is anchored on
// shared VLQ1 models; tests/test_gpu_train.py compares the
// quantization error with the reference's own Index.train).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
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


// ---- k-means++ seeding (seed_centroids, kmeans.cpp:54-102) ------------------

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
// uniform double in [0, 1) from (seed, counter)
__device__ __forceinline__ double u01(uint64_t seed, uint64_t ctr) {
    return (double)(mix64(seed ^ mix64(ctr)) >> 11) * 0x1.0p-53;
}

__global__ void k_fill_f32(float* v, uint64_t n, float x) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = x;
}

__global__ void k_to_double(const float* __restrict__ v, uint64_t n, double* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (double)v[i];
}

// min_d[i] = min(min_d[i], sqdist(x_i, c)) over `cnt` new centres (the
// reference's update after each draw, kmeans.cpp:94-99; sqdist in reference
// order).  128 points per tile, staged transposed in shared memory; the
// centres (padded to a multiple of 8 with rows at FLT_MAX, whose distance is
// +inf) are read as shared-memory broadcasts.
constexpr int PPU_T = 128;
__global__ void __launch_bounds__(PPU_T) k_pp_update(const float* __restrict__ X, uint64_t n, uint32_t dim,
                                                     const float* __restrict__ Cn, uint32_t cnt,
                                                     float* __restrict__ min_d) {
    extern __shared__ float sm[];
    const uint32_t cpad = (cnt + 7) & ~7u;
    float* cs = sm;                          // [cpad][dim]
    float* xs = sm + (size_t)cpad * dim;     // [dim][PPU_T]
    for (uint32_t t = threadIdx.x; t < cpad * dim; t += PPU_T)
        cs[t] = (t < cnt * dim) ? Cn[t] : 3.0e38f;
    for (uint64_t base = (uint64_t)blockIdx.x * PPU_T; base < n; base += (uint64_t)gridDim.x * PPU_T) {
        __syncthreads();
        const uint32_t np = (uint32_t)umin64(PPU_T, n - base);
        for (uint32_t t = threadIdx.x; t < np * dim; t += PPU_T) {
            const uint32_t p = t / dim, d = t - p * dim;
            xs[d * PPU_T + p] = X[(base + p) * dim + d];
        }
        __syncthreads();
        if (threadIdx.x >= np) continue;
        const uint64_t i = base + threadIdx.x;
        float best = min_d[i];
        for (uint32_t c0 = 0; c0 < cpad; c0 += 8) {
            float acc[8];
#pragma unroll
            for (int g = 0; g < 8; g++) acc[g] = 0.0f;
            const float* cg = cs + (size_t)c0 * dim;
            for (uint32_t d = 0; d < dim; d++) {
                const float xv = xs[d * PPU_T + threadIdx.x];
#pragma unroll
                for (int g = 0; g < 8; g++) acc[g] = sq_step(acc[g], xv, cg[(size_t)g * dim + d]);
            }
#pragma unroll
            for (int g = 0; g < 8; g++) best = fminf(best, acc[g]);
        }
        min_d[i] = best;
    }
}

// Same update for wide points (dim > 256, where a transposed 128-point tile
// no longer fits in shared memory): thread per point, rows read from global.
__global__ void __launch_bounds__(PPU_T) k_pp_update_wide(const float* __restrict__ X, uint64_t n, uint32_t dim,
                                                          const float* __restrict__ Cn, uint32_t cnt,
                                                          float* __restrict__ min_d) {
    extern __shared__ float sm[];
    for (uint32_t t = threadIdx.x; t < cnt * dim; t += PPU_T) sm[t] = Cn[t];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * PPU_T + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PPU_T) {
        const float* x = X + i * dim;
        float best = min_d[i];
        for (uint32_t c = 0; c < cnt; c++) {
            float a = 0.0f;
            for (uint32_t d = 0; d < dim; d++) a = sq_step(a, x[d], sm[(size_t)c * dim + d]);
            best = fminf(best, a);
        }
        min_d[i] = best;
    }
}

// One round of D^2 draws: up to R new centres from the distribution
// proportional to min_d as of the round start (prefix = its inclusive double
// prefix sum), each draw accepted with probability min_d'/min_d, min_d' the
// distance also counting the centres accepted earlier in this round.  This
// is rejection sampling, so every accepted centre is an exact draw from the
// reference's sequential distribution (proportional to the CURRENT min_d):
// K sequential passes over the training set become K/R passes.  The pick
// for a target u*total is the first i with prefix[i] >= target (the
// reference's `acc >= target`, kmeans.cpp:84-90), n-1 if none; total <= 0 ->
// uniform (kmeans.cpp:79-80).
__global__ void __launch_bounds__(256) k_pp_round(const float* __restrict__ X, uint64_t n, uint32_t dim,
                                                  const double* __restrict__ prefix, const float* __restrict__ min_d,
                                                  uint64_t seed, uint64_t ctr0, uint32_t R, uint32_t max_draws,
                                                  float* __restrict__ C_out, uint32_t* __restrict__ count_out) {
    extern __shared__ float sm[];
    float* cs = sm;                       // [R][dim] centres accepted this round
    float* xs = sm + (size_t)R * dim;     // [dim] the drawn point
    __shared__ float red[8];
    __shared__ unsigned long long s_pick;
    __shared__ int s_accept;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double total = prefix[n - 1];
    uint32_t acc = 0;
    for (uint32_t draw = 0; draw < max_draws && acc < R; draw++) {
        const uint64_t ctr = ctr0 + 2ull * draw;
        const double u1 = u01(seed, ctr), u2 = u01(seed, ctr + 1);
        if (wid == 0) {
            uint64_t pick;
            if (!(total > 0.0)) {
                pick = umin64(n - 1, (uint64_t)(u1 * (double)n));
            } else {
                const double target = u1 * total;
                uint64_t lo = 0, hi = n;  // answer: first i in [lo, hi) with prefix[i] >= target, or hi
                while (hi - lo > 32) {
                    const uint64_t seg = (hi - lo + 31) / 32;
                    const uint64_t end = umin64(lo + (uint64_t)(lane + 1) * seg, hi);
                    const bool ok = (lo + (uint64_t)lane * seg < hi) && prefix[end - 1] >= target;
                    const unsigned m = __ballot_sync(0xffffffffu, ok);
                    if (m == 0) {
                        lo = hi;
                        break;
                    }
                    const uint32_t f = __ffs(m) - 1;
                    const uint64_t nlo = lo + (uint64_t)f * seg;
                    hi = umin64(nlo + seg, hi);
                    lo = nlo;
                }
                const bool ok = (lo + lane < hi) && prefix[lo + lane] >= target;
                const unsigned m = __ballot_sync(0xffffffffu, ok);
                pick = m ? lo + (__ffs(m) - 1) : hi;
                if (pick >= n) pick = n - 1;
            }
            if (lane == 0) s_pick = pick;
        }
        __syncthreads();
        const uint64_t pick = s_pick;
        for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) xs[d] = X[pick * dim + d];
        __syncthreads();
        float dmin = __int_as_float(0x7f800000);
        for (uint32_t j = threadIdx.x; j < acc; j += blockDim.x) {
            const float* c = cs + (size_t)j * dim;
            float a = 0.0f;
            for (uint32_t d = 0; d < dim; d++) a = sq_step(a, xs[d], c[d]);
            dmin = fminf(dmin, a);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        if (lane == 0) red[wid] = dmin;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = red[0];
            for (uint32_t w = 1; w < blockDim.x / 32; w++) m = fminf(m, red[w]);
            int accept;
            if (!(total > 0.0)) {
                accept = 1;
            } else {
                const float d_old = min_d[pick];
                const float d_new = fminf(d_old, m);
                accept = d_old > 0.0f && u2 * (double)d_old < (double)d_new;
            }
            s_accept = accept;
        }
        __syncthreads();
        if (s_accept) {
            for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) {
                cs[(size_t)acc * dim + d] = xs[d];
                C_out[(size_t)acc * dim + d] = xs[d];
            }
            acc++;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *count_out = acc;
}

// max_i |c_i|^2 (double, in order) for the TF32 certificate of the
// tensor-core assignment; non-negative doubles order like their bit patterns
__global__ void k_max_sqnorm(const float* __restrict__ C, uint32_t k, uint32_t dim, unsigned long long* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (uint32_t d = 0; d < dim; d++) s += (double)C[(size_t)i * dim + d] * C[(size_t)i * dim + d];
        atomicMax(out, (unsigned long long)__double_as_longlong(s));
    }
}

}  // namespace dev

namespace {

// Exact assign_nearest (kmeans.cpp:21-33) of n points against k device
// centroids: for k >= 1024 (and a tcgen05-supported dim) the tensor-core
// ARGMIN GEMM proposes candidates and k_refine_argmin settles the exact
// strict-'<' argmin under the TF32 error certificate, the rest take the
// exact CUDA-core scan -- the add path's assignment (Engine::assign_chunk)
// for centroids that change every Lloyd iteration.
struct Assigner {
    uint32_t dim, k;
    bool tc;
    DevBuf<float> cent_tc, cnorm, td, rows;
    DevBuf<uint32_t> tidx, flag, fbest;
    DevBuf<unsigned long long> mx;
    DevBuf<unsigned int> nflag;
    uint64_t fallbacks = 0;
    Assigner(uint32_t dim_, uint32_t k_, uint64_t n) : dim(dim_), k(k_) {
        tc = k >= 1024 && coarse_tc_supported(dim);
        if (!tc) return;
        const uint32_t ntiles = (k + 127) / 128;
        cent_tc.alloc((size_t)ntiles * 128 * dim);
        cnorm.alloc((size_t)ntiles * 128);
        tidx.alloc(n * 4);
        td.alloc(n * 4);
        flag.alloc(n);
        mx.alloc(1);
        nflag.alloc(1);
    }
    void run(const float* X, uint64_t n, const float* C, uint32_t* best, cudaStream_t st) {
        AddArgs a{};
        a.dim = dim;
        a.k = k;
        a.centroids = C;
        if (!tc) {
            launch_assign_nearest(a, X, n, best, st);
            return;
        }
        launch_relayout_centroids(C, k, dim, cent_tc.p, nullptr, cnorm.p, st);
        CUDA_CHECK(cudaMemsetAsync(mx.p, 0, 8, st));
        dev::k_max_sqnorm<<<(k + 255) / 256, 256, 0, st>>>(C, k, dim, mx.p);
        CUDA_LAUNCH_CHECK();
        unsigned long long bits = 0;
        CUDA_CHECK(cudaMemcpyAsync(&bits, mx.p, 8, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        double m2;
        std::memcpy(&m2, &bits, 8);
        const float cmax = (float)(std::sqrt(m2) * (1.0 + 1e-6)) + 1e-30f;  // as Engine::upload_model
        launch_coarse_tc(0, X, n, dim, cent_tc.p, nullptr, cnorm.p, k, nullptr, 0, tidx.p, td.p, st);
        CUDA_CHECK(cudaMemsetAsync(nflag.p, 0, 4, st));
        launch_refine_argmin(X, n, dim, C, tidx.p, td.p, cmax, best, flag.p, nflag.p, st);
        unsigned int nf = 0;
        CUDA_CHECK(cudaMemcpyAsync(&nf, nflag.p, 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        if (nf) {
            fallbacks += nf;
            rows.alloc((size_t)nf * dim);
            fbest.alloc(nf);
            launch_gather_rows_list(X, dim, flag.p, nf, rows.p, st);
            launch_assign_nearest(a, rows.p, nf, fbest.p, st);
            launch_scatter_u32(fbest.p, flag.p, nf, best, st);
        }
    }
};

// k-means++ seeding (seed_centroids, kmeans.cpp:54-102) -> dC[k, dim].
// Rounds of up to R rejection-sampled draws (k_pp_round), each followed by
// the exact min_d update for the round's new centres (k_pp_update) and a
// fresh double prefix sum.
void seed_pp(const float* dX, uint64_t n, uint32_t dim, uint32_t k, uint64_t seed, float* dC, cudaStream_t st) {
    const uint32_t Rmax = (uint32_t)std::max<uint64_t>(8, std::min<uint64_t>(256, (96u << 10) / (4ull * dim)) & ~7ull);
    DevBuf<float> min_d;
    DevBuf<double> dv, prefix;
    DevBuf<uint32_t> cnt;
    min_d.alloc(n);
    dv.alloc(n);
    prefix.alloc(n);
    cnt.alloc(1);
    size_t scan_bytes = 0;
    CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, dv.p, prefix.p, (int)n, st));
    DevBuf<unsigned char> temp;
    temp.alloc(std::max<size_t>(scan_bytes, 1));
    const bool wide = dim > 256;
    const size_t upd_smem = wide ? (size_t)Rmax * dim * 4 : ((size_t)((Rmax + 7) & ~7u) * dim + (size_t)dim * dev::PPU_T) * 4;
    const size_t round_smem = ((size_t)Rmax * dim + dim) * 4;
    if (upd_smem > (227u << 10) || round_smem > (227u << 10))
        throw std::runtime_error("train_kmeans: dimension too large for the device seeding");
    CUDA_CHECK(cudaFuncSetAttribute(wide ? dev::k_pp_update_wide : dev::k_pp_update,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem));
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_pp_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)round_smem));
    const unsigned upd_grid = (unsigned)std::min<uint64_t>((n + dev::PPU_T - 1) / dev::PPU_T, 148ull * 8);
    auto update = [&](const float* Cn, uint32_t c) {
        (wide ? dev::k_pp_update_wide : dev::k_pp_update)<<<upd_grid, dev::PPU_T, upd_smem, st>>>(dX, n, dim, Cn, c,
                                                                                                min_d.p);
        CUDA_LAUNCH_CHECK();
    };
    // first centre: uniform over the training set (kmeans.cpp:61-63)
    dev::k_fill_f32<<<592, 256, 0, st>>>(min_d.p, n, INFINITY);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaMemsetAsync(prefix.p + (n - 1), 0, 8, st));  // total 0 -> uniform pick
    dev::k_pp_round<<<1, 256, round_smem, st>>>(dX, n, dim, prefix.p, min_d.p, seed, 0, 1, 1, dC, cnt.p);
    CUDA_LAUNCH_CHECK();
    update(dC, 1);
    uint32_t t = 1;
    for (uint64_t round = 1; t < k; round++) {
        dev::k_to_double<<<592, 256, 0, st>>>(min_d.p, n, dv.p);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cub::DeviceScan::InclusiveSum(temp.p, scan_bytes, dv.p, prefix.p, (int)n, st));
        const uint32_t R = std::min(Rmax, k - t);
        dev::k_pp_round<<<1, 256, round_smem, st>>>(dX, n, dim, prefix.p, min_d.p, seed, round << 32, R, 4 * R,
                                                     dC + (size_t)t * dim, cnt.p);
        CUDA_LAUNCH_CHECK();
        uint32_t got = 0;
        CUDA_CHECK(cudaMemcpyAsync(&got, cnt.p, 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        if (got) update(dC + (size_t)t * dim, got);
        t += got;
    }
}

// train_kmeans (kmeans.cpp:104-185) on device data X[n, dim] -> C[k, dim].
// `init` (device, nullable) replaces the k-means++ seeding with given
// centroids: the Lloyd iterations and the repair are then deterministic and
// equal the reference's bit for bit (tests/test_gpu_train.py).
void kmeans(const float* dX, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed, float* dC,
            const float* init, cudaStream_t st) {
    if (k == 0 || n < k) throw std::runtime_error("train_kmeans: need at least k training points");
    if (iters == 0) throw std::runtime_error("train_kmeans: iters must be >= 1");
    if (init)
        CUDA_CHECK(cudaMemcpyAsync(dC, init, (size_t)k * dim * 4, cudaMemcpyDeviceToDevice, st));
    else
        seed_pp(dX, n, dim, k, seed, dC, st);
    Assigner asg(dim, k, n);
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
    std::vector<uint32_t> hempty(k), hassign;
    std::vector<float> hdist;
    for (uint32_t it = 0; it < iters; it++) {
        asg.run(dX, n, dC, best.p, st);
        // dist[i] of the assignment (kmeans.cpp:123-127), before the update
        dev::k_point_dist<<<592, 256, 0, st>>>(dX, dC, best.p, n, dim, pdist.p);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp.p, sort_bytes, best.p, best_sorted.p, iota.p, order.p, n, 0,
                                                   end_bit, st));
        CUDA_CHECK(cudaMemsetAsync(counts.p, 0, ((size_t)k + 1) * 8, st));
        launch_histogram(best_sorted.p, n, counts.p, st);
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp.p, scan_bytes, counts.p, off.p, (int)(k + 1), st));
        dev::k_segment_mean<<<k, 128, 0, st>>>(dX, dim, order.p, off.p, dC, empty.p);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaMemcpyAsync(hempty.data(), empty.p, k * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        bool any = false;
        for (uint32_t c = 0; c < k && !any; c++) any = hempty[c] != 0;
        if (!any) continue;
        // repair (kmeans.cpp:157-181), sequential on the host exactly as the
        // reference: donor = first cluster of maximal error, its farthest
        // member (strict '>' from index 0) moves to the empty cluster
        hassign.resize(n);
        hdist.resize(n);
        CUDA_CHECK(cudaMemcpyAsync(hassign.data(), best.p, n * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(hdist.data(), pdist.p, n * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        std::vector<double> err(k, 0.0);
        std::vector<uint64_t> moff((size_t)k + 1, 0);
        for (uint64_t i = 0; i < n; i++) {
            err[hassign[i]] += hdist[i];
            moff[hassign[i] + 1]++;
        }
        for (uint32_t c = 0; c < k; c++) moff[c + 1] += moff[c];
        std::vector<uint32_t> members(n);
        {
            std::vector<uint64_t> pos(moff.begin(), moff.end() - 1);
            for (uint64_t i = 0; i < n; i++) members[pos[hassign[i]]++] = (uint32_t)i;  // ascending per cluster
        }
        for (uint32_t c = 0; c < k; c++) {
            if (!hempty[c]) continue;
            const uint32_t donor = (uint32_t)(std::max_element(err.begin(), err.end()) - err.begin());
            uint64_t far_i = 0;
            float far_d = -1.0f;
            for (uint64_t t = moff[donor]; t < moff[donor + 1]; t++) {
                const uint32_t i = members[t];
                if (hassign[i] == donor && hdist[i] > far_d) {
                    far_d = hdist[i];
                    far_i = i;
                }
            }
            CUDA_CHECK(cudaMemcpyAsync(dC + (size_t)c * dim, dX + far_i * dim, (size_t)dim * 4,
                                       cudaMemcpyDeviceToDevice, st));
            hassign[far_i] = c;
            err[donor] -= far_d;
            hdist[far_i] = 0.0f;
            err[c] = 0.0;
        }
    }
    CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace

// train_kmeans (kmeans.hpp) on host arrays: X[n, dim] -> out[k, dim];
// init (host, nullable) replaces the seeding.
void train_kmeans_host(int device, const float* X, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters,
                       uint64_t seed, const float* init, float* out) {
    if (dim == 0) throw std::runtime_error("train_kmeans: dimension mismatch");
    if (k == 0 || n < k) throw std::runtime_error("train_kmeans: need at least k training points");
    if (iters == 0) throw std::runtime_error("train_kmeans: iters must be >= 1");
    DeviceGuard g(device);
    cudaStream_t st;
    CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamFree {
        cudaStream_t s;
        ~StreamFree() { cudaStreamDestroy(s); }
    } sf{st};
    DevBuf<float> dX, dC, dI;
    dX.alloc(n * dim);
    dC.alloc((size_t)k * dim);
    CUDA_CHECK(cudaMemcpyAsync(dX.p, X, n * dim * 4, cudaMemcpyHostToDevice, st));
    if (init) {
        dI.alloc((size_t)k * dim);
        CUDA_CHECK(cudaMemcpyAsync(dI.p, init, (size_t)k * dim * 4, cudaMemcpyHostToDevice, st));
    }
    kmeans(dX.p, n, dim, k, iters, seed, dC.p, init ? dI.p : nullptr, st);
    CUDA_CHECK(cudaMemcpyAsync(out, dC.p, (size_t)k * dim * 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
}

// Returns a trained model (t3 left empty: computed on upload).
HostModel train_model_device(int device, const float* train, uint64_t nt, uint32_t dim, uint32_t k, uint32_t n,
                             uint32_t m, uint32_t iters, uint64_t seed, bool clamp) {
    if (m == 0 || dim % m != 0) throw std::runtime_error("m must divide the vector dimension");
    if (k == 0 || nt < k) throw std::runtime_error("train_kmeans: need at least k training points");
    if (iters == 0) throw std::runtime_error("train_kmeans: iters must be >= 1");
    if (n == 0 || n >= k) throw std::runtime_error("build_nn_graph: need 0 < n < k");
    DeviceGuard g(device);
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
        kmeans(X.p, nt, dim, k, iters, seed, C.p, nullptr, st);
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
    return hm;
}

}  // namespace vlq
