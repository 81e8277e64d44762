// IVFADC comparison baseline (proj/src/ivf_baseline.cpp) on the GPU.
//
// The paper's Faiss-style baseline: ONE level of K lists holding (id, PQ code
// of x - c_i), built with the VLQ model's codebook and PQ (eval.cpp:182), and
// searched by scanning the w nearest regions with a per-(query, region)
// residual lookup table.  Unlike VLQ-ADC, every step here is directly the
// reference's arithmetic, so the GPU distances are the reference's bit for
// bit and the top-k needs no re-score:
//
//   build:  assign_nearest (exact, strict '<')  -> residual x - c (fp32 sub)
//           -> pq_encode (256-way sequential-sqdist argmin per sub-space)
//           -> stable bucketing by region (ids ascend within a list)
//   search: first_level_scan's exact top-w (the engine's coarse stage) ->
//           per region: residual y - c, LUT[p][j] = sqdist(residual_p, PQ_pj)
//           in order, d = sum_p LUT[p][code_p] in order (d starts at 0) ->
//           block-shared candidate buffer of (d, id) keys, radix-select
//           flushes, exact (dist, id) top-k (select_topk, search.cpp:122-140).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <cstring>
#include <stdexcept>

#include "engine.h"
#include "select.cuh"

namespace vlq {
namespace dev {

__device__ __forceinline__ uint64_t ivf_argmin_key(float d, uint32_t idx) {  // strict '<' from FLT_MAX
    return (d < FLT_MAX) ? make_key(d, idx) : ~0ull;
}

// residual + pq_encode of one point per warp, given its region
__global__ void __launch_bounds__(256) k_ivf_encode(const float* __restrict__ X, uint64_t nx, uint32_t dim,
                                                    uint32_t m, const float* __restrict__ centroids,
                                                    const float* __restrict__ pq, const uint32_t* __restrict__ region,
                                                    uint8_t* __restrict__ codes) {
    extern __shared__ float rsm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t dsub = dim / m;
    float* rs = rsm + (size_t)warp * dim;
    const uint64_t pt = (uint64_t)blockIdx.x * 8 + warp;
    if (pt >= nx) return;
    const float* c = centroids + (uint64_t)region[pt] * dim;
    for (uint32_t d = lane; d < dim; d += 32) rs[d] = __fsub_rn(X[pt * dim + d], c[d]);  // ivf_baseline.cpp:33-35
    __syncwarp();
    for (uint32_t p = 0; p < m; p++) {  // pq_encode (pq.cpp:52-67)
        uint64_t bk = ~0ull;
        for (uint32_t j = lane; j < VLQ_KSUB; j += 32) {
            const float* sc = pq + ((uint64_t)p * VLQ_KSUB + j) * dsub;
            float acc = 0.0f;
            for (uint32_t t = 0; t < dsub; t++) acc = sq_step(acc, rs[p * dsub + t], __ldg(sc + t));
            const uint64_t key = ivf_argmin_key(acc, j);
            bk = key < bk ? key : bk;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, bk, o);
            bk = w < bk ? w : bk;
        }
        if (lane == 0) codes[pt * m + p] = (uint8_t)((bk == ~0ull) ? 0u : (uint32_t)bk);
    }
}

__global__ void k_ivf_gather(const uint32_t* __restrict__ order, uint64_t n, uint32_t m,
                             const uint8_t* __restrict__ codes_pt, uint32_t* __restrict__ ids,
                             uint8_t* __restrict__ codes) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t pt = order[e];
        ids[e] = pt;
        for (uint32_t p = 0; p < m; p++) codes[e * m + p] = codes_pt[(uint64_t)pt * m + p];
    }
}

__device__ __forceinline__ uint64_t ivf_key(float d, uint32_t id) {
    uint32_t ub = __float_as_uint(d);
    ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;  // order-preserving
    return ((uint64_t)ub << 32) | id;
}

// Keeps exactly the `keep` smallest keys of cbuf[0..n) (compacted, unordered);
// returns the largest kept key.  Same radix select as the VLQ fast scan.
__device__ uint64_t ivf_select_keep(uint64_t* cbuf, uint32_t n, uint32_t keep, uint32_t* hist, unsigned int* s_misc) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint64_t prefix = 0, pmask = 0;
    uint32_t remaining = keep;
    int sh = 56;
    for (; sh >= 0; sh -= 8) {
        for (uint32_t b = tid; b < 256; b += nt) hist[b] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += nt) {
            const uint64_t k = cbuf[i];
            if ((k & pmask) == prefix) atomicAdd(&hist[(uint32_t)(k >> sh) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t v[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                v[j] = hist[tid * 8 + j];
                s += v[j];
            }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= (uint32_t)o) incl += y;
            }
            uint32_t run = incl - s;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (run < remaining && remaining <= run + v[j]) {
                    s_misc[0] = tid * 8 + j;
                    s_misc[1] = run;
                    s_misc[2] = v[j];
                }
                run += v[j];
            }
        }
        __syncthreads();
        const uint32_t b = s_misc[0], before = s_misc[1], inbin = s_misc[2];
        __syncthreads();
        prefix |= (uint64_t)b << sh;
        pmask |= 0xFFull << sh;
        remaining -= before;
        if (inbin == remaining) break;
    }
    const uint64_t T = sh > 0 ? (prefix | ((1ull << sh) - 1ull)) : prefix;
    uint32_t written = 0;
    for (uint32_t base = 0; base < n; base += nt) {
        const uint32_t i = base + tid;
        const uint64_t k = i < n ? cbuf[i] : ~0ull;
        const uint32_t take = (i < n && k <= T) ? 1u : 0u;
        uint32_t total;
        const uint32_t ex = block_excl_scan_u32(take, s_misc + 8, &total);
        if (take) cbuf[written + ex] = k;
        written += total;
        __syncthreads();
    }
    return T;
}

// One CTA (256 threads) per query: search_ivf_baseline (ivf_baseline.cpp:53-126).
constexpr uint32_t IVF_ROUND = 4;  // entries per thread between candidate-buffer checks

template <int M>  // M = 0: generic m (byte loads)
__global__ void __launch_bounds__(256) k_ivf_scan(const float* __restrict__ Y, uint32_t dim, uint32_t m,
                                                  const float* __restrict__ centroids, const float* __restrict__ pq,
                                                  const uint64_t* __restrict__ off, const uint32_t* __restrict__ ids,
                                                  const uint8_t* __restrict__ codes, const uint32_t* __restrict__ top,
                                                  uint32_t w, uint32_t topk, uint32_t cap,
                                                  int64_t* __restrict__ out_ids, float* __restrict__ out_d,
                                                  uint64_t* __restrict__ out_scanned) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t mm = M ? (uint32_t)M : m;
    const uint32_t dsub = dim / mm;
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(smem);                    // cap keys
    float* lut = reinterpret_cast<float*>(cbuf + cap);                     // m * 256
    float* res = lut + (size_t)mm * VLQ_KSUB;                              // dim
    __shared__ uint32_t hist[256];
    __shared__ unsigned int s_misc[48];
    __shared__ unsigned int s_count;
    __shared__ unsigned long long s_tau;
    const uint64_t q = blockIdx.x;
    const float* y = Y + q * dim;
    if (threadIdx.x == 0) {
        s_count = 0;
        s_tau = ~0ull;
    }
    uint64_t scanned = 0;
    const uint32_t per_round = blockDim.x * IVF_ROUND;
    for (uint32_t r = 0; r < w; r++) {
        const uint32_t region = top[q * w + r];
        const uint64_t b0 = off[region], b1 = off[region + 1];
        scanned += b1 - b0;
        if (b0 == b1) continue;  // ivf_baseline.cpp:92-94
        __syncthreads();         // previous region's LUT readers are done
        const float* ctr = centroids + (uint64_t)region * dim;
        for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) res[d] = __fsub_rn(y[d], ctr[d]);
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < mm * VLQ_KSUB; t += blockDim.x) {
            const uint32_t p = t >> 8;
            const float* sc = pq + (uint64_t)t * dsub;  // sub_centroid(p, j), t = p*256 + j
            float acc = 0.0f;
            for (uint32_t u = 0; u < dsub; u++) acc = sq_step(acc, res[p * dsub + u], __ldg(sc + u));
            lut[t] = acc;
        }
        __syncthreads();
        for (uint64_t e0 = b0; topk > 0 && e0 < b1; e0 += per_round) {
            // make room for a whole round, then scan it
            if (s_count + per_round > cap) {  // block-uniform
                const uint64_t T = ivf_select_keep(cbuf, s_count, topk, hist, s_misc);
                __syncthreads();
                if (threadIdx.x == 0) {
                    s_count = topk;
                    s_tau = T + 1;  // insert only keys <= T
                }
                __syncthreads();
            }
            const uint64_t tau = s_tau;
            const float taud = tau == ~0ull ? __int_as_float(0x7f800000)
                                            : __uint_as_float(((uint32_t)(tau >> 32) & 0x80000000u)
                                                                  ? ((uint32_t)(tau >> 32) & 0x7fffffffu)
                                                                  : ~(uint32_t)(tau >> 32));
#pragma unroll
            for (uint32_t u = 0; u < IVF_ROUND; u++) {
                const uint64_t e = e0 + (uint64_t)u * blockDim.x + threadIdx.x;
                if (e < b1) {
                    float d = 0.0f;  // ivf_baseline.cpp:112-117: d += lut[p][code[p]]
                    const uint8_t* cp = codes + e * mm;
                    if constexpr (M == 16) {
                        const uint4 v = __ldg(reinterpret_cast<const uint4*>(cp));
                        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int p = 0; p < 16; p++) d = __fadd_rn(d, lut[p * 256 + ((wv[p >> 2] >> (8 * (p & 3))) & 255u)]);
                    } else if constexpr (M == 8) {
                        const uint2 v = __ldg(reinterpret_cast<const uint2*>(cp));
                        const uint32_t wv[2] = {v.x, v.y};
#pragma unroll
                        for (int p = 0; p < 8; p++) d = __fadd_rn(d, lut[p * 256 + ((wv[p >> 2] >> (8 * (p & 3))) & 255u)]);
                    } else {
                        for (uint32_t p = 0; p < mm; p++) d = __fadd_rn(d, lut[p * 256 + cp[p]]);
                    }
                    if (d <= taud) {
                        const uint64_t key = ivf_key(d, __ldg(ids + e));
                        if (key < tau) cbuf[atomicAdd(&s_count, 1u)] = key;
                    }
                }
            }
            __syncthreads();
        }
    }
    // final: the topk smallest (dist, id) keys, sorted, padded (bindings.cpp:116-124)
    __syncthreads();
    uint32_t n = s_count;
    if (n > topk) {
        ivf_select_keep(cbuf, n, topk, hist, s_misc);
        n = topk;
    }
    __syncthreads();
    uint32_t np2 = 1;
    while (np2 < topk) np2 <<= 1;
    for (uint32_t i = n + threadIdx.x; i < np2; i += blockDim.x) cbuf[i] = ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(cbuf, np2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        if (t < n) {
            const uint64_t k = cbuf[t];
            const uint32_t ub = (uint32_t)(k >> 32);
            out_ids[q * topk + t] = (int64_t)(uint32_t)k;
            out_d[q * topk + t] = __uint_as_float((ub & 0x80000000u) ? (ub & 0x7fffffffu) : ~ub);
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
    if (threadIdx.x == 0 && out_scanned) out_scanned[q] = scanned;
}

}  // namespace dev

// ---------------------------------------------------------------------------
// build_ivf_baseline (ivf_baseline.cpp:11-51)
// ---------------------------------------------------------------------------
void Engine::ivf_build_stream(uint64_t nb, uint64_t chunk, const ChunkSource& src) {
    if (!model_ok_) throw std::runtime_error("build_ivf_baseline: no model loaded");
    if (nb > 0xffffffffull) throw std::runtime_error("build_ivf_baseline: more than 2^32-1 points");
    DeviceGuard g(cfg_.device);
    cudaStream_t st = stream_;
    chunk = std::max<uint64_t>(1, std::min(chunk, std::max<uint64_t>(nb, 1)));
    DevBuf<float> X;
    DevBuf<uint32_t> region;
    DevBuf<uint8_t> codes_pt;
    X.alloc(chunk * dim_);
    region.alloc(std::max<uint64_t>(nb, 1));
    codes_pt.alloc(std::max<uint64_t>(nb * m_, 1));
    for (uint64_t f = 0; f < nb; f += chunk) {
        const uint64_t c = std::min(chunk, nb - f);
        src(f, c, X.p, st);
        assign_chunk(X.p, c, region.p + f, st);  // assign_nearest, exact (kmeans.cpp:21-33)
        dev::k_ivf_encode<<<(unsigned)((c + 7) / 8), 256, 8 * dim_ * sizeof(float), st>>>(
            X.p, c, dim_, m_, centroids_.p, pq_.p, region.p + f, codes_pt.p + f * m_);
        CUDA_LAUNCH_CHECK();
    }
    X.reset();
    // stable bucketing by region: ids ascend within a list
    int end_bit = 1;
    while ((1ull << end_bit) <= (uint64_t)k_) end_bit++;
    DevBuf<uint32_t> region_sorted, iota, order;
    region_sorted.alloc(std::max<uint64_t>(nb, 1));
    iota.alloc(std::max<uint64_t>(nb, 1));
    order.alloc(std::max<uint64_t>(nb, 1));
    ivf_off_.alloc((size_t)k_ + 1);
    if (nb) {
        launch_iota(iota.p, nb, st);
        size_t temp_bytes = 0;
        CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, region.p, region_sorted.p, iota.p, order.p, nb,
                                                   0, end_bit, st));
        DevBuf<unsigned char> temp;
        temp.alloc(temp_bytes);
        CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, region.p, region_sorted.p, iota.p, order.p, nb,
                                                   0, end_bit, st));
    }
    DevBuf<unsigned long long> counts;
    counts.alloc((size_t)k_ + 2);
    CUDA_CHECK(cudaMemsetAsync(counts.p, 0, ((size_t)k_ + 2) * 8, st));
    if (nb) launch_histogram(region_sorted.p, nb, counts.p, st);
    {
        size_t temp_bytes = 0;
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts.p,
                                                 reinterpret_cast<unsigned long long*>(ivf_off_.p), (int)(k_ + 1), st));
        DevBuf<unsigned char> temp;
        temp.alloc(temp_bytes);
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp.p, temp_bytes, counts.p,
                                                 reinterpret_cast<unsigned long long*>(ivf_off_.p), (int)(k_ + 1), st));
    }
    ivf_ids_.reset();
    ivf_codes_.reset();
    ivf_ids_.alloc(std::max<uint64_t>(nb, 1));
    ivf_codes_.alloc(std::max<uint64_t>(nb * m_, 1));
    if (nb) {
        dev::k_ivf_gather<<<1184, 256, 0, st>>>(order.p, nb, m_, codes_pt.p, ivf_ids_.p, ivf_codes_.p);
        CUDA_LAUNCH_CHECK();
    }
    CUDA_CHECK(cudaStreamSynchronize(st));
    ivf_n_ = nb;
    ivf_ok_ = true;
}

void Engine::ivf_build_host(const float* base, uint64_t nb) {
    DeviceGuard g(cfg_.device);
    const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / (4ull * std::max<uint32_t>(dim_, 1)));
    PinnedBuf stage;
    ivf_build_stream(nb, chunk, [&](uint64_t first, uint64_t count, float* dst, cudaStream_t st) {
        CUDA_CHECK(cudaMemcpyAsync(dst, base + first * dim_, count * dim_ * 4, cudaMemcpyHostToDevice, st));
    });
}

// ---------------------------------------------------------------------------
// search_ivf_baseline (ivf_baseline.cpp:53-126)
// ---------------------------------------------------------------------------
void Engine::ivf_search_device(const float* d_q, uint64_t nq, uint32_t w, uint32_t topk, int64_t* d_ids,
                               float* d_dists, uint64_t* d_scanned, cudaStream_t st) {
    if (!ivf_ok_) throw std::runtime_error("search_ivf_baseline: no baseline index built");
    if (w == 0 || w > k_) throw std::runtime_error("search_ivf_baseline: need 0 < w <= k");
    if (topk > 1024) throw std::runtime_error("search_ivf_baseline: k > 1024 is not supported by the GPU engine");
    if (nq == 0) return;
    DeviceGuard g(cfg_.device);
    uint32_t np2 = 1;
    while (np2 < std::max<uint32_t>(topk, 1)) np2 <<= 1;
    const uint32_t cap = np2 + 256 * dev::IVF_ROUND;
    const size_t smem = (size_t)cap * 8 + ((size_t)m_ * VLQ_KSUB + dim_) * 4;
    if (smem > 227 * 1024) throw std::runtime_error("search_ivf_baseline: m too large for the GPU scan");
    // the engine's first level: exact top-w by (dist, id), as order[] in
    // ivf_baseline.cpp:82-91 (identical to first_level_scan)
    const uint64_t per_q = 4ull * k_ + 8ull * w + 4ull * w * (n_ + 1) + 256;
    uint64_t tile = std::max<uint64_t>(1, cfg_.workspace_bytes / per_q);
    tile = std::min<uint64_t>(std::min<uint64_t>(tile, cfg_.max_tile), nq);
    ws_.alloc(tile * k_);
    top_.alloc(tile * w);
    cand_top_.alloc(tile * (uint64_t)std::min<uint32_t>(k_, w + std::max<uint32_t>(32, w / 2)));
    qlist_.alloc(tile);
    if (tc_) {
        const uint32_t tn = tc_split_ ? 64 : 128;
        tmin_.alloc(tile * (uint64_t)(((k_ + tn - 1) / tn) * (tn / 32)));
        tau_.alloc(tile);
        lcnt_.alloc(tile);
        lidx_.alloc(tile * (uint64_t)kListCap);
        ld_.alloc(tile * (uint64_t)kListCap);
    }
    const bool prof = profiling_;
    profiling_ = false;  // the per-phase profile describes VLQ searches only
    struct Restore {
        bool& f;
        bool v;
        ~Restore() { f = v; }
    } restore{profiling_, prof};
    for (uint64_t t0 = 0; t0 < nq; t0 += tile) {
        const uint64_t nt = std::min(tile, nq - t0);
        const float* q = d_q + t0 * dim_;
        uint64_t launches = 0;
        bool fused = false;
        coarse_tile(q, nt, w, /*w2=*/0, launches, st, &fused);  // first level only
#define VLQ_IVF(MM)                                                                                               \
    do {                                                                                                          \
        auto fn = dev::k_ivf_scan<MM>;                                                                            \
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));             \
        fn<<<(unsigned)nt, 256, smem, st>>>(q, dim_, m_, centroids_.p, pq_.p, ivf_off_.p, ivf_ids_.p,           \
                                            ivf_codes_.p, top_.p, w, topk, cap, d_ids + t0 * topk,               \
                                            d_dists + t0 * topk, d_scanned ? d_scanned + t0 : nullptr);          \
    } while (0)
        if (m_ == 16) VLQ_IVF(16);
        else if (m_ == 8) VLQ_IVF(8);
        else VLQ_IVF(0);
#undef VLQ_IVF
        CUDA_LAUNCH_CHECK();
    }
}

void Engine::ivf_search_host(const float* q, uint64_t nq, uint32_t w, uint32_t topk, int64_t* ids, float* dists,
                             uint64_t* scanned) {
    if (!ivf_ok_) throw std::runtime_error("search_ivf_baseline: no baseline index built");
    if (w == 0 || w > k_) throw std::runtime_error("search_ivf_baseline: need 0 < w <= k");
    if (nq == 0) return;
    DeviceGuard g(cfg_.device);
    cudaStream_t st = stream_;
    const size_t qb = nq * dim_ * 4, ib = nq * topk * 8, db = nq * topk * 4, sb = nq * 8;
    sq_.alloc(nq * dim_);
    si_.alloc(std::max<uint64_t>(nq * topk, 1));
    sd_.alloc(std::max<uint64_t>(nq * topk, 1));
    ss_.alloc(nq);
    pin_.alloc(qb + ib + db + sb);
    unsigned char* pq = pin_.p;
    unsigned char* pi = pq + qb;
    unsigned char* pd = pi + ib;
    unsigned char* ps = pd + db;
    std::memcpy(pq, q, qb);
    CUDA_CHECK(cudaMemcpyAsync(sq_.p, pq, qb, cudaMemcpyHostToDevice, st));
    ivf_search_device(sq_.p, nq, w, topk, si_.p, sd_.p, ss_.p, st);
    if (topk) {
        CUDA_CHECK(cudaMemcpyAsync(pi, si_.p, ib, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(pd, sd_.p, db, cudaMemcpyDeviceToHost, st));
    }
    CUDA_CHECK(cudaMemcpyAsync(ps, ss_.p, sb, cudaMemcpyDeviceToHost, st));
    check_device_errors(st);
    if (topk) {
        std::memcpy(ids, pi, ib);
        std::memcpy(dists, pd, db);
    }
    if (scanned) std::memcpy(scanned, ps, sb);
}

void Engine::ivf_get_lists(uint64_t* off, uint32_t* ids, uint8_t* codes) {
    if (!ivf_ok_) throw std::runtime_error("build_ivf_baseline: no baseline index built");
    DeviceGuard g(cfg_.device);
    if (off) CUDA_CHECK(cudaMemcpyAsync(off, ivf_off_.p, ((size_t)k_ + 1) * 8, cudaMemcpyDeviceToHost, stream_));
    if (ids && ivf_n_) CUDA_CHECK(cudaMemcpyAsync(ids, ivf_ids_.p, ivf_n_ * 4, cudaMemcpyDeviceToHost, stream_));
    if (codes && ivf_n_)
        CUDA_CHECK(cudaMemcpyAsync(codes, ivf_codes_.p, ivf_n_ * m_, cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
}

}  // namespace vlq
