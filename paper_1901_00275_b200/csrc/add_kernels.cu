// Add/encode-path kernels (Algorithms 1+2 of the paper; reference
// proj/src/index.cpp:54-203, line_quant.cpp:24-49, pq.cpp:11-18 and :52-67).
//
//   k_tables          t2 = |PQ[p][j]|^2 (pq.cpp:11-18), t3 = <c_i,p , PQ[p][j]>
//                     (index.cpp:54-74)
//   k_assign_nearest  exact nearest centroid, strict '<' from FLT_MAX so the
//                     lowest id wins (assign_point, index.cpp:86-106)
//   k_encode          best edge (assign_edge, line_quant.cpp:24-49), residual
//                     at the exact lambda (index.cpp:181-184), PQ encode
//                     (pq.cpp:52-67), lambda byte (index.cpp:12-17) and the
//                     query-independent ADC term e = sum2 + 2(1-l)sum3 + 2l sum4
//                     used by the fast scan.
#include <cfloat>

#include "kernels.h"

namespace vlq {
namespace dev {

__global__ void __launch_bounds__(256) k_tables(const float* __restrict__ centroids, uint32_t k, uint32_t dim,
                                                const float* __restrict__ pq, uint32_t m, float* __restrict__ t2,
                                                float* __restrict__ t3) {
    const uint32_t dsub = dim / m;
    const uint32_t i = blockIdx.x;  // i == k: the t2 block
    for (uint32_t p = 0; p < m; p++) {
        for (uint32_t j = threadIdx.x; j < VLQ_KSUB; j += blockDim.x) {
            const float* sc = pq + ((uint64_t)p * VLQ_KSUB + j) * dsub;
            float acc = 0.0f;
            if (i < k) {
                const float* ci = centroids + (uint64_t)i * dim + p * dsub;
                for (uint32_t t = 0; t < dsub; t++) acc = dot_step(acc, ci[t], sc[t]);
                t3[((uint64_t)i * m + p) * VLQ_KSUB + j] = acc;
            } else {
                for (uint32_t t = 0; t < dsub; t++) acc = dot_step(acc, sc[t], sc[t]);
                t2[p * VLQ_KSUB + j] = acc;
            }
        }
    }
}

// key for the reference argmin "if (d < best_d)" scanned from best_d =
// FLT_MAX: a candidate only qualifies when d < FLT_MAX; among qualifying
// candidates the smallest (d, index) wins; with none, index 0.
__device__ __forceinline__ uint64_t argmin_key(float d, uint32_t idx) {
    return (d < FLT_MAX) ? make_key(d, idx) : ~0ull;
}

// Exact nearest centroid for each point: 64 points x all centroids per CTA,
// 4x4 register tile per thread, D streamed through shared memory.
constexpr int AS_TILE = 64;
constexpr int AS_SLAB = 32;

__global__ void __launch_bounds__(256) k_assign_nearest(const float* __restrict__ X, uint64_t nx,
                                                        const float* __restrict__ C, uint32_t k, uint32_t dim,
                                                        uint32_t* __restrict__ best_out) {
    __shared__ __align__(16) float Xs[AS_SLAB][AS_TILE + 4];
    __shared__ __align__(16) float Cs[AS_SLAB][AS_TILE + 4];
    const uint32_t tid = threadIdx.x, tx = tid & 15u, ty = tid >> 4;
    const uint64_t x0 = (uint64_t)blockIdx.x * AS_TILE;
    uint64_t best[4] = {~0ull, ~0ull, ~0ull, ~0ull};
    for (uint32_t c0 = 0; c0 < k; c0 += AS_TILE) {
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) acc[a][b] = 0.0f;
        for (uint32_t d0 = 0; d0 < dim; d0 += AS_SLAB) {
            const uint32_t dn = min((uint32_t)AS_SLAB, dim - d0);
            for (uint32_t e = tid; e < AS_SLAB * AS_TILE; e += 256) {
                uint32_t row = e / AS_SLAB, dd = e % AS_SLAB;
                float xv = 0.0f, cv = 0.0f;
                if (dd < dn) {
                    if (x0 + row < nx) xv = X[(x0 + row) * dim + d0 + dd];
                    if (c0 + row < k) cv = C[(uint64_t)(c0 + row) * dim + d0 + dd];
                }
                Xs[dd][row] = xv;
                Cs[dd][row] = cv;
            }
            __syncthreads();
            for (uint32_t dd = 0; dd < dn; dd++) {
                float4 xv = *reinterpret_cast<const float4*>(&Xs[dd][ty * 4]);
                float4 cv = *reinterpret_cast<const float4*>(&Cs[dd][tx * 4]);
                float xa[4] = {xv.x, xv.y, xv.z, xv.w};
                float ca[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                for (int a = 0; a < 4; a++)
#pragma unroll
                    for (int b = 0; b < 4; b++) acc[a][b] = sq_step(acc[a][b], xa[a], ca[b]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) {
                uint32_t c = c0 + tx * 4 + b;
                if (c < k) {
                    uint64_t key = argmin_key(acc[a][b], c);
                    if (key < best[a]) best[a] = key;
                }
            }
    }
    // reduce over the 16 threads (tx) that share a point row (half-warp)
#pragma unroll
    for (int a = 0; a < 4; a++) {
        uint64_t v = best[a];
        for (int o = 8; o > 0; o >>= 1) {
            uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
            v = w < v ? w : v;
        }
        uint64_t p = x0 + ty * 4 + a;
        if (tx == 0 && p < nx) best_out[p] = (v == ~0ull) ? 0u : (uint32_t)v;
    }
}

// One warp per point.
constexpr int ENC_WARPS = 8;

__global__ void __launch_bounds__(ENC_WARPS * 32) k_encode(AddArgs a, const float* __restrict__ X, uint64_t nx,
                                                         const uint32_t* __restrict__ best_in, int clamp,
                                                         uint32_t* __restrict__ cell_out,
                                                         float* __restrict__ lam_out, uint8_t* __restrict__ codes_out,
                                                         uint8_t* __restrict__ lamb_out,
                                                         float* __restrict__ eterm_out,
                                                         unsigned int* __restrict__ emax_bits,
                                                         float* __restrict__ resid_out) {
    extern __shared__ float sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t dim = a.dim, n = a.n, m = a.m, dsub = dim / m;
    float* xs = sm + (size_t)warp * (2 * dim + n + 1 + 32);
    float* rs = xs + dim;
    float* dist = rs + dim;  // n+1: [0] = a (own centroid), [1+j] = neighbour j
    const uint64_t pt = (uint64_t)blockIdx.x * ENC_WARPS + warp;
    if (pt >= nx) return;
    for (uint32_t d = lane; d < dim; d += 32) xs[d] = X[pt * dim + d];
    const uint32_t best = best_in[pt];
    __syncwarp();
    // exact distances to the centroid and its n neighbours (sqdist in order)
    for (uint32_t t = lane; t <= n; t += 32) {
        uint32_t c = (t == 0) ? best : a.nbr[(uint64_t)best * n + (t - 1)];
        const float* cp = a.centroids + (uint64_t)c * dim;
        float acc = 0.0f;
        for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, xs[d], __ldg(cp + d));
        dist[t] = acc;
    }
    __syncwarp();
    // assign_edge (line_quant.cpp:24-49): sequential, strict '<' after the first
    uint32_t best_j = 0;
    float best_lam = 0.0f;
    if (lane == 0) {
        const float av = dist[0];
        bool have = false;
        float best_sq = 0.0f;
        for (uint32_t j = 0; j < n; j++) {
            const float bv = dist[1 + j];
            const float cv = a.elen[(uint64_t)best * n + j];
            if (!(cv > 0.0f)) atomicOr(a.error_flag, 1u);
            float lam = line_lambda(av, bv, cv);
            if (clamp) lam = clamp_std(lam, 0.0f, 1.0f);
            const float dd = line_sqdist(av, bv, cv, lam);
            if (!have || dd < best_sq) {
                have = true;
                best_j = j;
                best_lam = lam;
                best_sq = dd;
            }
        }
    }
    best_j = __shfl_sync(0xffffffffu, best_j, 0);
    best_lam = __shfl_sync(0xffffffffu, best_lam, 0);
    const uint32_t cell = best * n + best_j;
    if (!codes_out && !resid_out) {  // observe_lambda_range pre-pass: lambda only
        if (lane == 0) lam_out[pt] = best_lam;
        return;
    }
    // residual at the exact lambda (index.cpp:181-184; training
    // displacements, bindings.cpp:59-71)
    const float* ci = a.centroids + (uint64_t)best * dim;
    const float* sj = a.centroids + (uint64_t)a.nbr[cell] * dim;
    const float oml = __fsub_rn(1.0f, best_lam);
    for (uint32_t d = lane; d < dim; d += 32) {
        rs[d] = __fsub_rn(xs[d], __fadd_rn(__fmul_rn(oml, ci[d]), __fmul_rn(best_lam, sj[d])));
        if (resid_out) resid_out[pt * dim + d] = rs[d];
    }
    __syncwarp();
    if (!codes_out) return;
    // pq_encode (pq.cpp:52-67): per sub-space argmin over 256 sub-centroids
    uint8_t* code = codes_out + pt * m;
    for (uint32_t p = 0; p < m; p++) {
        uint64_t bk = ~0ull;
        for (uint32_t j = lane; j < VLQ_KSUB; j += 32) {
            const float* sc = a.pq + ((uint64_t)p * VLQ_KSUB + j) * dsub;
            float acc = 0.0f;
            for (uint32_t t = 0; t < dsub; t++) acc = sq_step(acc, rs[p * dsub + t], __ldg(sc + t));
            uint64_t key = argmin_key(acc, j);
            bk = key < bk ? key : bk;
        }
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t w = __shfl_xor_sync(0xffffffffu, bk, o);
            bk = w < bk ? w : bk;
        }
        const uint32_t cj = (bk == ~0ull) ? 0u : (uint32_t)bk;
        if (lane == 0) code[p] = (uint8_t)cj;  // re-read by lane 0 below (same thread)
    }
    __syncwarp();
    if (lane == 0) {
        const uint32_t lb = quantize_lambda(best_lam, a.lo, a.hi);
        lamb_out[pt] = (uint8_t)lb;
        cell_out[pt] = cell;
        if (lam_out) lam_out[pt] = best_lam;
        // query-independent part of adc_distance (search.cpp:101-119) at the
        // dequantized lambda the scan will use
        const float lh = dequantize_lambda(lb, a.lo, a.hi);
        const uint32_t s = a.nbr[cell];
        const float* t3i = a.t3 + (uint64_t)best * m * VLQ_KSUB;
        const float* t3s = a.t3 + (uint64_t)s * m * VLQ_KSUB;
        float s2 = 0.0f, s3 = 0.0f, s4 = 0.0f;
        for (uint32_t p = 0; p < m; p++) {
            const uint32_t c = code[p];
            s2 = __fadd_rn(s2, a.t2[p * VLQ_KSUB + c]);
            s3 = __fadd_rn(s3, t3i[p * VLQ_KSUB + c]);
            s4 = __fadd_rn(s4, t3s[p * VLQ_KSUB + c]);
        }
        const float p3 = __fmul_rn(__fmul_rn(2.0f, __fsub_rn(1.0f, lh)), s3);
        const float p4 = __fmul_rn(__fmul_rn(2.0f, lh), s4);
        eterm_out[pt] = __fadd_rn(__fadd_rn(s2, p3), p4);
        const float mag = fabsf(s2) + fabsf(p3) + fabsf(p4);
        atomicMax(emax_bits, __float_as_uint(mag));
    }
}

__global__ void k_minmax(const float* __restrict__ v, uint64_t n, float* out2) {
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        mn = fminf(mn, v[i]);
        mx = fmaxf(mx, v[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // order-preserving u32 so integer atomics implement float min/max
        atomicMin(reinterpret_cast<unsigned int*>(out2), ord_float(mn));
        atomicMax(reinterpret_cast<unsigned int*>(out2) + 1, ord_float(mx));
    }
}

__global__ void k_histogram(const uint32_t* __restrict__ cells, uint64_t n, unsigned long long* counts) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[cells[i]], 1ull);
}

__global__ void k_gather_entries(const uint32_t* __restrict__ order, uint64_t n, uint32_t m, uint64_t first_id,
                                 const uint8_t* __restrict__ codes_pt, const uint8_t* __restrict__ lamb_pt,
                                 const float* __restrict__ eterm_pt, uint32_t* __restrict__ ids,
                                 uint8_t* __restrict__ codes, uint8_t* __restrict__ lambdas,
                                 float* __restrict__ eterm) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = order[t];
        ids[t] = (uint32_t)(first_id + p);
        lambdas[t] = lamb_pt[p];
        eterm[t] = eterm_pt[p];
        for (uint32_t b = 0; b < m; b++) codes[t * m + b] = codes_pt[(uint64_t)p * m + b];
    }
}

}  // namespace dev

void launch_tables(const float* centroids, uint32_t k, uint32_t dim, const float* pq, uint32_t m, float* t2,
                   float* t3, cudaStream_t st) {
    dev::k_tables<<<k + 1, 256, 0, st>>>(centroids, k, dim, pq, m, t2, t3);
    CUDA_LAUNCH_CHECK();
}

void launch_assign_nearest(const AddArgs& a, const float* X, uint64_t nx, uint32_t* best, cudaStream_t st) {
    if (nx == 0) return;
    dev::k_assign_nearest<<<(unsigned)((nx + dev::AS_TILE - 1) / dev::AS_TILE), 256, 0, st>>>(X, nx, a.centroids, a.k,
                                                                                             a.dim, best);
    CUDA_LAUNCH_CHECK();
}

void launch_encode(const AddArgs& a, const float* X, uint64_t nx, const uint32_t* best, int clamp_for_edges,
                   uint32_t* cell_out, float* lam_out, uint8_t* codes_out, uint8_t* lamb_out, float* eterm_out,
                   unsigned int* emax_bits, cudaStream_t st, float* resid_out) {
    if (nx == 0) return;
    size_t smem = (size_t)dev::ENC_WARPS * (2 * a.dim + a.n + 1 + 32) * sizeof(float);
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_encode<<<(unsigned)((nx + dev::ENC_WARPS - 1) / dev::ENC_WARPS), dev::ENC_WARPS * 32, smem, st>>>(
        a, X, nx, best, clamp_for_edges, cell_out, lam_out, codes_out, lamb_out, eterm_out, emax_bits, resid_out);
    CUDA_LAUNCH_CHECK();
}

void launch_minmax(const float* v, uint64_t n, float* out2, cudaStream_t st) {
    dev::k_minmax<<<296, 256, 0, st>>>(v, n, out2);
    CUDA_LAUNCH_CHECK();
}

void launch_histogram(const uint32_t* cells, uint64_t n, unsigned long long* counts, cudaStream_t st) {
    if (n == 0) return;
    dev::k_histogram<<<592, 256, 0, st>>>(cells, n, counts);
    CUDA_LAUNCH_CHECK();
}

void launch_gather_entries(const uint32_t* order, uint64_t n, uint32_t m, uint64_t first_id, const uint8_t* codes_pt,
                           const uint8_t* lamb_pt, const float* eterm_pt, uint32_t* ids, uint8_t* codes,
                           uint8_t* lambdas, float* eterm, cudaStream_t st) {
    if (n == 0) return;
    dev::k_gather_entries<<<1184, 256, 0, st>>>(order, n, m, first_id, codes_pt, lamb_pt, eterm_pt, ids, codes,
                                                lambdas, eterm);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq

// ---------------------------------------------------------------------------
// e-term of already-bucketed entries (index loaded from a VLQ1 file).
// ---------------------------------------------------------------------------
namespace vlq {
namespace dev {

__global__ void k_eterm_lists(AddArgs a, const uint64_t* __restrict__ off, uint32_t ncell,
                              const uint8_t* __restrict__ codes, const uint8_t* __restrict__ lambdas, uint64_t nent,
                              float* __restrict__ eterm, unsigned int* __restrict__ emax_bits) {
    const uint32_t m = a.m;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nent; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = ncell;  // off[lo] <= e < off[hi]
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (off[mid] <= e) lo = mid;
            else hi = mid;
        }
        const uint32_t cell = lo, i = cell / a.n, s = a.nbr[cell];
        const float lh = dequantize_lambda(lambdas[e], a.lo, a.hi);
        const float* t3i = a.t3 + (uint64_t)i * m * VLQ_KSUB;
        const float* t3s = a.t3 + (uint64_t)s * m * VLQ_KSUB;
        float s2 = 0.0f, s3 = 0.0f, s4 = 0.0f;
        for (uint32_t p = 0; p < m; p++) {
            const uint32_t c = codes[e * m + p];
            s2 = __fadd_rn(s2, a.t2[p * VLQ_KSUB + c]);
            s3 = __fadd_rn(s3, t3i[p * VLQ_KSUB + c]);
            s4 = __fadd_rn(s4, t3s[p * VLQ_KSUB + c]);
        }
        const float p3 = __fmul_rn(__fmul_rn(2.0f, __fsub_rn(1.0f, lh)), s3);
        const float p4 = __fmul_rn(__fmul_rn(2.0f, lh), s4);
        eterm[e] = __fadd_rn(__fadd_rn(s2, p3), p4);
        atomicMax(emax_bits, __float_as_uint(fabsf(s2) + fabsf(p3) + fabsf(p4)));
    }
}

}  // namespace dev

void launch_eterm_lists(const AddArgs& a, const uint64_t* list_off, uint32_t ncell, const uint8_t* codes,
                        const uint8_t* lambdas, uint64_t nent, float* eterm, unsigned int* emax_bits, cudaStream_t st) {
    if (nent == 0) return;
    dev::k_eterm_lists<<<(unsigned)dev::umin64((nent + 255) / 256, 4736), 256, 0, st>>>(
        a, list_off, ncell, codes, lambdas, nent, eterm, emax_bits);
    CUDA_LAUNCH_CHECK();
}


namespace dev {

// key = cell << 40 | the entry's first 5 code bytes (m >= 5; fewer bytes for
// smaller m), value = canonical position; one warp per cell
__global__ void k_scan_order_keys(const uint64_t* __restrict__ list_off, uint32_t ncell, const uint8_t* __restrict__ codes,
                                  uint32_t m, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t c = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < ncell; c += nw) {
        const uint64_t b0 = list_off[c], b1 = list_off[c + 1];
        for (uint64_t e = b0 + lane; e < b1; e += 32) {
            uint64_t key = c << 40;
            const uint32_t nb = m < 5 ? m : 5;
            for (uint32_t b = 0; b < nb; b++) key |= (uint64_t)codes[e * m + b] << (32 - 8 * b);
            keys[e] = key;
            vals[e] = (uint32_t)e;
        }
    }
}

__global__ void k_gather_scan_order(const uint32_t* __restrict__ order, uint64_t n, uint32_t m,
                                    const uint8_t* __restrict__ codes, const uint32_t* __restrict__ ids,
                                    const uint32_t* __restrict__ eterm_lam, uint8_t* __restrict__ scodes,
                                    uint32_t* __restrict__ sids, uint32_t* __restrict__ seterm_lam) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = order[i];
        if (m == 16) {
            reinterpret_cast<uint4*>(scodes)[i] = reinterpret_cast<const uint4*>(codes)[o];
        } else if (m == 8) {
            reinterpret_cast<uint2*>(scodes)[i] = reinterpret_cast<const uint2*>(codes)[o];
        } else {
            for (uint32_t b = 0; b < m; b++) scodes[i * m + b] = codes[o * m + b];
        }
        sids[i] = ids[o];
        seterm_lam[i] = eterm_lam[o];
    }
}

// Co-occurrence of code values inside the fast scan's warp blocks (32
// consecutive entries of a list from its start, one per lane), sampled every
// `stride`-th list: cooc[p][a][b] (a < b) counts the blocks in which sub-space
// p's codes a and b both occur, cooc[p][a][a] the blocks holding a.  One warp
// per block; distinct values by __match_any_sync.
__global__ void k_code_cooc(const uint64_t* __restrict__ list_off, uint32_t ncell, uint32_t stride,
                            const uint8_t* __restrict__ codes, uint32_t m, unsigned int* __restrict__ cooc) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t c = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * stride; c < ncell;
         c += nw * stride) {
        const uint64_t b0 = list_off[c], b1 = list_off[c + 1];
        for (uint64_t e0 = b0; e0 < b1; e0 += 32) {
            const uint64_t e = e0 + lane;
            const bool on = e < b1;
            const unsigned act = __ballot_sync(0xffffffffu, on);
            for (uint32_t p = 0; p < m; p++) {
                const uint32_t v = on ? codes[e * m + p] : 256u + lane;
                const unsigned peers = __match_any_sync(0xffffffffu, v);
                const bool lead = on && (__ffs(peers) - 1) == (int)lane;
                const unsigned leaders = __ballot_sync(0xffffffffu, lead) & act;
                unsigned int* cp = cooc + (uint64_t)p * 65536u;
                if (lead) atomicAdd(cp + v * 256u + v, 1u);
                for (unsigned rest = leaders; rest; rest &= rest - 1) {  // warp-uniform loop
                    const int j = __ffs(rest) - 1;
                    const uint32_t o = __shfl_sync(0xffffffffu, v, j);
                    if (lead && j > (int)lane) atomicAdd(cp + min(v, o) * 256u + max(v, o), 1u);
                }
            }
        }
    }
}

// codes[e][p] <- perm[p][codes[e][p]] (the scan copy's code relabeling)
__global__ void k_relabel_codes(uint8_t* __restrict__ codes, uint64_t n, uint32_t m, const uint8_t* __restrict__ perm) {
    __shared__ uint8_t tab[16 * 256];
    for (uint32_t i = threadIdx.x; i < m * 256u; i += blockDim.x) tab[i] = perm[i];
    __syncthreads();
    const uint64_t total = n * m;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        codes[i] = tab[(uint32_t)(i % m) * 256u + codes[i]];
}

}  // namespace dev

void launch_code_cooc(const uint64_t* list_off, uint32_t ncell, uint32_t stride, const uint8_t* codes, uint32_t m,
                      unsigned int* cooc, cudaStream_t st) {
    if (ncell == 0) return;
    dev::k_code_cooc<<<4736, 256, 0, st>>>(list_off, ncell, stride, codes, m, cooc);
    CUDA_LAUNCH_CHECK();
}

void launch_relabel_codes(uint8_t* codes, uint64_t n, uint32_t m, const uint8_t* perm, cudaStream_t st) {
    if (n == 0) return;
    dev::k_relabel_codes<<<(unsigned)dev::umin64((n * m + 255) / 256, 4736 * 4), 256, 0, st>>>(codes, n, m, perm);
    CUDA_LAUNCH_CHECK();
}

void launch_scan_order_keys(const uint64_t* list_off, uint32_t ncell, const uint8_t* codes, uint32_t m, uint64_t n,
                            uint64_t* keys, uint32_t* vals, cudaStream_t st) {
    if (n == 0) return;
    dev::k_scan_order_keys<<<4736, 256, 0, st>>>(list_off, ncell, codes, m, keys, vals);
    CUDA_LAUNCH_CHECK();
}

void launch_gather_scan_order(const uint32_t* order, uint64_t n, uint32_t m, const uint8_t* codes, const uint32_t* ids,
                              const uint32_t* eterm_lam, uint8_t* scodes, uint32_t* sids, uint32_t* seterm_lam,
                              cudaStream_t st) {
    if (n == 0) return;
    dev::k_gather_scan_order<<<(unsigned)dev::umin64((n + 255) / 256, 4736 * 4), 256, 0, st>>>(order, n, m, codes, ids,
                                                                                              eterm_lam, scodes, sids,
                                                                                              seterm_lam);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq
