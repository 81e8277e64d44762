// Search-path kernels (Algorithm 3 of the paper; reference
// proj/src/search.cpp:11-191).
//
//   k_sqdist_matrix     exact centroid distances (first_level_scan :11-36)
//   k_first_level       top-w1 by (dist, id)
//   k_second_level      line-subregion distances + top-w2 by (dist, cell)
//                       (second_level_rank :38-78, line_quant.cpp:9-22)
//   k_term5             t5 = <y_p, PQ[p][j]> (query_term5 :80-90)
//   k_scan<...>         fused list scan + warp top-k' (adc_distance :92-120,
//                       scan loop :154-162, select_topk :122-140)
//   k_rescore           exact reference-order re-score of the k' survivors,
//                       final (dist, id) top-k and the certificate that the
//                       exact top-k is among them
#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

// ---------------------------------------------------------------------------
// Exact squared-distance matrix  out[q*ldo + c] = sqdist(Y[q], C[c]).
// 64x64 output tile per CTA, 4x4 per thread, D streamed through shared
// memory in 32-wide slabs.  Each output accumulates d = 0..D-1 in order with
// __f*_rn, so it is bit-identical to the sequential reference sqdist.
// ---------------------------------------------------------------------------
constexpr int SQ_TILE = 64;
constexpr int SQ_SLAB = 32;

__global__ void __launch_bounds__(256) k_sqdist_matrix(const float* __restrict__ Y, uint64_t ny,
                                                       const float* __restrict__ C, uint64_t nc,
                                                       uint32_t dim, float* __restrict__ out,
                                                       uint64_t ldo) {
    __shared__ __align__(16) float Ys[SQ_SLAB][SQ_TILE + 4];
    __shared__ __align__(16) float Cs[SQ_SLAB][SQ_TILE + 4];
    const uint32_t tid = threadIdx.x;
    const uint32_t tx = tid & 15u, ty = tid >> 4;
    const uint64_t q0 = (uint64_t)blockIdx.y * SQ_TILE, c0 = (uint64_t)blockIdx.x * SQ_TILE;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.0f;
    for (uint32_t d0 = 0; d0 < dim; d0 += SQ_SLAB) {
        const uint32_t dn = min((uint32_t)SQ_SLAB, dim - d0);
        for (uint32_t e = tid; e < SQ_SLAB * SQ_TILE; e += 256) {
            uint32_t row = e / SQ_SLAB, dd = e % SQ_SLAB;
            float yv = 0.0f, cv = 0.0f;
            if (dd < dn) {
                if (q0 + row < ny) yv = Y[(q0 + row) * dim + d0 + dd];
                if (c0 + row < nc) cv = C[(c0 + row) * dim + d0 + dd];
            }
            Ys[dd][row] = yv;
            Cs[dd][row] = cv;
        }
        __syncthreads();
        for (uint32_t dd = 0; dd < dn; dd++) {
            float4 yv = *reinterpret_cast<const float4*>(&Ys[dd][ty * 4]);
            float4 cv = *reinterpret_cast<const float4*>(&Cs[dd][tx * 4]);
            float ya[4] = {yv.x, yv.y, yv.z, yv.w};
            float ca[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = sq_step(acc[a][b], ya[a], ca[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        uint64_t q = q0 + ty * 4 + a;
        if (q >= ny) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            uint64_t c = c0 + tx * 4 + b;
            if (c < nc) out[q * ldo + c] = acc[a][b];
        }
    }
}

// ---------------------------------------------------------------------------
// First level: top-w1 centroids of each query's distance row, ascending ids.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_first_level(const float* __restrict__ ws, uint32_t k,
                                                     uint32_t w1, uint32_t* __restrict__ top) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t scan[40];
    const uint64_t q = blockIdx.x;
    block_select_ordered(ws + q * k, k, w1, top + q * w1, hist, scan);
}

// ---------------------------------------------------------------------------
// Second level: line-subregion distances of the w1*n edges, top-w2 by
// (dist, centroid_id, edge_rank).  `top` is ascending, so edge position
// r*n + j is ascending in cell id i*n + j and the positional tie-break of
// block_select_ordered is exactly the reference's.  Also produces, per query,
// the scanned-candidate count and the |term1| bound of the certificate.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_second_level(SearchArgs a, uint32_t w1, uint32_t w2) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t scan[40];
    __shared__ unsigned long long s_scanned;
    __shared__ float s_dmax;
    const uint64_t q = blockIdx.x;
    const uint32_t n = a.n;
    const uint32_t total = w1 * n;
    const float* wsq = a.ws + q * a.k;
    const uint32_t* topq = a.top + q * w1;
    float* dq = a.dbuf + q * (uint64_t)total;
    if (threadIdx.x == 0) {
        s_scanned = 0;
        s_dmax = 0.0f;
    }
    extern __shared__ float ys2[];  // query vector (tensor-core mode)
    if (a.Y) {
        for (uint32_t d = threadIdx.x; d < a.dim; d += blockDim.x) ys2[d] = a.Y[q * a.dim + d];
        __syncthreads();
    }
    for (uint32_t e = threadIdx.x; e < total; e += blockDim.x) {
        uint32_t i = topq[e / n], j = e % n;
        float av = wsq[i];
        const uint32_t s = a.nbr[(uint64_t)i * n + j];
        float bv;
        if (a.Y) {  // ws[s] may be approximate: recompute exactly and publish it
            const float* cp = a.centroids + (uint64_t)s * a.dim;
            float acc = 0.0f;
            for (uint32_t d = 0; d < a.dim; d++) acc = sq_step(acc, ys2[d], cp[d]);
            bv = acc;
            const_cast<float*>(wsq)[s] = acc;
        } else {
            bv = wsq[s];
        }
        float cv = a.elen[(uint64_t)i * n + j];
        if (!(cv > 0.0f)) atomicOr(a.error_flag, 1u);  // line_quant.cpp:10-12
        float lam = clamp_std(line_lambda(av, bv, cv), 0.0f, 1.0f);
        dq[e] = line_sqdist(av, bv, cv, lam);
    }
    __syncthreads();
    uint32_t* selq = a.sel + q * w2;
    block_select_ordered(dq, total, w2, selq, hist, scan);
    __syncthreads();
    // positions -> cell ids; scanned count; |d| bound for the certificate
    const float lmax = a.lam_absmax;  // max |lambda| over dequantized values
    unsigned long long cnt = 0;
    float dmax = 0.0f;
    for (uint32_t t = threadIdx.x; t < w2; t += blockDim.x) {
        uint32_t e = selq[t];
        uint32_t i = topq[e / n], j = e % n;
        uint32_t cell = i * n + j;
        selq[t] = cell;
        cnt += a.list_off[cell + 1] - a.list_off[cell];
        float av = wsq[i], bv = wsq[a.nbr[cell]], cv = a.elen[cell];
        // |(1-l)a + (l^2-l)c + l b| <= (1+L)a + (L^2+L)c + L b for |l| <= L
        float bound = (1.0f + lmax) * fabsf(av) + (lmax * lmax + lmax) * fabsf(cv) + lmax * fabsf(bv);
        dmax = fmaxf(dmax, bound);
    }
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_scanned, cnt);
        atomicMax(reinterpret_cast<unsigned int*>(&s_dmax), __float_as_uint(dmax));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.meta[q].scanned = s_scanned;
        a.meta[q].dmax = s_dmax;
        a.meta[q].flag = 0;  // the fast scan may set 2 (candidate overflow)
    }
}

// ---------------------------------------------------------------------------
// Select-split multi-GPU schedule (dist.py): the rank that ran
// first_level_scan + second_level_rank for a query slice publishes, per
// selected cell, (a, b) = (ws[i], ws[nbr(cell)]) -- the only coarse values the
// later stages read -- and every shard engine applies the gathered selection:
// the cells into sel, a and b back into its ws rows, and the LOCAL scanned
// count and |term1| bound (exactly k_second_level's formulas) into meta.
// ---------------------------------------------------------------------------
__global__ void k_pack_selection(SearchArgs a, uint32_t w2, uint32_t* __restrict__ sel_out, float* __restrict__ ab) {
    const uint64_t q = blockIdx.x;
    const float* wsq = a.ws + q * a.k;
    for (uint32_t t = threadIdx.x; t < w2; t += blockDim.x) {
        const uint32_t cell = a.sel[q * w2 + t];
        sel_out[q * w2 + t] = cell;
        ab[(q * w2 + t) * 2] = wsq[cell / a.n];
        ab[(q * w2 + t) * 2 + 1] = wsq[a.nbr[cell]];
    }
}

__global__ void __launch_bounds__(256) k_apply_selection(SearchArgs a, uint32_t w2, SelParts parts, uint64_t q0) {
    __shared__ unsigned long long s_scanned;
    __shared__ float s_dmax;
    const uint64_t q = blockIdx.x;
    float* wsq = a.ws + q * a.k;
    // this query's row of the gathered selection: part (q0 + q) / per, possibly
    // on a peer GPU (read over NVLink)
    const uint64_t gq = q0 + q;
    const uint32_t part = parts.per ? (uint32_t)(gq / parts.per) : 0u;
    const uint64_t row = parts.per ? gq % parts.per : gq;
    const uint32_t* sel_in = parts.sel[part] + row * w2;
    const float* ab = parts.ab[part] + row * w2 * 2;
    if (threadIdx.x == 0) {
        s_scanned = 0;
        s_dmax = 0.0f;
    }
    __syncthreads();
    const float lmax = a.lam_absmax;
    unsigned long long cnt = 0;
    float dmax = 0.0f;
    for (uint32_t t = threadIdx.x; t < w2; t += blockDim.x) {
        const uint32_t cell = sel_in[t];
        a.sel[q * w2 + t] = cell;
        const float av = ab[t * 2], bv = ab[t * 2 + 1], cv = a.elen[cell];
        // equal values from every writer: both are the exact reference-order
        // distance to that centroid
        wsq[cell / a.n] = av;
        wsq[a.nbr[cell]] = bv;
        cnt += a.list_off[cell + 1] - a.list_off[cell];
        const float bound = (1.0f + lmax) * fabsf(av) + (lmax * lmax + lmax) * fabsf(cv) + lmax * fabsf(bv);
        dmax = fmaxf(dmax, bound);
    }
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_scanned, cnt);
        atomicMax(reinterpret_cast<unsigned int*>(&s_dmax), __float_as_uint(dmax));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.meta[q].scanned = s_scanned;
        a.meta[q].dmax = s_dmax;
        a.meta[q].flag = 0;
    }
}

// ---------------------------------------------------------------------------
// term5 table (query_term5): t5[q][p][j] = dot(y_p, PQ[p][j]) in order; also
// S5max = sum_p max_j |t5| for the certificate.
// ---------------------------------------------------------------------------
template <int DS>  // sub-space width when known at compile time (unrolled dot products), else 0
__global__ void __launch_bounds__(256) k_term5(float cert_slack, const float* __restrict__ Y, const float* __restrict__ pqT,
                                               uint32_t dim, uint32_t m, float* __restrict__ t5,
                                               QueryMeta* __restrict__ meta) {
    // thread j computes t5[p][j] for every sub-space p (sequential fp32 dot,
    // search.cpp:80-90 / vecset.cpp:39-45), reading the PQ codebook from its
    // transposed copy pqT[(p*dsub + t)*256 + j], so every load and every t5
    // store is warp-coalesced; S5max = sum_p max_j |t5[p][j]| for the
    // certificate.  blockDim.x == 256 (one thread per codeword).
    extern __shared__ float ys[];
    __shared__ float s_max[8 * 16];
    const uint64_t q = blockIdx.x;
    const uint32_t dsub = DS > 0 ? (uint32_t)DS : dim / m, j = threadIdx.x, lane = j & 31u, warp = j >> 5;
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) ys[d] = Y[q * dim + d];
    __syncthreads();
    float s5 = 0.0f;  // thread 0's running S5max
    for (uint32_t p0 = 0; p0 < m; p0 += 16) {  // sub-spaces in groups of 16 (register maxima)
        float mx[16];
#pragma unroll
        for (int pp = 0; pp < 16; pp++) {
            mx[pp] = 0.0f;
            const uint32_t p = p0 + pp;
            if (p < m) {
                const float* c = pqT + (uint64_t)p * dsub * VLQ_KSUB + j;
                const float* y = ys + p * dsub;
                float acc = 0.0f;
                if constexpr (DS > 0) {
                    float cv[DS];
#pragma unroll
                    for (int t = 0; t < DS; t++) cv[t] = __ldg(c + t * VLQ_KSUB);
#pragma unroll
                    for (int t = 0; t < DS; t++) acc = dot_step(acc, y[t], cv[t]);
                } else {
                    for (uint32_t t = 0; t < dsub; t++) acc = dot_step(acc, y[t], c[(uint64_t)t * VLQ_KSUB]);
                }
                t5[(q * m + p) * VLQ_KSUB + j] = acc;
                mx[pp] = fabsf(acc);
            }
        }
#pragma unroll
        for (int pp = 0; pp < 16; pp++) {
            if (p0 + pp < m) {
                float v = mx[pp];
                for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) s_max[warp * 16 + pp] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (uint32_t pp = 0; pp < 16 && p0 + pp < m; pp++) {
                float v = 0.0f;
                for (uint32_t w = 0; w < 8; w++) v = fmaxf(v, s_max[w * 16 + pp]);
                s5 += v;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        meta[q].s5max = s5;
        meta[q].qerr = cert_slack;  // 0 unless a test widens the certificate (engine knob cert_slack)
    }
}

// ---------------------------------------------------------------------------
// Fused list scan.  One CTA per query, warps take the query's selected
// cells round-robin, lanes take consecutive posting entries (coalesced code /
// lambda / e loads).  Per entry:
//   kFast:  dist = (term1 + e) - 2*sum5   with e = sum2 + 2(1-l)sum3 + 2l sum4
//           precomputed at add time (query independent); key = (dist, pos)
//   exact:  the reference's adc_distance op-for-op; key = (dist, id)
// Every warp keeps its kKeep smallest keys in a shared buffer (threshold
// insert + bitonic flush); warps share the best threshold seen so far (the
// min over warps of their kKeep-th key bounds the block's kKeep-th key).
// The warps' survivors are block-merged and the kKeep smallest written out.
// ---------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ void load_code(const uint8_t* __restrict__ codes, uint64_t e, uint32_t m,
                                          uint8_t* out) {
    if constexpr (M == 16) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(codes + e * 16));
        *reinterpret_cast<uint4*>(out) = v;
    } else if constexpr (M == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2*>(codes + e * 8));
        *reinterpret_cast<uint2*>(out) = v;
    } else if constexpr (M == 4) {
        uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(codes + e * 4));
        *reinterpret_cast<uint32_t*>(out) = v;
    } else {
        for (uint32_t p = 0; p < m; p++) out[p] = __ldg(codes + e * m + p);
    }
}

struct ScanShared {
    unsigned long long tau;  // shared threshold (min over warps)
};

template <int M, bool kFast>
__global__ void __launch_bounds__(256) k_scan(SearchArgs a, uint32_t w2, uint32_t keep, uint32_t buf,
                                              const uint32_t* __restrict__ qlist,
                                              const unsigned int* __restrict__ qcount) {
    extern __shared__ __align__(16) unsigned char smem[];

    const uint32_t _nb = qcount ? *qcount : gridDim.x;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint32_t m = (M > 0) ? (uint32_t)M : a.m;
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t q = qlist ? qlist[_b] : _b;
    float* lut = reinterpret_cast<float*>(smem);                        // m*256
    uint64_t* bufs = reinterpret_cast<uint64_t*>(smem + (size_t)m * VLQ_KSUB * 4);  // nwarps*buf
    __shared__ unsigned long long s_tau;
    uint64_t* wbuf = bufs + (size_t)warp * buf;

    const float* t5q = a.t5 + q * m * VLQ_KSUB;
    for (uint32_t i = threadIdx.x; i < m * VLQ_KSUB; i += blockDim.x) lut[i] = t5q[i];
    for (uint32_t i = threadIdx.x; i < nwarps * buf; i += blockDim.x) bufs[i] = ~0ull;
    if (threadIdx.x == 0) s_tau = ~0ull;
    __syncthreads();

    const float* wsq = a.ws + q * a.k;
    const uint32_t* selq = a.sel + q * w2;
    const float lo = a.lo, hi = a.hi;
    uint32_t cnt = 0;
    uint64_t tau = ~0ull;

    auto flush = [&]() {
        // sort the warp buffer, keep the `keep` smallest, update thresholds
        for (uint32_t i = cnt + lane; i < buf; i += 32) wbuf[i] = ~0ull;
        __syncwarp();
        bitonic_sort_u64<true>(wbuf, buf, lane, 32);
        cnt = min(cnt, keep);
        if (cnt == keep) {
            uint64_t t = wbuf[keep - 1];
            if (t < tau) tau = t;
            if (lane == 0) atomicMin(&s_tau, (unsigned long long)t);
        }
        __syncwarp();
    };

    for (uint32_t ci = warp; ci < w2; ci += nwarps) {
        const uint32_t cell = selq[ci];
        const uint64_t b0 = a.list_off[cell], b1 = a.list_off[cell + 1];
        if (b0 == b1) continue;
        const uint32_t i = cell / a.n;
        const uint32_t s = a.nbr[cell];
        const float av = wsq[i], bv = wsq[s], cv = a.elen[cell];
        const float* t3i = a.t3 + (uint64_t)i * m * VLQ_KSUB;
        const float* t3s = a.t3 + (uint64_t)s * m * VLQ_KSUB;
        for (uint64_t e0 = b0; e0 < b1; e0 += 32) {
            const uint64_t e = e0 + lane;
            uint64_t key = ~0ull;
            if (e < b1) {
                uint8_t code[(M > 0) ? M : 128];
                load_code<M>(a.codes, e, m, code);
                const uint32_t lb = __ldg(a.lambdas + e);
                const float lam = dequantize_lambda(lb, lo, hi);
                const float d = line_sqdist(av, bv, cv, lam);
                if constexpr (kFast) {
                    float sum5 = 0.0f;
#pragma unroll
                    for (uint32_t p = 0; p < ((M > 0) ? (uint32_t)M : m); p++)
                        sum5 = __fadd_rn(sum5, lut[p * VLQ_KSUB + code[p]]);
                    const float et = __ldg(a.eterm + e);
                    const float dist = __fsub_rn(__fadd_rn(d, et), __fmul_rn(2.0f, sum5));
                    key = make_key(dist, (uint32_t)e);
                } else {
                    float s2 = 0.0f, s3 = 0.0f, s4 = 0.0f, s5 = 0.0f;
                    for (uint32_t p = 0; p < m; p++) {
                        const uint32_t c = code[p];
                        s2 = __fadd_rn(s2, __ldg(a.t2 + p * VLQ_KSUB + c));
                        s3 = __fadd_rn(s3, __ldg(t3i + p * VLQ_KSUB + c));
                        s4 = __fadd_rn(s4, __ldg(t3s + p * VLQ_KSUB + c));
                        s5 = __fadd_rn(s5, lut[p * VLQ_KSUB + c]);
                    }
                    float r = __fadd_rn(d, s2);
                    r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, __fsub_rn(1.0f, lam)), s3));
                    r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, lam), s4));
                    r = __fsub_rn(r, __fmul_rn(2.0f, s5));
                    key = make_key(r, __ldg(a.ids + e));
                }
            }
            const uint64_t shared_tau = *reinterpret_cast<volatile unsigned long long*>(&s_tau);
            const uint64_t th = tau < shared_tau ? tau : shared_tau;
            const bool take = key < th;
            const uint32_t bal = __ballot_sync(0xffffffffu, take);
            if (bal) {
                if (take) wbuf[cnt + __popc(bal & ((1u << lane) - 1u))] = key;
                cnt += __popc(bal);
                __syncwarp();
                if (cnt > buf - 32) flush();
            }
        }
    }
    flush();
    __syncthreads();
    // block merge: every warp buffer now holds its sorted survivors then +inf
    const uint32_t total = nwarps * buf;
    bitonic_sort_u64<false>(bufs, total, threadIdx.x, blockDim.x);
    uint64_t* candq = a.cand + q * keep;
    for (uint32_t t = threadIdx.x; t < keep; t += blockDim.x) candq[t] = bufs[t];
    __syncthreads();  // shared memory is reused by the next query
    }
}

// ---------------------------------------------------------------------------
// Exact re-score of the fast-scan survivors (adc_distance op-for-op on the
// global t2/t3/t5 tables), final (dist, id) top-k, padding, and the
// certificate: with eps bounding |fast - exact| for every scanned entry,
// fast_k' - eps > exact_k proves that no dropped entry can enter the top-k.
// ---------------------------------------------------------------------------

// Exact re-score of the k' fast-scan survivors.  The survivor's cell is found
// by a binary search over the query's OWN selected cells' list starts (staged
// in shared memory: ~9 steps) instead of all K n list offsets in global memory
// (~21 dependent loads), and for m in {4, 8, 16} the 4 m table gathers of a
// survivor are unrolled so they are all in flight at once; the sums keep the
// reference's sequential order (adc_distance, search.cpp:92-120).
template <int M>
__global__ void __launch_bounds__(256) k_rescore(SearchArgs a, uint32_t w2, uint32_t keep, uint32_t topk,
                                                 int64_t* __restrict__ out_ids, float* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);  // keep (power of two)
    uint64_t* cstart = keys + keep;                        // w2: list start of selected cell t
    uint32_t* ccell = reinterpret_cast<uint32_t*>(cstart + w2);
    __shared__ float s_fast_last;
    __shared__ uint8_t s_inv[16 * VLQ_KSUB];  // code_inv (relabeled scan codes -> canonical codes)
    if (a.code_inv)
        for (uint32_t i = threadIdx.x; i < a.m * VLQ_KSUB; i += blockDim.x) s_inv[i] = a.code_inv[i];
    __syncthreads();

    const uint32_t _nb = a.qlist ? *a.qcount : gridDim.x;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint64_t q = a.qlist ? a.qlist[_b] : _b;
    const uint32_t m = M > 0 ? (uint32_t)M : a.m;
    const uint64_t* candq = a.cand + (a.qlist ? (uint64_t)_b : q) * keep;
    const float* wsq = a.ws + q * a.k;
    const float* t5q = a.t5 + q * m * VLQ_KSUB;
    const uint64_t scanned = a.meta[q].scanned;
    const uint32_t have = (uint32_t)dev::umin64(scanned, keep);
    const uint32_t* selq = a.sel + q * w2;
    for (uint32_t t = threadIdx.x; t < w2; t += blockDim.x) {
        const uint32_t c = selq[t];  // ascending cell ids, so ascending list starts
        ccell[t] = c;
        cstart[t] = a.list_off[c];
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < keep; t += blockDim.x) {
        uint64_t key = ~0ull;
        if (t < have) {
            const uint64_t ck = candq[t];
            const uint64_t pos = (uint32_t)ck;
            uint32_t lo = 0, hi = w2;  // the last selected cell whose list starts at or before pos
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (cstart[mid] <= pos) lo = mid;
                else hi = mid;
            }
            const uint32_t cell = ccell[lo];
            const uint32_t i = cell / a.n;
            const uint32_t s = a.nbr[cell];
            // reordered scan copy: the lambda byte is the packed word's low byte, the id in sids
            const uint32_t lbyte = a.scodes ? (a.eterm_lam[pos] & 0xffu) : (uint32_t)a.lambdas[pos];
            const float lam = dequantize_lambda(lbyte, a.lo, a.hi);
            const float d = line_sqdist(wsq[i], wsq[s], a.elen[cell], lam);
            const float* t3i = a.t3 + (uint64_t)i * m * VLQ_KSUB;
            const float* t3s = a.t3 + (uint64_t)s * m * VLQ_KSUB;
            float s2 = 0.0f, s3 = 0.0f, s4 = 0.0f, s5 = 0.0f;
            const uint8_t* codes = a.scodes ? a.scodes : a.codes;
            if constexpr (M > 0) {
                uint8_t code[M];
                if constexpr (M == 16) *reinterpret_cast<uint4*>(code) = __ldg(reinterpret_cast<const uint4*>(codes + pos * 16));
                else if constexpr (M == 8) *reinterpret_cast<uint2*>(code) = __ldg(reinterpret_cast<const uint2*>(codes + pos * 8));
                else *reinterpret_cast<uint32_t*>(code) = __ldg(reinterpret_cast<const uint32_t*>(codes + pos * 4));
                float v2[M], v3[M], v4[M], v5[M];
#pragma unroll
                for (int p = 0; p < M; p++) {  // every gather in flight at once
                    const uint32_t c = a.code_inv ? s_inv[p * VLQ_KSUB + code[p]] : code[p];
                    v2[p] = __ldg(a.t2 + p * VLQ_KSUB + c);
                    v3[p] = __ldg(t3i + p * VLQ_KSUB + c);
                    v4[p] = __ldg(t3s + p * VLQ_KSUB + c);
                    v5[p] = t5q[p * VLQ_KSUB + c];
                }
#pragma unroll
                for (int p = 0; p < M; p++) {
                    s2 = __fadd_rn(s2, v2[p]);
                    s3 = __fadd_rn(s3, v3[p]);
                    s4 = __fadd_rn(s4, v4[p]);
                    s5 = __fadd_rn(s5, v5[p]);
                }
            } else {
                const uint8_t* code = codes + pos * m;
                for (uint32_t p = 0; p < m; p++) {
                    const uint32_t c = a.code_inv ? s_inv[p * VLQ_KSUB + code[p]] : code[p];
                    s2 = __fadd_rn(s2, a.t2[p * VLQ_KSUB + c]);
                    s3 = __fadd_rn(s3, t3i[p * VLQ_KSUB + c]);
                    s4 = __fadd_rn(s4, t3s[p * VLQ_KSUB + c]);
                    s5 = __fadd_rn(s5, t5q[p * VLQ_KSUB + c]);
                }
            }
            float r = __fadd_rn(d, s2);
            r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, __fsub_rn(1.0f, lam)), s3));
            r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, lam), s4));
            r = __fsub_rn(r, __fmul_rn(2.0f, s5));
            key = make_key(r, a.scodes ? a.sids[pos] : a.ids[pos]);
            if (t == have - 1) s_fast_last = unord_float((uint32_t)(ck >> 32));
        }
        keys[t] = key;
    }
    __syncthreads();
    bitonic_sort_u64<false>(keys, keep, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        if (t < have) {
            out_ids[q * topk + t] = (int64_t)(uint32_t)keys[t];
            out_d[q * topk + t] = unord_float((uint32_t)(keys[t] >> 32));
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
    if (threadIdx.x == 0) {
        uint32_t flag = a.meta[q].flag == 2 ? 1u : 0u;
        if (!flag && scanned > keep && topk > 0) {
            // every scanned entry x satisfies |fast_x - exact_x| <= eps
            const QueryMeta mt = a.meta[q];
            const double u = 5.9604644775390625e-08;  // 2^-24
            // |term1_fast - term1_exact| <= 19u*Dmax (FFMA lambda/term1 vs the
            // reference op order), the reassociated e-sum 8u*(Dmax+Emax), the
            // final subtraction 4u*S5max; 1.25x margin
            const double eps = 1.25 * u * (27.0 * (double)mt.dmax + 8.0 * (double)a.emax + 4.0 * (double)mt.s5max) +
                               1.25 * (double)a.e_pack_err + (double)mt.qerr + 1e-30;
            const double exact_k = (double)unord_float((uint32_t)(keys[topk - 1] >> 32));
            const double fast_last = (double)s_fast_last;
            if (!(fast_last - eps > exact_k)) flag = 1;
        }
        a.meta[q].flag = flag;
    }
    __syncthreads();  // shared memory is reused by the next query
    }
}

}  // namespace dev
}  // namespace vlq

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
namespace vlq {

void launch_sqdist_matrix(const float* Y, uint64_t ny, const float* C, uint64_t nc, uint32_t dim, float* out,
                          uint64_t ldo, cudaStream_t st) {
    if (ny == 0 || nc == 0) return;
    dim3 grid((unsigned)((nc + dev::SQ_TILE - 1) / dev::SQ_TILE), (unsigned)((ny + dev::SQ_TILE - 1) / dev::SQ_TILE));
    dev::k_sqdist_matrix<<<grid, 256, 0, st>>>(Y, ny, C, nc, dim, out, ldo);
    CUDA_LAUNCH_CHECK();
}

void launch_first_level(const float* ws, uint64_t nq, uint32_t k, uint32_t w1, uint32_t* top, cudaStream_t st) {
    dev::k_first_level<<<(unsigned)nq, 512, 0, st>>>(ws, k, w1, top);
    CUDA_LAUNCH_CHECK();
}

void launch_second_level(const SearchArgs& a, uint64_t nq, uint32_t w1, uint32_t w2, cudaStream_t st) {
    dev::k_second_level<<<(unsigned)nq, 512, a.Y ? a.dim * sizeof(float) : 0, st>>>(a, w1, w2);
    CUDA_LAUNCH_CHECK();
}

void launch_pack_selection(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t* sel_out, float* ab,
                           cudaStream_t st) {
    dev::k_pack_selection<<<(unsigned)nq, 256, 0, st>>>(a, w2, sel_out, ab);
    CUDA_LAUNCH_CHECK();
}

void launch_apply_selection(const SearchArgs& a, uint64_t nq, uint32_t w2, const uint32_t* sel_in, const float* ab,
                            cudaStream_t st) {
    SelParts p{};
    p.sel[0] = sel_in;
    p.ab[0] = ab;
    p.nparts = 1;
    p.per = 0;  // one part holding every row
    launch_apply_selection_parts(a, nq, w2, p, 0, st);
}

void launch_apply_selection_parts(const SearchArgs& a, uint64_t nq, uint32_t w2, const SelParts& p, uint64_t q0,
                                  cudaStream_t st) {
    if (nq == 0) return;
    dev::k_apply_selection<<<(unsigned)nq, 256, 0, st>>>(a, w2, p, q0);
    CUDA_LAUNCH_CHECK();
}

void launch_term5(float cert_slack, const float* Y, const float* pqT, uint32_t dim, uint32_t m, float* t5, QueryMeta* meta,
                  uint64_t nq, cudaStream_t st) {
    const uint32_t ds = dim / m;
    auto fn = ds == 4 ? dev::k_term5<4> : ds == 6 ? dev::k_term5<6> : ds == 8 ? dev::k_term5<8>
              : ds == 16 ? dev::k_term5<16> : dev::k_term5<0>;
    fn<<<(unsigned)nq, 256, dim * sizeof(float), st>>>(cert_slack, Y, pqT, dim, m, t5, meta);
    CUDA_LAUNCH_CHECK();
}

size_t scan_smem_bytes(uint32_t m, uint32_t nwarps, uint32_t buf) {
    return (size_t)m * VLQ_KSUB * 4 + (size_t)nwarps * buf * 8;
}

template <int M, bool kFast>
static void launch_scan_t(const SearchArgs& a, uint64_t nblocks, uint32_t w2, uint32_t keep, uint32_t buf,
                          uint32_t nwarps, const uint32_t* qlist, const unsigned int* qcount, cudaStream_t st) {
    size_t smem = scan_smem_bytes(a.m, nwarps, buf);
    auto fn = dev::k_scan<M, kFast>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<list_grid(nblocks, qcount != nullptr), nwarps * 32, smem, st>>>(a, w2, keep, buf, qlist, qcount);
    CUDA_LAUNCH_CHECK();
}

void launch_scan(const SearchArgs& a, uint64_t nblocks, uint32_t w2, uint32_t keep, uint32_t buf, uint32_t nwarps,
                 bool fast, const uint32_t* qlist, const unsigned int* qcount, cudaStream_t st) {
    if (fast) {
        switch (a.m) {
            case 16: launch_scan_t<16, true>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            case 8: launch_scan_t<8, true>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            case 4: launch_scan_t<4, true>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            default: launch_scan_t<0, true>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
        }
    } else {
        switch (a.m) {
            case 16: launch_scan_t<16, false>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            case 8: launch_scan_t<8, false>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            case 4: launch_scan_t<4, false>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
            default: launch_scan_t<0, false>(a, nblocks, w2, keep, buf, nwarps, qlist, qcount, st); break;
        }
    }
}

void launch_rescore(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, uint32_t topk, int64_t* out_ids,
                    float* out_d, cudaStream_t st) {
    const size_t smem = keep * sizeof(uint64_t) + (size_t)w2 * 12;
    auto fn = a.m == 16 ? dev::k_rescore<16> : a.m == 8 ? dev::k_rescore<8> : a.m == 4 ? dev::k_rescore<4>
                                                                                          : dev::k_rescore<0>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // one thread per survivor: 128-thread CTAs for k' <= 128 (twice the CTAs
    // resident, every thread gathering), 256 above
    const unsigned threads = keep <= 128 ? 128u : 256u;
    fn<<<list_grid(nq, a.qlist != nullptr && !a.qorder), threads, smem, st>>>(a, w2, keep, topk, out_ids, out_d);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq

// ---------------------------------------------------------------------------
// Exact-fallback emit and the cross-shard (dist, id) merge (K9).
// ---------------------------------------------------------------------------
namespace vlq {
namespace dev {

__global__ void k_emit_exact(SearchArgs a, const uint32_t* __restrict__ qlist, const unsigned int* __restrict__ qcount,
                             uint32_t keep, uint32_t topk, int64_t* __restrict__ out_ids, float* __restrict__ out_d) {

    const uint32_t _nb = qcount ? *qcount : gridDim.x;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint64_t q = qlist ? qlist[_b] : _b;
    const uint64_t have = dev::umin64(a.meta[q].scanned, keep);
    const uint64_t* candq = a.cand + q * keep;
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        if (t < have) {
            out_ids[q * topk + t] = (int64_t)(uint32_t)candq[t];
            out_d[q * topk + t] = unord_float((uint32_t)(candq[t] >> 32));
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
    __syncthreads();  // shared memory is reused by the next query
    }
}

// Merges nparts per-shard top-k rows (each ascending by (dist, id), padded
// with -1/+inf) into the global top-k under the same total order.
// K9 on sorted parts (every search output row is ascending by (dist, id),
// padded with -1 / +inf): the merged position of a part's r-th key is r plus
// the number of smaller keys in every other part (a binary search each;
// keys are unique since every id lives in exactly one shard).  No sort, two
// block barriers.
__global__ void __launch_bounds__(256) k_merge_sorted(TopkParts parts, uint64_t row0, uint32_t topk,
                                                      int64_t* __restrict__ out_ids, float* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t nparts = parts.nparts;
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);  // [nparts][topk]
    uint64_t* res = keys + (size_t)nparts * topk;         // [topk]
    const uint64_t q = blockIdx.x;
    const uint32_t total = nparts * topk;
    for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {  // parts may live on peer GPUs (P2P loads)
        const uint32_t part = t / topk, r = t % topk;
        const uint64_t src = (row0 + q) * topk + r;
        const int64_t id = parts.ids[part][src];
        keys[t] = id >= 0 ? make_key(parts.d[part][src], (uint32_t)id) : ~0ull;
    }
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) res[t] = ~0ull;
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint64_t key = keys[t];
        if (key == ~0ull) continue;
        const uint32_t part = t / topk;
        uint32_t pos = t % topk;
        for (uint32_t g = 0; g < nparts && pos < topk; g++) {
            if (g == part) continue;
            const uint64_t* row = keys + (size_t)g * topk;
            uint32_t lo = 0, hi = topk;  // count of keys < key in row g
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (row[mid] < key) lo = mid + 1;
                else hi = mid;
            }
            pos += lo;
        }
        if (pos < topk) res[pos] = key;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        const uint64_t key = res[t];
        if (key != ~0ull) {
            out_ids[q * topk + t] = (int64_t)(uint32_t)key;
            out_d[q * topk + t] = unord_float((uint32_t)(key >> 32));
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
}

__global__ void k_merge_topk(const int64_t* __restrict__ in_ids, const float* __restrict__ in_d, uint32_t nparts,
                             uint64_t nq, uint32_t topk, uint32_t npow2, int64_t* __restrict__ out_ids,
                             float* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    const uint64_t q = blockIdx.x;
    for (uint32_t t = threadIdx.x; t < npow2; t += blockDim.x) {
        uint64_t key = ~0ull;
        if (t < nparts * topk) {
            const uint32_t part = t / topk, r = t % topk;
            const uint64_t src = ((uint64_t)part * nq + q) * topk + r;
            const int64_t id = in_ids[src];
            if (id >= 0) key = make_key(in_d[src], (uint32_t)id);
        }
        keys[t] = key;
    }
    __syncthreads();
    bitonic_sort_u64<false>(keys, npow2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        const uint64_t key = keys[t];
        if (key != ~0ull) {
            out_ids[q * topk + t] = (int64_t)(uint32_t)key;
            out_d[q * topk + t] = unord_float((uint32_t)(key >> 32));
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
}

}  // namespace dev

void launch_emit_exact(const SearchArgs& a, const uint32_t* qlist, const unsigned int* qcount, uint64_t nblocks,
                       uint32_t keep, uint32_t topk, int64_t* out_ids, float* out_d, cudaStream_t st) {
    if (nblocks == 0) return;
    dev::k_emit_exact<<<list_grid(nblocks, qcount != nullptr), 128, 0, st>>>(a, qlist, qcount, keep, topk, out_ids,
                                                                         out_d);
    CUDA_LAUNCH_CHECK();
}

void launch_merge_topk_parts(const TopkParts& p, uint64_t row0, uint64_t nrows, uint32_t topk, int64_t* out_ids,
                             float* out_d, cudaStream_t st) {
    if (nrows == 0 || topk == 0) return;
    const size_t smem = ((size_t)p.nparts + 1) * topk * 8;
    if (smem > 200 * 1024) throw std::runtime_error("merge_topk: nparts * k too large");
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_merge_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_merge_sorted<<<(unsigned)nrows, 256, smem, st>>>(p, row0, topk, out_ids, out_d);
    CUDA_LAUNCH_CHECK();
}

void launch_merge_topk(const int64_t* in_ids, const float* in_d, uint32_t nparts, uint64_t nq, uint32_t topk,
                       int64_t* out_ids, float* out_d, cudaStream_t st) {
    if (nq == 0 || topk == 0) return;
    const size_t smem_sorted = ((size_t)nparts + 1) * topk * 8;
    if (smem_sorted <= 200 * 1024 && nparts <= VLQ_MAX_PARTS) {
        TopkParts p{};
        for (uint32_t g = 0; g < nparts; g++) {
            p.ids[g] = in_ids + (uint64_t)g * nq * topk;
            p.d[g] = in_d + (uint64_t)g * nq * topk;
        }
        p.nparts = nparts;
        launch_merge_topk_parts(p, 0, nq, topk, out_ids, out_d, st);
        return;
    }
    uint32_t n = 1;
    while (n < nparts * topk) n <<= 1;
    size_t smem = (size_t)n * 8;
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_merge_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_merge_topk<<<(unsigned)nq, 256, smem, st>>>(in_ids, in_d, nparts, nq, topk, n, out_ids, out_d);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq

// ---------------------------------------------------------------------------
// small helpers: flagged-query compaction and per-query scanned counts
// ---------------------------------------------------------------------------
namespace vlq {
namespace dev {

__global__ void k_compact_flags(const QueryMeta* __restrict__ meta, uint64_t nq, uint32_t* __restrict__ qlist,
                                unsigned int* __restrict__ count) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x)
        if (meta[q].flag) qlist[atomicAdd(count, 1u)] = (uint32_t)q;
}

// Longest-processing-time-first order of the tile's queries for the fast
// scan (one CTA per query, dispatched in block order as SM slots free up):
// queries bucketed by their scanned-entry count, largest first, so the batch
// does not end on a few long queries.  One block.
__global__ void __launch_bounds__(1024) k_lpt_order(const QueryMeta* __restrict__ meta, uint32_t nq,
                                                    uint32_t* __restrict__ order, unsigned int* __restrict__ count) {
    constexpr uint32_t NB = 256;
    __shared__ unsigned long long s_max;
    __shared__ uint32_t hist[NB], offs[NB];
    if (threadIdx.x == 0) s_max = 0;
    for (uint32_t b = threadIdx.x; b < NB; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    unsigned long long mx = 0;
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) mx = max(mx, meta[q].scanned);
    atomicMax(&s_max, mx);
    __syncthreads();
    const unsigned long long m1 = s_max + 1;
    auto bucket = [&](uint32_t q) { return NB - 1 - (uint32_t)((meta[q].scanned * NB) / m1); };
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) atomicAdd(&hist[bucket(q)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t b = 0; b < NB; b++) {
            offs[b] = run;
            run += hist[b];
        }
        *count = nq;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) order[atomicAdd(&offs[bucket(q)], 1u)] = q;
}

__global__ void k_copy_scanned(const QueryMeta* __restrict__ meta, uint64_t nq, uint64_t* __restrict__ out) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x)
        out[q] = meta[q].scanned;
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

}  // namespace dev

void launch_compact_flags(const QueryMeta* meta, uint64_t nq, uint32_t* qlist, unsigned int* count, cudaStream_t st) {
    dev::k_compact_flags<<<(unsigned)dev::umin64((nq + 255) / 256, 1184), 256, 0, st>>>(meta, nq, qlist, count);
    CUDA_LAUNCH_CHECK();
}

void launch_lpt_order(const QueryMeta* meta, uint64_t nq, uint32_t* order, unsigned int* count, cudaStream_t st) {
    if (nq == 0) return;
    dev::k_lpt_order<<<1, 1024, 0, st>>>(meta, (uint32_t)nq, order, count);
    CUDA_LAUNCH_CHECK();
}

void launch_copy_scanned(const QueryMeta* meta, uint64_t nq, uint64_t* out, cudaStream_t st) {
    dev::k_copy_scanned<<<(unsigned)dev::umin64((nq + 255) / 256, 1184), 256, 0, st>>>(meta, nq, out);
    CUDA_LAUNCH_CHECK();
}

void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st) {
    if (n == 0) return;
    dev::k_iota<<<(unsigned)dev::umin64((n + 255) / 256, 4736), 256, 0, st>>>(v, n);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq

// ---------------------------------------------------------------------------
// brute-force ground truth helpers (dataset.cpp:46-92): per-row ordered
// selection and a (dist, id) merge into each query's running top-k.
// ---------------------------------------------------------------------------
namespace vlq {
namespace dev {

__global__ void __launch_bounds__(512) k_select_rows(const float* __restrict__ vals, uint64_t ld, uint32_t len,
                                                     uint32_t L, uint32_t* __restrict__ out) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t scan[40];
    const uint64_t r = blockIdx.x;
    block_select_ordered(vals + r * ld, len, L, out + r * L, hist, scan);
}

__global__ void k_gt_merge(const float* __restrict__ dist, uint64_t ldd, uint32_t k, uint32_t npos,
                           const uint32_t* __restrict__ sel_pos, uint64_t base_id, uint64_t* __restrict__ running,
                           uint32_t npow2) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    const uint64_t q = blockIdx.x;
    const uint32_t L = min(k, npos);
    for (uint32_t t = threadIdx.x; t < npow2; t += blockDim.x) {
        uint64_t key = ~0ull;
        if (t < k) key = running[q * k + t];
        else if (t < k + L) {
            const uint32_t pos = sel_pos[q * L + (t - k)];
            key = make_key(dist[q * ldd + pos], (uint32_t)(base_id + pos));
        }
        keys[t] = key;
    }
    __syncthreads();
    bitonic_sort_u64<false>(keys, npow2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) running[q * k + t] = keys[t];
}

}  // namespace dev

void launch_select_rows(const float* vals, uint64_t ld, uint64_t nrows, uint32_t len, uint32_t L, uint32_t* out,
                        cudaStream_t st) {
    if (nrows == 0) return;
    dev::k_select_rows<<<(unsigned)nrows, 512, 0, st>>>(vals, ld, len, L, out);
    CUDA_LAUNCH_CHECK();
}

void launch_gt_merge(const float* dist, uint64_t ldd, uint64_t nq, uint32_t k, uint32_t npos, const uint32_t* sel_pos,
                     uint64_t base_id, uint64_t* running, cudaStream_t st) {
    if (nq == 0) return;
    uint32_t n = 1;
    while (n < 2 * k) n <<= 1;
    size_t smem = (size_t)n * 8;
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_gt_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_gt_merge<<<(unsigned)nq, 256, smem, st>>>(dist, ldd, k, npos, sel_pos, base_id, running, n);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq
