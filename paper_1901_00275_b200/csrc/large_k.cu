// select_topk for k > 1024 (search.cpp:122-140 has no cap on k): every
// scanned entry of a query gets its exact reference-order adc_distance
// (search.cpp:92-120), the (dist, id) keys of the query are sorted as one
// segment (CUB segmented radix sort), and the first k are emitted with the
// binding's -1 / +inf padding (bindings.cpp:111-125).  The keys of a group of
// queries live in HBM at once (sum of their scanned counts x 8 bytes), so the
// engine runs this path over query groups sized to a memory budget.  Rare
// path: the fast scan (k <= 768) and the exact scan (k <= 1024) cover the
// common cases.
#include <cub/device/device_segmented_radix_sort.cuh>

#include <vector>

#include "engine.h"

namespace vlq {
namespace dev {

// One CTA per query q = q0 + blockIdx.x: cell t of the query's selection
// writes its entries' keys at out + off[b] + cpre[t] + (entry - list start).
template <int M>
__global__ void __launch_bounds__(256) k_emit_all_exact(SearchArgs a, uint32_t w2, uint64_t q0,
                                                         const uint64_t* __restrict__ off,
                                                         uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t m = (M > 0) ? (uint32_t)M : a.m;
    const uint64_t q = q0 + blockIdx.x;
    float* lut = reinterpret_cast<float*>(smem);                                   // m * 256
    uint64_t* cpre = reinterpret_cast<uint64_t*>(smem + (size_t)m * VLQ_KSUB * 4);  // w2 + 1
    const float* t5q = a.t5 + q * m * VLQ_KSUB;
    for (uint32_t i = threadIdx.x; i < m * VLQ_KSUB; i += blockDim.x) lut[i] = t5q[i];
    const uint32_t* selq = a.sel + q * w2;
    if (threadIdx.x == 0) {  // cell prefix over the selection order (w2 <= a few thousand)
        uint64_t run = 0;
        for (uint32_t t = 0; t < w2; t++) {
            cpre[t] = run;
            run += a.list_off[selq[t] + 1] - a.list_off[selq[t]];
        }
        cpre[w2] = run;
    }
    __syncthreads();
    uint64_t* outq = out + off[blockIdx.x];
    const float* wsq = a.ws + q * a.k;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
    for (uint32_t ci = warp; ci < w2; ci += nwarps) {
        const uint32_t cell = selq[ci];
        const uint64_t b0 = a.list_off[cell], b1 = a.list_off[cell + 1];
        const uint32_t i = cell / a.n;
        const uint32_t s = a.nbr[cell];
        const float av = wsq[i], bv = wsq[s], cv = a.elen[cell];
        const float* t3i = a.t3 + (uint64_t)i * m * VLQ_KSUB;
        const float* t3s = a.t3 + (uint64_t)s * m * VLQ_KSUB;
        for (uint64_t e = b0 + lane; e < b1; e += 32) {
            const float lam = dequantize_lambda(__ldg(a.lambdas + e), a.lo, a.hi);
            const float d = line_sqdist(av, bv, cv, lam);
            float s2 = 0.0f, s3 = 0.0f, s4 = 0.0f, s5 = 0.0f;
            for (uint32_t p = 0; p < m; p++) {  // adc_distance, reference order
                const uint32_t c = __ldg(a.codes + e * m + p);
                s2 = __fadd_rn(s2, __ldg(a.t2 + p * VLQ_KSUB + c));
                s3 = __fadd_rn(s3, __ldg(t3i + p * VLQ_KSUB + c));
                s4 = __fadd_rn(s4, __ldg(t3s + p * VLQ_KSUB + c));
                s5 = __fadd_rn(s5, lut[p * VLQ_KSUB + c]);
            }
            float r = __fadd_rn(d, s2);
            r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, __fsub_rn(1.0f, lam)), s3));
            r = __fadd_rn(r, __fmul_rn(__fmul_rn(2.0f, lam), s4));
            r = __fsub_rn(r, __fmul_rn(2.0f, s5));
            outq[cpre[ci] + (e - b0)] = make_key(r, __ldg(a.ids + e));
        }
    }
}

// the first k keys of every sorted segment, -1 / +inf padded
__global__ void k_emit_sorted(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ off, uint64_t q0,
                              uint32_t topk, int64_t* __restrict__ out_ids, float* __restrict__ out_d) {
    const uint64_t b = blockIdx.x, q = q0 + b;
    const uint64_t have = off[b + 1] - off[b];
    for (uint32_t t = threadIdx.x; t < topk; t += blockDim.x) {
        if (t < have) {
            const uint64_t key = keys[off[b] + t];
            out_ids[q * topk + t] = (int64_t)(uint32_t)key;
            out_d[q * topk + t] = unord_float((uint32_t)(key >> 32));
        } else {
            out_ids[q * topk + t] = -1;
            out_d[q * topk + t] = __int_as_float(0x7f800000);
        }
    }
}

}  // namespace dev

void launch_topk_large(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t topk, const uint64_t* h_scanned,
                       uint64_t budget_keys, int64_t* out_ids, float* out_d, cudaStream_t st) {
    uint64_t q0 = 0;
    std::vector<uint64_t> off;
    DevBuf<uint64_t> d_off, keys, sorted;
    DevBuf<unsigned char> temp;
    while (q0 < nq) {
        // the next group of queries whose keys fit the budget (at least one query)
        off.assign(1, 0);
        uint64_t q1 = q0;
        while (q1 < nq && (q1 == q0 || off.back() + h_scanned[q1] <= budget_keys)) {
            off.push_back(off.back() + h_scanned[q1]);
            q1++;
        }
        const uint64_t ng = q1 - q0, total = off.back();
        d_off.alloc(ng + 1);
        CUDA_CHECK(cudaMemcpyAsync(d_off.p, off.data(), (ng + 1) * 8, cudaMemcpyHostToDevice, st));
        keys.alloc(std::max<uint64_t>(1, total));
        sorted.alloc(std::max<uint64_t>(1, total));
        const size_t smem = (size_t)a.m * VLQ_KSUB * 4 + ((size_t)w2 + 1) * 8;
        auto fn = a.m == 16 ? dev::k_emit_all_exact<16> : a.m == 8 ? dev::k_emit_all_exact<8> : dev::k_emit_all_exact<0>;
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        fn<<<(unsigned)ng, 256, smem, st>>>(a, w2, q0, d_off.p, keys.p);
        CUDA_LAUNCH_CHECK();
        if (total > 0) {
            size_t tb = 0;
            CUDA_CHECK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, keys.p, sorted.p, (int64_t)total, (int64_t)ng,
                                                               d_off.p, d_off.p + 1, 0, 64, st));
            temp.alloc(std::max<size_t>(1, tb));
            CUDA_CHECK(cub::DeviceSegmentedRadixSort::SortKeys(temp.p, tb, keys.p, sorted.p, (int64_t)total, (int64_t)ng,
                                                               d_off.p, d_off.p + 1, 0, 64, st));
        }
        dev::k_emit_sorted<<<(unsigned)ng, 256, 0, st>>>(sorted.p, d_off.p, q0, topk, out_ids, out_d);
        CUDA_LAUNCH_CHECK();
        CUDA_CHECK(cudaStreamSynchronize(st));  // the group's buffers are reused
        q0 = q1;
    }
}

}  // namespace vlq
