// Fused PQ-ADC list scan, fast path (K4 of DESIGN.md).
//
// One CTA per query.  Warps take the query's selected cells round-robin;
// lanes take posting entries (U per lane per iteration, strided by 32 so
// every load instruction is warp-coalesced: 16 B codes, 1 B lambda, 4 B e).
// Per entry:
//     lambda  = lambda0 + b * delta                      (FFMA)
//     term1   = A + lambda * (B + lambda * C)            (2 FFMA; per-cell A=a,
//               B=b-a-c, C=c from the query's exact centroid distances)
//     sum5    = sum_p LUT[p][code_p]                      (m shared lookups)
//     dist    = (term1 + e) - 2 sum5                      (e precomputed at add)
// The key (dist, position) goes through a warp-private top-k' buffer with a
// block-shared threshold; survivors are merged by a warp merge tree and
// re-scored exactly by k_rescore, whose certificate bounds |fast - exact|.
//
// LUT bank replication: a random 8-bit index into one 256-entry fp32 table
// costs ~3.2 shared-memory wavefronts per warp access.  Sub-space p is stored
// as C_p interleaved copies (word (j*C_p + c) for copy c); lane l reads copy
// (l mod C_p), so lane groups hit disjoint bank sets.  C_p = 16 gives exactly
// 2 wavefronts, 32 gives 1.  The copy budget per M fills <= 160 KB of smem.
#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

template <int M>
struct LutPlan {
    // log2(copies) of sub-space p
    __host__ __device__ static constexpr int lg(int p) {
        return M == 16 ? (p < 8 ? 4 : 2) : (M == 8 ? 4 : (M == 4 ? 5 : (M == 2 ? 5 : 5)));
    }
    __host__ __device__ static constexpr int copies(int p) { return 1 << lg(p); }
    __host__ __device__ static constexpr int off(int p) {  // word offset of sub-space p
        int o = 0;
        for (int q = 0; q < p; q++) o += 256 * copies(q);
        return o;
    }
    __host__ __device__ static constexpr int words() { return off(M); }
};

template <int M>
__device__ __forceinline__ void load_code_vec(const uint8_t* __restrict__ p, uint32_t (&w)[(M + 3) / 4]) {
    if constexpr (M == 16) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
        w[0] = v.x;
        w[1] = v.y;
        w[2] = v.z;
        w[3] = v.w;
    } else if constexpr (M == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = v.x;
        w[1] = v.y;
    } else if constexpr (M == 4) {
        w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
    } else {
        w[0] = 0;
        for (int b = 0; b < M; b++) w[0] |= (uint32_t)__ldg(p + b) << (8 * b);
    }
}

// byte k of code word -> byte offset of LUT[p][byte] for this lane's copy
template <int LG>
__device__ __forceinline__ uint32_t lut_index(uint32_t w, int k, uint32_t lane_off) {
    constexpr uint32_t mask = 0xFFu << (2 + LG);
    const int sh = 8 * k - (2 + LG);
    const uint32_t v = sh >= 0 ? (w >> sh) : (w << (-sh));
    return (v & mask) | lane_off;
}

template <int M>
__device__ __forceinline__ float lut_sum(const unsigned char* lut, const uint32_t (&w)[(M + 3) / 4], uint32_t lane) {
    float s = 0.0f;
#pragma unroll
    for (int p = 0; p < M; p++) {
        constexpr int dummy = 0;
        (void)dummy;
        const int LG = LutPlan<M>::lg(p);
        const uint32_t lane_off = (lane & ((1u << LG) - 1u)) << 2;
        uint32_t idx;
        if (LG == 5) idx = lut_index<5>(w[p >> 2], p & 3, lane_off);
        else if (LG == 4) idx = lut_index<4>(w[p >> 2], p & 3, lane_off);
        else idx = lut_index<2>(w[p >> 2], p & 3, lane_off);
        s = __fadd_rn(s, *reinterpret_cast<const float*>(lut + 4 * LutPlan<M>::off(p) + idx));
    }
    return s;
}

// bitonic merge of a bitonic sequence of n u64 keys (ascending), warp-only
__device__ __forceinline__ void bitonic_merge_warp(uint64_t* a, uint32_t n, uint32_t lane) {
    for (uint32_t stride = n >> 1; stride > 0; stride >>= 1) {
        for (uint32_t p = lane; p < (n >> 1); p += 32) {
            uint32_t lo = 2 * p - (p & (stride - 1));
            uint32_t hi = lo + stride;
            uint64_t x = a[lo], y = a[hi];
            if (x > y) {
                a[lo] = y;
                a[hi] = x;
            }
        }
        __syncwarp();
    }
}

template <int M, int U>
__global__ void __launch_bounds__(512, 1) k_scan_fast(SearchArgs a, uint32_t w2, uint32_t keep) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = (M + 3) / 4;
    const uint32_t buf = 2 * keep;
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t q = blockIdx.x;
    unsigned char* lut = smem;
    uint64_t* bufs = reinterpret_cast<uint64_t*>(smem + 4 * LutPlan<M>::words());
    uint64_t* wbuf = bufs + (size_t)warp * buf;
    __shared__ unsigned long long s_tau;

    // replicate the query's term5 table into the banked LUT
    const float* t5q = a.t5 + q * M * VLQ_KSUB;
    float* lutf = reinterpret_cast<float*>(lut);
#pragma unroll 1
    for (int p = 0; p < M; p++) {
        const int lg = LutPlan<M>::lg(p);
        const int base = LutPlan<M>::off(p);
        for (uint32_t i = threadIdx.x; i < (256u << lg); i += blockDim.x)
            lutf[base + i] = t5q[p * VLQ_KSUB + (i >> lg)];
    }
    for (uint32_t i = threadIdx.x; i < nwarps * buf; i += blockDim.x) bufs[i] = ~0ull;
    if (threadIdx.x == 0) s_tau = ~0ull;
    __syncthreads();

    const float* wsq = a.ws + q * a.k;
    const uint32_t* selq = a.sel + q * w2;
    const float delta = (a.hi - a.lo) * (1.0f / 256.0f);
    const float lam0 = a.lo + 0.5f * delta;
    uint32_t cnt = 0;
    uint64_t tau = ~0ull;

    auto flush = [&]() {
        for (uint32_t i = cnt + lane; i < buf; i += 32) wbuf[i] = ~0ull;
        __syncwarp();
        bitonic_sort_u64<true>(wbuf, buf, lane, 32);
        cnt = min(cnt, keep);
        if (cnt == keep) {
            const uint64_t t = wbuf[keep - 1];
            if (t < tau) tau = t;
            if (lane == 0) atomicMin(&s_tau, (unsigned long long)t);
        }
        __syncwarp();
    };

    for (uint32_t ci = warp; ci < w2; ci += nwarps) {
        const uint32_t cell = selq[ci];
        const uint64_t b0 = a.list_off[cell];
        const uint32_t L = (uint32_t)(a.list_off[cell + 1] - b0);
        if (L == 0) continue;
        const uint32_t i = cell / a.n;
        const float av = wsq[i], bv = wsq[a.nbr[cell]], cv = a.elen[cell];
        const float Bc = (bv - av) - cv;
        const uint8_t* codes_c = a.codes + b0 * M;
        const uint8_t* lam_c = a.lambdas + b0;
        const float* e_c = a.eterm + b0;
        const uint32_t pos0 = (uint32_t)b0;
        for (uint32_t o = 0; o < L; o += 32 * U) {
            uint32_t cw[U][NW];
            uint32_t lb[U];
            float ev[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t idx = o + u * 32 + lane;
                if (idx < L) {
                    load_code_vec<M>(codes_c + (size_t)idx * M, cw[u]);
                    lb[u] = __ldg(lam_c + idx);
                    ev[u] = __ldg(e_c + idx);
                } else {
#pragma unroll
                    for (int t = 0; t < NW; t++) cw[u][t] = 0;
                    lb[u] = 0;
                    ev[u] = 0.0f;
                }
            }
            uint64_t key[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t idx = o + u * 32 + lane;
                const float lam = fmaf((float)lb[u], delta, lam0);
                const float t1 = fmaf(lam, fmaf(lam, cv, Bc), av);
                const float s5 = lut_sum<M>(lut, cw[u], lane);
                const float dist = fmaf(-2.0f, s5, t1 + ev[u]);
                uint32_t ub = __float_as_uint(dist);
                ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;  // order-preserving
                key[u] = idx < L ? (((uint64_t)ub << 32) | (pos0 + idx)) : ~0ull;
            }
            const uint64_t st = *reinterpret_cast<volatile unsigned long long*>(&s_tau);
            const uint64_t th = tau < st ? tau : st;
            bool any = false;
#pragma unroll
            for (int u = 0; u < U; u++) any |= key[u] < th;
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const bool take = key[u] < th;
                    const uint32_t bal = __ballot_sync(0xffffffffu, take);
                    if (bal) {
                        if (take) wbuf[cnt + __popc(bal & ((1u << lane) - 1u))] = key[u];
                        cnt += __popc(bal);
                        __syncwarp();
                        if (cnt > buf - 32) flush();
                    }
                }
            }
        }
    }
    flush();
    __syncthreads();
    // merge tree: after round s, warp w (w % 2s == 0) holds the sorted best
    // `keep` of warps [w, w + 2s) in wbuf[0, keep)
    for (uint32_t s = 1; s < nwarps; s <<= 1) {
        if ((warp % (2 * s)) == 0 && warp + s < nwarps) {
            const uint64_t* other = bufs + (size_t)(warp + s) * buf;
            for (uint32_t t = lane; t < keep; t += 32) wbuf[keep + t] = other[keep - 1 - t];
            __syncwarp();
            bitonic_merge_warp(wbuf, buf, lane);
        }
        __syncthreads();
    }
    uint64_t* candq = a.cand + q * keep;
    for (uint32_t t = threadIdx.x; t < keep; t += blockDim.x) candq[t] = bufs[t];
}

}  // namespace dev

template <int M>
static void launch_fast_t(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, cudaStream_t st) {
    constexpr int U = 2;
    const uint32_t nwarps = 16;
    const size_t smem = 4 * (size_t)dev::LutPlan<M>::words() + (size_t)nwarps * 2 * keep * 8;
    auto fn = dev::k_scan_fast<M, U>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)nq, nwarps * 32, smem, st>>>(a, w2, keep);
    CUDA_LAUNCH_CHECK();
}

bool launch_scan_fast(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, cudaStream_t st) {
    if (keep > 256) return false;
    switch (a.m) {
        case 16: launch_fast_t<16>(a, nq, w2, keep, st); return true;
        case 8: launch_fast_t<8>(a, nq, w2, keep, st); return true;
        case 4: launch_fast_t<4>(a, nq, w2, keep, st); return true;
        default: return false;
    }
}

}  // namespace vlq
