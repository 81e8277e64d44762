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
#include <algorithm>
#include <cstdlib>

#include "async.cuh"

#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

template <int M, int R = 2>
struct LutPlan {
    // log2(copies) of sub-space p.  R = 2: full replication (<= 160 KB, one
    // CTA per SM); R = 1: 4 copies; R = 0: a single table (several CTAs/SM)
    __host__ __device__ static constexpr int lg(int p) {
        return R == 0 ? 0 : (R == 1 ? 2 : (M == 16 ? (p < 8 ? 4 : 2) : (M == 8 ? 4 : 5)));
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

template <int M, int R>
__device__ __forceinline__ float lut_sum(const unsigned char* lut, const uint32_t (&w)[(M + 3) / 4], uint32_t lane) {
    float s = 0.0f;
#pragma unroll
    for (int p = 0; p < M; p++) {
        constexpr int dummy = 0;
        (void)dummy;
        const int LG = LutPlan<M, R>::lg(p);
        const uint32_t lane_off = (lane & ((1u << LG) - 1u)) << 2;
        uint32_t idx;
        if (LG == 5) idx = lut_index<5>(w[p >> 2], p & 3, lane_off);
        else if (LG == 4) idx = lut_index<4>(w[p >> 2], p & 3, lane_off);
        else if (LG == 2) idx = lut_index<2>(w[p >> 2], p & 3, lane_off);
        else idx = lut_index<0>(w[p >> 2], p & 3, lane_off);
        s = __fadd_rn(s, *reinterpret_cast<const float*>(lut + 4 * LutPlan<M, R>::off(p) + idx));
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

// Block-wide radix select over the block-shared candidate buffer: keeps
// exactly the `keep` smallest u64 keys (compacted, unordered) and returns the
// largest kept key.  Keys are unique (dist bits | entry position).  Digits of
// 8 bits from the first byte in which the keys differ (an AND / OR reduction
// skips the common leading bytes -- the sign/exponent byte every distance of
// a query shares, whose histogram was one fully contended bin); histogram
// atomics are aggregated per warp (__match_any_sync); stops early once the
// selected bin is taken whole; compaction reserves output slots per warp.
// `hist` >= 256 words, `s_misc` >= 48 words of shared scratch.
// max_keep > 0 (intermediate flushes): stop after the first digit pass when
// the keys up to and including the crossing bin number <= max_keep, and keep
// them all (>= keep keys: the threshold stays a valid bound, one pass instead
// of several); *kept receives the number of keys kept.
__device__ uint64_t block_select_keep(uint64_t* cbuf, uint32_t n, uint32_t keep, uint32_t* hist,
                                      unsigned int* s_misc, bool agg = false, uint32_t max_keep = 0,
                                      uint32_t* kept = nullptr) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31u, warp = tid >> 5, nwarps = nt >> 5;
    // 0. common leading bits of all keys
    uint64_t kand = ~0ull, kor = 0;
    for (uint32_t i = tid; i < n; i += nt) {
        const uint64_t k = cbuf[i];
        kand &= k;
        kor |= k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, o);
        kor |= __shfl_xor_sync(0xffffffffu, kor, o);
    }
    if (lane == 0) {  // hist as scratch: 4 words per warp (hist is only 4-byte aligned)
        hist[4 * warp] = (uint32_t)kand;
        hist[4 * warp + 1] = (uint32_t)(kand >> 32);
        hist[4 * warp + 2] = (uint32_t)kor;
        hist[4 * warp + 3] = (uint32_t)(kor >> 32);
    }
    __syncthreads();
    kand = ~0ull;
    kor = 0;
    for (uint32_t w = 0; w < nwarps; w++) {
        kand &= ((uint64_t)hist[4 * w + 1] << 32) | hist[4 * w];
        kor |= ((uint64_t)hist[4 * w + 3] << 32) | hist[4 * w + 2];
    }
    __syncthreads();  // hist is reused below
    const uint64_t diff = kand ^ kor;
    int sh = diff ? ((63 - __clzll((long long)diff)) & ~7) : 0;
    uint64_t pmask = sh >= 56 ? 0ull : ~((1ull << (sh + 8)) - 1ull);
    uint64_t prefix = kand & pmask;
    uint32_t remaining = keep;
    const uint32_t n_all = ((n + nt - 1) / nt) * nt;  // every lane runs the same trip count (match_any)
    for (; sh >= 0; sh -= 8) {
        for (uint32_t b = tid; b < 256; b += nt) hist[b] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n_all; i += nt) {
            const uint64_t k = i < n ? cbuf[i] : 0ull;
            const bool valid = i < n && (k & pmask) == prefix;
            const uint32_t d = valid ? ((uint32_t)(k >> sh) & 255u) : (256u + lane);  // invalid: no peers
            if (agg) {
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                if (valid && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&hist[d], (uint32_t)__popc(peers));
            } else if (valid) {
                atomicAdd(&hist[d], 1u);
            }
        }
        __syncthreads();
        if (tid < 32) {  // warp 0: scan 256 bins (8 per lane), find the crossing bin
            uint32_t v[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                v[j] = hist[tid * 8 + j];
                s += v[j];
            }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
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
        if (inbin == remaining) break;  // the whole bin is kept
        if (max_keep && keep - remaining + inbin <= max_keep) break;  // approximate: keep the whole bin
    }
    const uint64_t T = sh > 0 ? (prefix | ((1ull << sh) - 1ull)) : prefix;  // keep keys <= T
    // in-place compaction in chunks of 8 keys per thread: the chunk is read
    // into registers before any slot is written, and every written slot lies
    // below the chunk's end, so no unread key is overwritten
    constexpr uint32_t R = 8;
    if (tid == 0) s_misc[3] = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += R * nt) {
        uint64_t k[R];
        uint32_t take = 0;
#pragma unroll
        for (uint32_t r = 0; r < R; r++) {
            const uint32_t i = base + r * nt + tid;
            k[r] = i < n ? cbuf[i] : ~0ull;
            take |= (i < n && k[r] <= T ? 1u : 0u) << r;
        }
        __syncthreads();
#pragma unroll
        for (uint32_t r = 0; r < R; r++) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (take >> r) & 1u);
            uint32_t slot = 0;
            if (lane == 0 && bal) slot = atomicAdd(&s_misc[3], (uint32_t)__popc(bal));
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if ((take >> r) & 1u) cbuf[slot + __popc(bal & ((1u << lane) - 1u))] = k[r];
        }
        __syncthreads();
    }
    if (kept) *kept = s_misc[3];
    return T;
}

template <int M, int U, int R>
__global__ void __launch_bounds__(R == 2 ? 512 : 256, R == 2 ? 1 : (R == 1 || U > 6 ? 2 : 3)) k_scan_fast(SearchArgs a, uint32_t w2, uint32_t keep,
                                                                      uint32_t cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Plan = LutPlan<M, R>;
    constexpr int NW = (M + 3) / 4;
    constexpr uint32_t CH = 32 * U;  // entries per chunk
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t q = blockIdx.x;
    unsigned char* lut = smem;
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(smem + 4 * Plan::words());   // cap keys
    uint32_t* cpref = reinterpret_cast<uint32_t*>(cbuf + cap);                 // w2 + 1
    __shared__ uint32_t hist[256];
    __shared__ unsigned int s_misc[48];
    __shared__ unsigned int s_count;
    __shared__ unsigned long long s_tau;

    // 1. replicate the query's term5 table into the banked LUT (4 copies per STS.128)
    const float* t5q = a.t5 + q * M * VLQ_KSUB;
    float4* lut4 = reinterpret_cast<float4*>(lut);
#pragma unroll
    for (int p = 0; p < M; p++) {
        const int lg = Plan::lg(p);
        if (lg >= 2) {
            const int base4 = Plan::off(p) >> 2;
            const uint32_t n4 = 256u << (lg - 2);
            for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) {
                const float v = __ldg(t5q + p * VLQ_KSUB + (i >> (lg - 2)));
                lut4[base4 + i] = make_float4(v, v, v, v);
            }
        } else {
            float* lutf = reinterpret_cast<float*>(lut) + Plan::off(p);
            for (uint32_t i = threadIdx.x; i < 256u; i += blockDim.x) lutf[i] = __ldg(t5q + p * VLQ_KSUB + i);
        }
    }
    // 2. chunk prefix over the selected cells (chunks never straddle cells)
    const uint32_t* selq = a.sel + q * w2;
    {
        const uint32_t per = (w2 + blockDim.x - 1) / blockDim.x;
        uint32_t local = 0;
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = selq[t];
            const uint32_t len = (uint32_t)(a.list_off[c + 1] - a.list_off[c]);
            cpref[t] = (len + CH - 1) / CH;
            local += cpref[t];
        }
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, s_misc + 8, &total);
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = cpref[t];
            cpref[t] = run;
            run += c;
        }
        if (threadIdx.x == 0) {
            cpref[w2] = total;
            s_count = 0;
            s_tau = ~0ull;
        }
    }
    __syncthreads();
    const uint32_t nchunks = cpref[w2];
    // balanced contiguous chunk range per warp
    const uint32_t c_lo = (uint32_t)(((uint64_t)nchunks * warp) / nwarps);
    const uint32_t c_hi = (uint32_t)(((uint64_t)nchunks * (warp + 1)) / nwarps);
    uint32_t t = 0;
    {
        uint32_t lo = 0, hi = w2;  // largest t with cpref[t] <= c_lo
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cpref[mid] <= c_lo) lo = mid;
            else hi = mid;
        }
        t = lo;
    }
    const float* wsq = a.ws + q * a.k;
    const float delta = a.lam_delta, lam0 = a.lam0;  // dequantization affine map
    uint32_t L = 0, pos0 = 0;
    const uint8_t* codes_c = nullptr;
    const uint8_t* lam_c = nullptr;
    const float* e_c = nullptr;
    float av = 0.f, Bc = 0.f, cv = 0.f;
    uint32_t loaded_t = 0xffffffffu;

    auto locate = [&](uint32_t g) {  // walks t forward to the cell holding chunk g
        while (cpref[t + 1] <= g) t++;
        if (t != loaded_t) {
            loaded_t = t;
            const uint32_t cell = selq[t];
            const uint64_t b0 = a.list_off[cell];
            L = (uint32_t)(a.list_off[cell + 1] - b0);
            pos0 = (uint32_t)b0;
            const uint32_t i = cell / a.n;
            av = wsq[i];
            const float bv = wsq[a.nbr[cell]];
            cv = a.elen[cell];
            Bc = (bv - av) - cv;
            codes_c = a.codes + b0 * M;
            lam_c = a.lambdas + b0;
            e_c = a.eterm + b0;
        }
        return (g - cpref[t]) * CH;
    };

    uint32_t done = 0;        // chunks consumed by this warp
    uint64_t n_seen = 0;      // block-wide entries processed before this round (estimate)
    uint32_t rlen = 1;
    const uint32_t my_total = c_hi - c_lo;
    // Rounds: every warp processes up to rlen chunks, then the block meets
    // and flushes the shared buffer if needed.  A warp whose insertions do not
    // fit the buffer writes nothing for that chunk and redoes it next round,
    // so nothing is ever dropped.
    while (__syncthreads_or(done < my_total)) {
        for (uint32_t r = 0; r < rlen && done < my_total; r++) {
            const uint32_t o = locate(c_lo + done);
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
                    for (int w = 0; w < NW; w++) cw[u][w] = 0;
                    lb[u] = 0;
                    ev[u] = 0.0f;
                }
            }
            const uint64_t tau = *reinterpret_cast<volatile unsigned long long*>(&s_tau);
            uint64_t key[U];
            uint32_t tk = 0;
#pragma unroll
            for (int u = 0; u < U; u++) {
                key[u] = ~0ull;
                if (o + u * 32 < L) {  // warp-uniform: skip fully empty slots
                    const uint32_t idx = o + u * 32 + lane;
                    const float lam = fmaf((float)lb[u], delta, lam0);
                    const float t1 = fmaf(lam, fmaf(lam, cv, Bc), av);
                    const float s5 = lut_sum<M, R>(lut, cw[u], lane);
                    const float dist = fmaf(-2.0f, s5, t1 + ev[u]);
                    uint32_t ub = __float_as_uint(dist);
                    ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;  // order-preserving
                    if (idx < L) key[u] = ((uint64_t)ub << 32) | (pos0 + idx);
                }
                tk |= (key[u] < tau ? 1u : 0u) << u;
            }
            uint32_t wtot = 0;
            uint32_t bal[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                bal[u] = __ballot_sync(0xffffffffu, (tk >> u) & 1u);
                wtot += __popc(bal[u]);
            }
            if (wtot) {
                uint32_t base = 0;
                if (lane == 0) {
                    // reserve only if the whole chunk fits
                    unsigned int cur = *reinterpret_cast<volatile unsigned int*>(&s_count);
                    base = 0xffffffffu;
                    while (cur + wtot <= cap) {
                        const unsigned int prev = atomicCAS(&s_count, cur, cur + wtot);
                        if (prev == cur) {
                            base = cur;
                            break;
                        }
                        cur = prev;
                    }
                }
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base == 0xffffffffu) break;  // buffer full: redo this chunk after the flush
                const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if ((tk >> u) & 1u) cbuf[base + __popc(bal[u] & lt)] = key[u];
                    base += __popc(bal[u]);
                }
            }
            done++;
        }
        __syncthreads();
        n_seen += rlen * nwarps * CH;
        const uint32_t cnt = s_count;
        if (cnt > keep && cnt > cap / 2) {  // block-uniform
            const uint64_t T = block_select_keep(cbuf, cnt, keep, hist, s_misc, a.sel_agg);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_count = keep;
                s_tau = T + 1;  // insert only keys <= T
            }
            __syncthreads();
        }
        // next round length: expected insertions ~ keep * (new entries) / n_seen
        // with a 4x margin; an underestimate only costs a redone chunk
        const uint32_t free_slots = cap - s_count;
        const uint64_t per_chunk_round = (uint64_t)nwarps * CH;
        uint64_t rn = (s_tau == ~0ull) ? free_slots / per_chunk_round
                                       : ((uint64_t)free_slots * n_seen) / (4ull * keep * per_chunk_round);
        rlen = (uint32_t)(rn < 1 ? 1ull : (rn > 32 ? 32ull : rn));
    }
    // final: exactly min(count, keep) smallest keys, sorted, padded with +inf
    uint32_t n = s_count;
    if (n > keep) {
        block_select_keep(cbuf, n, keep, hist, s_misc, a.sel_agg);
        n = keep;
    }
    __syncthreads();
    for (uint32_t i = n + threadIdx.x; i < keep; i += blockDim.x) cbuf[i] = ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(cbuf, keep, threadIdx.x, blockDim.x);
    uint64_t* candq = a.cand + q * keep;
    for (uint32_t i = threadIdx.x; i < keep; i += blockDim.x) candq[i] = cbuf[i];
}

__global__ void k_pack_eterm_lam(const float* __restrict__ eterm, const uint8_t* __restrict__ lambdas, uint64_t n,
                                 uint32_t* __restrict__ out) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
        out[e] = (__float_as_uint(eterm[e]) & ~0xffu) | (uint32_t)lambdas[e];
}

// v6: the v5 schedule (balanced chunk ranges, block-shared candidate buffer,
// adaptive rounds) with the per-entry arithmetic halved by the sm_100
// packed fp32 pipe.  Entries are taken in pairs (slot u, u+1 of a lane):
//     lambda, term1, term1 + e, the m-term LUT sum and the final -2 sum5 FFMA
// run as FFMA2 / FADD2 on (entry u, entry u+1), each element with exactly the
// rounding of the scalar v5 code (per-entry operation order unchanged, so the
// certificate of k_rescore holds as is).  Loads are unconditional at a
// clamped index (no zero-fill moves), and the threshold test is one float
// compare against the threshold key's distance; the exact 64-bit
// (dist, position) key is formed only for entries that pass it.
// LUT[p][code_p]: the byte is extracted with one LOP3 / PRMT / SHF and the
// shared load scales it (LDS [R.X4 + imm]), so a lookup is 2 instructions
template <int M>
__device__ __forceinline__ float lut_at(const unsigned char* lut, const uint32_t (&w)[(M + 3) / 4], int p) {
    const uint32_t word = w[p >> 2];
    const int k = p & 3;
    const uint32_t b = k == 0 ? (word & 0xffu) : (k == 3 ? (word >> 24) : __byte_perm(word, 0u, 0x4440u + k));
    return reinterpret_cast<const float*>(lut)[p * 256 + b];
}

__device__ __forceinline__ float key_dist(uint64_t key) {  // distance of an order-preserving key (upper 32 bits)
    const uint32_t ub = (uint32_t)(key >> 32);
    return __uint_as_float((ub & 0x80000000u) ? (ub & 0x7fffffffu) : ~ub);
}

// warp-cooperative L2 prefetch of [p, p + bytes): one 128-byte line per lane
__device__ __forceinline__ void prefetch_l2_range(const void* p, size_t bytes, uint32_t lane) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)127;
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(p) + bytes;
    for (uintptr_t x = a0 + 128u * lane; x < a1; x += 128u * 32u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x));
}

// Q8: the query's term5 table is quantized to u8 in shared memory (one scale
// for all sub-spaces, a per-sub-space offset), so a lookup is one PRMT and one
// LDS.U8, the m-term sum is exact integer arithmetic and the table is 4x
// smaller (fewer bank conflicts).  The quantization error (at most half a step
// per term) is written to meta[q].qerr and added to the re-score certificate.
template <int M>
__device__ __forceinline__ uint32_t lut8_at(const unsigned char* lq, const uint32_t (&w)[(M + 3) / 4], int p) {
    const uint32_t word = w[p >> 2];
    const int k = p & 3;
    const uint32_t b = k == 0 ? (word & 0xffu) : (k == 3 ? (word >> 24) : __byte_perm(word, 0u, 0x4440u + k));
    return lq[p * 256 + b];
}

// The query's term5 table quantized to u8 (all threads of the CTA): one step
// `scale` for all sub-spaces (the widest range / 255) and per-sub-space offsets,
// LUT_q8[p][j] = rint((t5[p][j] - min_p) / scale), so that
//     sum5 ~= smin + scale * sum_p LUT_q8[p][code_p]        (smin = sum_p min_p)
// with |error| <= m * scale / 2.  meta->qerr receives the resulting bound on
// |dist_q8 - dist| (x2 for the -2 sum5 of adc_distance) plus a generous
// allowance for the fp32 rounding of the reconstruction.  Ends synchronised.
template <int M>
__device__ void build_q8_lut(const float* __restrict__ t5f, unsigned char* lq, float* s_qmin, float* s_qrng,
                             QueryMeta* meta, float& scale, float& smin) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
    for (uint32_t p = warp; p < (uint32_t)M; p += nwarps) {  // per-sub-space range
        float mn = __int_as_float(0x7f800000), mx = -mn;
        for (uint32_t j = lane; j < VLQ_KSUB; j += 32) {
            const float v = __ldg(t5f + p * VLQ_KSUB + j);
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
        for (int o = 16; o > 0; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            s_qmin[p] = mn;
            s_qrng[p] = mx - mn;
        }
    }
    __syncthreads();
    float rng = 0.0f, sabs = 0.0f;
    smin = 0.0f;
#pragma unroll
    for (int p = 0; p < M; p++) {
        rng = fmaxf(rng, s_qrng[p]);
        smin += s_qmin[p];
        sabs += fabsf(s_qmin[p]);
    }
    scale = rng > 0.0f ? rng / 255.0f : 1.0f;
    const float inv = 1.0f / scale;
    for (uint32_t i = threadIdx.x; i < 256u * M; i += blockDim.x) {
        const float v = __ldg(t5f + i);
        const int qv = __float2int_rn((v - s_qmin[i >> 8]) * inv);
        lq[i] = (unsigned char)min(255, max(0, qv));
    }
    if (threadIdx.x == 0) {
        const float span = sabs + scale * 255.0f * M;
        meta->qerr = 2.0f * (0.5f * M * scale * 1.001f) + 1e-5f * span;
    }
    __syncthreads();
}

// LM = 2 (q8x32): the u8 table replicated once per lane so that every lane
// reads its own bank -- conflict-free LUT loads (one wavefront per warp
// lookup) at the price of 32x the table (64 KB per 8 sub-spaces, one CTA of
// 16 warps per SM).  Row (g, j) is 256 bytes: [half h][lane l][byte b] holds
// LUT[8g + 4h + b][j], so the address of LUT[p][j] for lane l is
//     (j << 8 | l << 2) + 65536 (p / 8) + 128 ((p / 4) % 2) + p % 4,
// where the first term is ONE PRMT of the code word with the lane's base and
// the rest is the LDS immediate; bank = l for every p and j.
template <int M>
__device__ __forceinline__ uint32_t lut8x32_at(const unsigned char* lq, const uint32_t (&w)[(M + 3) / 4], int p,
                                               uint32_t lane4) {
    const uint32_t a = __byte_perm(w[p >> 2], lane4, 0x7604u | ((uint32_t)(p & 3) << 4));
    return lq[a + 65536u * (p >> 3) + 128u * ((p >> 2) & 1) + (p & 3)];
}

template <int M>
__host__ __device__ constexpr uint32_t lut_bytes(int lm) {
    return lm == 0 ? 4 * 256 * M : (lm == 1 ? 256 * M : 65536u * ((M + 7) / 8));
}

template <int M, int U, int MINB, int LM = 0, int NT = 256>
__global__ void __launch_bounds__(NT, MINB) k_scan_fast2(SearchArgs a, uint32_t w2, uint32_t keep, uint32_t cap,
                                                         uint32_t pf) {
    static_assert(U % 2 == 0, "entries are processed in pairs");
    constexpr bool Q8 = LM != 0;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = (M + 3) / 4;
    constexpr uint32_t CH = 32 * U;  // entries per chunk
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    if (a.qlist && blockIdx.x >= *a.qcount) return;
    const uint64_t q = a.qlist ? a.qlist[blockIdx.x] : blockIdx.x;
    unsigned char* lut = smem;
    constexpr uint32_t LUT_B = lut_bytes<M>(LM);
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(smem + LUT_B);        // cap keys
    uint32_t* cpref = reinterpret_cast<uint32_t*>(cbuf + cap);         // w2 + 1
    __shared__ uint32_t hist[256];
    __shared__ unsigned int s_misc[48];
    __shared__ unsigned int s_count;
    __shared__ unsigned long long s_tau;
    __shared__ float s_qmin[Q8 ? M : 1], s_qrng[Q8 ? M : 1];

    // 1. the query's term5 table (one copy per sub-space)
    const float4* t5q = reinterpret_cast<const float4*>(a.t5 + q * M * VLQ_KSUB);
    float2 qs2 = make_float2(0.f, 0.f), qc2 = qs2;  // Q8: dist = qs * isum + (te + qc)
    if constexpr (!Q8) {
        for (uint32_t i = threadIdx.x; i < 64u * M; i += blockDim.x) reinterpret_cast<float4*>(lut)[i] = __ldg(t5q + i);
    } else {
        const float* t5f = a.t5 + q * M * VLQ_KSUB;
        float scale, smin;
        // LM = 2: quantize into the (not yet used) candidate buffer, then replicate
        unsigned char* lq = LM == 2 ? reinterpret_cast<unsigned char*>(cbuf) : lut;
        build_q8_lut<M>(t5f, lq, s_qmin, s_qrng, a.meta + q, scale, smin);
        if constexpr (LM == 2) {
            __syncthreads();
            for (uint32_t r = threadIdx.x; r < 256u * ((M + 7) / 8); r += blockDim.x) {
                const uint32_t g = r >> 8, j = r & 255u;
                uint32_t hw[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    hw[h] = 0;
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        const uint32_t p = 8 * g + 4 * h + b;
                        if (p < (uint32_t)M) hw[h] |= (uint32_t)lq[p * 256 + j] << (8 * b);
                    }
                }
                uint4* row = reinterpret_cast<uint4*>(lut + 65536u * g + 256u * j);
#pragma unroll
                for (int i = 0; i < 16; i++) row[i] = make_uint4(hw[i >> 3], hw[i >> 3], hw[i >> 3], hw[i >> 3]);
            }
            __syncthreads();  // the staging bytes in cbuf are dead from here on
        }
        qs2 = make_float2(-2.0f * scale, -2.0f * scale);
        qc2 = make_float2(-2.0f * smin, -2.0f * smin);
    }
    // 2. chunk prefix over the selected cells (chunks never straddle cells)
    const uint32_t* selq = a.sel + q * w2;
    {
        const uint32_t per = (w2 + blockDim.x - 1) / blockDim.x;
        uint32_t local = 0;
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = selq[t];
            const uint32_t len = (uint32_t)(a.list_off[c + 1] - a.list_off[c]);
            cpref[t] = (len + CH - 1) / CH;
            local += cpref[t];
        }
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, s_misc + 8, &total);
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = cpref[t];
            cpref[t] = run;
            run += c;
        }
        if (threadIdx.x == 0) {
            cpref[w2] = total;
            s_count = 0;
            s_tau = ~0ull;
        }
    }
    __syncthreads();
    const uint32_t nchunks = cpref[w2];
    const uint32_t c_lo = (uint32_t)(((uint64_t)nchunks * warp) / nwarps);
    const uint32_t c_hi = (uint32_t)(((uint64_t)nchunks * (warp + 1)) / nwarps);
    uint32_t t = 0;
    {
        uint32_t lo = 0, hi = w2;  // largest t with cpref[t] <= c_lo
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cpref[mid] <= c_lo) lo = mid;
            else hi = mid;
        }
        t = lo;
    }
    const float* wsq = a.ws + q * a.k;
    const float2 delta2 = make_float2(a.lam_delta, a.lam_delta), lam02 = make_float2(a.lam0, a.lam0);
    const float2 m2 = make_float2(-2.0f, -2.0f);
    uint32_t L = 0, pos0 = 0;
    const uint8_t* codes_c = nullptr;
    const uint8_t* lam_c = nullptr;
    const float* e_c = nullptr;
    float2 av2 = make_float2(0.f, 0.f), Bc2 = av2, cv2 = av2;
    uint32_t loaded_t = 0xffffffffu;
    const bool packed = a.eterm_lam != nullptr;
    const uint32_t* el_c = nullptr;

    auto locate = [&](uint32_t g) {  // walks t forward to the cell holding chunk g
        while (cpref[t + 1] <= g) t++;
        if (t != loaded_t) {
            loaded_t = t;
            const uint32_t cell = selq[t];
            const uint64_t b0 = a.list_off[cell];
            L = (uint32_t)(a.list_off[cell + 1] - b0);
            pos0 = (uint32_t)b0;
            const uint32_t i = cell / a.n;
            const float av = wsq[i];
            const float bv = wsq[a.nbr[cell]];
            const float cv = a.elen[cell];
            av2 = make_float2(av, av);
            Bc2 = make_float2((bv - av) - cv, (bv - av) - cv);
            cv2 = make_float2(cv, cv);
            codes_c = a.codes + b0 * M;
            lam_c = a.lambdas + b0;
            e_c = a.eterm + b0;
            if (packed) el_c = a.eterm_lam + b0;
        }
        return (g - cpref[t]) * CH;
    };

    uint32_t done = 0;
    uint64_t n_seen = 0;
    uint32_t rlen = 1;
    const uint32_t my_total = c_hi - c_lo;
    while (__syncthreads_or(done < my_total)) {
        for (uint32_t r = 0; r < rlen && done < my_total; r++) {
            const uint32_t o = locate(c_lo + done);
            if (pf) {  // L2 prefetch of the chunk pf ahead in this cell (off the critical path)
                const uint32_t s0 = o + pf * CH;
                if (s0 < L) {
                    const uint32_t n0 = min(L - s0, CH);
                    prefetch_l2_range(codes_c + (size_t)s0 * M, (size_t)n0 * M, lane);
                    prefetch_l2_range(lam_c + s0, n0, lane);
                    prefetch_l2_range(e_c + s0, (size_t)n0 * 4, lane);
                }
            }
            uint32_t cw[U][NW];
            uint32_t lb[U];
            float ev[U];
            // (warp-uniform variants hoisted out of the slot loop so each
            // issues its U x 2-3 loads back to back)
            if (packed) {  // one 4-byte word: e-term (low 8 mantissa bits dropped) | lambda byte
                uint32_t le[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t ic = min(o + u * 32 + lane, L - 1);  // clamped: the tail re-reads entry L-1
                    load_code_vec<M>(codes_c + (size_t)ic * M, cw[u]);
                    le[u] = __ldg(el_c + ic);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    lb[u] = le[u] & 0xffu;
                    ev[u] = __uint_as_float(le[u] & ~0xffu);
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t ic = min(o + u * 32 + lane, L - 1);
                    load_code_vec<M>(codes_c + (size_t)ic * M, cw[u]);
                    lb[u] = __ldg(lam_c + ic);
                    ev[u] = __ldg(e_c + ic);
                }
            }
            const uint64_t tau = *reinterpret_cast<volatile unsigned long long*>(&s_tau);
            const float taud = tau == ~0ull ? __int_as_float(0x7f800000) : key_dist(tau);
            uint32_t tk = 0;
            float dist[U];
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                dist[u] = dist[u + 1] = __int_as_float(0x7fffffff);
                if (o + u * 32 < L) {  // warp-uniform: skip fully empty pairs
                    const float2 lam = __ffma2_rn(make_float2((float)lb[u], (float)lb[u + 1]), delta2, lam02);
                    const float2 t1 = __ffma2_rn(lam, __ffma2_rn(lam, cv2, Bc2), av2);
                    const float2 te = __fadd2_rn(t1, make_float2(ev[u], ev[u + 1]));
                    float2 d;
                    if constexpr (Q8) {
                        uint32_t i0 = 0, i1 = 0;
#pragma unroll
                        for (int p = 0; p < M; p++) {
                            if constexpr (LM == 2) {
                                i0 += lut8x32_at<M>(lut, cw[u], p, lane << 2);
                                i1 += lut8x32_at<M>(lut, cw[u + 1], p, lane << 2);
                            } else {
                                i0 += lut8_at<M>(lut, cw[u], p);
                                i1 += lut8_at<M>(lut, cw[u + 1], p);
                            }
                        }
                        d = __ffma2_rn(qs2, make_float2((float)i0, (float)i1), __fadd2_rn(te, qc2));
                    } else {
                        float2 s = make_float2(lut_at<M>(lut, cw[u], 0), lut_at<M>(lut, cw[u + 1], 0));
#pragma unroll
                        for (int p = 1; p < M; p++)
                            s = __fadd2_rn(s, make_float2(lut_at<M>(lut, cw[u], p), lut_at<M>(lut, cw[u + 1], p)));
                        d = __ffma2_rn(m2, s, te);
                    }
                    dist[u] = d.x;
                    dist[u + 1] = d.y;
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t idx = o + u * 32 + lane;
                if (idx < L && dist[u] <= taud) {  // rare after the first rounds: exact key test
                    uint32_t ub = __float_as_uint(dist[u]);
                    ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;  // order-preserving
                    const uint64_t key = ((uint64_t)ub << 32) | (pos0 + idx);
                    if (key < tau) tk |= 1u << u;
                }
            }
            const uint32_t any = __ballot_sync(0xffffffffu, tk != 0);
            if (any) {
                uint32_t wtot = 0;
                uint32_t bal[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    bal[u] = __ballot_sync(0xffffffffu, (tk >> u) & 1u);
                    wtot += __popc(bal[u]);
                }
                uint32_t base = 0;
                if (lane == 0) {
                    unsigned int cur = *reinterpret_cast<volatile unsigned int*>(&s_count);
                    base = 0xffffffffu;
                    while (cur + wtot <= cap) {
                        const unsigned int prev = atomicCAS(&s_count, cur, cur + wtot);
                        if (prev == cur) {
                            base = cur;
                            break;
                        }
                        cur = prev;
                    }
                }
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base == 0xffffffffu) break;  // buffer full: redo this chunk after the flush
                const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if ((tk >> u) & 1u) {
                        uint32_t ub = __float_as_uint(dist[u]);
                        ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;
                        cbuf[base + __popc(bal[u] & lt)] = ((uint64_t)ub << 32) | (pos0 + o + u * 32 + lane);
                    }
                    base += __popc(bal[u]);
                }
            }
            done++;
        }
        __syncthreads();
        n_seen += rlen * nwarps * CH;
        const uint32_t cnt = s_count;
        if (cnt > keep && cnt > cap / 2) {  // block-uniform
            uint32_t kept = keep;
            const uint64_t T = block_select_keep(cbuf, cnt, keep, hist, s_misc, a.sel_agg,
                                                 a.flush_exact ? 0u : cap / 4, &kept);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_count = kept;  // >= keep after an approximate flush
                s_tau = T + 1;   // insert only keys <= T
            }
            __syncthreads();
        }
        const uint32_t free_slots = cap - s_count;
        const uint64_t per_chunk_round = (uint64_t)nwarps * CH;
        uint64_t rn = (s_tau == ~0ull) ? free_slots / per_chunk_round
                                       : ((uint64_t)free_slots * n_seen) / (4ull * keep * per_chunk_round);
        rlen = (uint32_t)(rn < 1 ? 1ull : (rn > 32 ? 32ull : rn));
    }
    uint32_t n = s_count;
    if (n > keep) {
        block_select_keep(cbuf, n, keep, hist, s_misc, a.sel_agg);
        n = keep;
    }
    __syncthreads();
    for (uint32_t i = n + threadIdx.x; i < keep; i += blockDim.x) cbuf[i] = ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(cbuf, keep, threadIdx.x, blockDim.x);
    uint64_t* candq = a.cand + (a.qlist ? (uint64_t)blockIdx.x : q) * keep;
    for (uint32_t i = threadIdx.x; i < keep; i += blockDim.x) candq[i] = cbuf[i];
}

// v7: the v6 arithmetic and candidate handling, with the entry stream staged
// into shared memory by the bulk-async copy engine instead of per-lane LDGs.
// Every warp owns a ring of NS stages (one chunk of 32 U entries each: the
// codes and the packed e-term | lambda words, both contiguous in HBM since a
// chunk never straddles a cell).  Lane 0 issues `cp.async.bulk` for chunk
// g + NS as soon as chunk g is consumed, so each warp keeps NS - 1 chunks in
// flight while it computes; consumers wait on the stage's mbarrier and read
// the entries with conflict-free LDS.  The per-cell parameters (list position
// and length, A = a, B = (b - a) - c, C = c) are computed once per query in the
// prologue, so the loop issues no dependent global loads at cell changes.
template <int M>
__device__ __forceinline__ void load_code_smem(const unsigned char* p, uint32_t (&w)[(M + 3) / 4]) {
    if constexpr (M == 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        w[0] = v.x;
        w[1] = v.y;
        w[2] = v.z;
        w[3] = v.w;
    } else if constexpr (M == 8) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        w[0] = v.x;
        w[1] = v.y;
    } else {
        static_assert(M == 4, "bulk scan: m in {4, 8, 16}");
        w[0] = *reinterpret_cast<const uint32_t*>(p);
    }
}

template <int M, int U>
struct BulkPlan {
    static constexpr uint32_t CH = 32 * U;
    static constexpr uint32_t CODE_B = CH * M + 16;  // + the 16-byte alignment slack of the source
    static constexpr uint32_t EL_B = CH * 4 + 16;
    static constexpr uint32_t STAGE_B = CODE_B + EL_B;
    static_assert(STAGE_B % 16 == 0, "stages stay 16-byte aligned");
};

template <int M, int U, int NS, int LM>
__host__ __device__ constexpr size_t bulk_smem_bytes(uint32_t w2, uint32_t cap) {
    return (size_t)lut_bytes<M>(LM) + 8 * (size_t)NS * (BulkPlan<M, U>::STAGE_B + 16 + 8) + (size_t)cap * 8 +
           (size_t)w2 * 24 + ((size_t)w2 + 1) * 4;
}

// LM = 1: the u8-quantized LUT of k_scan_fast2<.., 1> (4x smaller table, so
// the ring fits at 3 CTAs per SM)
template <int M, int U, int NS, int MINB, int LM = 0>
__global__ void __launch_bounds__(256, MINB) k_scan_bulk(SearchArgs a, uint32_t w2, uint32_t keep, uint32_t cap) {
    static_assert(U % 2 == 0, "entries are processed in pairs");
    static_assert(LM == 0 || LM == 1, "bulk scan: fp32 or u8 LUT");
    using P = BulkPlan<M, U>;
    constexpr uint32_t CH = P::CH;
    constexpr int NW = (M + 3) / 4;
    constexpr uint32_t NWARPS = 8;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t q = blockIdx.x;
    unsigned char* lut = smem;
    unsigned char* ring = smem + lut_bytes<M>(LM);                                 // [warp][stage]
    uint4* smeta = reinterpret_cast<uint4*>(ring + NWARPS * NS * P::STAGE_B);       // [warp][stage]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smeta + NWARPS * NS);              // [warp][stage]
    uint64_t* cbuf = bars + NWARPS * NS;                                            // cap keys
    float4* cpar = reinterpret_cast<float4*>(cbuf + cap);                           // [w2] (A, B, C, -)
    uint2* cpos = reinterpret_cast<uint2*>(cpar + w2);                              // [w2] (position, length)
    uint32_t* cpref = reinterpret_cast<uint32_t*>(cpos + w2);                       // [w2 + 1] chunk prefix
    __shared__ uint32_t hist[256];
    __shared__ unsigned int s_misc[48];
    __shared__ unsigned int s_count;
    __shared__ unsigned long long s_tau;

    __shared__ float s_qmin[LM ? M : 1], s_qrng[LM ? M : 1];

    // 1. the query's term5 table (one copy per sub-space)
    float2 qs2 = make_float2(0.f, 0.f), qc2 = qs2;  // LM = 1: dist = qs * isum + (te + qc)
    if constexpr (LM == 0) {
        const float4* t5q = reinterpret_cast<const float4*>(a.t5 + q * M * VLQ_KSUB);
        for (uint32_t i = threadIdx.x; i < 64u * M; i += blockDim.x) reinterpret_cast<float4*>(lut)[i] = __ldg(t5q + i);
    } else {
        float scale, smin;
        build_q8_lut<M>(a.t5 + q * M * VLQ_KSUB, lut, s_qmin, s_qrng, a.meta + q, scale, smin);
        qs2 = make_float2(-2.0f * scale, -2.0f * scale);
        qc2 = make_float2(-2.0f * smin, -2.0f * smin);
    }
    // 2. per-cell parameters and the chunk prefix (chunks never straddle cells)
    const uint32_t* selq = a.sel + q * w2;
    const float* wsq = a.ws + q * a.k;
    {
        const uint32_t per = (w2 + blockDim.x - 1) / blockDim.x;
        uint32_t local = 0;
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = selq[t];
            const uint64_t b0 = a.list_off[c];
            const uint32_t len = (uint32_t)(a.list_off[c + 1] - b0);
            const float av = wsq[c / a.n];
            const float bv = wsq[a.nbr[c]];
            const float cv = a.elen[c];
            cpar[t] = make_float4(av, (bv - av) - cv, cv, 0.0f);
            cpos[t] = make_uint2((uint32_t)b0, len);
            cpref[t] = (len + CH - 1) / CH;
            local += cpref[t];
        }
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, s_misc + 8, &total);
        for (uint32_t t = threadIdx.x * per; t < min(w2, (threadIdx.x + 1) * per); t++) {
            const uint32_t c = cpref[t];
            cpref[t] = run;
            run += c;
        }
        if (threadIdx.x == 0) {
            cpref[w2] = total;
            s_count = 0;
            s_tau = ~0ull;
        }
        if (lane == 0) {
            for (int s = 0; s < NS; s++) mbar_init(&bars[warp * NS + s], 1);
            mbar_fence_init();
        }
    }
    __syncthreads();
    const uint32_t nchunks = cpref[w2];
    const uint32_t c_lo = (uint32_t)(((uint64_t)nchunks * warp) / NWARPS);
    const uint32_t c_hi = (uint32_t)(((uint64_t)nchunks * (warp + 1)) / NWARPS);
    const uint32_t my_total = c_hi - c_lo;
    uint32_t tp = 0;  // producer cursor: cell of the next chunk to stage
    {
        uint32_t lo = 0, hi = w2;  // largest t with cpref[t] <= c_lo
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cpref[mid] <= c_lo) lo = mid;
            else hi = mid;
        }
        tp = lo;
    }
    unsigned char* wring = ring + warp * NS * P::STAGE_B;
    uint4* wmeta = smeta + warp * NS;
    uint64_t* wbar = bars + warp * NS;
    // lane 0: stage chunk (c_lo + d) into slot d % NS
    auto fill = [&](uint32_t d) {
        const uint32_t g = c_lo + d, s = d % NS;
        while (cpref[tp + 1] <= g) tp++;
        const uint2 cp = cpos[tp];
        const uint32_t o = (g - cpref[tp]) * CH;
        const uint32_t n = min(CH, cp.y - o);
        const uint32_t pos = cp.x + o;
        const uint64_t cb = (uint64_t)pos * M;                     // code bytes: align the source down to 16
        const uint32_t csh = (uint32_t)(cb & 15u);
        const uint32_t cbytes = (csh + n * M + 15u) & ~15u;
        const uint32_t esh = pos & 3u;                             // packed words: 4 per 16 bytes
        const uint32_t ebytes = ((esh + n) * 4u + 15u) & ~15u;
        wmeta[s] = make_uint4(tp, pos, n, (csh / M) | (esh << 8));
        unsigned char* st = wring + s * P::STAGE_B;
        mbar_expect_tx(&wbar[s], cbytes + ebytes);
        bulk_g2s(st, a.codes + (cb - csh), cbytes, &wbar[s]);
        bulk_g2s(st + P::CODE_B, a.eterm_lam + (pos - esh), ebytes, &wbar[s]);
    };
    if (lane == 0)
        for (uint32_t d = 0; d < (uint32_t)NS && d < my_total; d++) fill(d);

    const float2 delta2 = make_float2(a.lam_delta, a.lam_delta), lam02 = make_float2(a.lam0, a.lam0);
    const float2 m2 = make_float2(-2.0f, -2.0f);
    uint32_t done = 0;
    uint64_t n_seen = 0;
    uint32_t rlen = 1;
    while (__syncthreads_or(done < my_total)) {
        for (uint32_t r = 0; r < rlen && done < my_total; r++) {
            const uint32_t s = done % NS;
            mbar_wait(&wbar[s], (done / NS) & 1u);
            const uint4 mt = wmeta[s];
            const float4 cp = cpar[mt.x];
            const uint32_t pos = mt.y, n = mt.z, csh = mt.w & 0xffu, esh = mt.w >> 8;
            const float2 av2 = make_float2(cp.x, cp.x), Bc2 = make_float2(cp.y, cp.y), cv2 = make_float2(cp.z, cp.z);
            const unsigned char* st = wring + s * P::STAGE_B;
            const uint32_t* els = reinterpret_cast<const uint32_t*>(st + P::CODE_B) + esh;
            uint32_t cw[U][NW];
            uint32_t lb[U];
            float ev[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t idx = u * 32 + lane;  // entries >= n hold stale bytes; masked below
                load_code_smem<M>(st + (csh + idx) * M, cw[u]);
                const uint32_t le = els[idx];
                lb[u] = le & 0xffu;
                ev[u] = __uint_as_float(le & ~0xffu);
            }
            const uint64_t tau = *reinterpret_cast<volatile unsigned long long*>(&s_tau);
            const float taud = tau == ~0ull ? __int_as_float(0x7f800000) : key_dist(tau);
            uint32_t tk = 0;
            float dist[U];
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                dist[u] = dist[u + 1] = __int_as_float(0x7fffffff);
                if (u * 32 < n) {  // warp-uniform: skip fully empty pairs
                    const float2 lam = __ffma2_rn(make_float2((float)lb[u], (float)lb[u + 1]), delta2, lam02);
                    const float2 t1 = __ffma2_rn(lam, __ffma2_rn(lam, cv2, Bc2), av2);
                    const float2 te = __fadd2_rn(t1, make_float2(ev[u], ev[u + 1]));
                    float2 d;
                    if constexpr (LM == 1) {
                        uint32_t i0 = 0, i1 = 0;
#pragma unroll
                        for (int p = 0; p < M; p++) {
                            i0 += lut8_at<M>(lut, cw[u], p);
                            i1 += lut8_at<M>(lut, cw[u + 1], p);
                        }
                        d = __ffma2_rn(qs2, make_float2((float)i0, (float)i1), __fadd2_rn(te, qc2));
                    } else {
                        float2 sm = make_float2(lut_at<M>(lut, cw[u], 0), lut_at<M>(lut, cw[u + 1], 0));
#pragma unroll
                        for (int p = 1; p < M; p++)
                            sm = __fadd2_rn(sm, make_float2(lut_at<M>(lut, cw[u], p), lut_at<M>(lut, cw[u + 1], p)));
                        d = __ffma2_rn(m2, sm, te);
                    }
                    dist[u] = d.x;
                    dist[u + 1] = d.y;
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t idx = u * 32 + lane;
                if (idx < n && dist[u] <= taud) {
                    uint32_t ub = __float_as_uint(dist[u]);
                    ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;
                    const uint64_t key = ((uint64_t)ub << 32) | (pos + idx);
                    if (key < tau) tk |= 1u << u;
                }
            }
            const uint32_t any = __ballot_sync(0xffffffffu, tk != 0);
            if (any) {
                uint32_t wtot = 0;
                uint32_t bal[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    bal[u] = __ballot_sync(0xffffffffu, (tk >> u) & 1u);
                    wtot += __popc(bal[u]);
                }
                uint32_t base = 0;
                if (lane == 0) {
                    unsigned int cur = *reinterpret_cast<volatile unsigned int*>(&s_count);
                    base = 0xffffffffu;
                    while (cur + wtot <= cap) {
                        const unsigned int prev = atomicCAS(&s_count, cur, cur + wtot);
                        if (prev == cur) {
                            base = cur;
                            break;
                        }
                        cur = prev;
                    }
                }
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base == 0xffffffffu) break;  // buffer full: redo this chunk (still staged) after the flush
                const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if ((tk >> u) & 1u) {
                        uint32_t ub = __float_as_uint(dist[u]);
                        ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;
                        cbuf[base + __popc(bal[u] & lt)] = ((uint64_t)ub << 32) | (pos + u * 32 + lane);
                    }
                    base += __popc(bal[u]);
                }
            }
            __syncwarp();  // every lane has read slot s: refill it
            if (lane == 0 && done + NS < my_total) fill(done + NS);
            done++;
        }
        __syncthreads();
        n_seen += rlen * NWARPS * CH;
        const uint32_t cnt = s_count;
        if (cnt > keep && cnt > cap / 2) {  // block-uniform
            const uint64_t T = block_select_keep(cbuf, cnt, keep, hist, s_misc, a.sel_agg);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_count = keep;
                s_tau = T + 1;
            }
            __syncthreads();
        }
        const uint32_t free_slots = cap - s_count;
        const uint64_t per_chunk_round = (uint64_t)NWARPS * CH;
        uint64_t rn = (s_tau == ~0ull) ? free_slots / per_chunk_round
                                       : ((uint64_t)free_slots * n_seen) / (4ull * keep * per_chunk_round);
        rlen = (uint32_t)(rn < 1 ? 1ull : (rn > 64 ? 64ull : rn));
    }
    uint32_t n = s_count;
    if (n > keep) {
        block_select_keep(cbuf, n, keep, hist, s_misc, a.sel_agg);
        n = keep;
    }
    __syncthreads();
    for (uint32_t i = n + threadIdx.x; i < keep; i += blockDim.x) cbuf[i] = ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(cbuf, keep, threadIdx.x, blockDim.x);
    uint64_t* candq = a.cand + q * keep;
    for (uint32_t i = threadIdx.x; i < keep; i += blockDim.x) candq[i] = cbuf[i];
}

}  // namespace dev

// v7 launcher: su = slots per lane (2 / 4), stages per warp and CTAs per SM
// chosen so the ring fits the shared-memory budget; false if it cannot fit
template <int M, int U, int NS, int MINB, int LM = 0>
static bool launch_bulk_cfg(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, uint32_t cap,
                            cudaStream_t st) {
    const size_t smem = dev::bulk_smem_bytes<M, U, NS, LM>(w2, cap);
    if (smem > (size_t)(228 * 1024) / MINB - 2048) return false;
    auto fn = dev::k_scan_bulk<M, U, NS, MINB, LM>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)nq, 256, smem, st>>>(a, w2, keep, cap);
    CUDA_LAUNCH_CHECK();
    return true;
}

template <int M>
static bool launch_bulk(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int cfg, cudaStream_t st) {
    const uint32_t cap = std::max<uint32_t>(a.scan_cap ? a.scan_cap : 1024u, 2 * keep + 512);
    switch (cfg) {
        case 4: return launch_bulk_cfg<M, 4, 2, 3, 1>(a, nq, w2, keep, cap, st);  // u8 LUT, 3 CTAs/SM
        case 5: return launch_bulk_cfg<M, 4, 3, 2, 1>(a, nq, w2, keep, cap, st);  // u8 LUT, 2 CTAs/SM
        case 1: return launch_bulk_cfg<M, 2, 3, 3>(a, nq, w2, keep, cap, st);
        case 2: return launch_bulk_cfg<M, 4, 2, 2>(a, nq, w2, keep, cap, st);
        case 3: return launch_bulk_cfg<M, 2, 2, 3>(a, nq, w2, keep, cap, st);
        default: return launch_bulk_cfg<M, 4, 3, 2>(a, nq, w2, keep, cap, st);
    }
}

template <int M, int R, int U>
static void launch_fast_u(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, cudaStream_t st) {
    const uint32_t nwarps = R == 2 ? 16 : 8;
    const uint32_t cap = 2048;  // block-shared candidate buffer (keys)
    const size_t smem = 4 * (size_t)dev::LutPlan<M, R>::words() + (size_t)cap * 8 + ((size_t)w2 + 1) * 4;
    auto fn = dev::k_scan_fast<M, U, R>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)nq, nwarps * 32, smem, st>>>(a, w2, keep, cap);
    CUDA_LAUNCH_CHECK();
}

template <int M, int R>
static void launch_fast_t(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int su, cudaStream_t st) {
    if (R == 0 && su == 6) launch_fast_u<M, R, 6>(a, nq, w2, keep, st);
    else if (R == 0 && su == 8) launch_fast_u<M, R, 8>(a, nq, w2, keep, st);
    else launch_fast_u<M, R, 4>(a, nq, w2, keep, st);
}

void launch_pack_eterm_lam(const float* eterm, const uint8_t* lambdas, uint64_t n, uint32_t* out, cudaStream_t st) {
    if (n == 0) return;
    dev::k_pack_eterm_lam<<<(unsigned)dev::umin64((n + 255) / 256, 4736), 256, 0, st>>>(eterm, lambdas, n, out);
    CUDA_LAUNCH_CHECK();
}

template <int M>
static void launch_fast2(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int su, int pf,
                         cudaStream_t st, int q8 = 0) {
    // block-shared candidate buffer (keys): 2048 unless the scan_cap knob says otherwise
    const uint32_t cap = std::max<uint32_t>(a.scan_cap ? a.scan_cap : 2048u, 4 * keep);
    if (q8 == 2) {  // lane-replicated u8 LUT: one CTA of 16 warps (su 6) or 8 warps (su 106) per SM
        const size_t smem = dev::lut_bytes<M>(2) + (size_t)cap * 8 + ((size_t)w2 + 1) * 4;
        if (smem > 220 * 1024) throw std::runtime_error("scan q8x32: shared memory does not fit");
        const unsigned nt = su == 106 ? 256 : 512;
        auto fn = su == 106 ? dev::k_scan_fast2<M, 6, 1, 2, 256> : dev::k_scan_fast2<M, 6, 1, 2, 512>;
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        fn<<<(unsigned)nq, nt, smem, st>>>(a, w2, keep, cap, 0u);
        CUDA_LAUNCH_CHECK();
        return;
    }
    if (q8) {  // u8 LUT: su 6 (3 CTAs/SM), 8, 104 / 106 (4 CTAs/SM)
        const size_t smem = 256 * (size_t)M + (size_t)cap * 8 + ((size_t)w2 + 1) * 4;
        auto fn = su == 8 ? dev::k_scan_fast2<M, 8, 3, 1>
                  : su == 104 ? dev::k_scan_fast2<M, 4, 4, 1>
                  : su == 106 ? dev::k_scan_fast2<M, 6, 4, 1>
                              : dev::k_scan_fast2<M, 6, 3, 1>;
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        fn<<<(unsigned)nq, 256, smem, st>>>(a, w2, keep, cap, 0u);
        CUDA_LAUNCH_CHECK();
        return;
    }
    const size_t smem = 4 * 256 * (size_t)M + (size_t)cap * 8 + ((size_t)w2 + 1) * 4;
    // su: slots per lane (4/6/8); su + 100: the same with 4 CTAs/SM register budget (64 regs)
    auto fn = su == 4 ? dev::k_scan_fast2<M, 4, 3>
              : su == 8 ? dev::k_scan_fast2<M, 8, 3>
              : su == 104 ? dev::k_scan_fast2<M, 4, 4>
              : su == 106 ? dev::k_scan_fast2<M, 6, 4>
                          : dev::k_scan_fast2<M, 6, 3>;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)nq, 256, smem, st>>>(a, w2, keep, cap, (uint32_t)pf);
    CUDA_LAUNCH_CHECK();
}

// su: entry-slots per lane per chunk (4 / 6 / 8; 6 default, measured best on deep100m)
// pf: L2 prefetch distance of the v6 scan in chunks (0 = off)
bool launch_scan_fast(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int variant, int su, int pf,
                      cudaStream_t st) {
    // variant: 0 = default (v6: packed-fp32 pairs, single-table LUT),
    // 1 = generic warp-buffer scan (not here), 2 = fully replicated LUT (v5),
    // 3 = four copies (v5), 4 = single table (v5)
    if (keep > 512 || w2 > 4096 || variant == 1) return false;
    if (((variant >= 5 && variant <= 8) || variant == 11 || variant == 12) && a.eterm_lam) {
        // v7: bulk-async staged entry stream (11 / 12: with the u8 LUT)
        if (variant >= 11) variant -= 2;
        bool ok = false;
        switch (a.m) {
            case 16: ok = launch_bulk<16>(a, nq, w2, keep, variant - 5, st); break;
            case 8: ok = launch_bulk<8>(a, nq, w2, keep, variant - 5, st); break;
            case 4: ok = launch_bulk<4>(a, nq, w2, keep, variant - 5, st); break;
            default: break;
        }
        if (ok) return true;
        variant = 0;  // the ring does not fit (very large w2): v6
    }
    if ((variant == 9 || variant == 10) && a.eterm_lam) {  // v6 with the u8-quantized LUT (10: lane-replicated)
        const int lm = variant == 9 ? 1 : 2;
        switch (a.m) {
            case 16: launch_fast2<16>(a, nq, w2, keep, su, pf, st, lm); return true;
            case 8: launch_fast2<8>(a, nq, w2, keep, su, pf, st, lm); return true;
            case 4: launch_fast2<4>(a, nq, w2, keep, su, pf, st, lm); return true;
            default: variant = 0; break;
        }
    }
    if (variant == 0) {
        switch (a.m) {
            case 16: launch_fast2<16>(a, nq, w2, keep, su, pf, st); return true;
            case 8: launch_fast2<8>(a, nq, w2, keep, su, pf, st); return true;
            case 4: launch_fast2<4>(a, nq, w2, keep, su, pf, st); return true;
            default: break;  // other m: the v5 path below (or the generic scan)
        }
    }
    const int r = variant == 2 ? 2 : (variant == 3 ? 1 : 0);  // default: single table (measured best)
#define VLQ_FAST(MM)                                                  \
    do {                                                              \
        if (r == 2) launch_fast_t<MM, 2>(a, nq, w2, keep, su, st);        \
        else if (r == 1) launch_fast_t<MM, 1>(a, nq, w2, keep, su, st);   \
        else launch_fast_t<MM, 0>(a, nq, w2, keep, su, st);               \
        return true;                                                  \
    } while (0)
    switch (a.m) {
        case 16: VLQ_FAST(16);
        case 8: VLQ_FAST(8);
        case 4: VLQ_FAST(4);
        default: return false;
    }
#undef VLQ_FAST
}

}  // namespace vlq
