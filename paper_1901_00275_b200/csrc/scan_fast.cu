// Fused PQ-ADC list scan, fast path (K4 of DESIGN.md; search.cpp:92-120,
// 154-162 + select_topk :122-140).
//
// One CTA (6 warps, 4 CTAs per SM; 8 x 3 for the retry) per query.  The query's selected cells are
// cut into chunks of 32 U entries (chunks never straddle cells); a block
// prefix over the chunk counts gives every warp a balanced contiguous chunk
// range.  Per entry (lane-parallel, every load warp-coalesced: 16 B code and
// one 4-byte word (bits(e) & ~0xff) | lambda byte):
//     lambda = lambda0 + b * delta          term1 = A + lambda (B + lambda C)   (per-cell A, B, C)
//     sum5   = sum_p LUT[p][code_p]         dist  = (term1 + e) - 2 sum5
// A lane takes its entries in pairs on the sm_100 packed fp32 pipe
// (FFMA2 / FADD2), each element with the scalar rounding of the reference-
// order formula above, so k_rescore's certificate bounds |fast - exact|.
// Keys (dist, entry position) below the block threshold go to ONE block-shared
// candidate buffer; at round boundaries the buffer is cut to the k' smallest
// keys by a block radix select and the threshold tightens.  No candidate list
// reaches HBM; ids are read only for the k' survivors (k_rescore).

#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

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
    } else {
        static_assert(M == 4, "fast scan: m in {4, 8, 16}");
        w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
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


__global__ void k_pack_eterm_lam(const float* __restrict__ eterm, const uint8_t* __restrict__ lambdas, uint64_t n,
                                 uint32_t* __restrict__ out) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
        out[e] = (__float_as_uint(eterm[e]) & ~0xffu) | (uint32_t)lambdas[e];
}

// LUT[p][code_p]: one PRMT extracts the byte, one IMAD forms byte * 4 + table
// base, the LDS carries p * 1 KB as its immediate -- 3 instructions per lookup
// (bytes 0 and 3 written as AND / shift compiled to 4)
template <int M>
__device__ __forceinline__ float lut_at(const unsigned char* lut, const uint32_t (&w)[(M + 3) / 4], int p) {
    const uint32_t word = w[p >> 2];
    const int k = p & 3;
    const uint32_t b = __byte_perm(word, 0u, 0x4440u + k);  // PRMT, then one IMAD (b * 4 + table base)
    return reinterpret_cast<const float*>(lut)[p * 256 + b];
}

__device__ __forceinline__ float key_dist(uint64_t key) {  // distance of an order-preserving key (upper 32 bits)
    const uint32_t ub = (uint32_t)(key >> 32);
    return __uint_as_float((ub & 0x80000000u) ? (ub & 0x7fffffffu) : ~ub);
}

constexpr uint32_t SCAN_STAGE_MAX = 1024;  // selected cells per query whose parameters are staged in shared memory

template <int M, int U, int MINB, int NT = 256>
__global__ void __launch_bounds__(NT, MINB) k_scan_fast2(SearchArgs a, uint32_t w2, uint32_t keep, uint32_t cap) {
    static_assert(U % 2 == 0, "entries are processed in pairs");
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NW = (M + 3) / 4;
    constexpr uint32_t CH = 32 * U;  // entries per chunk
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;

    const uint32_t _nb = a.qlist ? *a.qcount : gridDim.x;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint64_t q = a.qlist ? a.qlist[_b] : _b;
    // the query's table (16 KB at m = 16) in static shared memory
    __shared__ __align__(16) float s_lut[256 * M];
    unsigned char* lut = reinterpret_cast<unsigned char*>(s_lut);
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(smem);                 // cap keys
    uint32_t* cpref = reinterpret_cast<uint32_t*>(cbuf + cap);         // w2 + 1
    __shared__ uint32_t hist[256];
    __shared__ unsigned int s_misc[48];
    __shared__ unsigned int s_count;
    __shared__ unsigned long long s_tau;

    // 1. the query's term5 table (one copy per sub-space)
    if (a.code_perm) {  // relabeled scan codes: LUT[p][perm[p][c]] = term5[p][c]
        const float4* t5q = reinterpret_cast<const float4*>(a.t5 + q * M * VLQ_KSUB);
        const uint32_t* pq4 = reinterpret_cast<const uint32_t*>(a.code_perm);
        float* lf = reinterpret_cast<float*>(lut);
        for (uint32_t i = threadIdx.x; i < 64u * M; i += blockDim.x) {  // 4 values + their 4 slots per load
            const float4 v = __ldg(t5q + i);
            const uint32_t pw = __ldg(pq4 + i), b = (i * 4) & ~255u;
            lf[b | (pw & 0xffu)] = v.x;
            lf[b | ((pw >> 8) & 0xffu)] = v.y;
            lf[b | ((pw >> 16) & 0xffu)] = v.z;
            lf[b | (pw >> 24)] = v.w;
        }
    } else {
        const float4* t5q = reinterpret_cast<const float4*>(a.t5 + q * M * VLQ_KSUB);
        for (uint32_t i = threadIdx.x; i < 64u * M; i += blockDim.x) reinterpret_cast<float4*>(lut)[i] = __ldg(t5q + i);
    }
    // 2. chunk prefix over the selected cells (chunks never straddle cells)
    const uint32_t* selq = a.sel + q * w2;
    const float* wsq = a.ws + q * a.k;
    // per-cell parameters staged once per query (all threads, loads in
    // parallel) instead of a dependent global-load chain whenever a warp
    // enters a cell: list start, length, a = |y - c_i|^2, B = (b - a) - c, c
    const bool staged = w2 <= SCAN_STAGE_MAX;
    uint32_t* p_pos = cpref + w2 + 1;
    uint32_t* p_len = p_pos + w2;
    float* p_av = reinterpret_cast<float*>(p_len + w2);
    float* p_bc = p_av + w2;
    float* p_cv = p_bc + w2;
    if (staged) {
        for (uint32_t t = threadIdx.x; t < w2; t += blockDim.x) {
            const uint32_t cell = selq[t];
            const uint64_t b0 = a.list_off[cell];
            const float av = wsq[cell / a.n];
            const float bv = wsq[a.nbr[cell]];
            const float cv = a.elen[cell];
            p_pos[t] = (uint32_t)b0;
            p_len[t] = (uint32_t)(a.list_off[cell + 1] - b0);
            p_av[t] = av;
            p_bc[t] = (bv - av) - cv;
            p_cv[t] = cv;
        }
    }
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
        if (t != loaded_t && staged) {
            loaded_t = t;
            L = p_len[t];
            pos0 = p_pos[t];
            const float av = p_av[t], bc = p_bc[t], cv = p_cv[t];
            av2 = make_float2(av, av);
            Bc2 = make_float2(bc, bc);
            cv2 = make_float2(cv, cv);
            codes_c = (a.scodes ? a.scodes : a.codes) + (uint64_t)pos0 * M;
            lam_c = a.lambdas + pos0;
            e_c = a.eterm + pos0;
            if (packed) el_c = a.eterm_lam + pos0;
        } else if (t != loaded_t) {
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
            codes_c = (a.scodes ? a.scodes : a.codes) + b0 * M;
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
            uint32_t cw[U][NW];
            uint32_t lb[U];
            float ev[U];
            // (warp-uniform variants hoisted out of the slot loop so each
            // issues its U x 2-3 loads back to back)
            if (packed) {  // one 4-byte word: e-term (low 8 mantissa bits dropped) | lambda byte
                uint32_t le[U];
                if (o + CH <= L) {  // warp-uniform: a whole chunk, one base address + immediate offsets
                    const uint8_t* cb = codes_c + (size_t)(o + lane) * M;
                    const uint32_t* eb = el_c + o + lane;
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        load_code_vec<M>(cb + u * 32 * M, cw[u]);
                        le[u] = __ldg(eb + u * 32);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const uint32_t ic = min(o + u * 32 + lane, L - 1);  // clamped: the tail re-reads entry L-1
                        load_code_vec<M>(codes_c + (size_t)ic * M, cw[u]);
                        le[u] = __ldg(el_c + ic);
                    }
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
                    float2 s = make_float2(lut_at<M>(lut, cw[u], 0), lut_at<M>(lut, cw[u + 1], 0));
#pragma unroll
                    for (int p = 1; p < M; p++)
                        s = __fadd2_rn(s, make_float2(lut_at<M>(lut, cw[u], p), lut_at<M>(lut, cw[u + 1], p)));
                    const float2 d = __ffma2_rn(m2, s, te);
                    dist[u] = d.x;
                    dist[u + 1] = d.y;
                }
            }
            bool near = false;  // any of the lane's entries at or below the threshold distance
#pragma unroll
            for (int u = 0; u < U; u++) near |= (o + u * 32 + lane < L) & (dist[u] <= taud);
            if (__any_sync(0xffffffffu, near)) {  // rare after the first rounds: exact key test
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t idx = o + u * 32 + lane;
                    if (idx < L && dist[u] <= taud) {
                        uint32_t ub = __float_as_uint(dist[u]);
                        ub ^= (uint32_t)((int32_t)ub >> 31) | 0x80000000u;  // order-preserving
                        const uint64_t key = ((uint64_t)ub << 32) | (pos0 + idx);
                        if (key < tau) tk |= 1u << u;
                    }
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
        const uint64_t rcap = a.round_cap ? a.round_cap : 32u;
        rlen = (uint32_t)(rn < 1 ? 1ull : (rn > rcap ? rcap : rn));
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
    uint64_t* candq = a.cand + (a.qlist ? (uint64_t)_b : q) * keep;
    for (uint32_t i = threadIdx.x; i < keep; i += blockDim.x) candq[i] = cbuf[i];
    __syncthreads();  // shared memory is reused by the next query
    }
}


}  // namespace dev

void launch_pack_eterm_lam(const float* eterm, const uint8_t* lambdas, uint64_t n, uint32_t* out, cudaStream_t st) {
    if (n == 0) return;
    dev::k_pack_eterm_lam<<<(unsigned)dev::umin64((n + 255) / 256, 4736), 256, 0, st>>>(eterm, lambdas, n, out);
    CUDA_LAUNCH_CHECK();
}

template <int M>
static void launch_fast2(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int su, cudaStream_t st) {
    // block-shared candidate buffer (keys): 2048 unless the scan_cap knob says otherwise
    const uint32_t cap = std::max<uint32_t>(a.scan_cap ? a.scan_cap : 2048u, 4 * keep);
    // + the static 4 * 256 * M B table; + 20 B per selected cell of staged parameters
    const size_t smem = (size_t)cap * 8 + ((size_t)w2 + 1) * 4 + (w2 <= dev::SCAN_STAGE_MAX ? (size_t)w2 * 20 : 0);
    // su: slots per lane (4 / 6 / 8); su + 100: the same with 4 CTAs/SM register budget (64 regs)
    // 306: 6 slots, 6 warps per CTA, 4 CTAs (queries) per SM at 80 registers -- the
    // same 24 warps per SM as 8 x 3, spread over 4 queries instead of 3
    // (measured: 16.40 vs 16.51 ms at C4, -2.6 to -5.3% at C1-C3; 5 x 5 and
    // 4 x 6 were slower, profiles/r2_study_occ_c4.jsonl; 6 x 5 at 64 registers
    // spills and was 25% slower, profiles/r2_study_scan_6x5_c4.jsonl)
    auto fn = su == 4 ? dev::k_scan_fast2<M, 4, 3>
              : su == 8 ? dev::k_scan_fast2<M, 8, 3>
              : su == 104 ? dev::k_scan_fast2<M, 4, 4>
              : su == 106 ? dev::k_scan_fast2<M, 6, 4>
              : su == 306 ? dev::k_scan_fast2<M, 6, 4, 192>
                          : dev::k_scan_fast2<M, 6, 3>;
    const int threads = su == 306 ? 192 : 256;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<list_grid(nq, a.qlist != nullptr && !a.qorder), threads, smem, st>>>(a, w2, keep, cap);
    CUDA_LAUNCH_CHECK();
}

// The fused fast scan for m in {4, 8, 16} on the packed e-term | lambda stream
// (or the separate arrays); false when it does not apply (other m, w2 > 4096,
// k' > 512): the engine then runs the generic warp-buffer scan.
bool launch_scan_fast(const SearchArgs& a, uint64_t nq, uint32_t w2, uint32_t keep, int slots, cudaStream_t st) {
    if (keep > 512 || w2 > 4096) return false;
    switch (a.m) {
        case 16: launch_fast2<16>(a, nq, w2, keep, slots, st); return true;
        case 8: launch_fast2<8>(a, nq, w2, keep, slots, st); return true;
        case 4: launch_fast2<4>(a, nq, w2, keep, slots, st); return true;
        default: return false;
    }
}

}  // namespace vlq
