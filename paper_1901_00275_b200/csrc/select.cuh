// Block- and warp-level selection primitives (top-L smallest under the
// reference's total orders).
#pragma once

#include "common.cuh"

namespace vlq {
namespace dev {

// Block-wide exclusive scan of a packed u32 (two 16-bit counters).  Returns
// the exclusive prefix for this thread; *total receives the block total.
// `ws` must hold >= 33 u32 of shared scratch.  All threads must call.
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* ws, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t nwarps = (blockDim.x + 31u) >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nwarps ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        if (lane < nwarps) ws[lane] = w;  // inclusive per-warp totals
        if (lane == nwarps - 1) ws[32] = w;
    }
    __syncthreads();
    uint32_t excl = x - v + (warp ? ws[warp - 1] : 0u);
    *total = ws[32];
    __syncthreads();
    return excl;
}

// Order-preserving key (ord_float) of the L-th smallest of vals[0..len)
// (1 <= L <= len): radix select in three digit passes (11/11/10 bits).
// *rank_in_key receives how many keys equal to the result belong to the L
// smallest.  Shared scratch: hist[2048] + scan[40].  All threads call.
__device__ __noinline__ static uint32_t block_kth_ord(const float* __restrict__ vals, uint32_t len, uint32_t L,
                                                      uint32_t* hist, uint32_t* scan, uint32_t* rank_in_key) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint32_t prefix = 0, pmask = 0, remaining = L;  // remaining: 1-based rank inside the prefix group
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; pass++) {
        const int sh = shifts[pass];
        const uint32_t nb = 1u << widths[pass], dmask = nb - 1u;
        for (uint32_t b = tid; b < nb; b += nt) hist[b] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < len; i += nt) {
            uint32_t k = ord_float(vals[i]);
            if ((k & pmask) == prefix) atomicAdd(&hist[(k >> sh) & dmask], 1u);
        }
        __syncthreads();
        // exclusive scan of the histogram, 'per' bins per thread
        const uint32_t per = (nb + nt - 1) / nt;
        uint32_t local = 0;
        for (uint32_t b = tid * per; b < min(nb, (tid + 1) * per); b++) local += hist[b];
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, scan, &total);
        // the bin where the cumulative count crosses `remaining`
        for (uint32_t b = tid * per; b < min(nb, (tid + 1) * per); b++) {
            uint32_t h = hist[b];
            if (run < remaining && remaining <= run + h) {
                scan[34] = b;
                scan[35] = run;
            }
            run += h;
        }
        __syncthreads();
        const uint32_t bsel = scan[34];
        remaining -= scan[35];
        prefix |= bsel << sh;
        pmask |= dmask << sh;
        __syncthreads();
    }
    *rank_in_key = remaining;
    return prefix;
}

// Selects the L smallest of vals[0..len) under the order (value, position)
// -- the reference's (dist, id) comparator when position == id
// (proj/src/search.cpp:28-33) -- and writes their positions to out[0..L) in
// ASCENDING position order: the L-th smallest key T (block_kth_ord), then one
// ordered collection pass that keeps every key < T and the first r keys == T
// in position order.  Shared scratch: hist[2048] + scan[40].  All threads of
// the block call.
__device__ __noinline__ static void block_select_ordered(const float* __restrict__ vals, uint32_t len, uint32_t L,
                                     uint32_t* __restrict__ out, uint32_t* hist, uint32_t* scan) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    if (L >= len) {
        for (uint32_t i = tid; i < len; i += nt) out[i] = i;
        return;
    }
    uint32_t remaining;
    const uint32_t prefix = block_kth_ord(vals, len, L, hist, scan, &remaining);
    const uint32_t T = prefix;  // exact key of the L-th smallest value
    const uint32_t r = remaining;  // how many keys == T to take (in position order)
    uint32_t lt_run = 0, eq_run = 0;
    for (uint32_t base = 0; base < len; base += nt) {
        uint32_t i = base + tid;
        uint32_t k = i < len ? ord_float(vals[i]) : 0xffffffffu;
        uint32_t lt = (i < len && k < T) ? 1u : 0u;
        uint32_t eq = (i < len && k == T) ? 1u : 0u;
        uint32_t total;
        uint32_t ex = block_excl_scan_u32(lt | (eq << 16), scan, &total);
        uint32_t lt_before = lt_run + (ex & 0xffffu);
        uint32_t eq_before = eq_run + (ex >> 16);
        if (lt || (eq && eq_before < r)) out[lt_before + min(eq_before, r)] = i;
        lt_run += total & 0xffffu;
        eq_run += total >> 16;
    }
}

// The same selection (L smallest of vals[0..len) by (value, position), output
// positions ascending) with far fewer block barriers, for the fused coarse
// stage's small selections (~10^3 values): min / max, ONE histogram of 1024
// equal-width bins over [min, max] (a monotone binning, so every value in a
// lower bin is strictly smaller), the crossing bin b, then the members of bin
// b ranked exactly by (value, position) (counting, at most 256 of them) and
// one ordered compaction.  Falls back to block_select_ordered when bin b
// holds more than 256 values (e.g. massive ties).  Scratch: hist >= 1024 +
// 256 words, scan[40].  All threads of the block call.
__device__ __noinline__ static void block_select_ordered_range(const float* __restrict__ vals, uint32_t len,
                                                               uint32_t L, uint32_t* __restrict__ out,
                                                               uint32_t* hist, uint32_t* scan) {
    constexpr uint32_t NB = 1024, MAXB = 256;
    const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31u;
    if (L >= len) {
        for (uint32_t i = tid; i < len; i += nt) out[i] = i;
        return;
    }
    uint32_t* memb = hist + NB;  // crossing-bin members (positions), then their ranks
    const float INF = __int_as_float(0x7f800000);
    float mn = INF, mx = -INF;
    for (uint32_t i = tid; i < len; i += nt) {
        const float v = vals[i];
        mn = fminf(mn, v);
        if (v < INF) mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    for (uint32_t b = tid; b < NB; b += nt) hist[b] = 0;
    if (tid == 0) {
        scan[36] = 0xffffffffu;
        scan[37] = 0u;
        scan[38] = 0u;
    }
    __syncthreads();
    if (lane == 0) {
        atomicMin(&scan[36], ord_float(mn));
        atomicMax(&scan[37], ord_float(mx));
    }
    __syncthreads();
    const float lo = unord_float(scan[36]), hi = fmaxf(unord_float(scan[37]), lo);
    const float inv = hi > lo ? (float)(NB - 1) / (hi - lo) : 0.0f;
    auto bin_of = [&](float x) -> uint32_t {
        const float t = (fmaxf(x, lo) - lo) * inv;  // monotone in x
        return t < (float)(NB - 1) ? (uint32_t)t : NB - 1;  // +inf / NaN -> the last bin
    };
    for (uint32_t i = tid; i < len; i += nt) atomicAdd(&hist[bin_of(vals[i])], 1u);
    __syncthreads();
    const uint32_t per = (NB + nt - 1) / nt;
    {
        uint32_t local = 0;
        for (uint32_t b = tid * per; b < min(NB, (tid + 1) * per); b++) local += hist[b];
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, scan, &total);
        for (uint32_t b = tid * per; b < min(NB, (tid + 1) * per); b++) {
            if (run < L && L <= run + hist[b]) {
                scan[34] = b;
                scan[35] = run;
            }
            run += hist[b];
        }
    }
    __syncthreads();
    const uint32_t bsel = scan[34], before = scan[35], hb = hist[bsel];
    if (hb > min(MAXB, nt)) {  // block-uniform
        __syncthreads();
        block_select_ordered(vals, len, L, out, hist, scan);
        return;
    }
    const uint32_t r = L - before;  // members of bin b to take, by (value, position)
    for (uint32_t i = tid; i < len; i += nt)
        if (bin_of(vals[i]) == bsel) memb[atomicAdd(&scan[38], 1u)] = i;
    __syncthreads();
    // rank of member t among the members by (value, position); taken iff rank < r
    uint32_t take_pos = 0xffffffffu;
    if (tid < hb) {
        const uint32_t pi = memb[tid];
        const uint32_t ki = ord_float(vals[pi]);
        uint32_t rank = 0;
        for (uint32_t u = 0; u < hb; u++) {
            const uint32_t pu = memb[u];
            const uint32_t ku = ord_float(vals[pu]);
            rank += (ku < ki || (ku == ki && pu < pi)) ? 1u : 0u;
        }
        if (rank < r) take_pos = pi;
    }
    __syncthreads();
    if (tid < hb) memb[tid] = take_pos;  // the taken members' positions (others: ~0)
    __syncthreads();
    // ordered compaction: contiguous position ranges per thread
    const uint32_t pp = (len + nt - 1) / nt;
    const uint32_t i0 = min(len, tid * pp), i1 = min(len, i0 + pp);
    auto taken = [&](uint32_t i) -> bool {
        const uint32_t b = bin_of(vals[i]);
        if (b != bsel) return b < bsel;
        for (uint32_t u = 0; u < hb; u++)
            if (memb[u] == i) return true;
        return false;
    };
    uint32_t mine = 0;
    for (uint32_t i = i0; i < i1; i++) mine += taken(i) ? 1u : 0u;
    uint32_t total;
    uint32_t slot = block_excl_scan_u32(mine, scan, &total);
    for (uint32_t i = i0; i < i1; i++)
        if (taken(i)) out[slot++] = i;
}

// In-shared-memory bitonic sort (ascending) of n = power of two u64 keys by
// the calling threads [t0, t0+nthreads).  `sync` is either a warp or block
// barrier supplied by the caller through the template parameter.
template <bool kWarpOnly>
__device__ __forceinline__ void bitonic_sort_u64(uint64_t* a, uint32_t n, uint32_t t, uint32_t nthreads) {
    for (uint32_t size = 2; size <= n; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t p = t; p < (n >> 1); p += nthreads) {
                uint32_t lo = 2 * p - (p & (stride - 1));
                uint32_t hi = lo + stride;
                bool up = ((lo & size) == 0);
                uint64_t x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            if (kWarpOnly) __syncwarp();
            else __syncthreads();
        }
    }
}

}  // namespace dev
}  // namespace vlq
