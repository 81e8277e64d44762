// K1: query/point -> first-level-centroid distances on the 5th-gen tensor
// cores (tcgen05.mma kind::tf32, fp32 accumulators in TMEM).
//
//   approx(x, c) = |c|^2 - 2 <x, c>        (|x|^2 is row-constant, omitted)
//
// One CTA per 128 rows of X.  X's tile stays resident in shared memory; the
// centroid matrix streams through a 3-stage ring of 128-centroid tiles
// (cp.async.bulk into mbarrier-tracked stages).  The centroids are stored
// once, at model upload, in the UMMA K-major "interleaved" core-matrix layout
// ([tile][row/8][k/4][row%8][4 floats]), so every stage is ONE contiguous bulk
// copy.  Warp 0 = producer, warp 1 = MMA issuer (one elected lane, 12
// tcgen05.mma per tile at D = 96), warps 2..9 = epilogue (TMEM lane quadrant =
// warp % 4, two warps per quadrant split the 128 accumulator columns); TMEM
// holds two 128-column accumulators so tile t+1's MMAs overlap tile t's
// epilogue.
//
// Epilogues:  ARGMIN keeps each row's 4 smallest (approx, centroid) pairs
// (add path: assign_point, index.cpp:86-106);  STORE writes the approximate
// row (coarse search stage: first_level_scan, search.cpp:11-36).  Neither is
// the final answer: the refine kernels recompute exact reference-order
// distances for every candidate within the TF32 error bound of the best and
// certify that no other centroid can win (else an exact CUDA-core fallback).
#include <algorithm>
#include <cfloat>
#include <stdexcept>

#include "async.cuh"
#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

constexpr int TC_M = 128;      // rows of X per CTA (UMMA M)
constexpr int TC_N = 128;      // centroids per tile (UMMA N)
constexpr int TC_THREADS = 320;  // 10 warps

// bulk copy of any size: cp.async.bulk takes < 64 KB per instruction (a 64 KB
// centroid tile at D = 128 must be split)
__device__ __forceinline__ void bulk_g2s_any(unsigned char* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const unsigned char* s = static_cast<const unsigned char*>(src);
    for (uint32_t off = 0; off < bytes; off += 32768u)
        bulk_g2s(dst + off, s + off, min(32768u, bytes - off), bar);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE K-major canonical layout, Blackwell descriptor version 1
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int TC_MAX_STAGES = 4;  // centroid-tile ring depth: as many as fit in 227 KB, 2 to 4
// (a template parameter: a runtime ring depth made nvcc 12.9 drop the high
// half of the bulk-copy source address in the producer loop)

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// SPLIT = 3xTF32: x = hi + lo with hi = tf32(x); <x, c> ~= hi.hi + hi.lo + lo.hi
// (error ~2^-21 relative instead of 2^-9), three MMAs per K step, 64-centroid tiles.
// MODE 2 = TILEMIN: per row, the min of every 32-centroid column chunk
//   (out_row[row * ldo + chunk]).  The L-th smallest chunk minimum bounds the
//   row's L-th smallest value from above (L distinct elements lie below it).
// MODE 4 = TILEMIN8: per row, the min of every 8-centroid column chunk
//   (out_row[row * ldo + centroid / 8]); the chunk-select search path.
// MODE 3 = FILTER: per row, append every (approx, centroid) with approx <=
//   tau[row] to the row's candidate list (top_d/top_idx, capacity cap,
//   count in cnt[row]).
// PERSIST (search modes 1-3): a persistent grid of one CTA per SM walks a
// balanced contiguous range of (row block, centroid tile) units, so the
// nq = 10k batch (79 row blocks) keeps all 148 SMs busy.  Rows come
// pre-laid-out in the UMMA layout (Xtc / Xlo_tc, k_relayout_centroids); the
// producer bulk-copies a row block's A tile whenever the range enters a new
// one, after the MMA warp's commit on `aempty` shows the old A is consumed.
template <int MODE, bool SPLIT, int TC_STAGES, bool PERSIST>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_coarse_tc(const float* __restrict__ X, uint64_t nx, uint32_t dim, const float* __restrict__ cent_tc,
                const float* __restrict__ cent_lo, const float* __restrict__ cnorm_pad, uint32_t ntiles,
                uint32_t kvalid, float* __restrict__ out_row, uint64_t ldo, uint32_t* __restrict__ top_idx,
                float* __restrict__ top_d, const float* __restrict__ tau, uint32_t* __restrict__ cnt, uint32_t cap,
                const float* __restrict__ Xtc, const float* __restrict__ Xlo_tc, uint32_t nrb) {
    extern __shared__ __align__(128) unsigned char smem[];
    static_assert(!PERSIST || MODE != 0, "ARGMIN merges per row block: not persistent");
    constexpr int TN = SPLIT ? 64 : TC_N;  // centroids per tile (UMMA N)
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t tile_bytes = TN * dim * 4;  // one centroid tile (one precision)
    const uint32_t a_bytes = TC_M * dim * 4;
    unsigned char* sA = smem;
    unsigned char* sAlo = smem + a_bytes;  // SPLIT only
    constexpr int NB = SPLIT ? 2 : 1;
    // Ring stage = tile_bytes.  1xTF32: one whole centroid tile.  3xTF32: one
    // K half of a tile, hi and lo halves side by side (the centroids are laid
    // out as [tile][K half][row/8][k/4][row%8][4], k_relayout_khalf), so twice
    // as many stages are in flight and D = 128 fits beside its 128 KB A tile.
    const uint32_t half_bytes = tile_bytes / 2;
    unsigned char* sB = smem + a_bytes * NB;                              // STAGES x tile_bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + TC_STAGES * tile_bytes);
    uint64_t* full = bars;                   // [STAGES]
    uint64_t* empty = bars + TC_STAGES;      // [STAGES]
    uint64_t* tfull = bars + 2 * TC_STAGES;  // [2]
    uint64_t* tempty = tfull + 2;            // [2]
    uint64_t* afull = tempty + 2;            // A tile landed (PERSIST)
    uint64_t* aempty = afull + 1;            // A tile consumed by every MMA (PERSIST)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
    float* sMerge = reinterpret_cast<float*>(tmem_slot + 4);  // ARGMIN: 128 x 4 d + 128 x 4 idx; STORE: 8 x 32 x 33 transpose

    // unit u = rb * ntiles + t; this CTA's contiguous range [u0, u1)
    uint64_t u0, u1;
    if constexpr (PERSIST) {
        const uint64_t U = (uint64_t)nrb * ntiles;
        u0 = U * blockIdx.x / gridDim.x;
        u1 = U * (blockIdx.x + 1) / gridDim.x;
    } else {
        u0 = (uint64_t)blockIdx.x * ntiles;
        u1 = u0 + ntiles;
    }
    const uint32_t nchunk = dim / 4;  // 16-byte chunks per row
    if constexpr (!PERSIST) {
        // ---- A tile: row-major global -> interleaved K-major smem (all threads)
        const uint64_t row0 = (uint64_t)blockIdx.x * TC_M;
        for (uint32_t t = threadIdx.x; t < TC_M * nchunk; t += blockDim.x) {
            const uint32_t r = t / nchunk, c = t % nchunk;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row0 + r < nx) v = __ldg(reinterpret_cast<const float4*>(X + (row0 + r) * dim) + c);
            const uint32_t off = (r >> 3) * (nchunk * 128) + c * 128 + (r & 7) * 16;
            if constexpr (SPLIT) {
                const float4 hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
                *reinterpret_cast<float4*>(sA + off) = hi;
                *reinterpret_cast<float4*>(sAlo + off) = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
            } else if constexpr (MODE == 4) {  // the chunk-select bound assumes TF32-exact (RNA) operands
                *reinterpret_cast<float4*>(sA + off) =
                    make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
            } else {
                *reinterpret_cast<float4*>(sA + off) = v;
            }
        }
    }
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < TC_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);
        }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: two 128-column fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));  // >= 2 x TN
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A tile -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: (A tiles +) centroid tiles -> smem ring
        if (lane == 0) {
            uint32_t cur_rb = 0xffffffffu, aloads = 0;
            for (uint64_t u = u0; u < u1; u++) {
                const uint32_t i = (uint32_t)(u - u0);
                const uint32_t t = (uint32_t)(u % ntiles);
                if constexpr (PERSIST) {
                    const uint32_t rb = (uint32_t)(u / ntiles);
                    if (rb != cur_rb) {
                        if (aloads > 0) mbar_wait(aempty, (aloads - 1) & 1u);
                        mbar_expect_tx(afull, NB * a_bytes);
                        bulk_g2s_any(sA, Xtc + (size_t)rb * TC_M * dim, a_bytes, afull);
                        if constexpr (SPLIT) bulk_g2s_any(sAlo, Xlo_tc + (size_t)rb * TC_M * dim, a_bytes, afull);
                        cur_rb = rb;
                        aloads++;
                    }
                }
                if constexpr (SPLIT) {
                    for (uint32_t h = 0; h < 2; h++) {
                        const uint32_t i2 = 2 * i + h;
                        const uint32_t s = i2 % TC_STAGES, ph = (i2 / TC_STAGES) & 1u;
                        mbar_wait(&empty[s], ph ^ 1u);
                        mbar_expect_tx(&full[s], tile_bytes);
                        const size_t src = ((size_t)t * 2 + h) * (TN * dim / 2);
                        bulk_g2s_any(sB + s * tile_bytes, cent_tc + src, half_bytes, &full[s]);
                        bulk_g2s_any(sB + s * tile_bytes + half_bytes, cent_lo + src, half_bytes, &full[s]);
                    }
                } else {
                    const uint32_t s = i % TC_STAGES, ph = (i / TC_STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_expect_tx(&full[s], tile_bytes);
                    bulk_g2s_any(sB + s * tile_bytes, cent_tc + (size_t)t * TN * dim, tile_bytes, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) |
                               ((uint32_t)(TC_M >> 4) << 24);
        const uint32_t sbo = nchunk * 128, lbo = 128;
        const uint32_t a_addr = smem_u32(sA);
        uint32_t cur_rb = 0xffffffffu, aloads = 0;
        for (uint64_t u = u0; u < u1; u++) {
            const uint32_t i = (uint32_t)(u - u0);
            if constexpr (PERSIST) {
                const uint32_t rb = (uint32_t)(u / ntiles);
                if (rb != cur_rb) {
                    if (aloads > 0 && lane == 0) umma_commit(aempty);  // fires when the old A's MMAs are done
                    __syncwarp();
                    mbar_wait(afull, aloads & 1u);
                    cur_rb = rb;
                    aloads++;
                }
            }
            const uint32_t b = i & 1u, bph = (i >> 1) & 1u;
            mbar_wait(&tempty[b], bph ^ 1u);
            if constexpr (SPLIT) {
                const uint32_t sbo_b = (nchunk / 2) * 128;  // row-group stride inside a K half
                const uint32_t kh = dim / 16;               // MMAs (K = 8) per K half
                for (uint32_t h = 0; h < 2; h++) {
                    const uint32_t i2 = 2 * i + h;
                    const uint32_t s = i2 % TC_STAGES, ph = (i2 / TC_STAGES) & 1u;
                    mbar_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (lane == 0) {
                        const uint32_t b_addr = smem_u32(sB + s * tile_bytes);
                        for (uint32_t kk = 0; kk < kh; kk++) {
                            const uint32_t k = h * kh + kk;
                            const uint64_t ad = umma_desc(a_addr + k * 256, lbo, sbo);
                            const uint64_t al = umma_desc(smem_u32(sAlo) + k * 256, lbo, sbo);
                            const uint64_t bd = umma_desc(b_addr + kk * 256, lbo, sbo_b);
                            const uint64_t bl = umma_desc(b_addr + half_bytes + kk * 256, lbo, sbo_b);
                            umma_tf32(tmem_base + b * TN, ad, bd, idesc, k > 0 ? 1u : 0u);  // hi . hi
                            umma_tf32(tmem_base + b * TN, ad, bl, idesc, 1u);               // hi . lo
                            umma_tf32(tmem_base + b * TN, al, bd, idesc, 1u);               // lo . hi
                        }
                        umma_commit(&empty[s]);
                        if (h == 1) umma_commit(&tfull[b]);
                    }
                    __syncwarp();
                }
            } else {
                const uint32_t s = i % TC_STAGES, ph = (i / TC_STAGES) & 1u;
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t b_addr = smem_u32(sB + s * tile_bytes);
                    for (uint32_t k = 0; k < dim / 8; k++) {  // K = 8 tf32 per MMA = two 16-B chunks
                        const uint64_t ad = umma_desc(a_addr + k * 256, lbo, sbo);
                        const uint64_t bd = umma_desc(b_addr + k * 256, lbo, sbo);
                        umma_tf32(tmem_base + b * TN, ad, bd, idesc, k > 0 ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                    umma_commit(&tfull[b]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue warps 2..9
        const uint32_t quad = warp & 3u;            // TMEM lanes 32*quad ..
        const uint32_t half = (warp - 2u) >> 2;     // column half 0/1
        const uint32_t r = quad * 32 + lane;        // row within the tile
        float bd[4] = {FLT_MAX, FLT_MAX, FLT_MAX, FLT_MAX};
        uint32_t bi[4] = {0, 0, 0, 0};
        uint32_t cur_rb = 0xffffffffu;
        uint64_t grow = 0, row0 = 0;
        float tau_r = 0.0f;
        for (uint64_t u = u0; u < u1; u++) {
            const uint32_t i = (uint32_t)(u - u0);
            const uint32_t t = (uint32_t)(u % ntiles);
            const uint32_t rb = (uint32_t)(u / ntiles);
            if (rb != cur_rb) {
                cur_rb = rb;
                row0 = (uint64_t)rb * TC_M;
                grow = row0 + r;
                tau_r = (MODE == 3 && grow < nx) ? tau[grow] : 0.0f;
            }
            const uint32_t b = i & 1u, bph = (i >> 1) & 1u;
            mbar_wait(&tfull[b], bph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const float* nrm = cnorm_pad + (size_t)t * TN;
#pragma unroll
            for (int h = 0; h < TN / 64; h++) {
                uint32_t acc[32];
                const uint32_t col = half * (TN / 2) + h * 32;
                // search modes: one coalesced load, broadcast by shuffles; the
                // add path's ARGMIN epilogue keeps broadcast L1 loads (measured faster there)
                const float nv = MODE == 0 ? 0.0f : __ldg(nrm + col + lane);
                tmem_ld32(tmem_base + ((quad * 32) << 16) + b * TN + col, acc);
                float* tr = sMerge + (warp - 2) * 32 * 33;  // STORE: this warp's transpose tile
                float cmin = __int_as_float(0x7f800000);
                float c8[4] = {cmin, cmin, cmin, cmin};  // MODE 4: minima of 8-column chunks
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    const uint32_t cidx = t * TN + col + j;
                    const float nj = MODE == 0 ? __ldg(nrm + col + j) : __shfl_sync(0xffffffffu, nv, j);
                    const float d = fmaf(-2.0f, __uint_as_float(acc[j]), nj);
                    if constexpr (MODE == 0) {
                        if (d < bd[3]) {  // sorted insert, ties keep the lower index (earlier)
                            if (d < bd[2]) {
                                bd[3] = bd[2]; bi[3] = bi[2];
                                if (d < bd[1]) {
                                    bd[2] = bd[1]; bi[2] = bi[1];
                                    if (d < bd[0]) { bd[1] = bd[0]; bi[1] = bi[0]; bd[0] = d; bi[0] = cidx; }
                                    else { bd[1] = d; bi[1] = cidx; }
                                } else { bd[2] = d; bi[2] = cidx; }
                            } else { bd[3] = d; bi[3] = cidx; }
                        }
                    } else if constexpr (MODE == 1) {
                        tr[lane * 33 + j] = d;
                    } else if constexpr (MODE == 2) {
                        cmin = fminf(cmin, d);
                    } else if constexpr (MODE == 4) {
                        c8[j >> 3] = fminf(c8[j >> 3], d);
                    } else {
                        if (d <= tau_r && grow < nx) {
                            const uint32_t slot = atomicAdd(&cnt[grow], 1u);
                            if (slot < cap) {
                                top_d[grow * cap + slot] = d;
                                top_idx[grow * cap + slot] = cidx;
                            }
                        }
                    }
                }
                if constexpr (MODE == 2) {
                    if (grow < nx) out_row[grow * ldo + t * (TN / 32) + col / 32] = cmin;
                }
                if constexpr (MODE == 4) {
                    if (grow < nx)
                        *reinterpret_cast<float4*>(out_row + grow * ldo + (t * TN + col) / 8) =
                            make_float4(c8[0], c8[1], c8[2], c8[3]);
                }
                if constexpr (MODE == 1) {  // coalesced: one 128-byte row segment per instruction
                    __syncwarp();
                    const uint32_t cidx = t * TN + col + lane;
#pragma unroll 4
                    for (int rr = 0; rr < 32; rr++) {
                        const uint64_t orow = row0 + quad * 32 + rr;
                        if (orow < nx && cidx < kvalid) out_row[orow * ldo + cidx] = tr[rr * 33 + lane];
                    }
                    __syncwarp();
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
        }
        if constexpr (MODE == 0) {
            // merge the two column halves' top-4 lists for each row
            float* md = sMerge;                 // [128][4]
            uint32_t* mi = reinterpret_cast<uint32_t*>(sMerge + TC_M * 4);
            if (half == 1) {
                for (int j = 0; j < 4; j++) {
                    md[r * 4 + j] = bd[j];
                    mi[r * 4 + j] = bi[j];
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
            if (half == 0 && grow < nx) {
                float od[4];
                uint32_t oi[4];
                int a = 0, c = 0;
                for (int j = 0; j < 4; j++) {  // merge two sorted lists by (d, idx)
                    const float xd = bd[a], yd = md[r * 4 + c];
                    const uint32_t xi = bi[a], yi = mi[r * 4 + c];
                    const bool takex = (xd < yd) || (xd == yd && xi < yi);
                    od[j] = takex ? xd : yd;
                    oi[j] = takex ? xi : yi;
                    if (takex) a++;
                    else c++;
                }
                for (int j = 0; j < 4; j++) {
                    top_d[grow * 4 + j] = od[j];
                    top_idx[grow * 4 + j] = oi[j];
                }
            }
        }
    }
    // every MMA completed (the epilogue waited on every tfull); the producer's
    // copies were all consumed
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

// Re-lay centroids [K, D] row-major into the UMMA interleaved K-major tile
// layout, padding rows to a multiple of 128 (zero rows, +inf norms).
// rna: store tf32_rna(x) (round to nearest; the MMA then sees exact TF32
// operands, <= 2^-11 relative each, instead of truncating them, <= 2^-10)
__global__ void k_relayout_centroids(const float* __restrict__ C, uint32_t k, uint32_t dim, uint32_t ntiles,
                                     float* __restrict__ out, float* __restrict__ out_lo, float* __restrict__ norm_out,
                                     int rna, const float* __restrict__ mu) {
    const uint32_t nchunk = dim / 4;
    const uint64_t total = (uint64_t)ntiles * TC_N * nchunk;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = t / nchunk;
        const uint32_t c = (uint32_t)(t % nchunk);
        const uint32_t tile = (uint32_t)(row / TC_N), r = (uint32_t)(row % TC_N);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < k) v = reinterpret_cast<const float4*>(C + row * dim)[c];
        if (mu && row < k) {  // centered copy: fl(x - mu) per component
            const float4 m = reinterpret_cast<const float4*>(mu)[c];
            v = make_float4(v.x - m.x, v.y - m.y, v.z - m.z, v.w - m.w);
        }
        const uint64_t off = (uint64_t)tile * TC_N * dim + (r >> 3) * (nchunk * 32) + c * 32 + (r & 7) * 4;
        *reinterpret_cast<float4*>(out + off) =
            rna ? make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w)) : v;
        if (out_lo) {  // 3xTF32 split of the centroids (hi stays in `out` unrounded: the MMA truncates)
            const float4 hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
            *reinterpret_cast<float4*>(out + off) = hi;
            *reinterpret_cast<float4*>(out_lo + off) = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
        }
    }
    for (uint64_t row = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; norm_out && row < (uint64_t)ntiles * TC_N;
         row += (uint64_t)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        if (row < k)
            for (uint32_t d = 0; d < dim; d++) {
                const float x = mu ? C[row * dim + d] - mu[d] : C[row * dim + d];
                acc = dot_step(acc, x, x);
            }
        if (norm_out) norm_out[row] = row < k ? acc : __int_as_float(0x7f800000);
    }
}

// Split (3xTF32) copy of the centroids for the search coarse stage: hi =
// tf32(x), lo = x - hi, laid out per 64-centroid tile and K half as
// [tile][h][row/8][k/4 within the half][row%8][4] (one bulk copy per half).
__global__ void k_relayout_khalf(const float* __restrict__ C, uint32_t k, uint32_t dim, uint32_t ntiles,
                                 float* __restrict__ out_hi, float* __restrict__ out_lo) {
    const uint32_t nchunk = dim / 4, hc = nchunk / 2;
    const uint64_t total = (uint64_t)ntiles * 64 * nchunk;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = t / nchunk;
        const uint32_t c = (uint32_t)(t % nchunk);
        const uint32_t tile = (uint32_t)(row / 64), r = (uint32_t)(row % 64);
        const uint32_t h = c / hc, cc = c % hc;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < k) v = reinterpret_cast<const float4*>(C + row * dim)[c];
        const uint64_t off = ((uint64_t)tile * 2 + h) * (64 * dim / 2) + (r >> 3) * (hc * 32) + cc * 32 + (r & 7) * 4;
        const float4 hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
        *reinterpret_cast<float4*>(out_hi + off) = hi;
        *reinterpret_cast<float4*>(out_lo + off) = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
    }
}

}  // namespace dev

void launch_relayout_khalf(const float* C, uint32_t k, uint32_t dim, float* out_hi, float* out_lo, cudaStream_t st) {
    const uint32_t ntiles = (k + 63) / 64;
    dev::k_relayout_khalf<<<1184, 256, 0, st>>>(C, k, dim, ntiles, out_hi, out_lo);
    CUDA_LAUNCH_CHECK();
}

static size_t coarse_tc_smem_at(uint32_t dim, int mode, bool split, uint32_t stages) {
    const size_t tail = mode == 1 ? (size_t)8 * 32 * 33 * 4 : (size_t)dev::TC_M * 8 * 4;
    const size_t tn = split ? 64 : dev::TC_N, nb = split ? 2 : 1;
    // stage = one tile (1xTF32) or one K half of a tile in hi + lo (3xTF32): tn * dim * 4 either way
    return (size_t)dev::TC_M * dim * 4 * nb + (size_t)stages * tn * dim * 4 + 2 * stages * 8 + 6 * 8 + 16 + tail +
           256;
}

// deepest centroid-tile ring (<= TC_MAX_STAGES) that fits 227 KB; 0 if not even 2
static uint32_t coarse_tc_stages(uint32_t dim, int mode, bool split) {
    for (uint32_t s = dev::TC_MAX_STAGES; s >= 2; s--)
        if (coarse_tc_smem_at(dim, mode, split, s) <= 227 * 1024) return s;
    return 0;
}

// every epilogue mode the engine may launch (add: 0 unsplit; search: 1, 2, 3)
static bool coarse_tc_fits(uint32_t dim, bool split) {
    if (dim % (split ? 16u : 8u) != 0 || dim < 8) return false;  // K = 8 per MMA; split: two K halves
    for (int mode = split ? 1 : 0; mode < 4; mode++)
        if (coarse_tc_stages(dim, mode, split) == 0) return false;
    return true;
}

bool coarse_tc_supported(uint32_t dim) { return coarse_tc_fits(dim, false); }

bool coarse_tc_split_supported(uint32_t dim) { return coarse_tc_fits(dim, true); }

void launch_relayout_centroids(const float* C, uint32_t k, uint32_t dim, float* out, float* out_lo, float* norm_out,
                               cudaStream_t st, int rna, const float* mu) {
    const uint32_t ntiles = (k + dev::TC_N - 1) / dev::TC_N;
    dev::k_relayout_centroids<<<1184, 256, 0, st>>>(C, k, dim, ntiles, out, out_lo, norm_out, rna, mu);
    CUDA_LAUNCH_CHECK();
}

void launch_coarse_tc(int mode, const float* X, uint64_t nx, uint32_t dim, const float* cent_tc, const float* cent_lo,
                      const float* cnorm, uint32_t k, float* out_row, uint64_t ldo, uint32_t* top_idx, float* top_d,
                      cudaStream_t st, const float* tau, uint32_t* cnt, uint32_t cap, const float* Xtc,
                      const float* Xlo_tc) {
    if (nx == 0) return;
    const bool split = cent_lo != nullptr;
    const bool persist = Xtc != nullptr && mode != 0;
    const uint32_t tn = split ? 64 : dev::TC_N;
    const uint32_t ntiles = (k + tn - 1) / tn;
    const uint32_t stages = coarse_tc_stages(dim, mode, split);
    if (stages == 0) throw std::runtime_error("coarse_tc: shared-memory ring does not fit for this dim");
    if (persist && split && !Xlo_tc) throw std::runtime_error("coarse_tc: split rows need the lo half");
    const size_t smem = coarse_tc_smem_at(dim, mode, split, stages);
    const uint32_t nrb = (uint32_t)((nx + dev::TC_M - 1) / dev::TC_M);
    unsigned grid = nrb;
    if (persist) {
        static int nsm = 0;
        if (!nsm) {
            int dev = 0;
            CUDA_CHECK(cudaGetDevice(&dev));
            CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        }
        grid = (unsigned)std::min<uint64_t>((uint64_t)nsm, (uint64_t)nrb * ntiles);
    }
#define VLQ_TC_LAUNCH(MODE_, SPLIT_, PERSIST_)                                                                   \
    do {                                                                                                         \
        auto fn = stages == 4   ? dev::k_coarse_tc<MODE_, SPLIT_, 4, PERSIST_>                                   \
                  : stages == 3 ? dev::k_coarse_tc<MODE_, SPLIT_, 3, PERSIST_>                                   \
                                : dev::k_coarse_tc<MODE_, SPLIT_, 2, PERSIST_>;                                  \
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));           \
        fn<<<grid, dev::TC_THREADS, smem, st>>>(X, nx, dim, cent_tc, cent_lo, cnorm, ntiles, k, out_row, ldo,    \
                                                top_idx, top_d, tau, cnt, cap, Xtc, Xlo_tc, nrb);                \
    } while (0)
#define VLQ_TC_MODE(MODE_)                                                         \
    do {                                                                           \
        if (persist) {                                                             \
            if (split) VLQ_TC_LAUNCH(MODE_, true, true);                           \
            else VLQ_TC_LAUNCH(MODE_, false, true);                                \
        } else {                                                                   \
            if (split) VLQ_TC_LAUNCH(MODE_, true, false);                          \
            else VLQ_TC_LAUNCH(MODE_, false, false);                               \
        }                                                                          \
    } while (0)
    switch (mode) {
        case 0:
            if (split) VLQ_TC_LAUNCH(0, true, false);
            else VLQ_TC_LAUNCH(0, false, false);
            break;
        case 1: VLQ_TC_MODE(1); break;
        case 2: VLQ_TC_MODE(2); break;
        case 4:  // chunk-select path: 1xTF32 only
            if (split) throw std::runtime_error("coarse_tc: TILEMIN8 is a 1xTF32 mode");
            if (persist) VLQ_TC_LAUNCH(4, false, true);
            else VLQ_TC_LAUNCH(4, false, false);
            break;
        default: VLQ_TC_MODE(3); break;
    }
#undef VLQ_TC_MODE
#undef VLQ_TC_LAUNCH
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq

// ---------------------------------------------------------------------------
// Exact refinement + certificate of the tensor-core candidates.
//
// |approx(x,c) + |x|^2 - sqdist(x,c)| <= eps(x) for every centroid c, with
//   eps = 2 (2^-9 + D 2^-24) |x| cmax + D 2^-24 ((|x| + cmax)^2 + cmax^2) + 2^-23 (|x| + cmax)^2
// (TF32 operands truncate to 10 mantissa bits: relative error <= 2^-10 per
// factor; fp32 accumulation; the fp32 norm and the exact sequential sqdist
// each add D u |.|), times a 1.5 safety factor.  So every centroid whose
// exact distance can beat the approximate best lies within 2 eps of it.
// ---------------------------------------------------------------------------
namespace vlq {
namespace dev {


// Add path: exact argmin among the 4 tensor-core candidates (strict '<' from
// FLT_MAX, lowest id on ties: index.cpp:96-103) when the candidate set is
// provably complete; otherwise the point goes to the exact full scan.
__global__ void k_refine_argmin(const float* __restrict__ X, uint64_t nx, uint32_t dim,
                                const float* __restrict__ C, const uint32_t* __restrict__ top_idx,
                                const float* __restrict__ top_d, float cmax, uint32_t* __restrict__ best,
                                uint32_t* __restrict__ flagged, unsigned int* __restrict__ nflag) {
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nx; p += (uint64_t)gridDim.x * blockDim.x) {
        const float* x = X + p * dim;
        float xn = 0.0f;
        for (uint32_t d = 0; d < dim; d++) xn = fmaf(x[d], x[d], xn);
        const float eps = tc_eps(xn, cmax, dim);
        const float lim = top_d[p * 4] + 2.0f * eps;
        if (top_d[p * 4 + 3] <= lim) {  // a 5th centroid could also be within the margin
            flagged[atomicAdd(nflag, 1u)] = (uint32_t)p;
            continue;
        }
        uint64_t bk = ~0ull;
        for (int j = 0; j < 4; j++) {
            if (top_d[p * 4 + j] > lim) break;
            const uint32_t c = top_idx[p * 4 + j];
            const float* cp = C + (uint64_t)c * dim;
            float acc = 0.0f;
            for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, x[d], cp[d]);
            const uint64_t key = (acc < FLT_MAX) ? make_key(acc, c) : ~0ull;
            bk = key < bk ? key : bk;
        }
        best[p] = bk == ~0ull ? 0u : (uint32_t)bk;
    }
}

__global__ void k_gather_rows_list(const float* __restrict__ X, uint32_t dim, const uint32_t* __restrict__ rows,
                                   uint32_t nr, float* __restrict__ out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (uint64_t)nr * dim;
         t += (uint64_t)gridDim.x * blockDim.x)
        out[t] = X[(uint64_t)rows[t / dim] * dim + t % dim];
}

__global__ void k_scatter_u32(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ rows, uint32_t nr,
                              uint32_t* __restrict__ out) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += gridDim.x * blockDim.x) out[rows[t]] = vals[t];
}

// Search path: exact top-w1 among the L approximate candidates of each query
// (top[q*L..]), written back as ascending ids, exact distances stored into
// the ws row; certificate: L-th approximate value + |y|^2 - eps > exact
// w1-th, else the query is listed for an exact full row.
__global__ void k_refine_first(const float* __restrict__ Y, uint32_t dim, const float* __restrict__ C,
                               float* __restrict__ ws, uint32_t k, const uint32_t* __restrict__ cand, uint32_t L,
                               uint32_t w1, float cmax, uint32_t* __restrict__ top, uint32_t* __restrict__ flagged,
                               unsigned int* __restrict__ nflag, int split) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);  // npow2
    float* ys = reinterpret_cast<float*>(smem + 8 * 2048);
    __shared__ unsigned int s_amax;  // order-preserving bits of the largest candidate approx
    __shared__ float s_yn;
    const uint64_t q = blockIdx.x;
    uint32_t np2 = 1;
    while (np2 < L) np2 <<= 1;
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) ys[d] = Y[q * dim + d];
    if (threadIdx.x == 0) s_amax = 0u;
    __syncthreads();
    float* wsq = ws + q * k;
    const uint32_t* cq = cand + q * L;
    float amax = -__int_as_float(0x7f800000);
    for (uint32_t t = threadIdx.x; t < np2; t += blockDim.x) {
        uint64_t key = ~0ull;
        if (t < L) {
            const uint32_t c = cq[t];
            amax = fmaxf(amax, wsq[c]);  // approximate value (before overwrite)
            const float* cp = C + (uint64_t)c * dim;
            float acc = 0.0f;
            for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, ys[d], cp[d]);
            key = make_key(acc, c);
        }
        keys[t] = key;
    }
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_amax, ord_float(amax));
    __syncthreads();
    bitonic_sort_u64<false>(keys, np2, threadIdx.x, blockDim.x);
    if (threadIdx.x == 0) {
        float yn = 0.0f;
        for (uint32_t d = 0; d < dim; d++) yn = fmaf(ys[d], ys[d], yn);
        s_yn = yn;
    }
    __syncthreads();
    // certificate (all non-candidates have approx >= the L-th candidate's)
    if (threadIdx.x == 0) {
        const float eps = tc_eps(s_yn, cmax, dim, split != 0);
        const float exact_w1 = unord_float((uint32_t)(keys[w1 - 1] >> 32));
        const double lower = (double)unord_float(s_amax) + (double)s_yn - (double)eps;
        if (!(L < k ? lower > (double)exact_w1 : true)) flagged[atomicAdd(nflag, 1u)] = (uint32_t)q;
    }
    // exact values into the ws row (the downstream kernels read them)
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
        const uint64_t key = keys[t];
        wsq[(uint32_t)key] = unord_float((uint32_t)(key >> 32));
    }
    __syncthreads();
    // the w1 winners, re-sorted by id (second_level_rank's tie order needs ascending ids)
    for (uint32_t t = threadIdx.x; t < np2; t += blockDim.x)
        keys[t] = t < w1 ? (uint64_t)(uint32_t)keys[t] : ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(keys, np2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < w1; t += blockDim.x) top[q * w1 + t] = (uint32_t)keys[t];
}

// Exact distances for every centroid the downstream stages read: the top-w1
// regions and all their neighbours (second_level_rank reads ws[nbr],
// search.cpp:57).  Needed ids are deduplicated through a shared bitmap,
// compacted, and processed 32 at a time: the warp stages 32 centroid rows with
// 16-byte loads (one thread per centroid), then the sequential
// reference-order sqdist.
__global__ void __launch_bounds__(256) k_exact_needed(const float* __restrict__ Y, uint32_t dim,
                                                      const float* __restrict__ C, uint32_t k, uint32_t n,
                                                      const uint32_t* __restrict__ nbr, float* __restrict__ ws,
                                                      const uint32_t* __restrict__ top, uint32_t w1) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t nwords = (k + 31) / 32;
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem);            // nwords
    uint32_t* ids = bitmap + nwords;                                  // up to w1*(n+1)
    const size_t head = ((size_t)(nwords + w1 * (n + 1)) * 4 + 15) & ~(size_t)15;
    float* ys = reinterpret_cast<float*>(smem + head);                // dim, 16-B aligned
    float* tiles = ys + ((dim + 3) & ~3u);                             // 8 warps x 16 rows x (dim + 4)
    __shared__ uint32_t s_scan[40];
    const uint64_t q = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) bitmap[i] = 0;
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) ys[d] = Y[q * dim + d];
    __syncthreads();
    const uint32_t* tq = top + q * w1;
    for (uint32_t e = threadIdx.x; e < w1 * (n + 1); e += blockDim.x) {
        const uint32_t r = e / (n + 1), j = e % (n + 1);
        const uint32_t c = j == 0 ? tq[r] : nbr[(uint64_t)tq[r] * n + (j - 1)];
        atomicOr(&bitmap[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    // compact set bits (ascending ids)
    const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
    uint32_t local = 0;
    for (uint32_t i = threadIdx.x * per; i < min(nwords, (threadIdx.x + 1) * per); i++) local += __popc(bitmap[i]);
    uint32_t total;
    uint32_t run = block_excl_scan_u32(local, s_scan, &total);
    for (uint32_t i = threadIdx.x * per; i < min(nwords, (threadIdx.x + 1) * per); i++) {
        uint32_t w = bitmap[i];
        while (w) {
            const uint32_t b = __ffs(w) - 1;
            ids[run++] = i * 32 + b;
            w &= w - 1;
        }
    }
    __syncthreads();
    // rows staged through shared memory, 16 per warp at a time: the warp reads
    // each row with coalesced 16-byte loads (one row per instruction), then
    // lanes 0..15 each run the sequential reference-order sqdist of one row
    // (row stride dim + 4 floats: conflict-free 128-bit stores and loads)
    float* wsq = ws + q * k;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
    if ((dim & 3u) == 0 && dim <= 128) {
        const uint32_t n4 = dim >> 2, stride = dim + 4;
        float* tile = tiles + (size_t)warp * 16 * stride;
        for (uint32_t b0 = warp * 16; b0 < total; b0 += nwarps * 16) {
            const uint32_t nb = min(16u, total - b0);
            for (uint32_t r = 0; r < nb; r++) {
                const float4* cp = reinterpret_cast<const float4*>(C + (uint64_t)ids[b0 + r] * dim);
                for (uint32_t c4 = lane; c4 < n4; c4 += 32)
                    *reinterpret_cast<float4*>(tile + r * stride + c4 * 4) = __ldg(cp + c4);
            }
            __syncwarp();
            if (lane < nb) {
                const float* row = tile + lane * stride;
                float acc = 0.0f;
                for (uint32_t c4 = 0; c4 < n4; c4++) {
                    const float4 v = *reinterpret_cast<const float4*>(row + c4 * 4);
                    const float4 yv = *reinterpret_cast<const float4*>(ys + c4 * 4);
                    acc = sq_step(acc, yv.x, v.x);
                    acc = sq_step(acc, yv.y, v.y);
                    acc = sq_step(acc, yv.z, v.z);
                    acc = sq_step(acc, yv.w, v.w);
                }
                wsq[ids[b0 + lane]] = acc;
            }
            __syncwarp();
        }
    } else {
        for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
            const uint32_t c = ids[t];
            const float* cp = C + (uint64_t)c * dim;
            float acc = 0.0f;
            for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, ys[d], cp[d]);
            wsq[c] = acc;
        }
    }
}

// tau[row] = the L-th smallest chunk minimum (an upper bound on the row's
// L-th smallest approximate value).
// Y != null: the chunk minima came from the 1xTF32 pass, and tau is raised by
// both passes' error bounds so it also bounds the L-th smallest 3xTF32 value
// the filter pass compares against (at least L centroids pass).
__global__ void __launch_bounds__(512) k_tau_rows(const float* __restrict__ tmin, uint32_t nchunk, uint32_t L,
                                                  uint32_t* __restrict__ scratch, float* __restrict__ tau,
                                                  const float* __restrict__ Y, uint32_t dim, float cmax,
                                                  int pass2_split) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t scan[40];
    __shared__ unsigned int s_max;
    const uint64_t q = blockIdx.x;
    const float* row = tmin + q * nchunk;
    uint32_t* pos = scratch + q * L;
    block_select_ordered(row, nchunk, L, pos, hist, scan);
    if (threadIdx.x == 0) s_max = 0u;
    __syncthreads();
    float mx = -__int_as_float(0x7f800000);
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) mx = fmaxf(mx, row[pos[t]]);
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, ord_float(mx));
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = unord_float(s_max);
        if (Y) {
            float yn = 0.0f;
            for (uint32_t d = 0; d < dim; d++) yn = fmaf(Y[q * dim + d], Y[q * dim + d], yn);
            // approx2 <= approx1 + eps1 + eps2: the L centroids under tau1
            // (1xTF32) are all under tau1 + eps1 + eps2, eps2 the bound of the
            // filter pass (3xTF32, or 1xTF32 again when pass2_split == 0)
            t += (tc_eps(yn, cmax, dim, false) + tc_eps(yn, cmax, dim, pass2_split != 0)) * 1.01f;
        }
        tau[q] = t;
    }
}

// Exact top-w1 from the filtered candidate list: exact reference-order
// sqdist of every listed centroid, (dist, id) order, certificate
// tau + |y|^2 - eps > exact_w1 (every unlisted centroid has approx > tau).
__global__ void k_refine_list(const float* __restrict__ Y, uint32_t dim, const float* __restrict__ C, uint32_t k,
                              const uint32_t* __restrict__ cand, const uint32_t* __restrict__ cnt, uint32_t cap,
                              const float* __restrict__ tau, uint32_t w1, float cmax, int split,
                              uint32_t* __restrict__ top, uint32_t* __restrict__ flagged,
                              unsigned int* __restrict__ nflag) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);  // pow2 >= cap
    float* ys = reinterpret_cast<float*>(smem + 8 * 2048);
    float* tiles = ys + ((dim + 3) & ~3u);               // 8 warps x 16 rows x (dim + 4)
    __shared__ float s_yn;
    const uint64_t q = blockIdx.x;
    const uint32_t n = cnt[q];
    if (n > cap || n < w1) {  // list overflow (or too short): exact full row
        if (threadIdx.x == 0) flagged[atomicAdd(nflag, 1u)] = (uint32_t)q;
        return;
    }
    uint32_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) ys[d] = Y[q * dim + d];
    __syncthreads();
    const uint32_t* cq = cand + q * cap;
    if ((dim & 3u) == 0 && dim <= 128) {
        // rows staged through shared memory, 16 per warp (coalesced 16-byte
        // loads), lanes 0..15 run the reference-order sqdist of one row each
        const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
        const uint32_t n4 = dim >> 2, stride = dim + 4;
        float* tile = tiles + (size_t)warp * 16 * stride;
        for (uint32_t t = n + threadIdx.x; t < np2; t += blockDim.x) keys[t] = ~0ull;
        for (uint32_t b0 = warp * 16; b0 < n; b0 += nwarps * 16) {
            const uint32_t nb = min(16u, n - b0);
            for (uint32_t r = 0; r < nb; r++) {
                const float4* cp = reinterpret_cast<const float4*>(C + (uint64_t)cq[b0 + r] * dim);
                for (uint32_t c4 = lane; c4 < n4; c4 += 32)
                    *reinterpret_cast<float4*>(tile + r * stride + c4 * 4) = __ldg(cp + c4);
            }
            __syncwarp();
            if (lane < nb) {
                const float* row = tile + lane * stride;
                float acc = 0.0f;
                for (uint32_t c4 = 0; c4 < n4; c4++) {
                    const float4 v = *reinterpret_cast<const float4*>(row + c4 * 4);
                    const float4 yv = *reinterpret_cast<const float4*>(ys + c4 * 4);
                    acc = sq_step(acc, yv.x, v.x);
                    acc = sq_step(acc, yv.y, v.y);
                    acc = sq_step(acc, yv.z, v.z);
                    acc = sq_step(acc, yv.w, v.w);
                }
                keys[b0 + lane] = make_key(acc, cq[b0 + lane]);
            }
            __syncwarp();
        }
    } else {
        for (uint32_t t = threadIdx.x; t < np2; t += blockDim.x) {
            uint64_t key = ~0ull;
            if (t < n) {
                const uint32_t c = cq[t];
                const float* cp = C + (uint64_t)c * dim;
                float acc = 0.0f;
                for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, ys[d], cp[d]);
                key = make_key(acc, c);
            }
            keys[t] = key;
        }
    }
    if (threadIdx.x == 0) {
        float yn = 0.0f;
        for (uint32_t d = 0; d < dim; d++) yn = fmaf(ys[d], ys[d], yn);
        s_yn = yn;
    }
    __syncthreads();
    bitonic_sort_u64<false>(keys, np2, threadIdx.x, blockDim.x);
    if (threadIdx.x == 0) {
        const float eps = tc_eps(s_yn, cmax, dim, split != 0);
        const float exact_w1 = unord_float((uint32_t)(keys[w1 - 1] >> 32));
        const double lower = (double)tau[q] + (double)s_yn - (double)eps;
        if (!(lower > (double)exact_w1)) flagged[atomicAdd(nflag, 1u)] = (uint32_t)q;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < np2; t += blockDim.x) keys[t] = t < w1 ? (uint64_t)(uint32_t)keys[t] : ~0ull;
    __syncthreads();
    bitonic_sort_u64<false>(keys, np2, threadIdx.x, blockDim.x);
    for (uint32_t t = threadIdx.x; t < w1; t += blockDim.x) top[q * w1 + t] = (uint32_t)keys[t];
}

// Exact full ws rows for the listed queries (certificate failures).
__global__ void k_exact_rows(const float* __restrict__ Y, uint32_t dim, const float* __restrict__ C, uint32_t k,
                             float* __restrict__ ws, const uint32_t* __restrict__ qlist,
                             const unsigned int* __restrict__ count) {
    extern __shared__ float ysm[];

    const uint32_t _nb = *count;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint64_t q = qlist[_b];
    for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) ysm[d] = Y[q * dim + d];
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < k; c += blockDim.x) {
        const float* cp = C + (uint64_t)c * dim;
        float acc = 0.0f;
        for (uint32_t d = 0; d < dim; d++) acc = sq_step(acc, ysm[d], cp[d]);
        ws[q * k + c] = acc;
    }
    __syncthreads();  // shared memory is reused by the next query
    }
}

__global__ void __launch_bounds__(512) k_first_level_list(const float* __restrict__ ws, uint32_t k, uint32_t w1,
                                                          uint32_t* __restrict__ top, const uint32_t* __restrict__ qlist,
                                                          const unsigned int* __restrict__ count) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t scan[40];

    const uint32_t _nb = *count;  // list launches: a small grid strides over the device-side count
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
    const uint64_t q = qlist[_b];
    block_select_ordered(ws + q * k, k, w1, top + q * w1, hist, scan);
    __syncthreads();  // shared memory is reused by the next query
    }
}

}  // namespace dev

void launch_refine_argmin(const float* X, uint64_t nx, uint32_t dim, const float* C, const uint32_t* top_idx,
                          const float* top_d, float cmax, uint32_t* best, uint32_t* flagged, unsigned int* nflag,
                          cudaStream_t st) {
    if (nx == 0) return;
    dev::k_refine_argmin<<<(unsigned)dev::umin64((nx + 127) / 128, 4736), 128, 0, st>>>(X, nx, dim, C, top_idx, top_d,
                                                                                     cmax, best, flagged, nflag);
    CUDA_LAUNCH_CHECK();
}

void launch_gather_rows_list(const float* X, uint32_t dim, const uint32_t* rows, uint32_t nr, float* out,
                             cudaStream_t st) {
    if (nr == 0) return;
    dev::k_gather_rows_list<<<1184, 256, 0, st>>>(X, dim, rows, nr, out);
    CUDA_LAUNCH_CHECK();
}

void launch_scatter_u32(const uint32_t* vals, const uint32_t* rows, uint32_t nr, uint32_t* out, cudaStream_t st) {
    if (nr == 0) return;
    dev::k_scatter_u32<<<(nr + 255) / 256, 256, 0, st>>>(vals, rows, nr, out);
    CUDA_LAUNCH_CHECK();
}

void launch_refine_first(const float* Y, uint64_t nq, uint32_t dim, const float* C, float* ws, uint32_t k,
                         const uint32_t* cand, uint32_t L, uint32_t w1, float cmax, uint32_t* top, uint32_t* flagged,
                         unsigned int* nflag, int split, cudaStream_t st) {
    if (nq == 0) return;
    const size_t smem = 8 * 2048 + (size_t)dim * 4;
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_refine_first, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_refine_first<<<(unsigned)nq, 256, smem, st>>>(Y, dim, C, ws, k, cand, L, w1, cmax, top, flagged, nflag,
                                                         split);
    CUDA_LAUNCH_CHECK();
}

size_t exact_needed_smem(uint32_t k, uint32_t n, uint32_t w1, uint32_t dim) {
    const size_t head = (size_t)((k + 31) / 32) * 4 + (size_t)w1 * (n + 1) * 4;
    const size_t tiles = ((dim & 3u) == 0 && dim <= 128) ? (size_t)8 * 16 * (dim + 4) * 4 : 0;
    return ((head + 15) & ~(size_t)15) + (size_t)((dim + 3) & ~3u) * 4 + tiles;
}

void launch_exact_needed(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, uint32_t n,
                         const uint32_t* nbr, float* ws, const uint32_t* top, uint32_t w1, cudaStream_t st) {
    if (nq == 0) return;
    const size_t smem = exact_needed_smem(k, n, w1, dim);
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_exact_needed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_exact_needed<<<(unsigned)nq, 256, smem, st>>>(Y, dim, C, k, n, nbr, ws, top, w1);
    CUDA_LAUNCH_CHECK();
}


void launch_tau_rows(const float* tmin, uint64_t nq, uint32_t nchunk, uint32_t L, uint32_t* scratch, float* tau,
                     cudaStream_t st, const float* Y, uint32_t dim, float cmax, int pass2_split) {
    if (nq == 0) return;
    dev::k_tau_rows<<<(unsigned)nq, 512, 0, st>>>(tmin, nchunk, L, scratch, tau, Y, dim, cmax, pass2_split);
    CUDA_LAUNCH_CHECK();
}

void launch_refine_list(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, const uint32_t* cand,
                        const uint32_t* cnt, uint32_t cap, const float* tau, uint32_t w1, float cmax, int split,
                        uint32_t* top, uint32_t* flagged, unsigned int* nflag, cudaStream_t st) {
    if (nq == 0) return;
    const size_t tiles = ((dim & 3u) == 0 && dim <= 128) ? (size_t)8 * 16 * (dim + 4) * 4 : 0;
    const size_t smem = 8 * 2048 + (size_t)((dim + 3) & ~3u) * 4 + tiles;
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_refine_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_refine_list<<<(unsigned)nq, 256, smem, st>>>(Y, dim, C, k, cand, cnt, cap, tau, w1, cmax, split, top,
                                                        flagged, nflag);
    CUDA_LAUNCH_CHECK();
}

void launch_exact_rows(const float* Y, uint64_t nq, uint32_t dim, const float* C, uint32_t k, float* ws,
                       const uint32_t* qlist, const unsigned int* count, cudaStream_t st) {
    if (nq == 0) return;
    dev::k_exact_rows<<<list_grid(nq, true), 256, dim * 4, st>>>(Y, dim, C, k, ws, qlist, count);
    CUDA_LAUNCH_CHECK();
}

void launch_first_level_list(const float* ws, uint64_t nq, uint32_t k, uint32_t w1, uint32_t* top,
                             const uint32_t* qlist, const unsigned int* count, cudaStream_t st) {
    if (nq == 0) return;
    dev::k_first_level_list<<<list_grid(nq, true), 512, 0, st>>>(ws, k, w1, top, qlist, count);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq
