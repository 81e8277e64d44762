// Chunk-select coarse stage: first_level_scan + second_level_rank
// (proj/src/search.cpp:11-78) from ONE 1xTF32 tensor-core pass.
//
//   k_coarse_tc<4> (TILEMIN8)  approx(y, c) = |c|^2 - 2 <y, c> on TF32 operands;
//                              per query the minimum of every 8-centroid chunk
//                              (tmin [nq, K/8]); no K-wide row in HBM
//   k_chunk_select             tau >= the w1-th smallest chunk minimum (histogram),
//                              T = tau + 2.02 eps (eps = tc_eps, the TF32 bound);
//                              compacts the chunks with minimum <= T
//   k_rows (chunks)            exact reference-order sqdist of every centroid in
//                              those chunks (barrier-free row kernel)
//   k_top_need                 exact top-w1 by (dist, id) with a certificate;
//                              the w1 regions' neighbours, bitmap-deduplicated
//   k_rows (needed ids)        their exact distances
//   k_second_sel               second_level_rank over the w1 n edges -> the
//                              selected cells, their (a, b) pairs, the scanned
//                              count and the |term1| bound
//
// Why the chunk set is complete (the certificate, checked per query): the w1
// chunks whose minimum is <= tau each hold a centroid with approx <= tau, i.e.
// exact <= tau + |y|^2 + eps, so the exact w1-th smallest over the evaluated
// centroids is <= tau + |y|^2 + eps.  Every centroid outside the selected
// chunks has approx > T, i.e. exact > T + |y|^2 - eps = tau + |y|^2 + 1.02 eps.
// The kernel checks T + |y|^2 - eps > exact_w1 explicitly (in double); a query
// that fails it (or whose chunk list overflows) is listed and takes the exact
// full-row path (k_exact_rows + k_first_level_list), then k_top_need in
// "top" mode from its exact top-w1.
//
// Versus the two-pass filter (1xTF32 chunk minima + 3xTF32 filter pass +
// exact refine + k_exact_needed writing ~2k exact distances into a K-wide ws
// row per query): one tensor-core pass instead of two (the 3xTF32 pass issued
// 3x the MMAs), and the needed exact distances live in shared memory only.
#include <stdexcept>

#include "async.cuh"
#include "kernels.h"
#include "select.cuh"

namespace vlq {
namespace dev {

constexpr uint32_t FS_THREADS = 256;  // k_second_sel
constexpr uint32_t TN_THREADS = 128;  // k_top_need
constexpr uint32_t FS_MAX_KEYS = 2048; // exactly evaluated chunk centroids per query
constexpr uint32_t FS_CS = 8;          // centroids per chunk (TILEMIN8)

// tau / T per query and the compacted list of selected chunks.  tau is an
// upper bound on the L-th smallest chunk minimum, found with ONE histogram
// pass over the row's value range: 2048 equal-width bins between the row's
// minimum and maximum (a monotone binning), the bin b where the cumulative
// count reaches L, and tau = the largest value in bin b -- at least the L-th
// smallest value, and within one bin width (~range / 2048) of it.  (A radix
// select on the float bits put every value of a row into a handful of
// first-pass bins -- same exponent -- and serialised on their atomics.)  The
// row lives in registers (VPT values per thread, coalesced); the list is
// compacted in ascending chunk order (ballots per (slot, warp) segment + one
// block scan over the segment counts).
template <int VPT, int NT>
__global__ void __launch_bounds__(NT) k_chunk_select(const float* __restrict__ tmin, uint32_t nchunk, uint32_t L,
                                                     const float* __restrict__ Y, uint32_t dim, float cmax,
                                                     uint32_t capc, uint32_t* __restrict__ clist,
                                                     uint32_t* __restrict__ ccnt, float* __restrict__ Tout,
                                                     const float* __restrict__ mu) {
    constexpr uint32_t NB = 2048, NWARP = NT / 32;
    __shared__ uint32_t hist[NB];
    __shared__ uint32_t scan[40];
    __shared__ uint32_t segc[VPT * NWARP];
    __shared__ float s_T, s_yn;
    __shared__ unsigned int s_mn, s_mx, s_bin, s_tau;
    const uint64_t q = blockIdx.x;
    const float* row = tmin + q * nchunk;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const float INF = __int_as_float(0x7f800000);
    float v[VPT];
#pragma unroll
    for (int j = 0; j < VPT; j++) {
        const uint32_t i = j * NT + tid;
        v[j] = i < nchunk ? row[i] : INF;
    }
    if (warp == 0) {  // |y'|^2 of the (centered) tensor-core operand, lane-parallel (any fp32 order: the
                      // bound's D u s^2 term covers its rounding), read by thread 0 after the barriers below
        float part = 0.0f;
        for (uint32_t d = lane; d < dim; d += 32) {
            const float y = mu ? Y[q * dim + d] - mu[d] : Y[q * dim + d];
            part = fmaf(y, y, part);
        }
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) s_yn = part;
    }
    for (uint32_t b = tid; b < NB; b += NT) hist[b] = 0;
    // row min / max over the finite values (padded centroids give +inf)
    float mn = INF, mx = -INF;
#pragma unroll
    for (int j = 0; j < VPT; j++) {
        mn = fminf(mn, v[j]);
        if (v[j] < INF) mx = fmaxf(mx, v[j]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) {
        s_mn = 0xffffffffu;  // order-preserving keys (approx values are |c|^2 - 2 <y, c>: often negative)
        s_mx = 0u;
        s_tau = 0u;
    }
    __syncthreads();
    if (lane == 0) {
        atomicMin(&s_mn, ord_float(mn));
        atomicMax(&s_mx, ord_float(mx));
    }
    __syncthreads();
    const float lo = unord_float(s_mn), hi = fmaxf(unord_float(s_mx), lo);
    const float inv = hi > lo ? (float)(NB - 1) / (hi - lo) : 0.0f;
    auto bin_of = [&](float x) -> uint32_t {
        const float t = (fmaxf(x, lo) - lo) * inv;  // monotone in x; +inf -> the last bin
        return t < (float)(NB - 1) ? (uint32_t)t : NB - 1;  // NaN (inf * 0) -> the last bin
    };
#pragma unroll
    for (int j = 0; j < VPT; j++)
        if (v[j] < INF) atomicAdd(&hist[bin_of(v[j])], 1u);
    __syncthreads();
    {
        constexpr uint32_t per = (NB + NT - 1) / NT;
        uint32_t local = 0;
        for (uint32_t b = tid * per; b < min(NB, (tid + 1) * per); b++) local += hist[b];
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, scan, &total);
        const uint32_t Lc = min(L, nchunk);
        for (uint32_t b = tid * per; b < min(NB, (tid + 1) * per); b++) {
            if (run < Lc && Lc <= run + hist[b]) s_bin = b;
            run += hist[b];
        }
    }
    __syncthreads();
    const uint32_t bsel = s_bin;
    uint32_t tmax = 0u;  // the largest value in the crossing bin (>= the L-th smallest), order-preserving
#pragma unroll
    for (int j = 0; j < VPT; j++)
        if (v[j] < INF && bin_of(v[j]) == bsel) tmax = max(tmax, ord_float(v[j]));
    for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if (lane == 0) atomicMax(&s_tau, tmax);
    __syncthreads();
    if (tid == 0) {
        s_T = unord_float(s_tau) + 2.02f * tc_eps(s_yn, cmax, dim, false, /*rna=*/true, mu != nullptr);
    }
    __syncthreads();
    const float T = s_T;
    // ordered compaction: element j * NT + warp * 32 + lane; segment (j, warp)
    uint32_t bal[VPT];
#pragma unroll
    for (int j = 0; j < VPT; j++) {
        bal[j] = __ballot_sync(0xffffffffu, v[j] <= T);
        if (lane == 0) segc[j * NWARP + warp] = __popc(bal[j]);
    }
    __syncthreads();
    uint32_t total;
    const uint32_t mine = tid < VPT * NWARP ? segc[tid] : 0u;
    const uint32_t ex = block_excl_scan_u32(mine, scan, &total);
    if (tid < VPT * NWARP) segc[tid] = ex;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VPT; j++) {
        if ((bal[j] >> lane) & 1u) {
            const uint32_t slot = segc[j * NWARP + warp] + __popc(bal[j] & ((1u << lane) - 1u));
            if (slot < capc) clist[q * capc + slot] = j * NT + warp * 32 + lane;
        }
    }
    if (tid == 0) {
        ccnt[q] = total;
        Tout[q] = T;
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Exact reference-order sqdist (vecset.cpp:22-29: acc += (y - c)^2 in order)
// of the rows id_of(0 .. cnt) (centroid ids; id >= k gives +inf), out(t, d).
// Each warp takes batches of 32 rows, lane l owning row l of the batch; the
// rows stream through shared memory in PW-dimension pieces (coalesced 16-byte
// cp.async, zero-filled for invalid rows), NB pieces per warp in flight, so
// the L2 latency of the gathered centroid rows overlaps the sequential sums.
// Warp-synchronous; `wbuf` is this warp's NB * 32 * (PW + 4) floats (row
// stride PW + 4: conflict-free LDS.128).  The loop keeps (batch, piece)
// counters instead of dividing; a lane's row bases are computed once per batch.
template <uint32_t PW, uint32_t NB, typename IdFn, typename OutFn>
__device__ __forceinline__ void exact_rows_pipe_t(const float* __restrict__ C, uint32_t k, uint32_t dim,
                                                  const float* ys, float* wbuf, uint32_t cnt, uint32_t warp,
                                                  uint32_t nwarps, IdFn&& id_of, OutFn&& out) {
    constexpr uint32_t RS = PW + 4, BUF = 32 * RS;
    constexpr uint32_t CPR = PW / 4, RPI = 32 / CPR, NI = CPR;  // chunks per row piece, rows per copy instr
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t npiece = (dim + PW - 1) / PW;
    const uint32_t nbatch = cnt > warp * 32 ? (cnt - warp * 32 + nwarps * 32 - 1) / (nwarps * 32) : 0;
    if (nbatch == 0) return;
    const uint32_t nu = nbatch * npiece;
    const uint32_t sub = lane % CPR, rsub = lane / CPR;  // copy role: chunk `sub` of rows RPI i + rsub
    const float* rb[NI];
    uint32_t rvalid = 0;
    uint32_t ib = 0, ip = 0, islot = 0;  // next unit to issue
    auto issue = [&]() {
        if (ip == 0) {
            const uint32_t r0 = (warp + ib * nwarps) * 32;
            const uint32_t my_id = r0 + lane < cnt ? id_of(r0 + lane) : 0xffffffffu;
            rvalid = 0;
#pragma unroll
            for (uint32_t i = 0; i < NI; i++) {
                const uint32_t id = __shfl_sync(0xffffffffu, my_id, RPI * i + rsub);
                const bool v = id < k;
                rvalid |= (v ? 1u : 0u) << i;
                rb[i] = C + (v ? (uint64_t)id * dim : 0ull) + sub * 4;
            }
        }
        float* buf = wbuf + islot * BUF + rsub * RS + sub * 4;
        const bool dval = ip * PW + sub * 4 < dim;
#pragma unroll
        for (uint32_t i = 0; i < NI; i++)
            cp_async16(buf + RPI * i * RS, rb[i] + ip * PW, dval && ((rvalid >> i) & 1u));
        cp_async_commit();
        islot = islot + 1 == NB ? 0 : islot + 1;
        if (++ip == npiece) {
            ip = 0;
            ib++;
        }
    };
#pragma unroll
    for (uint32_t u = 0; u + 1 < NB; u++) {
        if (u < nu) issue();
        else cp_async_commit();
    }
    float acc = 0.0f;
    uint32_t cb = 0, cp = 0, cslot = 0;  // unit being computed
    for (uint32_t u = 0; u < nu; u++) {
        if (u + NB - 1 < nu) issue();
        else cp_async_commit();
        cp_async_wait<NB - 1>();
        __syncwarp();
        const float* row = wbuf + cslot * BUF + lane * RS;
        const float* yp = ys + cp * PW;
        if (cp * PW + PW <= dim) {
#pragma unroll
            for (uint32_t c4 = 0; c4 < PW / 4; c4++) {
                const float4 v = *reinterpret_cast<const float4*>(row + c4 * 4);
                const float4 yv = *reinterpret_cast<const float4*>(yp + c4 * 4);
                acc = sq_step(acc, yv.x, v.x);
                acc = sq_step(acc, yv.y, v.y);
                acc = sq_step(acc, yv.z, v.z);
                acc = sq_step(acc, yv.w, v.w);
            }
        } else {
            for (uint32_t c4 = 0; c4 < (dim - cp * PW) / 4; c4++) {
                const float4 v = *reinterpret_cast<const float4*>(row + c4 * 4);
                const float4 yv = *reinterpret_cast<const float4*>(yp + c4 * 4);
                acc = sq_step(acc, yv.x, v.x);
                acc = sq_step(acc, yv.y, v.y);
                acc = sq_step(acc, yv.z, v.z);
                acc = sq_step(acc, yv.w, v.w);
            }
        }
        __syncwarp();
        cslot = cslot + 1 == NB ? 0 : cslot + 1;
        if (++cp == npiece) {
            const uint32_t t = (warp + cb * nwarps) * 32 + lane;
            if (t < cnt) out(t, id_of(t) < k ? acc : __int_as_float(0x7f800000));
            acc = 0.0f;
            cp = 0;
            cb++;
        }
    }
    cp_async_wait<0>();
}

struct FusedArgs {
    const float* Y;
    uint32_t w1, w2, cs;      // regions, cells, centroids per chunk
    const uint32_t* clist;    // [nq, capc] selected chunks (chunk mode)
    const uint32_t* ccnt;     // [nq]
    uint32_t capc;
    const float* T;           // [nq] chunk threshold (approx units, without |y|^2)
    float cmax;
    const uint32_t* qlist;    // top mode: block b handles query qlist[b] (b < *qcount) from a.top
    const unsigned int* qcount;
    uint32_t* flagged;        // chunk mode: queries whose certificate failed / list overflowed
    unsigned int* nflag;
    uint32_t* sel_out;        // optional select-split hand-off: cells [nq, w2]
    float* ab_out;            //                                 (a, b) [nq, w2, 2]
    const float* mu = nullptr;  // centered tensor-core operands (chunk mode): the common shift
};

__host__ __device__ inline uint32_t fs_nwords(uint32_t k) { return (k + 31) / 32; }
// ---------------------------------------------------------------------------
// The exact centroid rows run in kernels that do nothing else -- no block
// barriers, several CTAs per SM with NB row pieces in flight per warp, so the
// gathered rows stream at L2 speed -- and the selections run in light
// per-query kernels.  (A single fused per-query kernel doing all of it measured
// 1.55 ms at C4 against 1.39 ms for these four: its block-level selection
// phases left the row loads idle.)
//   k_rows (chunks)  exact distances of the kept chunks' centroids -> vals [q][t]
//   k_top_need       exact top-w1 + certificate (chunk mode) or the exact
//                    top-w1 of the fallback (top mode); the needed ids (regions
//                    and their neighbours, deduplicated, ascending) -> nid [q][t]
//   k_rows (list)    exact distances of the needed ids -> nval [q][t]
//   k_second_sel     second_level_rank from nid / nval -> selection, (a, b),
//                    scanned count, |term1| bound
// ---------------------------------------------------------------------------
constexpr uint32_t RW_WARPS = 4;   // warps per query CTA of the row kernels
// NB = 3 pieces in flight per warp (30 KB per CTA, 7 CTAs per SM): C3 first
// level 1.402 -> 1.376 ms against NB = 4 (5 CTAs per SM); 4 x 2, 8 x 2 equal,
// 2 x 4 and 2 x 2 slower (profiles/r2_study_rows_shape_c3.jsonl)
constexpr uint32_t RW_PW = 16, RW_NB = 3;

struct RowsArgs {
    const float* C;
    const float* Y;
    uint32_t k, dim;
    int chunks;               // 1: ids = list[q][t / 8] * 8 + t % 8 for t < 8 cnt[q] (cnt[q] <= capc); 0: ids = list[q][t]
    const uint32_t* list;
    const uint32_t* cnt;
    uint32_t ld;              // row stride of list (capc, or the needed-id capacity)
    uint32_t capc;
    float* out;
    uint32_t ldo;
};

template <int WARPS, int NB>
__global__ void __launch_bounds__(WARPS * 32) k_rows(RowsArgs r) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t q = blockIdx.x;
    const uint32_t dim = r.dim, dimp = (dim + RW_PW - 1) / RW_PW * RW_PW;
    float* ys = reinterpret_cast<float*>(smem);
    float* wbuf = ys + dimp + (threadIdx.x >> 5) * NB * 32 * (RW_PW + 4);
    for (uint32_t d = threadIdx.x; d < dimp; d += blockDim.x) ys[d] = d < dim ? r.Y[q * dim + d] : 0.0f;
    uint32_t cnt = r.cnt[q];
    if (r.chunks) cnt = (cnt > r.capc || cnt * FS_CS > FS_MAX_KEYS) ? 0u : cnt * FS_CS;  // overflow: k_top_need flags it
    __syncthreads();
    const uint32_t* lq = r.list + q * r.ld;
    float* oq = r.out + q * r.ldo;
    if (r.chunks)
        exact_rows_pipe_t<RW_PW, NB>(
            r.C, r.k, dim, ys, wbuf, cnt, threadIdx.x >> 5, WARPS,
            [&](uint32_t t) { return __ldg(lq + t / FS_CS) * FS_CS + (t & (FS_CS - 1)); },
            [&](uint32_t t, float v) { oq[t] = v; });
    else
        exact_rows_pipe_t<RW_PW, NB>(
            r.C, r.k, dim, ys, wbuf, cnt, threadIdx.x >> 5, WARPS, [&](uint32_t t) { return __ldg(lq + t); },
            [&](uint32_t t, float v) { oq[t] = v; });
}

struct NeedArgs {
    const float* vals;   // [nq][FS_MAX_KEYS] chunk-centroid distances (chunk mode)
    uint32_t* nid;       // [nq][ldn] needed ids, ascending
    uint32_t* nneed;     // [nq]
    uint32_t ldn;
};

__global__ void __launch_bounds__(TN_THREADS) k_top_need(SearchArgs a, FusedArgs f, NeedArgs na) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ float s_yn;
    __shared__ unsigned int s_w1max;
    const bool top_mode = f.qlist != nullptr;
    const uint32_t k = a.k, n = a.n, dim = a.dim, w1 = f.w1, nw = fs_nwords(k);
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint32_t* topS = reinterpret_cast<uint32_t*>(smem);                 // w1
    uint32_t* bitmap = topS + ((w1 + 3) & ~3u);                           // nw
    float* vals = reinterpret_cast<float*>(bitmap + nw);                  // FS_MAX_KEYS (chunk mode)
    uint32_t* topPos = reinterpret_cast<uint32_t*>(vals + FS_MAX_KEYS);  // w1
    uint32_t* hist = topPos + ((w1 + 3) & ~3u);                           // 1024 + 256 + 40 (range select)
    uint32_t* scan = hist + 2048;
    const uint32_t _nb = top_mode ? *f.qcount : gridDim.x;
    for (uint32_t _b = blockIdx.x; _b < _nb; _b += gridDim.x) {
        const uint64_t q = top_mode ? f.qlist[_b] : _b;
        if (!top_mode) {
            const uint32_t nc = f.ccnt[q];
            const uint32_t ncent = nc * FS_CS;
            if (nc > f.capc || ncent > FS_MAX_KEYS || nc < w1) {
                if (tid == 0) f.flagged[atomicAdd(f.nflag, 1u)] = (uint32_t)q;
                continue;
            }
            const float* vq = na.vals + q * FS_MAX_KEYS;
            for (uint32_t t = tid; t < ncent; t += nt) vals[t] = vq[t];
            if (tid < 32) {  // |y'|^2, lane-parallel (any fp32 order: covered by the bound's D u s^2 term)
                float part = 0.0f;
                for (uint32_t d = tid; d < dim; d += 32) {
                    const float y = f.mu ? f.Y[q * dim + d] - f.mu[d] : f.Y[q * dim + d];
                    part = fmaf(y, y, part);
                }
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                if (tid == 0) {
                    s_yn = part;
                    s_w1max = 0u;
                }
            }
            __syncthreads();
            // exact top-w1 by (dist, id): the chunk list is ascending, so position order == id order
            block_select_ordered_range(vals, ncent, w1, topPos, hist, scan);
            __syncthreads();
            const uint32_t* cl = f.clist + q * f.capc;
            float mx = 0.0f;
            for (uint32_t r = tid; r < w1; r += nt) {
                const uint32_t pos = topPos[r];
                topS[r] = cl[pos / FS_CS] * FS_CS + (pos & (FS_CS - 1));
                mx = fmaxf(mx, vals[pos]);  // +inf (a padded id) fails the certificate below
            }
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((tid & 31) == 0) atomicMax(&s_w1max, __float_as_uint(mx));  // distances >= 0
            __syncthreads();
            const float exact_w1 = __uint_as_float(s_w1max);
            const float eps = tc_eps(s_yn, f.cmax, dim, false, /*rna=*/true, f.mu != nullptr);
            const double lower = (double)f.T[q] + (double)s_yn - (double)eps;
            if (!(lower > (double)exact_w1)) {
                if (tid == 0) f.flagged[atomicAdd(f.nflag, 1u)] = (uint32_t)q;
                __syncthreads();
                continue;
            }
            for (uint32_t r = tid; r < w1; r += nt) a.top[q * w1 + r] = topS[r];
        } else {
            for (uint32_t t = tid; t < w1; t += nt) topS[t] = a.top[q * w1 + t];
        }
        // the regions and their neighbours, deduplicated through a bitmap,
        // compacted in ascending id order
        for (uint32_t i = tid; i < nw; i += nt) bitmap[i] = 0;
        __syncthreads();
        // regions, then their neighbour rows (coalesced, up to 8 loads in flight per thread)
        for (uint32_t r = tid; r < w1; r += nt) atomicOr(&bitmap[topS[r] >> 5], 1u << (topS[r] & 31));
        const uint32_t ne = w1 * n;
        for (uint32_t e0 = 0; e0 < ne; e0 += 8 * nt) {
            uint32_t c[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint32_t e = e0 + u * nt + tid;
                c[u] = e < ne ? __ldg(a.nbr + (uint64_t)topS[e / n] * n + e % n) : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (c[u] != 0xffffffffu) atomicOr(&bitmap[c[u] >> 5], 1u << (c[u] & 31));
        }
        __syncthreads();
        const uint32_t per = (nw + nt - 1) / nt;
        uint32_t local = 0;
        for (uint32_t i = tid * per; i < min(nw, (tid + 1) * per); i++) local += __popc(bitmap[i]);
        uint32_t total;
        uint32_t run = block_excl_scan_u32(local, scan, &total);
        uint32_t* nq_out = na.nid + q * na.ldn;
        for (uint32_t i = tid * per; i < min(nw, (tid + 1) * per); i++) {
            uint32_t w = bitmap[i];
            while (w) {
                const uint32_t b = __ffs(w) - 1;
                nq_out[run++] = i * 32 + b;
                w &= w - 1;
            }
        }
        if (tid == 0) na.nneed[q] = total;
        __syncthreads();
    }
}

struct SecondArgs {
    const uint32_t* nid;
    const float* nval;
    const uint32_t* nneed;
    uint32_t ldn;
};

__global__ void __launch_bounds__(FS_THREADS) k_second_sel(SearchArgs a, FusedArgs f, SecondArgs sa) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long s_scanned;
    __shared__ float s_dmax;
    const uint32_t k = a.k, n = a.n, w1 = f.w1, w2 = f.w2, nw = fs_nwords(k), total = w1 * n;
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const uint64_t q = blockIdx.x;
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem);          // nw
    uint16_t* wpref = reinterpret_cast<uint16_t*>(bitmap + nw);     // nw
    float* nval = reinterpret_cast<float*>(bitmap + nw + (nw + 1) / 2);  // ldn
    float* dq = nval + sa.ldn;                                      // w1 n
    uint32_t* selpos = reinterpret_cast<uint32_t*>(dq + total);     // w2
    uint32_t* topS = selpos + w2;                                   // w1
    uint32_t* hist = topS + w1;                                     // range select scratch
    uint32_t* scan = hist + 2048;
    for (uint32_t i = tid; i < nw; i += nt) bitmap[i] = 0;
    if (tid == 0) {
        s_scanned = 0;
        s_dmax = 0.0f;
    }
    const uint32_t cnt = sa.nneed[q];
    const uint32_t* idq = sa.nid + q * sa.ldn;
    const float* vq = sa.nval + q * sa.ldn;
    for (uint32_t r = tid; r < w1; r += nt) topS[r] = a.top[q * w1 + r];
    __syncthreads();
    for (uint32_t t = tid; t < cnt; t += nt) {
        const uint32_t c = idq[t];
        atomicOr(&bitmap[c >> 5], 1u << (c & 31));
        nval[t] = vq[t];  // ids are ascending: rank(c) = t
    }
    __syncthreads();
    {
        const uint32_t per = (nw + nt - 1) / nt;
        uint32_t local = 0;
        for (uint32_t i = tid * per; i < min(nw, (tid + 1) * per); i++) local += __popc(bitmap[i]);
        uint32_t tot;
        uint32_t run = block_excl_scan_u32(local, scan, &tot);
        for (uint32_t i = tid * per; i < min(nw, (tid + 1) * per); i++) {
            wpref[i] = (uint16_t)run;
            run += __popc(bitmap[i]);
        }
    }
    __syncthreads();
    auto val_of = [&](uint32_t c) -> float {
        const uint32_t w = c >> 5;
        return nval[wpref[w] + __popc(bitmap[w] & ((1u << (c & 31)) - 1u))];
    };
    // second_level_rank (search.cpp:38-78)
    for (uint32_t e = tid; e < total; e += nt) {
        const uint32_t i = topS[e / n], j = e % n;
        const float av = val_of(i);
        const uint32_t s = a.nbr[(uint64_t)i * n + j];
        const float bv = val_of(s);
        const float cv = a.elen[(uint64_t)i * n + j];
        if (!(cv > 0.0f)) atomicOr(a.error_flag, 1u);  // line_quant.cpp:10-12
        const float lam = clamp_std(line_lambda(av, bv, cv), 0.0f, 1.0f);
        dq[e] = line_sqdist(av, bv, cv, lam);
    }
    __syncthreads();
    block_select_ordered_range(dq, total, w2, selpos, hist, scan);
    __syncthreads();
    float* wsq = a.ws + q * a.k;
    const float lmax = a.lam_absmax;
    unsigned long long c2 = 0;
    float dmax = 0.0f;
    for (uint32_t t = tid; t < w2; t += nt) {
        const uint32_t e = selpos[t];
        const uint32_t i = topS[e / n], j = e % n;
        const uint32_t cell = i * n + j;
        const uint32_t s = a.nbr[cell];
        const float av = val_of(i), bv = val_of(s), cv = a.elen[cell];
        a.sel[q * w2 + t] = cell;
        wsq[i] = av;
        wsq[s] = bv;
        if (f.sel_out) {
            f.sel_out[q * w2 + t] = cell;
            f.ab_out[(q * w2 + t) * 2] = av;
            f.ab_out[(q * w2 + t) * 2 + 1] = bv;
        }
        c2 += a.list_off[cell + 1] - a.list_off[cell];
        const float bound = (1.0f + lmax) * fabsf(av) + (lmax * lmax + lmax) * fabsf(cv) + lmax * fabsf(bv);
        dmax = fmaxf(dmax, bound);
    }
    for (int o = 16; o > 0; o >>= 1) {
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if ((tid & 31) == 0) {
        atomicAdd(&s_scanned, c2);
        atomicMax(reinterpret_cast<unsigned int*>(&s_dmax), __float_as_uint(dmax));
    }
    __syncthreads();
    if (tid == 0) {
        a.meta[q].scanned = s_scanned;
        a.meta[q].dmax = s_dmax;
        a.meta[q].flag = 0;
    }
}

}  // namespace dev

void launch_chunk_select(const float* tmin, uint64_t nq, uint32_t nchunk, uint32_t L, const float* Y, uint32_t dim,
                         float cmax, uint32_t capc, uint32_t* clist, uint32_t* ccnt, float* T, cudaStream_t st,
                         const float* mu) {
    if (nq == 0) return;
    // K <= 65536: 32 values per thread in 256-thread CTAs (C3: 1.441 -> 1.424 ms of
    // first level vs 16 x 512; 8 x 1024 1.466 ms, profiles/r2_study_cs_shape_c3.jsonl)
    if (nchunk <= 32 * 256)
        dev::k_chunk_select<32, 256><<<(unsigned)nq, 256, 0, st>>>(tmin, nchunk, L, Y, dim, cmax, capc, clist, ccnt, T,
                                                                    mu);
    else if (nchunk <= 16 * 512)
        dev::k_chunk_select<16, 512><<<(unsigned)nq, 512, 0, st>>>(tmin, nchunk, L, Y, dim, cmax, capc, clist, ccnt, T,
                                                                    mu);
    else if (nchunk <= 32 * 1024)
        dev::k_chunk_select<32, 1024><<<(unsigned)nq, 1024, 0, st>>>(tmin, nchunk, L, Y, dim, cmax, capc, clist, ccnt,
                                                                      T, mu);
    else
        throw std::runtime_error("chunk_select: K above 262144");
    CUDA_LAUNCH_CHECK();
}


// ---- split form -------------------------------------------------------------
uint32_t select_need_capacity(uint32_t n, uint32_t w1) { return w1 * (n + 1); }
uint32_t select_chunk_keys() { return dev::FS_MAX_KEYS; }

static size_t top_need_smem(uint32_t k, uint32_t w1) {
    return ((size_t)((w1 + 3) & ~3u) * 2 + dev::fs_nwords(k) + dev::FS_MAX_KEYS + 2048 + 64) * 4;
}
static size_t second_sel_smem(uint32_t k, uint32_t n, uint32_t w1, uint32_t w2) {
    const uint32_t nw = dev::fs_nwords(k);
    return ((size_t)nw + (nw + 1) / 2 + select_need_capacity(n, w1) + (size_t)w1 * n + w2 + w1 + 2048 + 64) * 4;
}
static size_t rows_smem(uint32_t dim) {
    const uint32_t dimp = (dim + dev::RW_PW - 1) / dev::RW_PW * dev::RW_PW;
    return ((size_t)dimp + (size_t)dev::RW_WARPS * dev::RW_NB * 32 * (dev::RW_PW + 4)) * 4;
}

bool select_split_supported(uint32_t k, uint32_t n, uint32_t w1, uint32_t w2, uint32_t dim, uint32_t capc) {
    return dim % 4 == 0 && dim <= 1024 && w1 <= 256 && w2 <= w1 * n && (uint64_t)w1 * (n + 1) <= 16384 &&
           capc <= 1024 && top_need_smem(k, w1) <= 200 * 1024 && second_sel_smem(k, n, w1, w2) <= 200 * 1024;
}

void launch_rows(const float* C, const float* Y, uint32_t k, uint32_t dim, int chunks, const uint32_t* list,
                 const uint32_t* cnt, uint32_t ld, uint32_t capc, float* out, uint32_t ldo, uint64_t nq,
                 cudaStream_t st) {
    if (nq == 0) return;
    dev::RowsArgs r{C, Y, k, dim, chunks, list, cnt, ld, capc, out, ldo};
    auto fn = dev::k_rows<dev::RW_WARPS, dev::RW_NB>;
    const size_t smem = rows_smem(dim);
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)nq, dev::RW_WARPS * 32, smem, st>>>(r);
    CUDA_LAUNCH_CHECK();
}

void launch_top_need(const SearchArgs& a, uint64_t nblocks, const float* Y, uint32_t w1, uint32_t w2,
                     const uint32_t* clist, const uint32_t* ccnt, uint32_t capc, const float* T, float cmax,
                     const uint32_t* qlist, const unsigned int* qcount, uint32_t* flagged, unsigned int* nflag,
                     const float* vals, uint32_t* nid, uint32_t* nneed, uint32_t ldn, cudaStream_t st,
                     const float* mu) {
    if (nblocks == 0) return;
    dev::FusedArgs f{Y, w1, w2, dev::FS_CS, clist, ccnt, capc, T, cmax, qlist, qcount, flagged, nflag, nullptr, nullptr,
                     mu};
    dev::NeedArgs na{vals, nid, nneed, ldn};
    const size_t smem = top_need_smem(a.k, w1);
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_top_need, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // 128 threads: 64 registers per thread cap 256-thread CTAs at 4 queries per
    // SM; 8 x 4 warps run twice as many queries (C3 first level 1.424 -> 1.402
    // ms; k_second_sel at 128 was slower, profiles/r2_study_fs_threads_c3.jsonl)
    dev::k_top_need<<<list_grid(nblocks, qlist != nullptr), dev::TN_THREADS, smem, st>>>(a, f, na);
    CUDA_LAUNCH_CHECK();
}

void launch_second_sel(const SearchArgs& a, uint64_t nq, uint32_t w1, uint32_t w2, const uint32_t* nid,
                       const float* nval, const uint32_t* nneed, uint32_t ldn, uint32_t* sel_out, float* ab_out,
                       cudaStream_t st) {
    if (nq == 0) return;
    dev::FusedArgs f{nullptr, w1, w2, dev::FS_CS, nullptr, nullptr, 0, nullptr, 0.0f, nullptr, nullptr,
                     nullptr, nullptr, sel_out, ab_out};
    dev::SecondArgs sa{nid, nval, nneed, ldn};
    const size_t smem = second_sel_smem(a.k, a.n, w1, w2);
    CUDA_CHECK(cudaFuncSetAttribute(dev::k_second_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dev::k_second_sel<<<(unsigned)nq, dev::FS_THREADS, smem, st>>>(a, f, sa);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq
