// Shared device helpers for the VLQ-ADC B200 engine.
//
// Numeric contract: the reference (/root/reference/proj) is compiled -O3
// without -march, i.e. plain SSE2 fp32 with no FMA, every reduction a
// left-to-right scalar loop.  Every "exact" routine here
// reproduces that with __fadd_rn/__fsub_rn/__fmul_rn/__fdiv_rn, which nvcc
// never contracts into FFMA, in the reference's operation order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#define VLQ_KSUB 256u

namespace vlq {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw CudaError(std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                        "): " + cudaGetErrorString(e));
    }
}

}  // namespace vlq

#define CUDA_CHECK(x) ::vlq::cuda_check((x), #x, __FILE__, __LINE__)
#define CUDA_LAUNCH_CHECK() ::vlq::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

namespace vlq {
namespace dev {

// sqdist (proj/src/vecset.cpp:22-29): acc = acc + (a-b)*(a-b), in order.
__device__ __forceinline__ float sq_step(float acc, float a, float b) {
    float t = __fsub_rn(a, b);
    return __fadd_rn(acc, __fmul_rn(t, t));
}
// dot (vecset.cpp:39-45) / sqnorm (:31-37)
__device__ __forceinline__ float dot_step(float acc, float a, float b) {
    return __fadd_rn(acc, __fmul_rn(a, b));
}

// std::clamp semantics (returns v for NaN).
__device__ __forceinline__ float clamp_std(float v, float lo, float hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// line_lambda (proj/src/line_quant.cpp:9-14): (0.5f*((a+c)-b))/c.
__device__ __forceinline__ float line_lambda(float a, float b, float c) {
    return __fdiv_rn(__fmul_rn(0.5f, __fsub_rn(__fadd_rn(a, c), b)), c);
}

// line_sqdist (line_quant.cpp:20-22): (((1-l)*a) + ((l*l-l)*c)) + (l*b).
__device__ __forceinline__ float line_sqdist(float a, float b, float c, float l) {
    float t0 = __fmul_rn(__fsub_rn(1.0f, l), a);
    float t1 = __fmul_rn(__fsub_rn(__fmul_rn(l, l), l), c);
    return __fadd_rn(__fadd_rn(t0, t1), __fmul_rn(l, b));
}

// dequantize_lambda (proj/src/index.cpp:19-21): lo + (((b+0.5)*(hi-lo))/256).
// Division by 256 is an exact power-of-two scaling, so the multiply by
// 2^-8 below is bit-identical for every normal result.
__device__ __forceinline__ float dequantize_lambda(uint32_t b, float lo, float hi) {
    float t = __fmul_rn(__fadd_rn((float)b, 0.5f), __fsub_rn(hi, lo));
    return __fadd_rn(lo, __fdiv_rn(t, 256.0f));
}

// quantize_lambda (index.cpp:12-17).
__device__ __forceinline__ uint32_t quantize_lambda(float lam, float lo, float hi) {
    float c = clamp_std(lam, lo, hi);
    float step = __fdiv_rn(__fsub_rn(hi, lo), 256.0f);
    float q = __fdiv_rn(__fsub_rn(c, lo), step);
    int level = (int)q;  // C++ float->int truncation (cvt.rzi)
    level = level < 0 ? 0 : (level > 255 ? 255 : level);
    return (uint32_t)level;
}

// Order-preserving map of a float to u32; -0 is canonicalised to +0 so the
// reference comparators' (a == b) tie semantics hold.
__device__ __forceinline__ uint32_t ord_float(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u << 1) == 0) u = 0;  // +-0 -> +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_float(uint32_t u) {
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t make_key(float f, uint32_t idx) {
    return ((uint64_t)ord_float(f) << 32) | idx;
}

// |approx(x, c) + |x|^2 - sqdist(x, c)| <= tc_eps for every centroid c of the
// tensor-core coarse stage (approx = |c|^2 - 2 <x, c> on TF32 operands, fp32
// accumulation; sqdist the exact sequential reference sum): TF32 operands keep
// 10 mantissa bits (<= 2^-10 relative per factor); 3xTF32 (split) leaves
// <= 3 * 2^-21 from the dropped lo.lo term and truncated lo parts; the fp32
// norm and the sequential sqdist each add D u |.|; x 1.5 safety factor.
// rna: both operands were rounded to TF32 beforehand (cvt.rna, <= 2^-11 each).
// centered: both operands were shifted by a common mu in fp32 (y' = fl(y - mu),
// c' = fl(c - mu); xnorm2 = |y'|^2, cmax = max |c'|): | |y' - c'|^2 - |y - c|^2 |
// <= 2 u s |y - c| + u^2 s^2 <= 3 u s^2 more.
__device__ __forceinline__ float tc_eps(float xnorm2, float cmax, uint32_t dim, bool split = false,
                                        bool rna = false, bool centered = false) {
    // 1xTF32: each operand keeps 10 mantissa bits (<= 2^-10 relative per factor, truncated;
    // <= 2^-11 rounded); 3xTF32: the dropped lo.lo term and the truncated lo parts leave <= 3 * 2^-21
    const float xn = sqrtf(xnorm2);
    const float s = xn + cmax;
    const float u = 5.9604645e-08f;
    const float rel = split ? 1.430511474609375e-06f : (rna ? 9.765625e-4f : 1.953125e-3f);
    const float cu = centered ? 5.0f : 2.0f;
    return 1.5f * (2.0f * (rel + dim * u) * xn * cmax + dim * u * (s * s + cmax * cmax) + cu * u * s * s) + 1e-30f;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

}  // namespace dev
}  // namespace vlq
