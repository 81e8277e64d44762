// Device-side synthetic data of the reference's law (dataset.cpp:13-44):
// C centres ~ U[0,1]^D, each point picks a centre uniformly and adds
// N(0, spread^2) per coordinate.  The reference draws sequentially from one
// mt19937_64 stream (bit-identical host copy: vlq_gen_synthetic); at 1e8-1e9
// points that is hours of host time, so this generator is counter-based
// (a keyed 64-bit mix per (seed, row, column)), making any row regenerable
// independently on any device or on the host (SURVEY §8d "Generation").
#include "kernels.h"

namespace vlq {
namespace dev {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ float u01(uint64_t h) {  // (0, 1]
    return ((float)(uint32_t)(h >> 40) + 1.0f) * (1.0f / 16777216.0f);
}

__host__ __device__ __forceinline__ float center_coord(uint64_t seed, uint32_t c, uint32_t j) {
    return u01(mix64(seed ^ mix64(0xC0FFEEull + ((uint64_t)c << 20) + j))) - (1.0f / 16777216.0f);
}

__global__ void k_synth(uint64_t first, uint64_t count, uint32_t dim, uint32_t clusters, float spread, uint64_t seed,
                        float* __restrict__ out) {
    const uint64_t total = count * dim;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = first + t / dim;
        const uint32_t j = (uint32_t)(t % dim);
        const uint64_t rk = mix64(seed * 0x632be59bd9b4e019ull + row);
        const uint32_t c = (uint32_t)(mix64(rk) % clusters);
        // Box-Muller on two keyed uniforms
        const uint64_t h = mix64(rk ^ (0x5851f42d4c957f2dull * (uint64_t)(j + 1)));
        const float u1 = u01(h), u2 = u01(mix64(h));
        const float g = sqrtf(-2.0f * logf(u1)) * cosf(6.283185307179586f * u2);
        out[t] = center_coord(seed, c, j) + spread * g;
    }
}

}  // namespace dev

void launch_synth(uint64_t first, uint64_t count, uint32_t dim, uint32_t clusters, float spread, uint64_t seed,
                  float* out, cudaStream_t st) {
    if (count == 0) return;
    dev::k_synth<<<4736, 256, 0, st>>>(first, count, dim, clusters, spread, seed, out);
    CUDA_LAUNCH_CHECK();
}

}  // namespace vlq
