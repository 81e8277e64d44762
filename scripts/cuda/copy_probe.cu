// Pinned-copy probe: H2D 3.84 MB + D2H 12 MB timed with events on a
// non-blocking stream, after the host touched the pinned buffer from one or
// several threads (write before the H2D, read after the D2H), with and
// without flushing those lines from the CPU caches (clflushopt) or using
// non-temporal stores -- cache-resident dirty / shared lines make the DMA slow.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <cstdio>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>
__attribute__((target("clflushopt"))) static void flush(const unsigned char* p, size_t n) {
    for (size_t i = 0; i < n; i += 64) _mm_clflushopt((void*)(p + i));
    _mm_sfence();
}
static void nt_copy(unsigned char* d, const unsigned char* s, size_t n) {  // n multiple of 16, d 16-aligned
    for (size_t i = 0; i < n; i += 16) _mm_stream_si128((__m128i*)(d + i), _mm_loadu_si128((const __m128i*)(s + i)));
    _mm_sfence();
}
enum Mode { ST, MT, MT_FLUSH, MT_NT };
static void par(int nt, size_t n, const std::function<void(size_t, size_t)>& f) {
    std::vector<std::thread> th;
    size_t per = (n / nt + 63) & ~(size_t)63;
    for (int t = 0; t < nt; t++) th.emplace_back([=] { if (t * per < n) f(t * per, std::min(per, n - t * per)); });
    for (auto& x : th) x.join();
}
static void run(const char* name, unsigned char* h, unsigned char* d, cudaStream_t st, Mode m) {
    const size_t qb = 3840000, ob = 12000000;
    std::vector<unsigned char> src(qb, 1), dst(ob);
    cudaEvent_t e[3];
    for (auto& x : e) cudaEventCreate(&x);
    for (int it = 0; it < 6; it++) {
        if (m == ST) memcpy(h, src.data(), qb);
        else if (m == MT) par(8, qb, [&](size_t o, size_t n) { memcpy(h + o, src.data() + o, n); });
        else if (m == MT_FLUSH) par(8, qb, [&](size_t o, size_t n) { memcpy(h + o, src.data() + o, n); flush(h + o, n); });
        else par(8, qb, [&](size_t o, size_t n) { nt_copy(h + o, src.data() + o, n); });
        cudaEventRecord(e[0], st);
        cudaMemcpyAsync(d, h, qb, cudaMemcpyHostToDevice, st);
        cudaEventRecord(e[1], st);
        cudaMemcpyAsync(h + qb, d + qb, ob, cudaMemcpyDeviceToHost, st);
        cudaEventRecord(e[2], st);
        cudaStreamSynchronize(st);
        // copy-out of the D2H region (as the host API does), then the next iteration's D2H lands on it
        if (m == ST) memcpy(dst.data(), h + qb, ob);
        else if (m == MT) par(8, ob, [&](size_t o, size_t n) { memcpy(dst.data() + o, h + qb + o, n); });
        else par(8, ob, [&](size_t o, size_t n) { memcpy(dst.data() + o, h + qb + o, n); flush(h + qb + o, n); });
        float a, b;
        cudaEventElapsedTime(&a, e[0], e[1]);
        cudaEventElapsedTime(&b, e[1], e[2]);
        if (it >= 3) printf("%-22s h2d %.3f ms (%.1f GB/s)  d2h %.3f ms (%.1f GB/s)\n", name, a, qb / a / 1e6, b, ob / b / 1e6);
    }
}
int main() {
    unsigned char *h, *d;
    cudaMalloc(&d, 16000000);
    cudaMallocHost((void**)&h, 16000000);
    cudaStream_t nb;
    cudaStreamCreateWithFlags(&nb, cudaStreamNonBlocking);
    run("single thread", h, d, nb, ST);
    run("8 threads", h, d, nb, MT);
    run("8 threads + clflushopt", h, d, nb, MT_FLUSH);
    run("8 threads nt-store", h, d, nb, MT_NT);
    return 0;
}
