// TEST INFRASTRUCTURE -- C++ restatement of the reference's k-means
// (proj/src/kmeans.cpp) used only as a parity checker by tests/.  C++ (not C)
// because the reference's seeding draws from std::mt19937_64 through
// libstdc++'s uniform_int / uniform_real distributions; linking the same
// standard library reproduces its random stream exactly.
//
//   vo_train_kmeans  train_kmeans (kmeans.cpp:104-185): k-means++ seeding,
//                    Lloyd iterations, empty-cluster repair
//   vo_kmeans_seed   seed_centroids only (kmeans.cpp:54-102)
//   vo_kmeans_lloyd  the Lloyd + repair loop from given centroids
//                    (kmeans.cpp:117-183)
//
// Arithmetic follows SURVEY App. A: sequential fp32 sqdist without
// contraction (built with -ffp-contract=off), double sums in point order.
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

// sqdist (vecset.cpp:22-29)
float sqd(const float* a, const float* b, uint32_t d) {
    float acc = 0.0f;
    for (uint32_t i = 0; i < d; i++) {
        const float t = a[i] - b[i];
        acc = acc + t * t;
    }
    return acc;
}

// assign_nearest (kmeans.cpp:21-33): strict '<' from centroid 0
uint32_t nearest(const float* x, const float* C, uint32_t k, uint32_t dim, float* best_d) {
    uint32_t best = 0;
    float bd = std::numeric_limits<float>::max();
    for (uint32_t c = 0; c < k; c++) {
        const float d = sqd(x, C + (size_t)c * dim, dim);
        if (d < bd) {
            bd = d;
            best = c;
        }
    }
    *best_d = bd;
    return best;
}

// seed_centroids (kmeans.cpp:54-102): the first centre uniform, then D^2
// sampling; the running total is a fresh sequential double sum every step
void seed(const float* X, uint64_t n, uint32_t dim, uint32_t k, std::mt19937_64& rng, float* C) {
    std::uniform_int_distribution<size_t> first(0, n - 1);
    const size_t c0 = first(rng);
    std::memcpy(C, X + c0 * dim, (size_t)dim * 4);
    std::vector<float> md(n);
    for (uint64_t i = 0; i < n; i++) md[i] = sqd(X + i * dim, C, dim);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    for (uint32_t c = 1; c < k; c++) {
        double total = 0.0;
        for (uint64_t i = 0; i < n; i++) total += md[i];
        size_t pick;
        if (total <= 0) {
            pick = first(rng);
        } else {
            const double target = unif(rng) * total;
            double run = 0.0;
            pick = n - 1;
            for (uint64_t i = 0; i < n; i++) {
                run += md[i];
                if (run >= target) {
                    pick = i;
                    break;
                }
            }
        }
        float* dst = C + (size_t)c * dim;
        std::memcpy(dst, X + pick * dim, (size_t)dim * 4);
        for (uint64_t i = 0; i < n; i++) md[i] = std::min(md[i], sqd(X + i * dim, dst, dim));
    }
}

// Lloyd iterations + empty-cluster repair (kmeans.cpp:117-183)
void lloyd(const float* X, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, float* C) {
    std::vector<uint32_t> as(n);
    std::vector<float> dist(n);
    for (uint32_t it = 0; it < iters; it++) {
        for (uint64_t i = 0; i < n; i++) as[i] = nearest(X + i * dim, C, k, dim, &dist[i]);
        std::vector<double> sums((size_t)k * dim, 0.0), err(k, 0.0);
        std::vector<uint64_t> cnt(k, 0);
        for (uint64_t i = 0; i < n; i++) {
            const uint32_t c = as[i];
            cnt[c]++;
            err[c] += dist[i];
            for (uint32_t d = 0; d < dim; d++) sums[(size_t)c * dim + d] += X[i * dim + d];
        }
        for (uint32_t c = 0; c < k; c++) {
            if (!cnt[c]) continue;
            for (uint32_t d = 0; d < dim; d++)
                C[(size_t)c * dim + d] = (float)(sums[(size_t)c * dim + d] / (double)cnt[c]);
        }
        for (uint32_t c = 0; c < k; c++) {
            if (cnt[c]) continue;
            const uint32_t donor = (uint32_t)(std::max_element(err.begin(), err.end()) - err.begin());
            uint64_t far_i = 0;
            float far_d = -1.0f;
            for (uint64_t i = 0; i < n; i++)
                if (as[i] == donor && dist[i] > far_d) {
                    far_d = dist[i];
                    far_i = i;
                }
            std::memcpy(C + (size_t)c * dim, X + far_i * dim, (size_t)dim * 4);
            cnt[c] = 1;
            as[far_i] = c;
            err[donor] -= far_d;
            dist[far_i] = 0.0f;
            err[c] = 0.0;
        }
    }
}

int check(uint64_t n, uint32_t k, uint32_t iters) {
    if (k == 0 || n < k) {
        g_err = "train_kmeans: need at least k training points";
        return -1;
    }
    if (iters == 0) {
        g_err = "train_kmeans: iters must be >= 1";
        return -1;
    }
    return 0;
}

}  // namespace

extern "C" {

const char* vo_train_last_error(void) { return g_err.c_str(); }

int vo_train_kmeans(const float* X, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed_v,
                    float* out) {
    if (check(n, k, iters)) return -1;
    std::mt19937_64 rng(seed_v);
    seed(X, n, dim, k, rng, out);
    lloyd(X, n, dim, k, iters, out);
    return 0;
}

int vo_kmeans_seed(const float* X, uint64_t n, uint32_t dim, uint32_t k, uint64_t seed_v, float* out) {
    if (check(n, k, 1)) return -1;
    std::mt19937_64 rng(seed_v);
    seed(X, n, dim, k, rng, out);
    return 0;
}

int vo_kmeans_lloyd(const float* X, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, const float* init,
                    float* out) {
    if (check(n, k, iters)) return -1;
    std::memcpy(out, init, (size_t)k * dim * 4);
    lloyd(X, n, dim, k, iters, out);
    return 0;
}

// quantization_error (kmeans.cpp:35-51): sum of nearest squared distances
double vo_quantization_error(const float* X, uint64_t n, uint32_t dim, const float* C, uint32_t k) {
    double acc = 0.0;
    for (uint64_t i = 0; i < n; i++) {
        float d;
        nearest(X + i * dim, C, k, dim, &d);
        acc += d;
    }
    return acc;
}

}  // extern "C"
