// Host f32 -> f16 conversion rate (F16C, RN-even) with T threads on pinned-like memory: can the
// host halve the PCIe bytes of the end-to-end path faster than PCIe moves them?
//   g++ -O3 -mavx2 -mf16c -pthread -o tools/bin/f16c_probe tools/f16c_probe.cpp
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void conv(const float* src, uint16_t* dst, size_t n) {
    size_t i = 0;
    for (; i + 16 <= n; i += 16) {
        __m256 a = _mm256_loadu_ps(src + i), b = _mm256_loadu_ps(src + i + 8);
        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), _mm256_cvtps_ph(a, _MM_FROUND_TO_NEAREST_INT));
        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i + 8), _mm256_cvtps_ph(b, _MM_FROUND_TO_NEAREST_INT));
    }
    for (; i < n; ++i) dst[i] = _cvtss_sh(src[i], _MM_FROUND_TO_NEAREST_INT);
}

int main() {
    const size_t n = (size_t)1 << 28;  // 1 GiB of f32
    float* src = static_cast<float*>(aligned_alloc(64, n * 4));
    uint16_t* dst = static_cast<uint16_t*>(aligned_alloc(64, n * 2));
    for (size_t i = 0; i < n; ++i) src[i] = (float)(i % 1000) * 0.001f;
    memset(dst, 0, n * 2);
    for (int T : {1, 2, 4, 8, 12, 16}) {
        double best = 1e30;
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([=] {
                    const size_t a = n * t / T, b = n * (t + 1) / T;
                    conv(src + a, dst + a, b - a);
                });
            for (auto& x : th) x.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = s < best ? s : best;
        }
        printf("threads %2d: %.1f GB/s of f32 input (%.1f us per 4.19 MB cfg3 frame-set)\n", T, n * 4 / best / 1e9,
               4.19e6 / (n * 4 / best) * 1e6);
    }
    return 0;
}
