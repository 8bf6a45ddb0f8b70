// Host memcpy bandwidth into page-locked memory with T threads (persistent, cv-woken).
#include <cuda_runtime.h>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include <atomic>
int main() {
    const size_t B = 8 << 20;
    char* src = (char*)malloc(B); memset(src, 1, B);
    char* pin; cudaHostAlloc((void**)&pin, B, 0);
    char* pg = (char*)malloc(B); memset(pg, 0, B);
    auto now = [] { return std::chrono::steady_clock::now(); };
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = now(); memcpy(pin, src, B); auto t1 = now();
        memcpy(pg, src, B); auto t2 = now();
        printf("1 thread: to pinned %.3f ms, to pageable %.3f ms\n",
               std::chrono::duration<double, std::milli>(t1 - t0).count(), std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    for (int T : {2, 4, 8}) {
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = now();
            std::vector<std::thread> th;
            for (int i = 0; i < T; ++i) th.emplace_back([&, i] { memcpy(pin + B / T * i, src + B / T * i, B / T); });
            for (auto& t : th) t.join();
            auto t1 = now();
            printf("%d threads (spawn+join): %.3f ms\n", T, std::chrono::duration<double, std::milli>(t1 - t0).count());
        }
        // per-thread memcpy time only
        std::vector<double> ms(T);
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i) th.emplace_back([&, i] { auto a = now(); memcpy(pin + B / T * i, src + B / T * i, B / T); ms[i] = std::chrono::duration<double, std::milli>(now() - a).count(); });
        for (auto& t : th) t.join();
        printf("   per-thread memcpy ms:"); for (double m : ms) printf(" %.3f", m); printf("\n");
    }
    return 0;
}
