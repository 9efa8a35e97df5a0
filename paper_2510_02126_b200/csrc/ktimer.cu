// ktimer.cu -- optional CUDA-event timing of one kernel class on its launch
// stream (used by bench.py for the roofline of the dominant kernel).  When a
// class is enabled, every launch of that class is bracketed by two events on
// the launching stream; lyap_kernel_stats() sums the elapsed times.
#include <vector>
#include <mutex>
#include "common.cuh"
#include "ktimer.h"

namespace lyap {

namespace {
struct Pair { cudaEvent_t a, b; };
std::mutex g_mu;
int g_enabled = -1;
std::vector<Pair> g_pool;
size_t g_used = 0;
double g_ms = 0.0;
int64_t g_count = 0;

cudaEvent_t *slot(size_t i, int which) {
    while (g_pool.size() <= i) {
        Pair p;
        cudaEventCreate(&p.a);
        cudaEventCreate(&p.b);
        g_pool.push_back(p);
    }
    return which ? &g_pool[i].b : &g_pool[i].a;
}

void drain() {
    for (size_t i = 0; i < g_used; i++) {
        float ms = 0.f;
        cudaEventSynchronize(g_pool[i].b);
        cudaEventElapsedTime(&ms, g_pool[i].a, g_pool[i].b);
        g_ms += ms;
        g_count++;
    }
    g_used = 0;
}
}  // namespace

void ktimer_begin(int cls, cudaStream_t s) {
    if (cls != g_enabled) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_used >= 4096) drain();
    cudaEventRecord(*slot(g_used, 0), s);
}

double g_flops = 0.0, g_bytes = 0.0;
void ktimer_work(int cls, double flops, double bytes) {
    if (cls != g_enabled) return;
    std::lock_guard<std::mutex> lk(g_mu);
    g_flops += flops;
    g_bytes += bytes;
}

void ktimer_end(int cls, cudaStream_t s) {
    if (cls != g_enabled) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(*slot(g_used, 1), s);
    g_used++;
}

}  // namespace lyap

extern "C" int lyap_kernel_timing(int cls) {
    using namespace lyap;
    std::lock_guard<std::mutex> lk(g_mu);
    drain();
    g_enabled = cls;
    g_ms = 0.0;
    g_count = 0;
    g_flops = 0.0;
    g_bytes = 0.0;
    return LYAP_OK;
}

extern "C" int lyap_kernel_stats(double *ms, int64_t *launches) {
    using namespace lyap;
    std::lock_guard<std::mutex> lk(g_mu);
    drain();
    if (ms) *ms = g_ms;
    if (launches) *launches = g_count;
    return LYAP_OK;
}

extern "C" int lyap_kernel_work(double *flops, double *bytes) {
    using namespace lyap;
    std::lock_guard<std::mutex> lk(g_mu);
    if (flops) *flops = g_flops;
    if (bytes) *bytes = g_bytes;
    return LYAP_OK;
}
