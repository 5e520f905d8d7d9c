// Single frame-set latency through the C ABI from C++ (no Python): cfg1 and cfg3 plans, one
// resident frame-set, (a) CUDA events around one pnce_process_frames call after an idle gap,
// (b) host wall time of the call + synchronize, (c) the same launch replayed from a CUDA graph.
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../include/pnce_b200.h"

static double median(std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }

int main() {
    struct G { const char* name; int m, c, nt, nr, nb, l, deg; uint32_t mask; };
    G gs[] = {{"cfg1", 127, 16, 4, 4, 1, 16, 7, (1u << 6) | (1u << 5)}, {"cfg3", 1023, 64, 64, 64, 8, 64, 10, (1u << 9) | (1u << 2)}};
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (const G& g : gs) {
        pnce_cfg_t cfg{g.m, g.c, g.nt, g.nr, g.nb, g.l, g.deg, g.mask, 1u, 0};
        pnce_plan_t* plan = nullptr;
        if (pnce_plan_create(&cfg, &plan, st) != PNCE_OK) { printf("plan: %s\n", pnce_last_error()); return 1; }
        const int nbat = (g.nt + g.nb - 1) / g.nb;
        const size_t iq_n = (size_t)nbat * g.nr * (g.c + g.m + g.l - 1) * 2, taps_n = (size_t)g.nr * g.nt * g.l * 2;
        float *iq, *taps, *h;
        cudaMalloc(&iq, iq_n * 4);
        cudaMalloc(&taps, taps_n * 4);
        cudaMalloc(&h, taps_n * 4);
        pnce_draw_channel(plan, g.l, 1, h, 1, st);
        pnce_simulate_frames(plan, h, 10.0, 2, iq, 1, st);
        cudaStreamSynchronize(st);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        std::vector<double> ev, wall;
        for (int i = 0; i < 300; ++i) {
            cudaStreamSynchronize(st);
            auto t0 = std::chrono::steady_clock::now();
            cudaEventRecord(a, st);
            pnce_process_frames(plan, iq, taps, nullptr, nullptr, nullptr, 0, 1, st);
            cudaEventRecord(b, st);
            cudaStreamSynchronize(st);
            auto t1 = std::chrono::steady_clock::now();
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (i >= 50) { ev.push_back(ms * 1e3); wall.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count()); }
        }
        // graph replay of the same launch
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        pnce_process_frames(plan, iq, taps, nullptr, nullptr, nullptr, 0, 1, st);
        cudaStreamEndCapture(st, &graph);
        int gerr = cudaGraphInstantiate(&exec, graph, 0);
        std::vector<double> gev, gwall;
        for (int i = 0; gerr == 0 && i < 300; ++i) {
            cudaStreamSynchronize(st);
            auto t0 = std::chrono::steady_clock::now();
            cudaEventRecord(a, st);
            cudaGraphLaunch(exec, st);
            cudaEventRecord(b, st);
            cudaStreamSynchronize(st);
            auto t1 = std::chrono::steady_clock::now();
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (i >= 50) { gev.push_back(ms * 1e3); gwall.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count()); }
        }
        printf("%s: direct call: events %.1f us, host wall (call+sync) %.1f us | graph replay: events %.1f us, wall %.1f us (graph err %d)\n",
               g.name, median(ev), median(wall), gev.empty() ? -1.0 : median(gev), gwall.empty() ? -1.0 : median(gwall), gerr);
        pnce_plan_destroy(plan);
    }
    return 0;
}
