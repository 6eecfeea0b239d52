// Phase-timeline probe of qft_cdft_smem (tools only, not shipped): compiles the
// kernel with QFT_PROBE so thread 0 of every CTA records clock64() at each
// phase barrier, runs the config-2 (or -DPLOG2N=k) workload on random data and
// prints the median cycles per phase.  Build + run: tools/probe/run_probe.sh
#ifndef NOPROBE
#define QFT_PROBE 1
#endif
#ifdef PIPE2
#define QFT_PIPE 2
#endif
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstring>
#include "../../paper_1301_0763_b200/csrc/qft_pipe.cuh"

// qft_probe_buf is defined by qft_launch.cuh under QFT_PROBE

#ifndef PLOG2N
#define PLOG2N 12
#endif

int main(int argc, char **argv) {
    constexpr int LOG2N = PLOG2N, N = 1 << LOG2N;
    long long batch = argc > 1 ? atoll(argv[1]) : (LOG2N == 12 ? 16384 : 262144 / 4);
#ifdef PIPE2
    using K = qft::PCfg<LOG2N, float>;
#define LAUNCH qft::launch_pipe<LOG2N, float>
#elif defined(PIPE)
    using K = qft::PCfg<LOG2N, float>;
#define LAUNCH qft::launch_pipe<LOG2N, float>
#else
    using K = qft::KCfg<LOG2N, float>;
#define LAUNCH qft::launch_smem<LOG2N, float, 0>
#endif
    printf("N=2^%d batch=%lld TT=%d NW=%d SMEM=%d\n", LOG2N, batch, K::TT, K::NW, K::SMEM);
    size_t bytes = (size_t)batch * N * 8;
    float *in, *out, *U;
    cudaMalloc(&in, bytes);
    cudaMalloc(&out, bytes);
    cudaMalloc(&U, N / 4 * 4);
    std::vector<float> h(N / 4, 0.5f), hin(1 << 20);
    for (auto &v : hin) v = (float)rand() / RAND_MAX - 0.5f;
    for (size_t o = 0; o < bytes / 4; o += hin.size()) cudaMemcpy(in + o, hin.data(), std::min(hin.size(), bytes / 4 - o) * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(U, h.data(), N, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    qft::LaunchArgs a{in, out, batch, U, h.data(), sms, 0};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) LAUNCH(a);
    cudaEventRecord(e0);
    const int REP = 10;
    for (int i = 0; i < REP; ++i) LAUNCH(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= REP;
    printf("kernel %.3f ms  %.2f M tr/s  %.1f GB/s  err=%s\n", ms, batch / ms / 1e3, batch * N * 16.0 / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
#ifdef NOPROBE
    return 0;
#else
    std::vector<long long> b(160 * 16 * 64);
    cudaMemcpyFromSymbol(b.data(), qft_probe_buf, b.size() * 8);
#ifdef PIPE2
    // per warp, relative to warp 0's units start of the same iteration: units start / end,
    // after its wait (D: udone, A0: tma) / end of D or A0; CTA 0 and CTA 77, iterations 5..7
    for (int c : {0, 77})
        for (int it = 5; it < 8; ++it) {
            long long *m = &b[(c * 16 + it) * 64], t0 = m[24];
            printf("CTA %d it %d:", c, it);
            for (int w = 0; w < K::NW; ++w)
                printf(" w%d[%lld %lld %lld %lld]", w, m[24 + w] - t0, m[8 + w] - t0, m[40 + w] - t0, m[52 + w] - t0);
            printf("\n");
        }
    {
        std::vector<double> itv;
        for (int c = 0; c < sms; ++c)
            for (int it = 2; it < 14; ++it) itv.push_back(b[(c * 16 + it + 1) * 64 + 24] - b[(c * 16 + it) * 64 + 24]);
        std::sort(itv.begin(), itv.end());
        printf("median iteration (warp 0 units start to next) %.0f cycles\n", itv[itv.size() / 2]);
    }
    return 0;
#endif
#ifdef PIPE
    {   // bitwise check against the unpipelined kernel on the same input
        float *out2;
        cudaMalloc(&out2, bytes);
        qft::LaunchArgs a2{in, out2, batch, U, h.data(), sms, 0};
        qft::launch_smem<LOG2N, float, 0>(a2);
        std::vector<float> r1(bytes / 4), r2(bytes / 4);
        cudaMemcpy(r1.data(), out, bytes, cudaMemcpyDeviceToHost);
        cudaMemcpy(r2.data(), out2, bytes, cudaMemcpyDeviceToHost);
        size_t bad = 0;
        for (size_t i = 0; i < r1.size(); ++i) bad += memcmp(&r1[i], &r2[i], 4) != 0;
        printf("bitwise vs qft_cdft_smem: %zu differing words of %zu\n", bad, r1.size());
        cudaFree(out2);
    }
#endif

#ifdef PIPE
    {   // per warp: end of its phase-2 work (D or in-place A0) and, for A0 warps, the end of
        // the TMA wait, relative to the phase-2 start (mark 3); medians over CTAs, iterations 2..13
        printf("phase-2 per warp (median cycles after the units barrier): ");
        for (int w = 0; w < K::NW; ++w) {
            std::vector<double> e, wt;
            for (int c = 0; c < sms; ++c)
                for (int it = 2; it < 14; ++it) {
                    long long *m = &b[(c * 16 + it) * 64];
                    e.push_back(m[52 + w] - m[3]);
                    wt.push_back(m[40 + w] - m[3]);
                }
            std::sort(e.begin(), e.end());
            std::sort(wt.begin(), wt.end());
            const bool a0 = w >= K::NWD && w < K::NWD + K::NWA;
            if (a0) printf("w%d[A0 wait %.0f end %.0f] ", w, wt[wt.size() / 2], e[e.size() / 2]);
            else printf("w%d[D end %.0f] ", w, e[e.size() / 2]);
        }
        printf("\n");
    }
#endif
    // per-phase durations over CTAs < sms, iterations 2..13
#ifdef PIPE
    // pipe marks: 1 start, 3 after units, 4 D done (thread 0), 5 after phase-2 barrier
    for (int c = 0; c < sms; ++c)
        for (int it = 0; it < 16; ++it) {
            long long *m = &b[(c * 16 + it) * 64];
            m[0] = m[1];
            m[2] = m[1];
        }
    const char *names[] = {"-", "-", "units", "D(thr0)", "A0_extra", "loop"};
    for (int c = 0; c < sms; ++c)
        for (int it = 0; it < 15; ++it) b[(c * 16 + it) * 64 + 0] = b[(c * 16 + it) * 64 + 0];
#else
    const char *names[] = {"tma_wait", "A0", "units", "D(thr0)", "D_bar", "loop"};
#endif
    std::vector<double> ph[6], wspread, wmin;
    for (int c = 0; c < sms; ++c)
        for (int it = 2; it < 14; ++it) {
            long long *m = &b[(c * 16 + it) * 64], *mn = &b[(c * 16 + it + 1) * 64];
            ph[0].push_back(m[1] - m[0]);
            ph[1].push_back(m[2] - m[1]);
            ph[2].push_back(m[3] - m[2]);
            ph[3].push_back(m[4] - m[3]);
            ph[4].push_back(m[5] - m[4]);
#ifdef PIPE
            ph[5].push_back(mn[1] - m[5]);
#else
            ph[5].push_back(mn[0] - m[5]);
#endif
            long long lo = 1LL << 62, hi = 0;
            for (int w = 0; w < K::NW; ++w) {
                lo = std::min(lo, m[8 + w] - m[2]);
                hi = std::max(hi, m[8 + w] - m[2]);
            }
            wmin.push_back(lo);
            wspread.push_back(hi);
        }
    auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    };
    double tot = 0;
    for (int k = 0; k < 6; ++k) tot += med(ph[k]);
    for (int k = 0; k < 6; ++k) printf("  %-9s %7.0f cycles (%4.1f%%)\n", names[k], med(ph[k]), 100 * med(ph[k]) / tot);
    printf("  iteration %7.0f cycles = %.0f per transform; units: first warp done %.0f, last %.0f\n", tot, tot / K::TT,
           med(wmin), med(wspread));
    long long *u = &b[160 * 16 * 64 - 64];
    {
        long long *m = &b[(0 * 16 + 14) * 64];
        printf("  CTA 0 iteration 15: start %lld, unit start +%lld, units barrier +%lld\n", m[1], u[0] - m[1], m[3] - m[1]);
        printf("  m5 -> after TMA issue %lld -> m1(next) %lld\n", m[6] - m[5], (m + 64)[1] - m[5]);
        printf("  phase 2 per warp (rel. to units barrier m3): tma-wait-end/end:");
        for (int w = 0; w < K::NW; ++w) printf(" w%d %lld/%lld", w, m[40 + w] - m[3], m[52 + w] - m[3]);
        printf("\n");
        printf("  per-warp units start/end (rel. to the previous phase-2 barrier exit m5):");
        long long *mp = m - 64;
        for (int w = 0; w < K::NW; ++w) printf(" %lld/%lld", m[24 + w] - mp[5], m[8 + w] - mp[5]);
        printf("\n");
    }
    printf("  TMA issue (CTA 0 last): fence %lld, expect_tx %lld, copies %lld\n", u[11] - u[10], u[12] - u[11], u[13] - u[12]);
    printf("  unit_big (CTA 0 warp 0, last iteration): F load+fold %lld, F store %lld, Lee-32 %lld, C %lld cycles\n",
           u[1] - u[0], u[2] - u[1], u[3] - u[2], u[4] - u[3]);
    return 0;
#endif
}
