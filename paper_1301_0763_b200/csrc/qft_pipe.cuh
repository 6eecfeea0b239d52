// qft_pipe.cuh -- software-pipelined single-pass kernel (complex cdft, N <= 4096).
//
// Same phases and the same per-cell arithmetic as qft_cdft_smem (qft_launch.cuh),
// scheduled so that the latency-bound chain phase D of batch i overlaps the
// fold/route phase A0 of batch i+1 on other warps:
//
//   two buffer sets X[0], X[1] of TT signal slots each (a slot is one padded
//   working area, PADDED cells >= N, so the raw signal fits in it);
//   TMA bulk-loads the raw signals of batch i into set i&1;
//   A0 runs IN PLACE in the slot: a warp group loads the raw samples into
//   registers, synchronises on a named barrier, then stores the folded cells
//   (the loads of a slot all precede its stores);
//
//   per batch i:   units(i) on X[i&1]                      all warps
//                  __syncthreads
//                  D(i) from X[i&1] -> y                   warps [0, NWD)
//                  | wait TMA(i+1), A0(i+1) in X[(i+1)&1]  warps [NWD, NWD+NWA)
//                  __syncthreads
//                  TMA(i+2) -> X[i&1]                      thread 0
//
// The probe (tools/probe) measured D at ~30 % of the unpipelined iteration with
// only half the warps busy; here those idle warps fold the next batch.
#pragma once
#include "qft_launch.cuh"

#ifndef QFT_PIPE
#define QFT_PIPE 1  // serve fp32 N = 4096 cdft with the pipelined kernel (1: barrier-phased, 2: dataflow -- measured no faster)
#endif
#ifndef QFT_PIPE_DSPREAD
#define QFT_PIPE_DSPREAD 0  // phase-D items spread evenly over all non-A0 warps (measured -0.5 %)
#endif
#ifndef QFT_PIPE_NW_EXTRA
#define QFT_PIPE_NW_EXTRA 0  // extra warps (phase D with QFT_PIPE_DSPREAD)
#endif
#ifndef QFT_PIPE_NWA
#define QFT_PIPE_NWA 5  // warps running the in-place A0 of the next batch during D
#endif
#ifndef QFT_PIPE_TMA_EARLY
// refill TMA of the consumed buffer set issued by warp 0 as soon as the D warps
// are done (named barrier), instead of after the CTA barrier at the head of the
// next units phase (where warp 0 runs a unit on the critical path)
#define QFT_PIPE_TMA_EARLY 0
#endif
#ifndef QFT_PIPE_UMAP
#define QFT_PIPE_UMAP 1  // measured +0.3 % (55.13 vs 54.91M tr/s, 3 interleaved rounds)
#endif
#ifndef QFT_PIPE_SMALLD
#define QFT_PIPE_SMALLD 1  // blocks with L <= 16 in phase 2 (idle D lanes) instead of a divergent rest-unit lane
#endif
#ifndef QFT_PIPE_L2PF
#define QFT_PIPE_L2PF 0  // L2 bulk prefetch of the batch after the next
#endif
#ifndef QFT_PIPE_TMA_WARP
// warp issuing the refill TMA after the phase-2 barrier: an A0 warp has no
// outstanding global stores for its fence.proxy.async to drain (a D warp does)
#define QFT_PIPE_TMA_WARP 0
#endif
#ifndef QFT_PIPE_ITEMS
// A0 items n = 64c: their samples x[64c] / x[N-64c] come from the chunk loads
// (chunk c lane 0 / chunk c-1 lane 31) through a small per-slot array, instead of
// 32 loads at stride 64 cells (all in one bank: 16-way conflicts)
#define QFT_PIPE_ITEMS 0  // measured -6 % (51.6 vs 54.9M tr/s): the items then wait on the named barrier
#endif

// probe marks of the dataflow kernel, individually selectable (tools/probe)
#if defined(QFT_PROBE) && !defined(QFT_PMASK)
#define QFT_PMASK 15
#endif
#if defined(QFT_PROBE) && (QFT_PMASK & 1)
#define QFT_PMARK24() QFT_WMARK_AT(24)
#else
#define QFT_PMARK24() do {} while (0)
#endif
#if defined(QFT_PROBE) && (QFT_PMASK & 2)
#define QFT_PMARK8() QFT_WMARK_AT(8)
#else
#define QFT_PMARK8() do {} while (0)
#endif
#if defined(QFT_PROBE) && (QFT_PMASK & 4)
#define QFT_PMARK40() QFT_WMARK_AT(40)
#else
#define QFT_PMARK40() do {} while (0)
#endif
#if defined(QFT_PROBE) && (QFT_PMASK & 8)
#define QFT_PMARK52() QFT_WMARK_AT(52)
#else
#define QFT_PMARK52() do {} while (0)
#endif

namespace qft {

template <int LOG2N, typename T>
struct PCfg {
    using P = SPlan<LOG2N>;
    static constexpr int VB = (int)sizeof(vec2<T>);
    static constexpr int UB = P::UCELLS * (int)sizeof(T);
    static constexpr int BUDGET = 226 * 1024 - UB - 64;
    static constexpr int PER_W = P::PADDED * VB;  // slot: padded working area (>= N cells)
    static constexpr int TT0 = BUDGET / (2 * PER_W);
    static constexpr int TTC = P::n >= 12 ? QFT_TT_MAX : 64;
    static constexpr int TT = TT0 > TTC ? TTC : TT0;
    static constexpr bool FITS = TT >= 1 && P::m >= 64 && PER_W % 16 == 0;  // TMA slots 16-byte aligned
    static constexpr int mx(int a, int b) { return a > b ? a : b; }
    static constexpr int NU = 2 * (P::NU1 + 1);
    static constexpr int W_U = (TT > 0 ? TT : 1) * NU;
    static constexpr int DI = P::DT;
    static constexpr int NWD0 = ((TT > 0 ? TT : 1) * DI + 31) / 32;  // D warps needed
    static constexpr int NWA = QFT_PIPE_NWA;                          // A0 warps
    static constexpr int NW = mx(W_U, NWD0 + NWA) + QFT_PIPE_NW_EXTRA;
    // every warp not folding the next batch runs phase D; the items are spread
    // evenly (DPW consecutive items per warp) so no sub-partition carries a
    // full D warp more than another
    static constexpr int NWD = QFT_PIPE_DSPREAD ? NW - NWA : NWD0;
    static constexpr int DPW = ((TT > 0 ? TT : 1) * DI + NWD - 1) / NWD;
    static constexpr int NT = NW * 32;
    static constexpr int NC64 = P::m / 64;  // A0 chunks per signal
    static constexpr int RA = (NC64 + NWA - 1) / NWA;
    // small blocks in phase 2 on the D warps' idle lanes (QFT_PIPE_SMALLD)
    static constexpr bool SMALLD = QFT_PIPE_SMALLD && !QFT_PIPE_DSPREAD && P::JS >= 0 &&
                                   (TT > 0 ? TT : 1) * DI <= NWD * 32 - 2 * (TT > 0 ? TT : 1);
    static constexpr int X_OFF = 0;
    static constexpr int U_OFF = 2 * (TT > 0 ? TT : 1) * PER_W;
    static constexpr int ITM_OFF = (U_OFF + UB + 15) / 16 * 16;  // per slot: x[64c], x[N-64c], c < NC64
    static constexpr int ITM_BYTES = QFT_PIPE_ITEMS ? (TT > 0 ? TT : 1) * 2 * (P::m / 64) * VB : 0;
    static constexpr int BAR_OFF = (ITM_OFF + ITM_BYTES + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + 64;  // 5 mbarriers
};

template <int LOG2N, typename T>
constexpr bool pipe_fits() {
    return PCfg<LOG2N, T>::FITS && PCfg<LOG2N, T>::SMEM <= 227 * 1024 && PCfg<LOG2N, T>::NW <= 16;
}

// (LOG2N, T) instances served by the pipelined kernel (mode 0)
template <int LOG2N, typename T>
constexpr bool use_pipe() {
    return QFT_PIPE && pipe_fits<LOG2N, T>() && LOG2N == 12 && sizeof(T) == 4;
}

QFT_DEV void named_bar(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

// one warp: lane 0 arms bar with the bytes of ntr signals, then lane tau
// bulk-copies raw signal tau (N cells) into its slot (the copies issue in
// parallel; each issuing lane first orders the CTA's earlier generic accesses
// of the slots -- published to it by the preceding barrier -- before its
// async-proxy writes)
#ifndef QFT_PIPE_TMA_SPLIT
#define QFT_PIPE_TMA_SPLIT 8  // bulk copies per signal (issued by parallel lanes): measured 1 / 2 / 4 / 8 = 58.5 / 58.7 / 58.8 / 59.1M tr/s
#endif
template <int LOG2N, typename T>
QFT_DEV void tma_load_slots(vec2<T> *X, const vec2<T> *src, int ntr, uint64_t *bar, int lane) {
    using P = SPlan<LOG2N>;
    constexpr int K = QFT_PIPE_TMA_SPLIT;
    constexpr uint32_t BYTES = P::N * (uint32_t)sizeof(vec2<T>), PART = BYTES / K;
    static_assert(BYTES % K == 0 && PART % 16 == 0 && K <= 8, "16-byte bulk-copy parts, <= 8 per signal");
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(BYTES * ntr)
                     : "memory");
    __syncwarp();
    if (lane < ntr * K) {
        const int tau = lane / K, k = lane - tau * K;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(X + tau * P::PADDED) + k * PART),
                     "l"(reinterpret_cast<const char *>(src + (long long)tau * P::N) + (size_t)k * PART), "r"(PART),
                     "r"(smem_u32(bar))
                     : "memory");
    }
}

// In-place A0 of ntr signals (raw samples at the start of each slot) by the
// NWA-warp group; ga = thread index within the group.  Per signal: every load
// (chunks of 64 samples + the items n = 64c) into registers, named barrier,
// every store (same fold / route as a0_complex).
template <int LOG2N, typename T>
QFT_DEV void a0_inplace(vec2<T> *X, int ntr, int ga, const A0Lane64 &a0l64, vec2<T> *itm = nullptr) {
    using P = SPlan<LOG2N>;
    using C = PCfg<LOG2N, T>;
    constexpr int NWA = C::NWA, NC64 = C::NC64, RA = C::RA;
    const int lane = ga & 31, gw = ga >> 5;
    auto shfl_up = [](vec2<T> v) { return shfl_vec(v, false); };
    for (int tau = 0; tau < ntr; ++tau) {
        vec2<T> *s = X + tau * P::PADDED;
        A0Chunk64<T> ch[RA];
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            const int c = gw + r * NWA;
            if (c < NC64) ch[r].template load<LOG2N>(s, c, lane);
        }
        const bool item = ga < NC64;  // n = 64 ga (ga = 0: the base pair)
        vec2<T> ia, ib;
        if constexpr (QFT_PIPE_ITEMS) {
            // chunk c: lane 0 loaded x[64c] (xe), lane 31 loaded x[N - 64(c+1)] (mn),
            // the mirror of item c+1 (item 0's partner is x[m] = chunk NC64-1's mn)
            vec2<T> *ia_s = itm + tau * 2 * NC64, *ib_s = ia_s + NC64;
#pragma unroll
            for (int r = 0; r < RA; ++r) {
                const int c = gw + r * NWA;
                if (c < NC64) {
                    if (lane == 0) ia_s[c] = ch[r].xe;
                    if (lane == 31) ib_s[c + 1 < NC64 ? c + 1 : 0] = ch[r].mn;
                }
            }
            named_bar(1, NWA * 32);
            if (item) {
                ia = ia_s[ga];
                ib = ib_s[ga];
            }
        } else {
            if (item) {
                ia = s[64 * ga];
                ib = s[ga == 0 ? P::m : P::N - 64 * ga];
            }
            named_bar(1, NWA * 32);
        }
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            const int c = gw + r * NWA;  // warp-uniform: the store's shuffle sees the whole warp
            if (c < NC64) ch[r].template store<LOG2N>(s, c, lane, a0l64, shfl_up);
        }
        if (item) {
            if (ga == 0) {
                s[padx(P::BASE)] = ia;      // dc[0] = x[0]
                s[padx(P::BASE + 1)] = ib;  // dc[m] = x[m]
            } else {
                const int n = 64 * ga, j = ctz32((uint32_t)n);
                const int cell = P::m - (1 << (LOG2N - 1 - j)) + (n >> (j + 1));
                s[padx(cell)] = vadd(ia, ib);
                s[padx(P::S0 + cell)] = sine_cell(ia, ib, cell);
            }
        }
        // the next signal's loads read another slot: no barrier needed here
    }
}

template <int LOG2N, typename T>
__global__ void __launch_bounds__(PCfg<LOG2N, T>::NT, 1)
    qft_cdft_pipe(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out, long long batch, const T *__restrict__ Ug,
                  const __grid_constant__ LeeConst<T> kc) {
    using P = SPlan<LOG2N>;
    using C = PCfg<LOG2N, T>;
    constexpr int TT = C::TT, NT = C::NT, NW = C::NW, NWD = C::NWD, NWA = C::NWA;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    vec2<T> *X0 = reinterpret_cast<vec2<T> *>(smem_raw + C::X_OFF);
    T *U = reinterpret_cast<T *>(smem_raw + C::U_OFF);
    vec2<T> *itm = reinterpret_cast<vec2<T> *>(smem_raw + C::ITM_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::BAR_OFF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool a0_warp = warp >= NWD && warp < NWD + NWA;
    const int ga = tid - NWD * 32;
    const A0Lane64 a0l64 = a0_lane64<LOG2N>(lane);
    const long long nbatch = (batch + TT - 1) / TT, G = gridDim.x;
    auto ntr_of = [&](long long b) { return (int)((batch - b * TT) < TT ? (batch - b * TT) : TT); };
    auto set = [&](int s) { return X0 + s * TT * P::PADDED; };
    // unit of this warp in the units phase: warp w runs on SM sub-partition w % 4;
    // QFT_PIPE_UMAP rotates the unit kind (big cos / big sin / rest cos / rest sin)
    // by the signal index so no sub-partition gets three of the heavier rest units
    const int uwarp = (QFT_PIPE_UMAP && C::NU == 4 && NW == TT * 4) ? ((warp & ~3) | ((warp + (warp >> 2)) & 3)) : warp;

    for (int i = tid; i < P::UCELLS; i += NT) U[i] = Ug[i];
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    long long bt = blockIdx.x;
    if (bt >= nbatch) return;
    if (warp == 0) {
        tma_load_slots<LOG2N, T>(set(0), in + bt * TT * P::N, ntr_of(bt), &bar[0], lane);
        if (bt + G < nbatch) tma_load_slots<LOG2N, T>(set(1), in + (bt + G) * TT * P::N, ntr_of(bt + G), &bar[1], lane);
    }
    uint32_t ph0 = 0, ph1 = 0;
    // prologue: A0 of the first batch
    if (a0_warp) {
        mbar_wait(&bar[0], ph0);
        a0_inplace<LOG2N, T>(set(0), ntr_of(bt), ga, a0l64, itm);
    }
    ph0 ^= 1u;
    __syncthreads();
    int cur = 0;
    for (; bt < nbatch; bt += G) {
        const int ntr = ntr_of(bt);
        vec2<T> *W = set(cur);
        QFT_MARK(1);
        QFT_PMARK24();
        fused_units<LOG2N, T, 0, TT, NW, !C::SMALLD>(W, U, kc.u, ntr, uwarp, lane);
        QFT_WMARK();
        __syncthreads();
        QFT_MARK(3);
        if (warp < NWD) {
            if constexpr (C::SMALLD) {
                // the blocks with L <= 16 (both sides of every signal) on the last D warp's
                // idle lanes, then the D warps meet: every phase-D item reads them
                const int sl = tid - (NWD * 32 - 2 * TT);
                if (sl >= 0 && (sl >> 1) < ntr) {
                    vec2<T> *w = W + (sl >> 1) * P::PADDED;
                    if (QFT_SC) b_small<LOG2N, false, T>(w + ((sl & 1) ? padx(P::S0) : 0), kc.u, sl & 1);
                    else if (sl & 1) b_small<LOG2N, true, T>(w, kc.u);
                    else b_small<LOG2N, false, T>(w, kc.u);
                }
                named_bar(2, NWD * 32);
            }
            if (QFT_PIPE_DSPREAD) {
                const int it = warp * C::DPW + lane;  // DPW <= 32 consecutive items per warp
                const int tau = it / P::DT, ti = it - tau * P::DT;
                if (lane < C::DPW && it < TT * P::DT && tau < ntr)
                    Chain<LOG2N, T>::unit(W + tau * P::PADDED, out + (bt * TT + tau) * P::N, ti);
            } else {
                for (int it = tid; it < TT * P::DT; it += NWD * 32) {
                    const int tau = it / P::DT, ti = it - tau * P::DT;
                    if (tau < ntr) Chain<LOG2N, T>::unit(W + tau * P::PADDED, out + (bt * TT + tau) * P::N, ti);
                }
            }
            QFT_PMARK52();
#if QFT_PIPE_TMA_EARLY
            // the D warps are the only readers of set cur in this phase: once
            // they are all done, warp 0 refills it while the A0 group finishes
            named_bar(2, NWD * 32);
            if (warp == 0 && bt + 2 * G < nbatch)
                tma_load_slots<LOG2N, T>(W, in + (bt + 2 * G) * TT * P::N, ntr_of(bt + 2 * G), &bar[cur], lane);
#endif
        } else if (a0_warp && bt + G < nbatch) {
            uint32_t &ph = cur ? ph0 : ph1;  // the next batch sits in set cur^1
            mbar_wait(&bar[cur ^ 1], ph);
            QFT_PMARK40();
            a0_inplace<LOG2N, T>(set(cur ^ 1), ntr_of(bt + G), ga, a0l64, itm);
            QFT_PMARK52();
        }
        if (bt + G < nbatch) {
            if (cur) ph0 ^= 1u;
            else ph1 ^= 1u;
        }
        QFT_MARK(4);
        __syncthreads();
        QFT_MARK(5);
        // set cur is free: bring in batch bt + 2G
        if (!QFT_PIPE_TMA_EARLY && warp == QFT_PIPE_TMA_WARP && bt + 2 * G < nbatch)
            tma_load_slots<LOG2N, T>(W, in + (bt + 2 * G) * TT * P::N, ntr_of(bt + 2 * G), &bar[cur], lane);
#if QFT_PIPE_L2PF
        // the batch after that into L2, so its bulk copy one iteration later is served from L2
        if (warp == QFT_PIPE_TMA_WARP + 1 && lane < TT && bt + 3 * G < nbatch && lane < ntr_of(bt + 3 * G))
            l2_prefetch(in + ((bt + 3 * G) * TT + lane) * P::N, P::N * (uint32_t)sizeof(vec2<T>));
#endif
        QFT_MARK(6);
        cur ^= 1;
    }
}

// wait with a suspend-time hint: the waiting warp is parked by the hardware
// until the phase completes (up to the hint) instead of re-polling
QFT_DEV void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
QFT_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// Dataflow variant (QFT_PIPE == 2): no CTA-wide barrier inside the loop.  Four
// mbarriers carry exactly the dependencies of the schedule above:
//   adone   A0(i) stored                  -> every warp may start units(i)
//   udone   units(i) stored (all warps)   -> D warps may start D(i)
//   ddone   D(i) has read its set         -> warp 0 refills the set by TMA
//   tma[s]  raw signals of a batch landed -> A0 warps may fold them
// so the A0 warps fold batch i+1 and start units(i+1) while the D warps are
// still in D(i), and a D warp goes from D(i) straight into units(i+1).
// ---------------------------------------------------------------------------
template <int LOG2N, typename T>
__global__ void __launch_bounds__(PCfg<LOG2N, T>::NT, 1)
    qft_cdft_pipe2(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out, long long batch,
                   const T *__restrict__ Ug, const __grid_constant__ LeeConst<T> kc) {
    using P = SPlan<LOG2N>;
    using C = PCfg<LOG2N, T>;
    constexpr int TT = C::TT, NT = C::NT, NW = C::NW, NWD = C::NWD, NWA = C::NWA;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    vec2<T> *X0 = reinterpret_cast<vec2<T> *>(smem_raw + C::X_OFF);
    T *U = reinterpret_cast<T *>(smem_raw + C::U_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::BAR_OFF);
    uint64_t *tma = bar, *adone = bar + 2, *udone = bar + 3, *ddone = bar + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool dwarp = warp < NWD, awarp = warp >= NWD && warp < NWD + NWA;
    const int ga = tid - NWD * 32;
    const A0Lane64 a0l64 = a0_lane64<LOG2N>(lane);
    const long long nbatch = (batch + TT - 1) / TT, G = gridDim.x;
    auto ntr_of = [&](long long b) { return (int)((batch - b * TT) < TT ? (batch - b * TT) : TT); };
    auto set = [&](int s) { return X0 + s * TT * P::PADDED; };

    for (int i = tid; i < P::UCELLS; i += NT) U[i] = Ug[i];
    if (tid == 0) {
        mbar_init(&tma[0], 1);
        mbar_init(&tma[1], 1);
        mbar_init(adone, NWA * 32);
        (void)udone;
        (void)ddone;
    }
    __syncthreads();
    const long long b0 = blockIdx.x;
    if (b0 >= nbatch) return;
    if (warp == 0) {
        tma_load_slots<LOG2N, T>(set(0), in + b0 * TT * P::N, ntr_of(b0), &tma[0], lane);
        if (b0 + G < nbatch) tma_load_slots<LOG2N, T>(set(1), in + (b0 + G) * TT * P::N, ntr_of(b0 + G), &tma[1], lane);
    }
    if (awarp) {
        mbar_wait(&tma[0], 0);
        a0_inplace<LOG2N, T>(set(0), ntr_of(b0), ga, a0l64);
        mbar_arrive(adone);
    }
    uint32_t k = 0;
    for (long long bt = b0; bt < nbatch; bt += G, ++k) {
        const int cur = k & 1;
        const uint32_t ph = k & 1;
        const int ntr = ntr_of(bt);
        vec2<T> *W = set(cur);
        mbar_wait_sleep(adone, ph);  // A0(bt) is in set cur
        QFT_PMARK24();
        fused_units<LOG2N, T, 0, TT, NW>(W, U, kc.u, ntr, warp, lane);
        QFT_PMARK8();
        // all units of the batch stored (named barrier 2, every thread); the D
        // warps then need only each other (barrier 3) before the set is refilled,
        // and every warp only the A0 group (mbarrier adone) before units(i+1):
        // the A0 warps start units(i+1) while the D warps are still in D(i)
        named_bar(2, NT);
        if (dwarp) {
            QFT_PMARK40();
            for (int it = tid; it < TT * P::DT; it += NWD * 32) {
                const int tau = it / P::DT, ti = it - tau * P::DT;
                if (tau < ntr) Chain<LOG2N, T>::unit(W + tau * P::PADDED, out + (bt * TT + tau) * P::N, ti);
            }
            QFT_PMARK52();
            if (bt + 2 * G < nbatch) {
                named_bar(3, NWD * 32);  // set cur is no longer read
                if (warp == 0)
                    tma_load_slots<LOG2N, T>(W, in + (bt + 2 * G) * TT * P::N, ntr_of(bt + 2 * G), &tma[cur], lane);
            }
        } else if (awarp && bt + G < nbatch) {
            mbar_wait_sleep(&tma[cur ^ 1], ((k + 1) >> 1) & 1u);
            QFT_PMARK40();
            a0_inplace<LOG2N, T>(set(cur ^ 1), ntr_of(bt + G), ga, a0l64);
            QFT_PMARK52();
            mbar_arrive(adone);
        }
    }
}

// ---------------------------------------------------------------------------
// Group-pipelined variant (QFT_PIPE == 3): the CTA is NG independent groups of
// GW = 4 warps (one warp per fused unit of a signal); each group streams its
// own signals through two slots with named barriers of its own, so the groups
// drift out of phase and one group's shared-memory-heavy units overlap another
// group's latency-bound chain phase D (the lock-step kernels above leave the
// shared-memory pipe idle during D and at every CTA barrier).
//
//   per group, iteration k (signal s_k in slot k & 1):
//     wait TMA(s_k); A0 loads (registers)
//     group barrier      -- every A0 load done, every D(s_{k-1}) read done
//     TMA(s_{k+1}) -> slot (k+1) & 1; A0 stores (in place)
//     group barrier
//     units(s_k): one warp per unit
//     group barrier
//     D(s_k) on the warps that own items; the others go straight on to the
//     A0 loads of s_{k+1}
// ---------------------------------------------------------------------------
#ifndef QFT_GPIPE_NG
#define QFT_GPIPE_NG 3
#endif
#ifndef QFT_GPIPE_STAGGER
#define QFT_GPIPE_STAGGER 0  // ns group g waits before its first signal (g * this)
#endif
template <int LOG2N, typename T>
struct GCfg {
    using P = SPlan<LOG2N>;
    static constexpr int VB = (int)sizeof(vec2<T>);
    static constexpr int UB = P::UCELLS * (int)sizeof(T);
    static constexpr int PER_W = P::PADDED * VB;
    static constexpr int GW = 2 * (P::NU1 + 1);  // warps per group = fused units per signal
    static constexpr int NG = QFT_GPIPE_NG;
    static constexpr int NW = NG * GW, NT = NW * 32;
    static constexpr int NC64 = P::m / 64;
    static constexpr int RA = (NC64 + GW - 1) / GW;
    static constexpr int U_OFF = NG * 2 * PER_W;
    static constexpr int BAR_OFF = (U_OFF + UB + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + NG * 2 * 8;
    static constexpr bool FITS = P::n <= 12 && P::JF >= 1 && GW == 4 && PER_W % 16 == 0 && SMEM <= 227 * 1024 &&
                                 NW <= 16 && P::DT <= GW * 32;
};

// in-place A0 of one signal by the NWA warps of a group, split at the barrier
template <int LOG2N, typename T, int NWA>
struct A0Group {
    using P = SPlan<LOG2N>;
    static constexpr int NC64 = P::m / 64, RA = (NC64 + NWA - 1) / NWA;
    A0Chunk64<T> ch[RA];
    vec2<T> ia, ib;
    QFT_DEV void load(const vec2<T> *s, int ga) {
        const int lane = ga & 31, gw = ga >> 5;
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            const int c = gw + r * NWA;
            if (c < NC64) ch[r].template load<LOG2N>(s, c, lane);
        }
        if (ga < NC64) {
            ia = s[64 * ga];
            ib = s[ga == 0 ? P::m : P::N - 64 * ga];
        }
    }
    QFT_DEV void store(vec2<T> *s, int ga, const A0Lane64 &a0l64) const {
        const int lane = ga & 31, gw = ga >> 5;
        auto shfl_up = [](vec2<T> v) { return shfl_vec(v, false); };
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            const int c = gw + r * NWA;
            if (c < NC64) ch[r].template store<LOG2N>(s, c, lane, a0l64, shfl_up);
        }
        if (ga < NC64) {
            if (ga == 0) {
                s[padx(P::BASE)] = ia;
                s[padx(P::BASE + 1)] = ib;
            } else {
                const int n = 64 * ga, j = ctz32((uint32_t)n);
                const int cell = P::m - (1 << (LOG2N - 1 - j)) + (n >> (j + 1));
                s[padx(cell)] = vadd(ia, ib);
                s[padx(P::S0 + cell)] = sine_cell(ia, ib, cell);
            }
        }
    }
};

template <int LOG2N, typename T>
__global__ void __launch_bounds__(GCfg<LOG2N, T>::NT, 1)
    qft_cdft_gpipe(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out, long long batch,
                   const T *__restrict__ Ug, const __grid_constant__ LeeConst<T> kc) {
    using P = SPlan<LOG2N>;
    using C = GCfg<LOG2N, T>;
    constexpr int GW = C::GW, NG = C::NG, NT = C::NT;
    constexpr uint32_t BYTES = P::N * (uint32_t)sizeof(vec2<T>);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *U = reinterpret_cast<T *>(smem_raw + C::U_OFF);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + C::BAR_OFF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp / GW, gw = warp - g * GW, gt = tid - g * GW * 32;
    vec2<T> *slot0 = reinterpret_cast<vec2<T> *>(smem_raw) + (2 * g) * P::PADDED;
    uint64_t *bar = bars + 2 * g;
    const int bid = 1 + g;  // named barrier of the group
    const A0Lane64 a0l64 = a0_lane64<LOG2N>(lane);
    // the unit kind and the phase-D warps rotate with the group, so the heavier
    // units and the D warps spread over the four SM sub-partitions (warp w runs on w % 4)
    const int kind = (gw + g) % GW;
    const int ditem = ((gw - g + GW) % GW) * 32 + lane;

    for (int i = tid; i < P::UCELLS; i += NT) U[i] = Ug[i];
    if (tid < 2 * NG) mbar_init(&bars[tid], 1);
    __syncthreads();
    const long long G = gridDim.x;
    auto sig = [&](long long k) { return (blockIdx.x + k * G) * NG + g; };
    if (sig(0) >= batch) return;
    if (QFT_GPIPE_STAGGER && g > 0) __nanosleep(QFT_GPIPE_STAGGER * g);
    if (gt == 0) tma_bulk_load(slot0, in + sig(0) * P::N, BYTES, &bar[0]);
    uint32_t ph = 0;  // bit s: parity of slot s
    for (long long k = 0; sig(k) < batch; ++k) {
        const int s = (int)(k & 1);
        vec2<T> *W = slot0 + s * P::PADDED;
        mbar_wait(&bar[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        {
            A0Group<LOG2N, T, GW> a0;
            a0.load(W, gt);
            named_bar(bid, GW * 32);
            // every read of the other slot (D of s_{k-1}) is done: refill it
            if (gt == 0 && sig(k + 1) < batch)
                tma_bulk_load(slot0 + (s ^ 1) * P::PADDED, in + sig(k + 1) * P::N, BYTES, &bar[s ^ 1]);
            a0.store(W, gt, a0l64);
        }
        named_bar(bid, GW * 32);
        run_unit<LOG2N, T, 0>(W, kind, U, kc.u, lane);
        named_bar(bid, GW * 32);
        if (ditem < P::DT) Chain<LOG2N, T>::unit(W, out + sig(k) * P::N, ditem);
    }
}

template <int LOG2N, typename T>
cudaError_t launch_gpipe(const LaunchArgs &a) {
    using C = GCfg<LOG2N, T>;
    auto kern = qft_cdft_gpipe<LOG2N, T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const long long ngroups = (a.batch + C::NG - 1) / C::NG;
    long long grid = a.num_sms;
    if (grid > ngroups) grid = ngroups;
    if (grid < 1) grid = 1;
    LeeConst<T> kc;
    for (int i = 0; i < 32; ++i) kc.u[i] = ((const T *)a.Uhead)[i];
    kern<<<(unsigned)grid, C::NT, C::SMEM, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch,
                                                       (const T *)a.U, kc);
    return cudaGetLastError();
}

template <int LOG2N, typename T>
cudaError_t launch_pipe(const LaunchArgs &a) {
    if constexpr (QFT_PIPE == 3 && GCfg<LOG2N, T>::FITS) return launch_gpipe<LOG2N, T>(a);
    using C = PCfg<LOG2N, T>;
    auto kern = QFT_PIPE == 2 ? qft_cdft_pipe2<LOG2N, T> : qft_cdft_pipe<LOG2N, T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const long long nbatch = (a.batch + C::TT - 1) / C::TT;
    long long grid = a.num_sms;
    if (grid > nbatch) grid = nbatch;
    if (grid < 1) grid = 1;
    LeeConst<T> kc;
    for (int i = 0; i < 32; ++i) kc.u[i] = ((const T *)a.Uhead)[i];
    kern<<<(unsigned)grid, C::NT, C::SMEM, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch, (const T *)a.U,
                                                       kc);
    return cudaGetLastError();
}

}  // namespace qft
