// qft_launch.cuh -- the batched transform kernels and their launchers.
//   qft_cdft_reg   N <= 32     : one thread per signal, whole transform in registers
//   qft_cdft_smem  N = 64..16384: persistent CTAs (1 per SM); each CTA transforms
//                                TT signals per iteration through the phases of
//                                qft_smem.cuh while a TMA bulk copy prefetches the
//                                next TT signals into a staging buffer (or, when
//                                the staging buffer does not fit, an L2 prefetch)
// Each (precision, N) instance is compiled in its own translation unit
// (qft_inst.cu) so the build parallelises.
#pragma once
#include <cuda_runtime.h>

#include "qft_smem.cuh"

#ifndef QFT_CTAS_PER_SM
#define QFT_CTAS_PER_SM 1  // shared-memory budget split: CTAs resident per SM (N <= 4096)
#endif
#ifndef QFT_A0_TMA
#define QFT_A0_TMA 1       // A0 input: TMA bulk copy into a staging buffer when it fits (1), else L2-prefetched global loads
#endif
#ifndef QFT_A0_UNR
#define QFT_A0_UNR 8       // A0 from global memory: 64-sample chunks in flight per warp (fp32)
#endif
#ifndef QFT_D_HALF
#define QFT_D_HALF 0  // see KCfg::DHALF
#endif
#ifndef QFT_MIXED_STAGE
#define QFT_MIXED_STAGE 0  // see KCfg::MIXED
#endif
#ifndef QFT_A0_PRE
#define QFT_A0_PRE 0  // next signal's A0 chunks loaded by idle phase-D warps: measured slower (config 5: 9.7 / 10.9 / 8.0M for 2 / 4 / 8 chunks per warp vs 11.06M)
#endif
#ifndef QFT_A0_PRE_UNR
#define QFT_A0_PRE_UNR 4  // chunks per prefetching warp (8 spills at 128 registers)
#endif
#ifndef QFT_NW_MIN
#define QFT_NW_MIN 4       // lower bound on warps per CTA
#endif
#ifndef QFT_HALO_SHFL
#define QFT_HALO_SHFL 0    // phase-C halo column by warp shuffle (else a second shared-memory read)
#endif
#ifndef QFT_REST_FUSED
#define QFT_REST_FUSED 0   // rest unit: F / C levels of all its blocks together (measured slower: 54.0 vs 55.5M tr/s)
#endif
#ifndef QFT_UFENCE
#define QFT_UFENCE 0       // scheduling fences between the sub-phases of a warp unit (see QFT_UMARK)
#endif
#ifndef QFT_TT_MAX
#define QFT_TT_MAX 4       // cap on signals per CTA iteration
#endif

// Phase timestamps for tools/probe (compiled out unless QFT_PROBE is defined):
// per (CTA, iteration < 16) 8 CTA-level marks (thread 0, after each barrier)
// and one mark per warp when it leaves the fused-unit phase.
#ifdef QFT_PROBE
static __device__ long long qft_probe_buf[160 * 16 * 64];
#define QFT_MARK(k)                                                                       \
    do {                                                                                  \
        const int it_ = (int)(__fdividef((float)(bt - blockIdx.x), (float)gridDim.x) + 0.5f);                              \
        if (tid == 0 && blockIdx.x < 160 && it_ < 16) qft_probe_buf[(blockIdx.x * 16 + it_) * 64 + (k)] = clock64(); \
    } while (0)
#define QFT_WMARK()                                                                       \
    do {                                                                                  \
        const int it_ = (int)(__fdividef((float)(bt - blockIdx.x), (float)gridDim.x) + 0.5f);                              \
        if (lane == 0 && blockIdx.x < 160 && it_ < 16) qft_probe_buf[(blockIdx.x * 16 + it_) * 64 + 8 + warp] = clock64(); \
    } while (0)
#define QFT_WMARK_AT(o)                                                                   \
    do {                                                                                  \
        const int it_ = (int)(__fdividef((float)(bt - blockIdx.x), (float)gridDim.x) + 0.5f);                              \
        if (lane == 0 && blockIdx.x < 160 && it_ < 16) qft_probe_buf[(blockIdx.x * 16 + it_) * 64 + (o) + warp] = clock64(); \
    } while (0)
#define QFT_UMARK(k)                                                                      \
    do {                                                                                  \
        if (blockIdx.x == 0 && threadIdx.x == 0) qft_probe_buf[160 * 16 * 64 - 64 + (k)] = clock64(); \
    } while (0)
#else
#define QFT_WMARK_AT(o) \
    do {                \
    } while (0)
#if QFT_UFENCE == 1
// compiler-only memory fence between the sub-phases of a warp unit
#define QFT_UMARK(k) asm volatile("" ::: "memory")
#elif QFT_UFENCE == 2
// a never-taken branch: a basic-block boundary between the sub-phases
#define QFT_UMARK(k)                                     \
    do {                                                 \
        if (threadIdx.x == 0xffff) asm volatile("trap;"); \
    } while (0)
#elif QFT_UFENCE == 3
#define QFT_UMARK(k)                                     \
    do {                                                 \
        long long c_;                                    \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)); \
        if (c_ == -1) asm volatile("trap;");              \
    } while (0)
#else
#define QFT_UMARK(k) \
    do {             \
    } while (0)
#endif
#define QFT_MARK(k) \
    do {            \
    } while (0)
#define QFT_WMARK() \
    do {            \
    } while (0)
#endif

namespace qft {

struct LaunchArgs {
    const void *in;
    void *out;
    long long batch;
    const void *U;        // level table (device)
    const void *Uhead;    // host copy of U[0..32): the constants of every Lee block with L <= 32
    int num_sms;
    cudaStream_t stream;
    long long nreal = 0;  // real modes: number of real rows (batch = row pairs)
};

// U[0..32) as a kernel parameter: lives in the constant bank, so the Lee-32
// multiplies read it as an operand (no shared-memory traffic).
template <typename T>
struct LeeConst {
    T u[32];
};

// ------------------------------------------------------------ TMA / mbarrier
QFT_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
QFT_DEV void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
QFT_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one thread: order earlier generic-proxy accesses of the buffer, arm the
// barrier with the byte count and issue the bulk copy global -> shared
QFT_DEV void tma_bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

QFT_DEV void l2_prefetch(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ------------------------------------------------------------ configuration
#ifndef QFT_CPS_SMALL
// CTAs resident per SM for N <= 2048 (0: the measured per-size choice below).  The
// phases of a small transform are short and separated by CTA barriers (ncu:
// barrier was 36 % of the stall samples at N = 1024 with one CTA per SM); more
// resident CTAs fill them.  Measured 1 / 2 / 3 CTAs (tools/size_sweep.py, % of HBM):
// fp32 2^10 48.8 / 52.8 / 56.6, 2^11 50.3 / 52.4 / 50.0 (4 CTAs: 58.0 after the phase-D
// depth change, qft_smem.cuh QFT_RC_MID), 2^7 44.7 / 32.1 / 32.8;
// fp64 2^9 48.4 / 53.7 / 54.1, 2^11 49.8 / 45.6 / 51.9
#define QFT_CPS_SMALL 0
#endif
// the sizes whose working area is 67 KB (fp32 N = 8192, fp64 N = 4096): one signal
// per CTA iteration (QFT_TT_MID) and QFT_CPS_MID resident CTAs
#ifndef QFT_TT_MID
#define QFT_TT_MID 1
#endif
#ifndef QFT_U13_SPLIT
// fp32 N = 8192: only the constants of the Lee blocks of <= 1024 cells (U[0..1024), what
// the warp units read) live in shared memory; the top fold levels read theirs from
// global memory (L1-resident).  The 4 KB saved let a third CTA fit (3 x 72 KB).
// Measured slower (46.2 vs 50.1 % of HBM with 2 CTAs: 80 registers with spills, the top
// levels' constants from global memory); off.
#define QFT_U13_SPLIT 0
#endif
#ifndef QFT_CPS_MID
#define QFT_CPS_MID 2  // measured (TT, CTAs) = (3, 1) / (1, 1) / (1, 2): fp32 2^13 33.1 / 47.9 / 49.7 %, fp64 2^12 40.8 / 41.0 / 42.3 % of HBM
#endif
template <int LOG2N, typename T>
constexpr bool mid_class() {
    return (sizeof(T) == 4 && LOG2N == 13) || (sizeof(T) == 8 && LOG2N == 12);
}
template <int LOG2N, typename T>
constexpr int cps_for() {
    if (LOG2N <= 11) {
        if (QFT_CPS_SMALL > 0) return QFT_CPS_SMALL;
        // N <= 256, re-measured after the phase-D depth change (4 / 6 / 8 CTAs, % of HBM):
        // fp32 2^7 73.7 / 70.8 / 74.5, 2^8 56.6 / 55.8 / 56.6; fp64 2^6 61.9 / 59.2 / 69.0,
        // 2^7 70.4 / 59.5 / 68.2, 2^8 60.3 / 59.4 / 62.6 (3 CTAs: fp32 2^7 59.1, fp64 2^6 53.4)
        if (LOG2N <= 8) return (sizeof(T) == 8 && LOG2N != 7) ? 8 : 4;
        if (sizeof(T) == 4 && LOG2N == 11) return 4;  // with QFT_RC_MID = 4: 52.0 (2 CTAs) / 58.0 % (4 CTAs, one signal each)
        // fp64 2^10 measured 49.0 / 51.7 / 51.5 %; one CTA keeps the small-batch
        // latency of BASELINE config 1 (64 signals: one 12-warp CTA per signal)
        if (sizeof(T) == 8 && LOG2N == 10) return 1;
        return 3;
    }
    if (mid_class<LOG2N, T>()) return (QFT_U13_SPLIT && sizeof(T) == 4 && LOG2N == 13) ? 3 : QFT_CPS_MID;
    return (LOG2N <= 12 && QFT_CTAS_PER_SM > 1) ? QFT_CTAS_PER_SM : 1;
}
// level-table entries kept in shared memory (QFT_U13_SPLIT: the first 1024)
template <int LOG2N, typename T>
constexpr int ucells_smem() {
    return (QFT_U13_SPLIT && sizeof(T) == 4 && LOG2N == 13) ? 1024 : SPlan<LOG2N>::UCELLS;
}
template <int LOG2N, typename T>
struct KCfg {
    using P = SPlan<LOG2N>;
    static constexpr int VB = (int)sizeof(vec2<T>);
    static constexpr int UCS = ucells_smem<LOG2N, T>();
    static constexpr bool USPLIT = UCS < P::UCELLS;
    static constexpr int UB = UCS * (int)sizeof(T);
    // CTAs per SM: the QFT_CTAS_PER_SM split applies where one signal still fits
    static constexpr int CPS = cps_for<LOG2N, T>();
    static constexpr int BUDGET = (226 * 1024) / CPS - UB - 64;
    static constexpr int PER_W = P::PADDED * VB;        // working area per signal
    static constexpr int PER_S = P::N * VB + PER_W;     // + TMA staging
    static constexpr int TTC = mid_class<LOG2N, T>() ? QFT_TT_MID : (P::n >= 12 ? QFT_TT_MAX : 64);
    static constexpr int clampt(int t) { return t < 1 ? 1 : (t > TTC ? TTC : t); }
    // stage through TMA when the staging buffer still leaves room for 2 signals
    // (fp32) / 1 signal (fp64, whose global A0 path spills)
    static constexpr int TMA_MIN = (sizeof(T) == 8 || CPS > 1) ? 1 : (TTC < 2 ? TTC : 2);
    static constexpr bool TMA0 = QFT_A0_TMA && BUDGET / PER_S >= TMA_MIN;
    // mixed staging (QFT_MIXED_STAGE, fp32 N = 4096): more signals per iteration
    // than fit with staging; TS of them are TMA-staged, the rest are read from
    // L2-prefetched global memory
    static constexpr bool MIXED = QFT_MIXED_STAGE && sizeof(T) == 4 && P::n == 12;
    static constexpr int TT = MIXED ? clampt(BUDGET / PER_W) : clampt(BUDGET / (TMA0 ? PER_S : PER_W));
    static constexpr int TS0 = MIXED ? (BUDGET - TT * PER_W) / (P::N * VB) : (TMA0 ? TT : 0);
    static constexpr int TS = TS0 > TT ? TT : TS0;  // TMA-staged signals per iteration
    static constexpr bool TMA = TS > 0;
    static_assert(TT * PER_W <= BUDGET, "working area exceeds shared memory");
    static constexpr int mx(int a, int b) { return a > b ? a : b; }
    static constexpr int NU = 2 * (P::NU1 + 1);  // fused warp units per signal
    static constexpr int W_U = TT * NU;
    // phase D in half items (QFT_D_HALF): twice the items, each half the unfold
    static constexpr bool DHALF = QFT_D_HALF && P::RC >= 1;
    static constexpr int DI = DHALF ? 2 * P::DT : P::DT;  // phase-D items per signal
    static constexpr int W_D = (TT * DI + 31) / 32;
    static constexpr int NW0 = mx(W_U, W_D);
    // warps are spread over 4 SM sub-partitions of 16K registers each: 12 warps
    // keep 168 registers (fp64), 16 keep 128; 17 (fp32, N <= 4096) drop to 96
    static constexpr int NWMAX1 = sizeof(T) == 8 ? 12 : (P::n >= 13 ? 16 : 17);
    // several resident CTAs share the register file: 24 warps per SM keep 85 registers (fp32)
    static constexpr int NWMAX = CPS == 1 ? NWMAX1 : (sizeof(T) == 8 ? 12 : 24) / CPS;
    static constexpr int NWLO = QFT_NW_MIN > NWMAX ? NWMAX : QFT_NW_MIN;
    static constexpr int NW = NW0 < NWLO ? NWLO : (NW0 > NWMAX ? NWMAX : NW0);
    static constexpr int NT = NW * 32;
    static constexpr int STAGE_OFF = 0;
    static constexpr int W_OFF = TS * P::N * VB;
    static constexpr int U_OFF = W_OFF + TT * PER_W;
    static constexpr int BAR_OFF = (U_OFF + UB + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + 16;
    // top levels (N > 4096): items per thread of one huge block side
    static constexpr int TIT = (1024 + NT - 1) / NT;
};

// smem kernel available for (LOG2N, T)
template <int LOG2N, typename T>
constexpr bool smem_fits() {
    using P = SPlan<LOG2N>;
    return (P::PADDED * (int)sizeof(vec2<T>) + ucells_smem<LOG2N, T>() * (int)sizeof(T) + 64) <=
           (226 * 1024) / cps_for<LOG2N, T>();
}

// ------------------------------------------------------------ small N
// signals per CTA of the register kernel's complex mode (= its threads): 128, or 64
// where 128 rows of NN + 1 cells would exceed the 48 KB of static shared memory
template <int NN, typename T>
struct RegCfg {
    static constexpr int SIG = (128 * (NN + 1) * (int)sizeof(vec2<T>) + 1024 > 48 * 1024) ? 64 : 128;
};
template <int NN, typename T, int MODE = 0>
__global__ void __launch_bounds__(128) qft_cdft_reg(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out,
                                                    long long batch, const T *__restrict__ U, long long nreal = 0) {
    __shared__ T sU[NN / 4 >= 2 ? NN / 4 : 2];
    for (int i = threadIdx.x; i < (NN / 4 >= 2 ? NN / 4 : 2); i += blockDim.x) sU[i] = U[i];
    __syncthreads();
    constexpr int m = NN / 2;
    if constexpr (MODE == 0) {
        // the CTA's signals go through shared memory (rows of NN + 1 cells): coalesced
        // global loads / stores, conflict-free per-thread rows -- a thread reading its own
        // signal from global memory touched 32 sectors per load instruction (27 % of HBM
        // at N = 32 fp32; tools/size_sweep.py)
        constexpr int SIG = RegCfg<NN, T>::SIG;
        __shared__ vec2<T> stage[SIG * (NN + 1)];
        for (long long b0 = (long long)blockIdx.x * SIG; b0 < batch; b0 += (long long)gridDim.x * SIG) {
            const int cnt = (int)(batch - b0 < SIG ? batch - b0 : SIG);
            for (int i = threadIdx.x; i < cnt * NN; i += SIG) stage[(i / NN) * (NN + 1) + (i % NN)] = in[b0 * NN + i];
            __syncthreads();
            if ((int)threadIdx.x < cnt) {
                vec2<T> x[NN], y[NN];
                vec2<T> *row = stage + threadIdx.x * (NN + 1);
#pragma unroll
                for (int n = 0; n < NN; ++n) x[n] = row[n];
                cdft_reg<NN, T>(x, y, sU);
#pragma unroll
                for (int n = 0; n < NN; ++n) row[n] = y[n];
            }
            __syncthreads();
            for (int i = threadIdx.x; i < cnt * NN; i += SIG) out[b0 * NN + i] = stage[(i / NN) * (NN + 1) + (i % NN)];
            __syncthreads();
        }
        return;
    }
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (long long)gridDim.x * blockDim.x) {
        if constexpr (MODE != 0) {
            constexpr int RL = MODE == 1 ? NN : (MODE == 2 ? m + 1 : (m > 1 ? m - 1 : 1));
            const T *xr = reinterpret_cast<const T *>(in);
            const long long ra = 2 * b, rb = ra + 1 < nreal ? ra + 1 : ra;
            const bool has_b = ra + 1 < nreal;
            vec2<T> x[RL];
#pragma unroll
            for (int n = 0; n < RL; ++n) x[n] = {xr[ra * RL + n], xr[rb * RL + n]};
            if constexpr (MODE == 1) {  // rdft_packed (shared.py:21-43) per component
                vec2<T> *ya = out + ra * (m + 1);
                if constexpr (NN == 2) {
                    const vec2<T> s = vadd(x[0], x[1]), d = vsub(x[0], x[1]);
                    ya[0] = {s.x, (T)0};
                    ya[1] = {d.x, (T)0};
                    if (has_b) {
                        ya[2] = {s.y, (T)0};
                        ya[3] = {d.y, (T)0};
                    }
                } else {
                    vec2<T> dc[m + 1], ds[m - 1], C[m + 1], S[m - 1];
                    dc[0] = x[0];
                    dc[m] = x[m];
#pragma unroll
                    for (int n = 1; n < m; ++n) {
                        dc[n] = vadd(x[n], x[NN - n]);
                        ds[n - 1] = vsub(x[n], x[NN - n]);
                    }
                    dct0_reg<NN, T>(dc, C, sU);
                    dst0_reg<NN, T>(ds, S, sU);
#pragma unroll
                    for (int k = 0; k <= m; ++k) {
                        const bool edge = (k == 0) || (k == m);
                        ya[k] = {C[k].x, edge ? (T)0 : -S[edge ? 0 : k - 1].x};
                        if (has_b) ya[m + 1 + k] = {C[k].y, edge ? (T)0 : -S[edge ? 0 : k - 1].y};
                    }
                }
            } else if constexpr (MODE == 2) {
                vec2<T> C[m + 1];
                dct0_reg<NN, T>(x, C, sU);
                T *ya = reinterpret_cast<T *>(out) + ra * (m + 1);
#pragma unroll
                for (int k = 0; k <= m; ++k) {
                    ya[k] = C[k].x;
                    if (has_b) ya[m + 1 + k] = C[k].y;
                }
            } else {
                vec2<T> S[RL];
                dst0_reg<NN, T>(x, S, sU);
                T *ya = reinterpret_cast<T *>(out) + ra * RL;
#pragma unroll
                for (int k = 0; k < RL; ++k) {
                    ya[k] = S[k].x;
                    if (has_b) ya[RL + k] = S[k].y;
                }
            }
        }
    }
}

// ------------------------------------------------------------ phase drivers
template <int LOG2N, typename T, int J>
QFT_DEV void run_f_blocks(vec2<T> *w, const T *U, bool dst, int lane) {
    // blocks J, J+1, ... < JF of one side, sequentially (combined warp unit)
    if constexpr (J < SPlan<LOG2N>::JF) {
        if (dst) {
            FBlock<LOG2N, J, true, T> f;
            f.load(w, U, lane);
            __syncwarp();
            f.store(w, lane);
        } else {
            FBlock<LOG2N, J, false, T> f;
            f.load(w, U, lane);
            __syncwarp();
            f.store(w, lane);
        }
        __syncwarp();
        run_f_blocks<LOG2N, T, J + 1>(w, U, dst, lane);
    }
}

template <typename T>
QFT_DEV vec2<T> shfl_vec(vec2<T> v, bool down) {
    vec2<T> r;
    if (down) {
        r.x = __shfl_down_sync(0xffffffffu, v.x, 1);
        r.y = __shfl_down_sync(0xffffffffu, v.y, 1);
    } else {
        r.x = __shfl_up_sync(0xffffffffu, v.x, 1);
        r.y = __shfl_up_sync(0xffffffffu, v.y, 1);
    }
    return r;
}

// backward levels of one big block (padded pointer wb), one warp
template <int R, bool DST, typename T>
QFT_DEV void run_c_blockp(vec2<T> *wb, int lane) {
    CBlockP<R, DST, T> c;
    c.load(wb, lane);
    vec2<T> out[1 << R];
#if QFT_HALO_SHFL
    // the halo column is the neighbour lane's own column: a register shuffle
    // (the edge lane's value is unused -- it copies instead of adding)
    auto halo = [&](int p) { return shfl_vec(c.own[p], !DST); };
#else
    const vec2<T> *hc = CBlockP<R, DST, T>::halo_colp(wb, lane);
    auto halo = [&](int p) { return hc[33 * p]; };  // read before the __syncwarp below
#endif
    c.compute(lane, halo, out);
    __syncwarp();
    CBlockP<R, DST, T>::storep(wb, lane, out);
    __syncwarp();
}

template <int LOG2N, typename T, int J>
QFT_DEV void run_c_blocks(vec2<T> *w, bool dst, int lane) {
    using P = SPlan<LOG2N>;
    if constexpr (J < P::JF) {
        constexpr int b = P::off(J);
        if (dst) run_c_blockp<P::RF(J), true, T>(w + padx(P::S0 + b), lane);
        else run_c_blockp<P::RF(J), false, T>(w + padx(b), lane);
        run_c_blocks<LOG2N, T, J + 1>(w, dst, lane);
    }
}

// ---- fused forward / Lee-32 / backward work of one side of one signal, one warp.
// The F -> Lee-32 -> B work of a Lee block depends on no other block, so a warp
// runs it start to finish with __syncwarp only (no CTA barrier).
// big unit: a block of L = 32 << R cells at padded pointer wb (block 0 for
// N <= 4096, a 1024-cell (sub-)block for N > 4096): one Lee-32 per lane
template <int L, int R, typename T, bool DST, bool REV = false>
QFT_DEV void unit_big(vec2<T> *wb, const T *U, const T *kcu, int lane, int ub = DST ? 1 : 0) {
    QFT_UMARK(0);
    FBlockP<L, R, DST, T> f;
    f.template load<REV>(wb, U, lane);
    __syncwarp();
    QFT_UMARK(1);
    f.store(wb, lane);
    __syncwarp();
    QFT_UMARK(2);
    if (lane < (1 << R)) b_l32p<DST, T>(wb + 33 * lane, kcu, ub, lane & 1);
    __syncwarp();
    QFT_UMARK(3);
    run_c_blockp<R, DST, T>(wb, lane);
    QFT_UMARK(4);
}
// rest unit: blocks JR..JF-1, the L = 32 block and the blocks with L <= 16.
// QFT_REST_FUSED: the F levels of every block JR..JF-1 are loaded / folded
// together (one __syncwarp before their stores), and likewise the C levels,
// instead of block after block (more independent work per warp).
template <int LOG2N, typename T, bool DST, int J, bool = (J < SPlan<LOG2N>::JF)>
struct FRest {
    QFT_DEV void load(const vec2<T> *, const T *, int) {}
    QFT_DEV void store(vec2<T> *, int) const {}
};
template <int LOG2N, typename T, bool DST, int J>
struct FRest<LOG2N, T, DST, J, true> {
    FBlock<LOG2N, J, DST, T> f;
    FRest<LOG2N, T, DST, J + 1> next;
    QFT_DEV void load(const vec2<T> *w, const T *U, int lane) {
        f.load(w, U, lane);
        next.load(w, U, lane);
    }
    QFT_DEV void store(vec2<T> *w, int lane) const {
        f.store(w, lane);
        next.store(w, lane);
    }
};
template <int LOG2N, typename T, bool DST, int J, bool = (J < SPlan<LOG2N>::JF)>
struct CRest {
    QFT_DEV void compute(const vec2<T> *, int) {}
    QFT_DEV void store(vec2<T> *, int) const {}
};
template <int LOG2N, typename T, bool DST, int J>
struct CRest<LOG2N, T, DST, J, true> {
    using P = SPlan<LOG2N>;
    static constexpr int R = P::RF(J), base = (DST ? P::S0 : 0) + P::off(J);
    vec2<T> out[1 << R];
    CRest<LOG2N, T, DST, J + 1> next;
    QFT_DEV void compute(const vec2<T> *w, int lane) {
        const vec2<T> *wb = w + padx(base);
        CBlockP<R, DST, T> c;
        c.load(wb, lane);
        const vec2<T> *hc = CBlockP<R, DST, T>::halo_colp(wb, lane);
        auto halo = [&](int p) { return hc[33 * p]; };
        c.compute(lane, halo, out);
        next.compute(w, lane);
    }
    QFT_DEV void store(vec2<T> *w, int lane) const {
        CBlockP<R, DST, T>::storep(w + padx(base), lane, out);
        next.store(w, lane);
    }
};
// SMALL = false: the blocks with L <= 16 are left to the caller (the pipelined
// kernel runs them in phase 2 on idle lanes: here lane CNT would diverge from the
// Lee-32 lanes and serialise the warp)
template <int LOG2N, typename T, bool DST, bool SMALL = true>
QFT_DEV void unit_rest(vec2<T> *w, const T *U, const T *kcu, int lane, int ub = DST ? 1 : 0) {
    using P = SPlan<LOG2N>;
    constexpr int sb = DST ? P::S0 : 0;
    constexpr int CNT = P::NL32 - P::K0;
#if QFT_REST_FUSED
    {
        FRest<LOG2N, T, DST, P::JR> fr;
        fr.load(w, U, lane);
        __syncwarp();
        fr.store(w, lane);
    }
#else
    run_f_blocks<LOG2N, T, P::JR>(w, U, DST, lane);
#endif
    __syncwarp();
    if (lane < CNT) b_l32<DST, T>(w, sb + 32 * (P::K0 + lane), kcu, ub, (P::K0 + lane) & 1);
    else if (SMALL && lane == CNT) b_small<LOG2N, DST, T>(w, kcu, ub);
    __syncwarp();
#if QFT_REST_FUSED
    {
        CRest<LOG2N, T, DST, P::JR> cr;
        cr.compute(w, lane);
        __syncwarp();
        cr.store(w, lane);
        __syncwarp();
    }
#else
    run_c_blocks<LOG2N, T, P::JR>(w, DST, lane);
#endif
}

// ---- top levels of the huge blocks (N > 4096), whole CTA.  For one signal at
// a time, every thread holds its items of every huge block (both sides) in
// registers across one CTA barrier, because the levels permute cells across the
// whole block.  The next signal's loads touch other cells, so they need no
// barrier after the previous signal's stores.
template <int LOG2N, typename T, int MODE, int J>
QFT_DEV void top_f_sig(vec2<T> *w, const T *U, int tid) {
    using P = SPlan<LOG2N>;
    using K = KCfg<LOG2N, T>;
    if constexpr (J >= P::JH) {
        __syncthreads();
    } else {
        using TC = Top<LOG2N, J, false, T>;
        // QFT_SC: the sine side runs the cosine code on the sine region
        using TS = Top<LOG2N, J, !QFT_SC, T>;
        vec2<T> *const wsn = QFT_SC ? w + padx(P::S0) : w;
        constexpr int G = TC::G, IT = K::TIT, NT = K::NT;
        constexpr bool DOC = MODE != 3, DOS = MODE != 2;
        vec2<T> vc[IT][G], vs[IT][G];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int t = tid + k * NT;
            if (t < 1024) {
                if (DOC) TC::f_load(w, U, t, vc[k]);
                if (DOS) TS::f_load(wsn, U, t, vs[k]);
            }
        }
        top_f_sig<LOG2N, T, MODE, J + 1>(w, U, tid);
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int t = tid + k * NT;
            if (t < 1024) {
                if (DOC) TC::f_store(w, t, vc[k]);
                if (DOS) TS::f_store(wsn, t, vs[k]);
            }
        }
    }
}
template <int LOG2N, typename T, int MODE, int J>
QFT_DEV void top_b_sig(vec2<T> *w, int tid) {
    using P = SPlan<LOG2N>;
    using K = KCfg<LOG2N, T>;
    if constexpr (J >= P::JH) {
        __syncthreads();
    } else {
        using TC = Top<LOG2N, J, false, T>;
        using TS = Top<LOG2N, J, !QFT_SC, T>;
        vec2<T> *const wsn = QFT_SC ? w + padx(P::S0) : w;
        constexpr int G = TC::G, IT = K::TIT, NT = K::NT;
        constexpr bool DOC = MODE != 3, DOS = MODE != 2;
        vec2<T> oc[IT][G], os[IT][G];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int i = tid + k * NT;
            if (i < 1024) {
                if (DOC) TC::b_compute(w, i, oc[k]);
                if (DOS) TS::b_compute(wsn, i, os[k]);
            }
        }
        top_b_sig<LOG2N, T, MODE, J + 1>(w, tid);
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int i = tid + k * NT;
            if (i < 1024) {
                if (DOC) TC::b_store(w, i, oc[k]);
                if (DOS) TS::b_store(wsn, i, os[k]);
            }
        }
    }
}
// all signals; ends with a CTA barrier (ntr is CTA-uniform)
template <int LOG2N, typename T, int MODE>
QFT_DEV void top_f(vec2<T> *W, const T *U, int ntr, int tid) {
    for (int tau = 0; tau < ntr; ++tau) top_f_sig<LOG2N, T, MODE, 0>(W + tau * SPlan<LOG2N>::PADDED, U, tid);
    __syncthreads();
}
template <int LOG2N, typename T, int MODE>
QFT_DEV void top_b(vec2<T> *W, int ntr, int tid) {
    for (int tau = 0; tau < ntr; ++tau) top_b_sig<LOG2N, T, MODE, 0>(W + tau * SPlan<LOG2N>::PADDED, tid);
    __syncthreads();
}

// fused unit `kind` of the signal at w: side kind & 1, big unit kind >> 1 (or
// the rest unit when kind >> 1 == NU1)
template <int LOG2N, typename T, int MODE, bool SMALL = true>
QFT_DEV void run_unit(vec2<T> *w, int kind, const T *U, const T *kcu, int lane) {
    using P = SPlan<LOG2N>;
    const bool dst = kind & 1;
    if ((MODE == 2 && dst) || (MODE == 3 && !dst)) return;  // side not needed
    const int bu = kind >> 1;
    if constexpr (QFT_SC) {  // both sides through the cosine code (qft_smem.cuh QFT_SC)
        vec2<T> *ws = w + (dst ? padx(P::S0) : 0);
        if (bu < P::NU1) unit_big<P::LB, P::RB, T, false>(ws + padx(P::big_cell(bu)), U, kcu, lane, dst);
        else unit_rest<LOG2N, T, false, SMALL>(ws, U, kcu, lane, dst);
    } else if (bu < P::NU1) {
        vec2<T> *wb = w + padx((dst ? P::S0 : 0) + P::big_cell(bu));
        if (dst) unit_big<P::LB, P::RB, T, true>(wb, U, kcu, lane);
        else unit_big<P::LB, P::RB, T, false>(wb, U, kcu, lane);
    } else {
        if (dst) unit_rest<LOG2N, T, true>(w, U, kcu, lane);
        else unit_rest<LOG2N, T, false>(w, U, kcu, lane);
    }
}

// A+B+C of TT signals, one warp per (signal, side, unit)
template <int LOG2N, typename T, int MODE, int TT, int NW, bool SMALL = true>
QFT_DEV void fused_units(vec2<T> *W, const T *U, const T *kcu, int ntr, int warp, int lane) {
    using P = SPlan<LOG2N>;
    constexpr int NU = 2 * (P::NU1 + 1);
    for (int u = warp; u < TT * NU; u += NW) {
        const int tau = u / NU, kind = u - tau * NU;
        if (tau >= ntr) continue;
        run_unit<LOG2N, T, MODE, SMALL>(W + tau * P::PADDED, kind, U, kcu, lane);
        __syncwarp();
    }
}

// ---- phased units (N <= 2048): below 1024-cell blocks a fused warp unit leaves
// most lanes idle in its Lee-32 step (block 0 of N = 1024 has 8 sub-blocks: 8 of
// 32 lanes; N = 128 has one chunk per side), and that step is most of the
// unit's instructions.  Here the three steps are CTA phases instead: F by warp
// units, then the Lee-32 chunks (and the L <= 16 blocks) of ALL signals of the
// iteration flat over the CTA's threads (the chunks of a side are the cells
// [32k, 32k+32), k < NL32, after the sub-block-major F stores), then C by warp
// units.  Same per-cell operations, two more CTA barriers per iteration.
#ifndef QFT_SMEM_L2PF
#define QFT_SMEM_L2PF 0  // L2 bulk prefetch of the batch after the next (single-pass kernel with TMA staging): measured -0.6 % (fp32 2^10), -1 % (fp64 2^10), +0.9 % (fp32 2^11)
#endif
#ifndef QFT_PHASED
#define QFT_PHASED 1
#endif
template <int LOG2N>
constexpr bool use_phased() {
    return QFT_PHASED && QFT_SC && LOG2N <= 11;
}
template <int LOG2N, typename T, int MODE, int TT, int NW>
QFT_DEV void phased_units(vec2<T> *W, const T *U, const T *kcu, int ntr, int tid) {
    using P = SPlan<LOG2N>;
    constexpr int NU = 2 * (P::NU1 + 1), NT = NW * 32, NL = P::NL32;
    constexpr bool DOC = MODE != 3, DOS = MODE != 2;
    const int warp = tid >> 5, lane = tid & 31;
    auto side = [&](int tau, bool dst) { return W + tau * P::PADDED + (dst ? padx(P::S0) : 0); };
    if constexpr (P::JF >= 1) {
        for (int u = warp; u < TT * NU; u += NW) {
            const int tau = u / NU, kind = u - tau * NU;
            const bool dst = kind & 1;
            if (tau >= ntr || (dst ? !DOS : !DOC)) continue;
            vec2<T> *ws = side(tau, dst);
            if ((kind >> 1) < P::NU1) {
                FBlockP<P::LB, P::RB, false, T> f;
                f.load(ws, U, lane);
                __syncwarp();
                f.store(ws, lane);
            } else {
                run_f_blocks<LOG2N, T, P::JR>(ws, U, false, lane);
            }
            __syncwarp();
        }
        __syncthreads();
    }
    if constexpr (NL > 0) {
        // NL + 1 = m/32 slots per side (the last one idle): a side's chunks sit 33 cells
        // apart and the sine side starts padx(m) = m/32 (mod 16) cells after the cosine
        // side, so the 16 lanes of a half-warp -- one side, or 16 / (NL + 1) sides -- hit
        // 16 distinct bank pairs (ncu: 2-way conflicts with NL slots per side)
        constexpr int NLP = NL + 1;
        for (int it = tid; it < TT * 2 * NLP; it += NT) {
            const int tau = it / (2 * NLP), r = it & (2 * NLP - 1), k = r & (NLP - 1);
            const bool dst = r >= NLP;
            if (k == NL || tau >= ntr || (dst ? !DOS : !DOC)) continue;
            b_l32<false, T>(side(tau, dst), 32 * k, kcu, dst, k & 1);
        }
    }
    // the L <= 16 blocks of every side, on the threads with the fewest chunks (the last ones)
    for (int it = NT - 1 - tid; it < TT * 2; it += NT) {
        const int tau = it >> 1;
        const bool dst = it & 1;
        if (tau >= ntr || (dst ? !DOS : !DOC)) continue;
        b_small<LOG2N, false, T>(side(tau, dst), kcu, dst);
    }
    if constexpr (P::JF >= 1) {
        __syncthreads();
        for (int u = warp; u < TT * NU; u += NW) {
            const int tau = u / NU, kind = u - tau * NU;
            const bool dst = kind & 1;
            if (tau >= ntr || (dst ? !DOS : !DOC)) continue;
            vec2<T> *ws = side(tau, dst);
            if ((kind >> 1) < P::NU1) run_c_blockp<P::RB, false, T>(ws, lane);
            else run_c_blocks<LOG2N, T, P::JR>(ws, false, lane);
        }
    }
}

// A0 of TT complex signals from src (staging buffer or global memory): chunks
// of 64 consecutive n per warp, UNR chunks in flight; then the multiples of 64.
// first: chunks [0, first) of a single signal (TTn == 1) were loaded ahead (QFT_A0_PRE)
template <int LOG2N, typename T, int UNR>
QFT_DEV void a0_complex(const vec2<T> *src, vec2<T> *W, int ntr, int TTn, int tid, int NT, int NW,
                        const A0Lane64 &a0l64, int first = 0) {
    using P = SPlan<LOG2N>;
    const int lane = tid & 31, warp = tid >> 5;
    if constexpr (P::m >= 64) {
        constexpr int NC64 = P::m / 64;
        auto shfl_up = [](vec2<T> v) { return shfl_vec(v, false); };
        for (int u0 = first + warp; u0 < TTn * NC64; u0 += NW * UNR) {
            A0Chunk64<T> ch[UNR];
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                const int u = u0 + r * NW, tau = u / NC64, c = u - tau * NC64;
                if (u < TTn * NC64 && tau < ntr) ch[r].template load<LOG2N>(src + tau * P::N, c, lane);
            }
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                const int u = u0 + r * NW, tau = u / NC64, c = u - tau * NC64;
                // the shuffle inside store is warp-uniform (u, tau do not depend on the lane)
                if (u < TTn * NC64 && tau < ntr) ch[r].template store<LOG2N>(W + tau * P::PADDED, c, lane, a0l64, shfl_up);
            }
        }
        if constexpr (!QFT_A0_LANE0) {
            for (int it = tid; it < TTn * NC64; it += NT) {
                const int tau = it / NC64, c = it - tau * NC64;
                if (tau < ntr) a0_item<LOG2N, T>(src + tau * P::N, W + tau * P::PADDED, 64 * c);
            }
        }
    } else {
        for (int tau = 0; tau < ntr; ++tau)
            for (int nn = tid; nn < P::m; nn += NT) a0_item<LOG2N, T>(src + tau * P::N, W + tau * P::PADDED, nn);
    }
}

// MODE 0: complex cdft on (batch, N) complex rows.  MODE 1/2/3: rdft / dct0 /
// dst0 on real rows (nreal rows of the mode's stored length), two rows per vec2
// signal; `batch` then counts row pairs.
template <int LOG2N, typename T, int MODE = 0>
__global__ void __launch_bounds__(KCfg<LOG2N, T>::NT, KCfg<LOG2N, T>::CPS)
    qft_cdft_smem(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out, long long batch,
                  const T *__restrict__ Ug, const __grid_constant__ LeeConst<T> kc, long long nreal = 0,
                  int tt_arg = KCfg<LOG2N, T>::TT) {
    // tt <= TT: signals per CTA iteration (smaller for small batches, so that
    // the batch spreads over every SM; the shared-memory slots stay TT)
    const int tt = KCfg<LOG2N, T>::TT == 1 ? 1 : tt_arg;
    using P = SPlan<LOG2N>;
    using K = KCfg<LOG2N, T>;
    constexpr int TT = K::TT, NT = K::NT, NW = K::NW;
    constexpr bool TMA = K::TMA && MODE == 0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    vec2<T> *stage = reinterpret_cast<vec2<T> *>(smem_raw + K::STAGE_OFF);
    vec2<T> *W = reinterpret_cast<vec2<T> *>(smem_raw + K::W_OFF);
    T *U = reinterpret_cast<T *>(smem_raw + K::U_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + K::BAR_OFF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const long long nbatch = (batch + tt - 1) / tt;
    const A0Lane64 a0l64 = a0_lane64<LOG2N>(lane);
    for (int i = tid; i < K::UCS; i += NT) U[i] = Ug[i];
    if (TMA && tid == 0) mbar_init(bar, 1);
    __syncthreads();
    long long bt = blockIdx.x;
    constexpr int TS = K::TS;
    // TMA part of batch b: its first min(TS, count) signals
    auto stage_count = [&](long long b) -> long long {
        const long long nt = (batch - b * tt) < tt ? (batch - b * tt) : tt;
        return nt < TS ? nt : TS;
    };
    if (TMA && tid == 0 && bt < nbatch)
        tma_bulk_load(stage, in + bt * tt * P::N, (uint32_t)(stage_count(bt) * P::N * K::VB), bar);
    uint32_t parity = 0;
    // QFT_A0_PRE: one signal per iteration read from global memory (no staging room):
    // the warps without a phase-D item load the first PRE_C A0 chunks of the next
    // signal into registers during phase D, and store them at the next A0
    constexpr int WD = (TT * K::DI + 31) / 32, NPW = NW > WD ? NW - WD : 0;
    constexpr bool PRE = QFT_A0_PRE && MODE == 0 && TS == 0 && TT == 1 && sizeof(T) == 4 && P::m >= 64 && NPW > 0;
    constexpr int PU = QFT_A0_PRE_UNR;  // chunks per prefetching warp
    constexpr int PRE_C0 = PRE ? NPW * PU : 0;
    constexpr int PRE_C = PRE_C0 < P::m / 64 ? PRE_C0 : P::m / 64;
    A0Chunk64<T> pre[PRE ? PU : 1];
    bool pre_ok = false;
    for (; bt < nbatch; bt += gridDim.x) {
        const int ntr = (int)((batch - bt * tt) < tt ? (batch - bt * tt) : tt);
        QFT_MARK(0);
        if constexpr (TMA) {
            mbar_wait(bar, parity);
            parity ^= 1u;
        }
        QFT_MARK(1);
        if (MODE == 0 && TS < TT && tid == 0 && bt + gridDim.x < nbatch) {
            // pull the next batch's unstaged signals into L2 while this one is transformed
            const long long nb = bt + gridDim.x;
            const long long nt = (batch - nb * tt) < tt ? (batch - nb * tt) : tt;
            if (nt > TS) l2_prefetch(in + (nb * tt + TS) * P::N, (uint32_t)((nt - TS) * P::N * K::VB));
        }
        // A0: fold + route -> W
        if constexpr (MODE != 0) {
            // real modes: rows of the mode's stored length straight from global memory
            constexpr int RL = MODE == 1 ? P::N : (MODE == 2 ? P::m + 1 : P::m - 1);
            const T *xr = reinterpret_cast<const T *>(in);
            for (int tau = 0; tau < ntr; ++tau) {
                const long long ra = 2 * (bt * tt + tau), rb = ra + 1 < nreal ? ra + 1 : ra;
                for (int nn = tid; nn <= P::m; nn += NT)
                    a0_item_real<LOG2N, T, MODE>(xr + ra * RL, xr + rb * RL, W + tau * P::PADDED, nn);
            }
        } else {
            if constexpr (PRE) {
                if (pre_ok && warp >= WD) {
                    auto shfl_up = [](vec2<T> v) { return shfl_vec(v, false); };
#pragma unroll
                    for (int r = 0; r < PU; ++r) {
                        const int c = (warp - WD) + r * NPW;
                        if (c < PRE_C) pre[r].template store<LOG2N>(W, c, lane, a0l64, shfl_up);
                    }
                }
                a0_complex<LOG2N, T, QFT_A0_UNR>(in + bt * P::N, W, 1, 1, tid, NT, NW, a0l64, pre_ok ? PRE_C : 0);
            } else if constexpr (TS < TT) {
                if (ntr > TS)
                    a0_complex<LOG2N, T, sizeof(T) == 8 ? 1 : QFT_A0_UNR>(in + (bt * tt + TS) * P::N,
                                                                          W + TS * P::PADDED, ntr - TS, TT - TS, tid,
                                                                          NT, NW, a0l64);
            }
            if constexpr (TS > 0) a0_complex<LOG2N, T, 1>(stage, W, ntr < TS ? ntr : TS, TS, tid, NT, NW, a0l64);
        }
        __syncthreads();
        QFT_MARK(2);
        // the staging buffer is free: prefetch the next batch while we compute
        if (TMA && tid == 0 && bt + gridDim.x < nbatch) {
            const long long nb = bt + gridDim.x;
            tma_bulk_load(stage, in + nb * tt * P::N, (uint32_t)(stage_count(nb) * P::N * K::VB), bar);
#if QFT_SMEM_L2PF
            // and the batch after that into L2, so that its bulk copy one iteration later
            // is served from L2 (ncu at N = 1024: 22 % of the stall samples wait for the copy)
            const long long nb2 = nb + gridDim.x;
            if (nb2 < nbatch) l2_prefetch(in + nb2 * tt * P::N, (uint32_t)(stage_count(nb2) * P::N * K::VB));
#endif
        }
        // TF: top forward levels of the huge blocks (N > 4096; ends with a barrier)
        if constexpr (P::JH > 0) top_f<LOG2N, T, MODE>(W, K::USPLIT ? Ug : U, ntr, tid);
        // A+B+C fused: one warp per (signal, side, unit) -- no CTA barrier inside
        if constexpr (use_phased<LOG2N>()) phased_units<LOG2N, T, MODE, TT, NW>(W, U, kc.u, ntr, tid);
        else fused_units<LOG2N, T, MODE, TT, NW>(W, U, kc.u, ntr, warp, lane);
        QFT_WMARK();
        __syncthreads();
        QFT_MARK(3);
        // TB: top backward levels of the huge blocks (ends with a barrier)
        if constexpr (P::JH > 0) top_b<LOG2N, T, MODE>(W, ntr, tid);
        // D: chain + recombination -> global
        for (int it = tid; it < TT * K::DI; it += NT) {
            const int tau = it / K::DI, ti = it - tau * K::DI;
            if (tau >= ntr) continue;
            if constexpr (MODE == 0) {
                if constexpr (K::DHALF) {
                    const int h = ti >= P::DT, t = ti - (h ? P::DT : 0);
                    Chain<LOG2N, T>::unit_half(W + tau * P::PADDED, out + (bt * tt + tau) * P::N, t, h);
                } else {
                    Chain<LOG2N, T>::unit(W + tau * P::PADDED, out + (bt * tt + tau) * P::N, ti);
                }
            } else {
                const int t = K::DHALF ? (ti >= P::DT ? ti - P::DT : ti) : ti;
                const int h = K::DHALF ? (ti >= P::DT) : 0;
                // per-signal outputs: rdft packed half spectrum (shared.py:38-43 with
                // complex_from_packed, shared.py:94-101), dct0 / dst0 real spectra
                const long long ra = 2 * (bt * tt + tau);
                const bool has_b = ra + 1 < nreal;
                auto emit = [&](int k, vec2<T> cv, vec2<T> sv) {
                    if constexpr (MODE == 1) {
                        vec2<T> *ya = out + ra * (P::m + 1);
                        const bool edge = (k == 0) || (k == P::m);
                        ya[k] = {cv.x, edge ? (T)0 : -sv.x};
                        if (has_b) ya[P::m + 1 + k] = {cv.y, edge ? (T)0 : -sv.y};
                    } else if constexpr (MODE == 2) {
                        T *ya = reinterpret_cast<T *>(out) + ra * (P::m + 1);
                        ya[k] = cv.x;
                        if (has_b) ya[P::m + 1 + k] = cv.y;
                    } else {
                        if (k == 0 || k == P::m) return;
                        T *ya = reinterpret_cast<T *>(out) + ra * (P::m - 1);
                        ya[k - 1] = sv.x;
                        if (has_b) ya[P::m - 1 + k - 1] = sv.y;
                    }
                };
                if constexpr (K::DHALF) Chain<LOG2N, T>::unit_e_half(W + tau * P::PADDED, emit, t, h);
                else Chain<LOG2N, T>::unit_e(W + tau * P::PADDED, emit, t);
            }
        }
        if constexpr (PRE) {
            // warps with no phase-D item: the next signal's first A0 chunks into registers
            // (its L2 prefetch was issued at the top of this iteration)
            pre_ok = bt + gridDim.x < nbatch;
            if (pre_ok && warp >= WD) {
                const vec2<T> *nx = in + (bt + gridDim.x) * P::N;
#pragma unroll
                for (int r = 0; r < PU; ++r) {
                    const int c = (warp - WD) + r * NPW;
                    if (c < PRE_C) pre[r].template load<LOG2N>(nx, c, lane);
                }
            }
        }
        QFT_MARK(4);
        __syncthreads();
        QFT_MARK(5);
    }
}

inline int smem_bytes_for_cfg(int smem) { return smem; }

template <int LOG2N, typename T, int MODE = 0>
cudaError_t launch_smem(const LaunchArgs &a) {
    using K = KCfg<LOG2N, T>;
    auto kern = qft_cdft_smem<LOG2N, T, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::NT, K::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    // small batches: fewer signals per CTA iteration so every SM gets work
    const long long ctas = (long long)a.num_sms * per_sm;
    int tt = K::TT;
    if (a.batch < ctas * K::TT) tt = (int)((a.batch + ctas - 1) / ctas);
    if (tt < 1) tt = 1;
    const long long nbatch = (a.batch + tt - 1) / tt;
    long long grid = ctas;
    if (grid > nbatch) grid = nbatch;
    if (grid < 1) grid = 1;
    LeeConst<T> kc;
    for (int i = 0; i < 32; ++i) kc.u[i] = ((const T *)a.Uhead)[i];
    kern<<<(unsigned)grid, K::NT, K::SMEM, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch,
                                                       (const T *)a.U, kc, a.nreal, tt);
    return cudaGetLastError();
}

template <int LOG2N, typename T>
constexpr int smem_config_bytes() { return KCfg<LOG2N, T>::SMEM; }

template <int NN, typename T, int MODE = 0>
cudaError_t launch_reg(const LaunchArgs &a) {
    constexpr int NT = MODE == 0 ? RegCfg<NN, T>::SIG : 128;
    long long blocks = (a.batch + NT - 1) / NT;
    long long cap = (long long)a.num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    qft_cdft_reg<NN, T, MODE><<<(unsigned)blocks, NT, 0, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out,
                                                                      a.batch, (const T *)a.U, a.nreal);
    return cudaGetLastError();
}

}  // namespace qft
