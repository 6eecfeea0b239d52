// qft_launch.cuh -- the batched transform kernels and their launchers.
//   qft_cdft_reg   N <= 32     : one thread per signal, whole transform in registers
//   qft_cdft_smem  N = 64..4096: persistent CTAs (1 per SM); each CTA transforms
//                                TT signals per iteration through the phases of
//                                qft_smem.cuh while a TMA bulk copy prefetches the
//                                next TT signals into a staging buffer
// Each (precision, N) instance is compiled in its own translation unit
// (qft_inst.cu) so the build parallelises.
#pragma once
#include <cuda_runtime.h>

#include "qft_smem.cuh"

#ifndef QFT_CTAS_PER_SM
#define QFT_CTAS_PER_SM 1  // shared-memory budget split: CTAs resident per SM
#endif
#ifndef QFT_A0_TMA
#define QFT_A0_TMA 1       // A0 input: TMA bulk copy into a staging buffer (1) or L2-prefetched global loads (0)
#endif
#ifndef QFT_TT_MAX
#define QFT_TT_MAX 4       // cap on signals per CTA iteration
#endif
#ifndef QFT_A0_64
#define QFT_A0_64 1        // A0 by 64-sample chunks (conflict-free block-0 stores, paired loads)
#endif
#ifndef QFT_FUSED_ABC
#define QFT_FUSED_ABC 1    // phases A, B, C fused per warp (no CTA barriers between them)
#endif
#ifndef QFT_HALO_SHFL
#define QFT_HALO_SHFL 0    // phase-C halo by warp shuffle (1) or by a shared-memory read (0)
#endif
#ifndef QFT_A0_UNIT8
#define QFT_A0_UNIT8 0     // A0 with 8 pairs per thread (fewer instructions, more bank conflicts)
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
template <int LOG2N, typename T>
struct KCfg {
    using P = SPlan<LOG2N>;
    static constexpr int VB = (int)sizeof(vec2<T>);
    static constexpr int PER = (QFT_A0_TMA ? P::N * VB : 0) + P::PADDED * VB;  // (staging +) working per signal
    static constexpr int UB = P::UCELLS * (int)sizeof(T);
    static constexpr int BUDGET = (226 * 1024) / QFT_CTAS_PER_SM - UB - 64;
    static constexpr int TT0 = BUDGET / PER;
    static constexpr int TTC = P::n >= 12 ? QFT_TT_MAX : 64;
    static constexpr int TT = TT0 < 1 ? 1 : (TT0 > TTC ? TTC : TT0);  // signals per CTA iteration
    static constexpr int rup32(int x) { return (x + 31) / 32 * 32; }
    static constexpr int NB32 = rup32(TT * P::NL32);                 // phase-B Lee-32 lanes per side
    static constexpr int W_B = (2 * NB32 + rup32(2 * TT)) / 32;
    static constexpr int W_D = (TT * P::DT + 31) / 32;
    static constexpr int W_AC = TT * P::NWU + QFT_CHAIN_MID;  // + the chain-mid warp
    static constexpr int mx(int a, int b) { return a > b ? a : b; }
    static constexpr int NU = P::JF >= 1 ? 4 : 2;  // fused warp units per signal
    static constexpr int W_U = TT * NU;
    static constexpr int NW0 = QFT_FUSED_ABC ? mx(W_U, W_D) : mx(mx(W_B, W_D), W_AC);
    static constexpr int NWMAX = sizeof(T) == 8 ? 12 : 17;  // keep >= 168 (fp64) / 120 (fp32) registers
    static constexpr int NW = NW0 < 4 ? 4 : (NW0 > NWMAX ? NWMAX : NW0);
    static constexpr int NT = NW * 32;
    static constexpr int STAGE_OFF = 0;
    static constexpr int W_OFF = QFT_A0_TMA ? TT * P::N * VB : 0;
    static constexpr int U_OFF = W_OFF + TT * P::PADDED * VB;
    static constexpr int BAR_OFF = (U_OFF + UB + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + 16;
};

// ------------------------------------------------------------ small N
template <int NN, typename T, int MODE = 0>
__global__ void __launch_bounds__(128) qft_cdft_reg(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out,
                                                    long long batch, const T *__restrict__ U, long long nreal = 0) {
    __shared__ T sU[NN / 4 >= 2 ? NN / 4 : 2];
    for (int i = threadIdx.x; i < (NN / 4 >= 2 ? NN / 4 : 2); i += blockDim.x) sU[i] = U[i];
    __syncthreads();
    constexpr int m = NN / 2;
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (long long)gridDim.x * blockDim.x) {
        if constexpr (MODE == 0) {
            vec2<T> x[NN], y[NN];
#pragma unroll
            for (int n = 0; n < NN; ++n) x[n] = in[b * NN + n];
            cdft_reg<NN, T>(x, y, sU);
#pragma unroll
            for (int n = 0; n < NN; ++n) out[b * NN + n] = y[n];
        } else {
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

template <int LOG2N, typename T, int J, bool DST>
QFT_DEV void run_c_block(vec2<T> *w, int lane) {
    CBlock<LOG2N, J, DST, T> c;
    c.load(w, lane);
    constexpr int G = CBlock<LOG2N, J, DST, T>::G;
    vec2<T> out[G];
#if QFT_HALO_SHFL
    auto halo = [&](int p) { return shfl_vec(c.own[p], !DST); };
#else
    const vec2<T> *hc = CBlock<LOG2N, J, DST, T>::halo_col(w, lane);
    auto halo = [&](int p) { return hc[33 * p]; };  // read before the __syncwarp below
#endif
    c.compute(lane, halo, out);
    __syncwarp();
    c.store(w, lane, out);
    __syncwarp();
}

template <int LOG2N, typename T, int J>
QFT_DEV void run_c_blocks(vec2<T> *w, bool dst, int lane) {
    if constexpr (J < SPlan<LOG2N>::JF) {
        if (dst) run_c_block<LOG2N, T, J, true>(w, lane);
        else run_c_block<LOG2N, T, J, false>(w, lane);
        run_c_blocks<LOG2N, T, J + 1>(w, dst, lane);
    }
}

// chain-mid: one warp computes C_JM / S_JM of all signals, level by level
template <int LOG2N, typename T, int TT>
QFT_DEV void run_chain_mid(vec2<T> *W, int ntr, int lane) {
    using P = SPlan<LOG2N>;
    using C = Chain<LOG2N, T>;
    for (int it = lane; it < ntr; it += 32) C::mid_base(W + it * P::PADDED);
    __syncwarp();
    constexpr int RK = (P::MJM + 1 + 31) / 32;  // rounds of 32 lanes per signal and level
    for (int j = P::n - 2; j >= P::JM; --j) {
        const int cnt = 2 * C::qj(j) + 1;  // k in [0, m_j]
        vec2<T> cv[TT][RK], sv[TT][RK];
#pragma unroll
        for (int tau = 0; tau < TT; ++tau)
#pragma unroll
            for (int r = 0; r < RK; ++r) {
                const int k = lane + 32 * r;
                if (tau < ntr && k < cnt) C::mid_level_load(W + tau * P::PADDED, j, k, cv[tau][r], sv[tau][r]);
            }
        __syncwarp();
#pragma unroll
        for (int tau = 0; tau < TT; ++tau)
#pragma unroll
            for (int r = 0; r < RK; ++r) {
                const int k = lane + 32 * r;
                if (tau < ntr && k < cnt) C::mid_level_store(W + tau * P::PADDED, j, k, cv[tau][r], sv[tau][r]);
            }
        __syncwarp();
    }
}

// ---- fused forward / Lee-32 / backward work of one side of one signal, one warp.
// The F -> Lee-32 -> B work of a Lee block depends on no other block, so a warp
// runs it start to finish with __syncwarp only (no CTA barrier).
// unit 0: block 0 (its 2^RF(0) sub-blocks = one Lee-32 per lane)
template <int LOG2N, typename T, bool DST>
QFT_DEV void unit_block0(vec2<T> *w, const T *U, const T *kcu, int lane) {
    using P = SPlan<LOG2N>;
    if constexpr (P::JF >= 1) {
        constexpr int sb = DST ? P::S0 : 0;
        FBlock<LOG2N, 0, DST, T> f;
        f.load(w, U, lane);
        __syncwarp();
        f.store(w, lane);
        __syncwarp();
        if (lane < (1 << P::RF(0))) b_l32<DST, T>(w, sb + 32 * lane, kcu);
        __syncwarp();
        run_c_block<LOG2N, T, 0, DST>(w, lane);
    }
}
// unit 1: blocks 1..JF-1, the L = 32 block and the blocks with L <= 16
template <int LOG2N, typename T, bool DST>
QFT_DEV void unit_rest(vec2<T> *w, const T *U, const T *kcu, int lane) {
    using P = SPlan<LOG2N>;
    constexpr int sb = DST ? P::S0 : 0;
    constexpr int K0 = P::JF >= 1 ? (1 << P::RF(0)) : 0;  // first chunk after block 0
    constexpr int CNT = P::NL32 - K0;
    run_f_blocks<LOG2N, T, 1>(w, U, DST, lane);
    __syncwarp();
    if (lane < CNT) b_l32<DST, T>(w, sb + 32 * (K0 + lane), kcu);
    else if (lane == CNT) b_small<LOG2N, DST, T>(w, kcu);
    __syncwarp();
    run_c_blocks<LOG2N, T, 1>(w, DST, lane);
}

// MODE 0: complex cdft on (batch, N) complex rows.  MODE 1/2/3: rdft / dct0 /
// dst0 on real rows (nreal rows of the mode's stored length), two rows per vec2
// signal; `batch` then counts row pairs.
template <int LOG2N, typename T, int MODE = 0>
__global__ void __launch_bounds__(KCfg<LOG2N, T>::NT, QFT_CTAS_PER_SM)
    qft_cdft_smem(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out, long long batch,
                  const T *__restrict__ Ug, const __grid_constant__ LeeConst<T> kc, long long nreal = 0) {
    using P = SPlan<LOG2N>;
    using K = KCfg<LOG2N, T>;
    constexpr int TT = K::TT, NT = K::NT, NW = K::NW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
#if QFT_A0_TMA
    vec2<T> *stage = reinterpret_cast<vec2<T> *>(smem_raw + K::STAGE_OFF);
#endif
    vec2<T> *W = reinterpret_cast<vec2<T> *>(smem_raw + K::W_OFF);
    T *U = reinterpret_cast<T *>(smem_raw + K::U_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + K::BAR_OFF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const long long nbatch = (batch + TT - 1) / TT;
    const A0Lane a0l = a0_lane<LOG2N>(lane);
    const A0Lane64 a0l64 = a0_lane64<LOG2N>(lane);
    for (int i = tid; i < P::UCELLS; i += NT) U[i] = Ug[i];
#if QFT_A0_TMA
    if (tid == 0) mbar_init(bar, 1);
#else
    (void)bar;
#endif
    __syncthreads();
    long long bt = blockIdx.x;
#if QFT_A0_TMA
    if (MODE == 0 && tid == 0 && bt < nbatch) {
        const long long nt = (batch - bt * TT) < TT ? (batch - bt * TT) : TT;
        tma_bulk_load(stage, in + bt * TT * P::N, (uint32_t)(nt * P::N * K::VB), bar);
    }
    uint32_t parity = 0;
#endif
    for (; bt < nbatch; bt += gridDim.x) {
        const int ntr = (int)((batch - bt * TT) < TT ? (batch - bt * TT) : TT);
#if QFT_A0_TMA
        if constexpr (MODE == 0) {
            mbar_wait(bar, parity);
            parity ^= 1u;
        }
#else
        // pull the next batch into L2 while this one is transformed
        if (tid == 0 && bt + gridDim.x < nbatch) {
            const long long nb = bt + gridDim.x;
            const long long nt = (batch - nb * TT) < TT ? (batch - nb * TT) : TT;
            l2_prefetch(in + nb * TT * P::N, (uint32_t)(nt * P::N * K::VB));
        }
        const vec2<T> *stage = in + bt * TT * P::N;  // A0 reads global memory directly
#endif
        // A0: fold + route, staging -> W
        if constexpr (MODE != 0) {
            // real modes: rows of the mode's stored length straight from global memory
            constexpr int RL = MODE == 1 ? P::N : (MODE == 2 ? P::m + 1 : P::m - 1);
            const T *xr = reinterpret_cast<const T *>(in);
            for (int tau = 0; tau < ntr; ++tau) {
                const long long ra = 2 * (bt * TT + tau), rb = ra + 1 < nreal ? ra + 1 : ra;
                for (int nn = tid; nn <= P::m; nn += NT)
                    a0_item_real<LOG2N, T, MODE>(xr + ra * RL, xr + rb * RL, W + tau * P::PADDED, nn);
            }
        } else {
#if QFT_A0_UNIT8
        for (int it = tid; it < TT * (P::m / 8); it += NT) {
            const int tau = it / (P::m / 8), k = it - tau * (P::m / 8);
            if (tau < ntr) a0_unit8<LOG2N, T>(stage + tau * P::N, W + tau * P::PADDED, k);
        }
#else
        {
            // warps take chunks of 32 consecutive n; lane 0's multiples of 32 afterwards
            constexpr int NCH = P::m / 32;
#if !QFT_A0_TMA
            // global loads: 8 chunks in flight per lane (memory-level parallelism)
            constexpr int UNR = 8;
            for (int u0 = warp; u0 < TT * NCH; u0 += NW * UNR) {
                vec2<T> xa[UNR], xb[UNR];
#pragma unroll
                for (int r = 0; r < UNR; ++r) {
                    const int u = u0 + r * NW, tau = u / NCH, c = u - tau * NCH, n = 32 * c + lane;
                    if (u < TT * NCH && tau < ntr && lane) {
                        xa[r] = stage[tau * P::N + n];
                        xb[r] = stage[tau * P::N + P::N - n];
                    }
                }
#pragma unroll
                for (int r = 0; r < UNR; ++r) {
                    const int u = u0 + r * NW, tau = u / NCH, c = u - tau * NCH;
                    if (u < TT * NCH && tau < ntr && lane) {
                        vec2<T> *w = W + tau * P::PADDED;
                        const int cell = a0l.A + c * a0l.B;
                        w[padx(cell)] = vadd(xa[r], xb[r]);
                        w[padx(cell) + padx(P::S0)] = vsub(xa[r], xb[r]);
                    }
                }
            }
#else
#if QFT_A0_64
            // chunks of 64 consecutive n; the multiples of 64 (and n = 0) afterwards
            // (N = 64 has a single 32-sample half: one chunk of lanes 0..15 suffices
            //  only for m >= 64, so small N keep the 32-sample chunks below)
            if constexpr (P::m >= 64) {
            constexpr int NC64 = P::m / 64;
            auto shfl_up = [](vec2<T> v) { return shfl_vec(v, false); };
            for (int u = warp; u < TT * NC64; u += NW) {
                const int tau = u / NC64, c = u - tau * NC64;
                if (tau < ntr) a0_chunk64<LOG2N, T>(stage + tau * P::N, W + tau * P::PADDED, c, lane, a0l64, shfl_up);
            }
            for (int it = tid; it < TT * NC64; it += NT) {
                const int tau = it / NC64, c = it - tau * NC64;
                if (tau < ntr) a0_item<LOG2N, T>(stage + tau * P::N, W + tau * P::PADDED, 64 * c);
            }
            } else {
                for (int tau = 0; tau < ntr; ++tau)
                    for (int nn = tid; nn < P::m; nn += NT)
                        a0_item<LOG2N, T>(stage + tau * P::N, W + tau * P::PADDED, nn);
            }
#else
            // the warp walks its chunks of each signal with fixed per-lane constants
            for (int tau = 0; tau < ntr; ++tau) {
                const vec2<T> *xs = stage + tau * P::N;
                vec2<T> *ws = W + tau * P::PADDED;
                if (lane) {
#pragma unroll 4
                    for (int c = warp; c < NCH; c += NW) a0_chunk<LOG2N, T>(xs, ws, c, lane, a0l);
                }
            }
            for (int it = tid; it < TT * NCH; it += NT) {
                const int tau = it / NCH, c = it - tau * NCH;
                if (tau < ntr) a0_item<LOG2N, T>(stage + tau * P::N, W + tau * P::PADDED, 32 * c);
            }
#endif
#endif  // QFT_A0_TMA
        }
#endif  // QFT_A0_UNIT8
        }
        __syncthreads();
#if QFT_A0_TMA
        // the staging buffer is free: prefetch the next batch while we compute
        if (MODE == 0 && tid == 0 && bt + gridDim.x < nbatch) {
            const long long nb = bt + gridDim.x;
            const long long nt = (batch - nb * TT) < TT ? (batch - nb * TT) : TT;
            tma_bulk_load(stage, in + nb * TT * P::N, (uint32_t)(nt * P::N * K::VB), bar);
        }
#endif
#if QFT_FUSED_ABC
        // A+B+C fused: one warp per (signal, side, unit) -- no CTA barrier inside
        for (int u = warp; u < TT * K::NU; u += NW) {
            const int tau = u / K::NU, kind = u - tau * K::NU;
            if (tau >= ntr) continue;
            vec2<T> *w = W + tau * P::PADDED;
            const bool dst = kind & 1;
            if ((MODE == 2 && dst) || (MODE == 3 && !dst)) continue;  // side not needed
            if (K::NU == 4 && kind < 2) {
                if (dst) unit_block0<LOG2N, T, true>(w, U, kc.u, lane);
                else unit_block0<LOG2N, T, false>(w, U, kc.u, lane);
            } else {
                if (dst) unit_rest<LOG2N, T, true>(w, U, kc.u, lane);
                else unit_rest<LOG2N, T, false>(w, U, kc.u, lane);
            }
            __syncwarp();
        }
        __syncthreads();
#else
        // A: forward levels of the big blocks (warp units: side x {block 0, blocks 1..})
        if constexpr (P::NWU > 0) {
            for (int u = warp; u < TT * P::NWU; u += NW) {
                const int tau = u / P::NWU, kind = u - tau * P::NWU;
                if (tau >= ntr) continue;
                vec2<T> *w = W + tau * P::PADDED;
                const bool dst = kind & 1;
                if (kind < 2) {
                    if (dst) {
                        FBlock<LOG2N, 0, true, T> f;
                        f.load(w, U, lane);
                        __syncwarp();
                        f.store(w, lane);
                    } else {
                        FBlock<LOG2N, 0, false, T> f;
                        f.load(w, U, lane);
                        __syncwarp();
                        f.store(w, lane);
                    }
                } else {
                    run_f_blocks<LOG2N, T, 1>(w, U, dst, lane);
                }
                __syncwarp();
            }
            __syncthreads();
        }
        // B: Lee-32 on every 32-cell chunk (warp-uniform side), then the small blocks
        for (int u = tid; u < 2 * K::NB32 + 2 * TT; u += NT) {
            if (u < 2 * K::NB32) {
                const bool dst = u >= K::NB32;
                const int v = dst ? u - K::NB32 : u;
                const int tau = v / (P::NL32 > 0 ? P::NL32 : 1), k = v - tau * P::NL32;
                if (P::NL32 > 0 && tau < ntr) {
                    vec2<T> *w = W + tau * P::PADDED;
                    if (dst) b_l32<true, T>(w, P::S0 + 32 * k, kc.u);
                    else b_l32<false, T>(w, 32 * k, kc.u);
                }
            } else {
                const int v = u - 2 * K::NB32;
                const int tau = v >> 1;
                if (tau < ntr) {
                    vec2<T> *w = W + tau * P::PADDED;
                    if (v & 1) b_small<LOG2N, true, T>(w, kc.u);
                    else b_small<LOG2N, false, T>(w, kc.u);
                }
            }
        }
        __syncthreads();
        // C: backward levels of the big blocks; one more warp unit computes the
        // lower chain levels C_JM, S_JM of all signals (chain-mid)
        {
            for (int u = warp; u < TT * P::NWU + QFT_CHAIN_MID; u += NW) {
                if (QFT_CHAIN_MID && u == TT * P::NWU) {
                    run_chain_mid<LOG2N, T, TT>(W, ntr, lane);
                    continue;
                }
                if constexpr (P::NWU > 0) {
                    const int tau = u / P::NWU, kind = u - tau * P::NWU;
                    if (tau >= ntr) continue;
                    vec2<T> *w = W + tau * P::PADDED;
                    const bool dst = kind & 1;
                    if (kind < 2) {
                        if (dst) run_c_block<LOG2N, T, 0, true>(w, lane);
                        else run_c_block<LOG2N, T, 0, false>(w, lane);
                    } else {
                        run_c_blocks<LOG2N, T, 1>(w, dst, lane);
                    }
                }
            }
            __syncthreads();
        }
#endif
        // D: chain + recombination -> global
        for (int it = tid; it < TT * P::DT; it += NT) {
            const int tau = it / P::DT, t = it - tau * P::DT;
            if (tau >= ntr) continue;
            if constexpr (MODE == 0) {
                Chain<LOG2N, T>::unit(W + tau * P::PADDED, out + (bt * TT + tau) * P::N, t);
            } else {
                // per-signal outputs: rdft packed half spectrum (shared.py:38-43 with
                // complex_from_packed, shared.py:94-101), dct0 / dst0 real spectra
                const long long ra = 2 * (bt * TT + tau);
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
                Chain<LOG2N, T>::unit_e(W + tau * P::PADDED, emit, t);
            }
        }
        __syncthreads();
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
    const long long nbatch = (a.batch + K::TT - 1) / K::TT;
    long long grid = (long long)a.num_sms * per_sm;
    if (grid > nbatch) grid = nbatch;
    if (grid < 1) grid = 1;
    LeeConst<T> kc;
    for (int i = 0; i < 32; ++i) kc.u[i] = ((const T *)a.Uhead)[i];
    kern<<<(unsigned)grid, K::NT, K::SMEM, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch,
                                                       (const T *)a.U, kc, a.nreal);
    return cudaGetLastError();
}

template <int LOG2N, typename T>
constexpr int smem_config_bytes() { return KCfg<LOG2N, T>::SMEM; }

template <int NN, typename T, int MODE = 0>
cudaError_t launch_reg(const LaunchArgs &a) {
    long long blocks = (a.batch + 127) / 128;
    long long cap = (long long)a.num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    qft_cdft_reg<NN, T, MODE><<<(unsigned)blocks, 128, 0, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out,
                                                                      a.batch, (const T *)a.U, a.nreal);
    return cudaGetLastError();
}

}  // namespace qft
