// qft_large.cu -- plan builder and launchers of the multi-pass path (qft_large.cuh).
// Compiled once per precision (-DQFT_LARGE_PREC=32|64).
//
// The plan builder replays the improved recursion at the level of Lee blocks
// (improved.py:49-112: fold, secant-scale the odd child, recurse, neighbour
// sums) and cuts every block larger than the leaf size into passes of at most
// RG fold levels, tracking where each sub-block's cells are (runs) and in which
// scratch buffer each spectrum ends up.  This is the "fixed kernel schedule"
// compiled from the decomposition tree (SURVEY.md §2 plan builder).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "qft_large_api.h"
#include "qft_large_plan.h"
#include "qft_launch.cuh"
#include "qft_leaf.cuh"

#if !defined(QFT_LARGE_PREC)
#error "compile with -DQFT_LARGE_PREC=32|64"
#endif
#if QFT_LARGE_PREC == 32
using Real = float;
#define QFT_LG(name) name##_f32
#else
using Real = double;
#define QFT_LG(name) name##_f64
#endif

using namespace qft;

namespace {

// largest single-pass sub-signal / leaf: 2^14 cells fp32, 2^13 fp64 (128 KiB)
constexpr int kSubLogMax = QFT_LARGE_PREC == 32 ? 14 : 13;
#ifndef QFT_LEAF_PAIR_GATHER
#define QFT_LEAF_PAIR_GATHER 1  // the two fold-on-load leaves of a block share one gather of x
#endif
#ifndef QFT_FOLD64
#define QFT_FOLD64 0  // fp64 plans with J0 <= 2 (N = 2^14, 2^15) fold on load like the fp32 ones
#endif
constexpr int kRG = 5;  // fold levels per F/B pass (fp64 R = 5: lane pairs, lg_f_pair5 / lg_b_pair5_out)
constexpr int kRC = 4;                                    // chain levels unfolded per thread
constexpr int kChunk = 256;
constexpr int kBChunk = 128;  // columns per CTA of a backward pass (outputs staged in shared memory)

template <typename T>
struct LeeConstL {
    T u[32];
};

struct Chunk {
    int task, t0;
};

struct TaskSet {  // one launch: tasks of one kind and one R (or log2 L for leaves)
    int R = 0;
    int staged = 0;  // F: fp64 five-level first-touch tasks through lg_f_staged_kernel
    void *d_tasks = nullptr, *d_dsts = nullptr, *d_chunks = nullptr, *d_rs = nullptr;
    int ntasks = 0, nchunks = 0;
};

using Sched = LargeSchedule;

}  // namespace

// N = 2^n: the sub-signal has 2^sublog points, J0 = n - sublog
static int sublog_for(int log2n) { return log2n - 1 < kSubLogMax ? log2n - 1 : kSubLogMax; }

struct QFT_LG(LargePlan) {
    int sublog, J0;
    Sched s;
    std::vector<std::vector<TaskSet>> fset, bset;
    void *d_items = nullptr, *d_leaves = nullptr;
    int nitems = 0;
    int launches = 0;
    QFT_LG(LargePlan)(int log2n, bool real_modes)
        : sublog(sublog_for(log2n)),
          J0(log2n - sublog_for(log2n)),
          s(log2n, sublog_for(log2n), kRG, J0, real_modes || !fold_on_load(log2n), !real_modes) {}
    // fold_on_load: the complex plan has no fold pass -- whole-block leaves fold x
    // while loading (tf_load_x) and the sub-signal folds x[k 2^J0] while loading
    // (sub_item).  Those gathers read every sector of x several times from L2, so
    // this only pays where the fold pass is a large share of the step: measured
    // +3.7 % at fp32 N = 2^16 (config 3), -4 % at fp64 N = 2^20 (config 4).
    static bool fold_on_load(int log2n) {
        return (QFT_LARGE_PREC == 32 || QFT_FOLD64) && log2n - sublog_for(log2n) <= 2;
    }
};

template <typename TT>
static int upload(const std::vector<TT> &v, void **d) {
    if (v.empty()) return 0;
    if (cudaMalloc(d, v.size() * sizeof(TT)) != cudaSuccess) return -1;
    return cudaMemcpy(*d, v.data(), v.size() * sizeof(TT), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : -1;
}

// ------------------------------------------------------------------ kernels
// fold pass: x -> W0 in the Lee-block cell layout (shared.py:28-35; the time-
// parity routing of improved.py:43, :81).  A CTA folds 2048 consecutive n (and
// their mirrors N-n), coalesced loads; the stores of one warp land in a few
// contiguous segments (block j takes every 2^(j+1)-th n).
constexpr int kFoldN = 2048, kFoldT = 256;
// samples n = n' << sh for n' in [0, m >> sh): the blocks j >= sh (the blocks
// j < sh are folded on first touch by the F passes)
template <typename T>
__global__ void __launch_bounds__(kFoldT) lg_fold_kernel(const vec2<T> *__restrict__ x, vec2<T> *__restrict__ W0,
                                                         int log2n, int sh, long long batch, long long Ws) {
    const int N = 1 << log2n, m = N / 2, cnt = m >> sh;
    const int nch = (cnt + kFoldN - 1) / kFoldN;
    for (long long g = blockIdx.x; g < batch * nch; g += gridDim.x) {
        const long long b = g / nch;
        const int a = (int)(g - b * nch) * kFoldN;
        const vec2<T> *xb = x + b * N;
        vec2<T> *w = W0 + b * Ws;
        constexpr int UNR = kFoldN / kFoldT;
        vec2<T> u[UNR], v[UNR];
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
            const int n = (a + r * kFoldT + (int)threadIdx.x) << sh;
            if (n < m) {
                u[r] = xb[n];
                v[r] = xb[n == 0 ? m : N - n];
            }
        }
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
            const int n = (a + r * kFoldT + (int)threadIdx.x) << sh;
            if (n >= m) continue;
            if (n == 0) {
                w[N - 1] = u[r];  // s(0) = x[0], s(m) = x[m]
                w[N] = v[r];
            } else {
                const int j = ctz32((uint32_t)n);
                const int cell = m - (1 << (log2n - 1 - j)) + (n >> (j + 1));
                w[cell] = vadd(u[r], v[r]);
                w[m + cell] = vsub(u[r], v[r]);
            }
        }
    }
}

// real modes: two rows of the mode's stored length per vec2 signal (pairs
// (2p, 2p+1); an odd last row pairs with itself and only its lane is stored)
template <typename T, int MODE>
__global__ void __launch_bounds__(kFoldT) lg_fold_real_kernel(const T *__restrict__ xr, vec2<T> *__restrict__ W0,
                                                              int log2n, long long batch, long long nreal,
                                                              long long Ws) {
    const int N = 1 << log2n, m = N / 2;
    const long long RL = MODE == 1 ? N : (MODE == 2 ? m + 1 : m - 1);
    const int cnt = m + 1;  // n in [0, m]
    const int nch = (cnt + kFoldN - 1) / kFoldN;
    for (long long g = blockIdx.x; g < batch * nch; g += gridDim.x) {
        const long long b = g / nch;
        const int a = (int)(g - b * nch) * kFoldN;
        const long long ra = 2 * b, rb = ra + 1 < nreal ? ra + 1 : ra;
        vec2<T> *w = W0 + b * Ws;
        for (int n = a + threadIdx.x; n < a + kFoldN && n < cnt; n += kFoldT) {
            if (n == m) continue;  // rdft / dct0: s(m) is routed with n = 0; dst0 has no s(m)
            lg_fold_real_item<T, MODE>(xr + ra * RL, xr + rb * RL, w, n, N, log2n);
        }
    }
}

template <int R, typename T>
__device__ __forceinline__ void lg_f_dispatch_r(vec2<T> *w, const FTask &tk, int t, bool dst, const T *U,
                                                const vec2<T> *x, int N) {
    if (t >= (tk.L >> R)) return;
    if (dst) lg_f_group<R, T, true>(w, tk, t, U, x, N);
    else lg_f_group<R, T, false>(w, tk, t, U, x, N);
}

// all forward tasks of one depth in one launch (R per task, uniform per CTA):
// grid.x enumerates (signal, chunk) with the chunks of one signal adjacent, so
// the strided sample gathers of its blocks share L2-resident sectors
template <typename T>
__global__ void __launch_bounds__(kChunk) lg_f_kernel(vec2<T> *__restrict__ W0, const FTask *__restrict__ tasks,
                                                      const int *__restrict__ dsts, const int *__restrict__ rs,
                                                      const Chunk *__restrict__ chunks, int nchunks,
                                                      const T *__restrict__ U, long long batch, long long Ws,
                                                      const vec2<T> *__restrict__ x, int N) {
    for (long long g = blockIdx.x; g < (long long)nchunks * batch; g += gridDim.x) {
        const long long b = g / nchunks;
        const Chunk ch = chunks[g - b * nchunks];
        const FTask tk = tasks[ch.task];
        const int t = ch.t0 + threadIdx.x;
        const bool dst = dsts[ch.task];
        vec2<T> *w = W0 + b * Ws;
        const vec2<T> *xb = x + b * N;
#if QFT_LARGE_PREC == 64
        if (rs[ch.task] == 5) {  // lane pairs: lanes l and l+16 share reflection group t
            const int tp = ch.t0 + (threadIdx.x >> 5) * 16 + (threadIdx.x & 15), h = (threadIdx.x >> 4) & 1;
            if (tp < (tk.L >> 5)) {  // both lanes of a pair agree (warp-uniform per half)
                if (dst) lg_f_pair5<T, true>(w, tk, tp, h, U, xb, N);
                else lg_f_pair5<T, false>(w, tk, tp, h, U, xb, N);
            }
            continue;
        }
#endif
        switch (rs[ch.task]) {
            case 1: lg_f_dispatch_r<1, T>(w, tk, t, dst, U, xb, N); break;
            case 2: lg_f_dispatch_r<2, T>(w, tk, t, dst, U, xb, N); break;
            case 3: lg_f_dispatch_r<3, T>(w, tk, t, dst, U, xb, N); break;
            case 4: lg_f_dispatch_r<4, T>(w, tk, t, dst, U, xb, N); break;
#if QFT_LARGE_PREC == 32
            case 5: lg_f_dispatch_r<5, T>(w, tk, t, dst, U, xb, N); break;
#endif
        }
    }
}

template <int R, typename T>
__global__ void __launch_bounds__(kBChunk) lg_b_kernel(vec2<T> *W0, vec2<T> *W1, const BTask *__restrict__ tasks,
                                                      const Chunk *__restrict__ chunks, long long batch, long long Ws) {
    constexpr int G = 1 << R, CELLS = kBChunk * G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    vec2<T> *stg = reinterpret_cast<vec2<T> *>(smem_raw);  // padded: cell p at p + p/32
    const Chunk ch = chunks[blockIdx.x];
    const BTask tk = tasks[ch.task];
    const int i = ch.t0 + threadIdx.x;
    const int ncols = min(kBChunk, (tk.L >> R) - ch.t0);
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        vec2<T> *W[2] = {W0 + b * Ws, W1 + b * Ws};
        if (threadIdx.x < ncols) {
            vec2<T> out[G];
            if (tk.dst) lg_b_column_out<R, T, true>(W, tk, i, out);
            else lg_b_column_out<R, T, false>(W, tk, i, out);
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const int p = threadIdx.x * G + q;
                stg[p + (p >> 5)] = out[q];
            }
        }
        __syncthreads();
        // the chunk's outputs are the contiguous cells [out0 + t0*G, out0 + (t0+ncols)*G)
        vec2<T> *dst = W[tk.out_buf] + tk.out0 + ch.t0 * G;
        for (int p = threadIdx.x; p < ncols * G; p += kBChunk) dst[p] = stg[p + (p >> 5)];
        __syncthreads();
        (void)CELLS;
    }
}

// fp64 R = 5 backward levels: lanes l and l+16 share column i (lg_b_pair5_out);
// a CTA of kBChunk threads covers kBChunk / 2 columns
template <typename T>
__global__ void __launch_bounds__(kBChunk) lg_b_pair_kernel(vec2<T> *W0, vec2<T> *W1, const BTask *__restrict__ tasks,
                                                           const Chunk *__restrict__ chunks, long long batch,
                                                           long long Ws) {
    constexpr int G = 32, COLS = kBChunk / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    vec2<T> *stg = reinterpret_cast<vec2<T> *>(smem_raw);  // padded: cell p at p + p/32
    const Chunk ch = chunks[blockIdx.x];
    const BTask tk = tasks[ch.task];
    const int lc = (threadIdx.x >> 5) * 16 + (threadIdx.x & 15), h = (threadIdx.x >> 4) & 1;
    const int i = ch.t0 + lc;
    const int ncols = min(COLS, (tk.L >> 5) - ch.t0);
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        vec2<T> *W[2] = {W0 + b * Ws, W1 + b * Ws};
        if (lc < ncols) {  // ncols is a multiple of 16: whole warps agree
            vec2<T> out[G / 2];
            if (tk.dst) lg_b_pair5_out<T, true>(W, tk, i, h, out);
            else lg_b_pair5_out<T, false>(W, tk, i, h, out);
#pragma unroll
            for (int q = 0; q < G / 2; ++q) {
                const int p = lc * G + h * (G / 2) + q;
                stg[p + (p >> 5)] = out[q];
            }
        }
        __syncthreads();
        vec2<T> *dst = W[tk.out_buf] + tk.out0 + ch.t0 * G;
        for (int p = threadIdx.x; p < ncols * G; p += kBChunk) dst[p] = stg[p + (p >> 5)];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ item kernel
// One persistent kernel runs every CTA-resident work item of every signal,
// signal-major (the items of a signal run concurrently, so the strided input
// gathers of its sub-signal and leaves share L2-resident sectors):
//   SUB  the 2^SUBLOG-point improved transform of the sub-signal x[k 2^J0]
//        (blocks j >= J0 of the time-parity chain) through the single-pass
//        phases of qft_launch.cuh; phase D emits C_J0 / S_J0 instead of y
//   LEAF one Lee block (or two of half the size) of 2^SUBLOG cells: whole
//        blocks fold x on load, sub-blocks of the F passes come from W0;
//        TF / warp units / TB (qft_leaf.cuh), spectrum written along the run
struct Item {
    int kind, k0;  // kind 0: SUB, 1: leaf task k0, 2: leaf tasks k0 and k0+1
};

template <int SUBLOG, typename T>
struct ItemCfg {
    using K = KCfg<SUBLOG, T>;
    using P = SPlan<SUBLOG>;
    static constexpr int NT = K::NT, NW = K::NW, L = 1 << SUBLOG;
    static constexpr int VB = (int)sizeof(vec2<T>);
    static constexpr int LPAD = L + L / 32 + 1;
    static constexpr int WCELLS = P::PADDED > LPAD ? P::PADDED : LPAD;
    static constexpr int UCELLS = L;  // level constants of every block size <= L
    static constexpr int U_OFF = WCELLS * VB;
    static constexpr int BAR_OFF = (U_OFF + UCELLS * (int)sizeof(T) + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + 16;
};

// ------------------------------------------------------------------ TMA tiles (fp64)
// W0 viewed as a 2-D tensor of 32-cell rows (64 doubles; the per-signal stride Ws
// is a multiple of 32 cells, and every leaf run / sub-signal range starts on a
// row).  A box of kTmaBoxCols = 66 doubles x kTmaRows rows reads each row plus 2
// out-of-bounds doubles that the TMA unit zero-fills: in shared memory every
// row lands at a pitch of 33 cells, which is exactly the padded working layout
// (cell p at p + p/32) -- the tile arrives conflict-free-padded with no
// per-thread copies (cp.async.bulk.tensor, UTMALDG).
constexpr int kTmaRows = 64, kTmaBoxCols = 66;
constexpr unsigned kTmaBoxBytes = kTmaRows * kTmaBoxCols * 8;

QFT_DEV void tma_tile_load(void *dst, const CUtensorMap *map, int row, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(0), "r"(row), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}
// one thread: load `cells` (a multiple of 32 * kTmaRows) consecutive W0 cells from
// row0 into the padded layout at dst, completing on bar
QFT_DEV void tma_cells(vec2<double> *dst, const CUtensorMap *map, long long row0, int cells, uint64_t *bar) {
    const int rows = cells / 32;
    for (int r = 0; r < rows; r += kTmaRows) tma_tile_load(dst + 33 * r, map, (int)(row0 + r), bar);
}
// the reverse: padded shared-memory rows -> W0 rows (out-of-bounds box columns,
// i.e. the pad cell of every row, are not written by a tensor store)
#ifndef QFT_TB_ROT
#define QFT_TB_ROT 0  // fp64 leaf TB stores in a lane-rotated slot order: conflict-free (4x fewer wavefronts), measured neutral on config 4
#endif
#ifndef QFT_LEAF_TMA_STORE
#define QFT_LEAF_TMA_STORE 1
#endif
QFT_DEV void tma_tile_store(const void *src, const CUtensorMap *map, int row) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(0),
                 "r"(row), "r"((uint32_t)__cvta_generic_to_shared(src))
                 : "memory");
}
QFT_DEV void tma_cells_store(const vec2<double> *src, const CUtensorMap *map, long long row0, int cells) {
    const int rows = cells / 32;
    for (int r = 0; r < rows; r += kTmaRows) tma_tile_store(src + 33 * r, map, (int)(row0 + r));
}
QFT_DEV void tma_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// async 8/16-byte global -> shared copies (no registers, all in flight at once)
template <typename T>
QFT_DEV void cp_async_cell(vec2<T> *dst, const vec2<T> *src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(vec2<T>) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
QFT_DEV void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// fp64 first-touch F tasks with their x samples staged in shared memory by
// cp.async (QFT_F_STAGED).  The cosine and the sine task of a Lee block read the
// same samples (dc = x[n] + x[N-n], ds = x[n] - x[N-n]), so a CTA takes both: the
// strided first-touch gathers are L2-bound (ncu: ~2 L2 sectors per useful sample,
// 5.8 GB of L2 reads for 1.1 GB of DRAM at N = 2^20), and staging once for both
// sides halves them.  Chunks of one signal are adjacent in the grid, so the blocks'
// gathers share x's sectors in L2.  A CTA of 256 threads takes GP reflection groups
// of one (cosine, sine) task pair: R = 5, GP = 64, thread (role, g) is side role & 1,
// child role >> 1 (lane pairs as lg_f_pair5); R <= 4, GP = 128, thread (side, g) does
// the whole group (lg_f_group).  stage[s][g] = (x[n], x[N-n]), n = 2^j (2e+1).
#ifndef QFT_F_STAGED
#define QFT_F_STAGED 1
#endif
#ifndef QFT_F_STG_T
#define QFT_F_STG_T 256
#endif
constexpr int kStgT = QFT_F_STG_T;  // threads per CTA
constexpr int stg_groups(int R) { return R == 5 ? kStgT / 4 : kStgT / 2; }
template <int R, typename T>
__device__ __forceinline__ void f_staged_chunk(vec2<T> *stg, const int *runc, const int *runs, const FTask *tp,
                                               int t0, vec2<T> *w, const vec2<T> *xb, int N, const T *U) {
    constexpr int G = 1 << R, GP = stg_groups(R);
    const int tid = threadIdx.x;
    const int gg = tid & (GP - 1), role = tid / GP;
    const bool dst = role & 1;
    const FTask tk = tp[dst ? 1 : 0];  // cosine task, its sine partner next
    const int ng = min(GP, (tk.L >> R) - t0);
    for (int q = tid; q < G * GP * 2; q += kStgT) {
        const int half = q & 1, g2 = (q >> 1) % GP, s = (q >> 1) / GP;
        if (g2 < ng) {
            const int e = runc[s] + runs[s] * (t0 + g2);
            const int n = (2 * e + 1) << tk.j;
            cp_async_cell<T>(stg + q, xb + (half ? N - n : n));
        }
    }
    cp_async_wait_all();
    __syncthreads();
    if (gg < ng) {
        const int t = t0 + gg;
        auto ld = [&](int s, int) {
            const vec2<T> *p = stg + (s * GP + gg) * 2;
            return dst ? vsub(p[0], p[1]) : vadd(p[0], p[1]);  // ds / dc fold (shared.py:28-35)
        };
        if constexpr (R == 5) {
            const int h = role >> 1;
            if (dst) lg_f_pair5_ld<T, true>(w, tk, t, h, U, ld);
            else lg_f_pair5_ld<T, false>(w, tk, t, h, U, ld);
        } else {
            if (dst) lg_f_group_ld<R, T, true>(w, tk, t, U, ld);
            else lg_f_group_ld<R, T, false>(w, tk, t, U, ld);
        }
    }
}
template <typename T>
__global__ void __launch_bounds__(kStgT, 512 / kStgT) lg_f_staged_kernel(vec2<T> *__restrict__ W0, const FTask *__restrict__ tasks,
                                                              const int *__restrict__ rs, const Chunk *__restrict__ chunks,
                                                              int nchunks, const T *__restrict__ U, long long batch,
                                                              long long Ws, const vec2<T> *__restrict__ x, int N) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    vec2<T> *stg = reinterpret_cast<vec2<T> *>(smem_raw);
    __shared__ int runc[32], runs[32];
    const int tid = threadIdx.x;
    for (long long g = blockIdx.x; g < (long long)nchunks * batch; g += gridDim.x) {
        const long long b = g / nchunks;
        const Chunk ch = chunks[g - b * nchunks];
        const int R = rs[ch.task];
        const FTask *tp = tasks + ch.task;
        if (tid < (1 << R)) {
            int c, sg;
            run_of(R, tp->L, tid, c, sg);
            runc[tid] = c;
            runs[tid] = sg;
        }
        __syncthreads();
        vec2<T> *w = W0 + b * Ws;
        const vec2<T> *xb = x + b * N;
        switch (R) {
            case 5: f_staged_chunk<5, T>(stg, runc, runs, tp, ch.t0, w, xb, N, U); break;
            case 4: f_staged_chunk<4, T>(stg, runc, runs, tp, ch.t0, w, xb, N, U); break;
            case 3: f_staged_chunk<3, T>(stg, runc, runs, tp, ch.t0, w, xb, N, U); break;
            case 2: f_staged_chunk<2, T>(stg, runc, runs, tp, ch.t0, w, xb, N, U); break;
            case 1: f_staged_chunk<1, T>(stg, runc, runs, tp, ch.t0, w, xb, N, U); break;
        }
        __syncthreads();  // the next chunk's copies overwrite the stage and the run table
    }
}

// the W0 cells an item reads, as up to 3 runs (lowest cell, count) -- for the
// L2 prefetch of the next item
template <int SUBLOG>
QFT_DEV int item_runs(const Item &it, const LeafTask *tasks, int N, long long *lo, int *cnt) {
    const int m = N / 2, mp = 1 << (SUBLOG - 1);
    if (it.kind == 0) {
        lo[0] = m - mp;
        cnt[0] = mp;
        lo[1] = N - mp;
        cnt[1] = mp + 2;
        return 2;
    }
    const int K = it.kind == 1 ? 1 : 2;
    for (int k = 0; k < K; ++k) {
        const LeafTask tk = tasks[it.k0 + k];
        lo[k] = tk.sg > 0 ? tk.c : tk.c - (tk.L - 1);
        cnt[k] = tk.L;
    }
    return K;
}

// Leaf item: K leaves of 2^A cells from W0 runs -> their spectra along the runs.
// KC: the caller's K when it is a compile-time fact (2: the pair gather may apply), else 0
// FX: the plan folds x on load (no fold pass): only then do leaves with j >= 0 occur
template <int A, typename T, int NT, int NW, int KC = 0, bool FX = true>
QFT_DEV void leaf_item(const LeafTask *tks, int K, vec2<T> *S, const T *U, const T *kcu, vec2<T> *wb, int tid,
                       const vec2<T> *xb, int N, const CUtensorMap *tmap = nullptr, long long wrow = 0,
                       uint64_t *bar = nullptr, uint32_t *phase = nullptr) {
    constexpr int L = 1 << A;
    const int warp = tid >> 5, lane = tid & 31;
    // fp64 with a tensor map: the runs arrive by TMA in memory order (a reversed
    // run's element e at position L-1-e, handled by the TF loads)
    const bool use_tma = tmap != nullptr;
    if (use_tma) {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            uint32_t bytes = 0;
            for (int k = 0; k < K; ++k)
                if (tks[k].j < 0) bytes += (uint32_t)(L / 32 / kTmaRows) * kTmaBoxBytes;
            if (bytes) {
                tma_expect(bar, bytes);
                for (int k = 0; k < K; ++k) {
                    const LeafTask tk = tks[k];
                    if (tk.j >= 0) continue;
                    const int lo = tk.sg > 0 ? tk.c : tk.c - (L - 1);
                    tma_cells(reinterpret_cast<vec2<double> *>(S + padx(k * L)), tmap, wrow + lo / 32, L, bar);
                }
            }
        }
        bool any = false;
        for (int k = 0; k < K; ++k) any |= tks[k].j < 0;
        if (any) {
            mbar_wait(bar, *phase);
            *phase ^= 1u;
        }
    }
    // load: async cell copies along the (forward or reversed) runs; with NT a
    // multiple of 32 dividing L, thread tid's cells are tid + k NT and their padded
    // addresses advance by NT + NT/32: pointer increments only
    constexpr bool LIN = (L % NT) == 0 && (NT % 32) == 0;
    for (int k = 0; k < K && !use_tma; ++k) {
        const LeafTask tk = tks[k];
        if (tk.j >= 0) continue;  // whole Lee block j: TF reads (and folds) x directly
        vec2<T> *s = S + padx(k * L);
        const vec2<T> *src = wb + tk.c;
        if constexpr (LIN) {
            vec2<T> *d = s + padx(tid);
            const vec2<T> *q = src + tk.sg * tid;
            const long long step = (long long)tk.sg * NT;
#pragma unroll 8
            for (int r = 0; r < L / NT; ++r, d += NT + NT / 32, q += step) cp_async_cell<T>(d, q);
        } else {
            for (int e = tid; e < L; e += NT) cp_async_cell<T>(s + padx(e), src + tk.sg * e);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // TF: top fold levels, held across one barrier, stored sub-block-major
    constexpr int G = LeafTop<A, false, T>::G, IT = (2 * 1024 + NT - 1) / NT;
    {
        vec2<T> v[IT][G];
        // two fold-on-load leaves of one block (its cosine and its sine side): thread tid
        // holds reflection group t of the first leaf in round r and of the second in
        // round r + IT/2 -- one gather of x feeds both (QFT_LEAF_PAIR_GATHER)
        constexpr bool HALVES = (IT % 2 == 0) && (NT * (IT / 2) == 1024);
        constexpr bool PAIR_OK = QFT_LEAF_PAIR_GATHER && HALVES && KC == 2 && FX;
        const bool pair = PAIR_OK && K == 2 && tks[0].j >= 0 && tks[1].j == tks[0].j && tks[0].dst != tks[1].dst;
        if constexpr (PAIR_OK) if (pair) {
            constexpr int H2 = HALVES ? IT / 2 : 0;  // rounds [0, H2): first leaf, [H2, IT): second leaf
            if (!tks[0].dst) {
#pragma unroll
                for (int r = 0; r < H2; ++r) tf_load_x_pair<A, T>(xb, N, tks[0].j, U, tid + r * NT, v[r], v[H2 + r]);
            } else {
#pragma unroll
                for (int r = 0; r < H2; ++r) tf_load_x_pair<A, T>(xb, N, tks[0].j, U, tid + r * NT, v[H2 + r], v[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < IT; ++r) {
            const int it = tid + r * NT;
            if (!pair && it < K * 1024) {
                const int k = it >> 10, t = it & 1023;
                const vec2<T> *s = S + padx(k * L);
                const int j = tks[k].j;
                if (FX && j >= 0) {
                    if (tks[k].dst) LeafTop<A, true, T>::tf_load_x(xb, N, j, U, t, v[r]);
                    else LeafTop<A, false, T>::tf_load_x(xb, N, j, U, t, v[r]);
                } else {
                    const bool rev = use_tma && tks[k].sg < 0;
                    if (tks[k].dst) LeafTop<A, true, T>::tf_load(s, U, t, v[r], rev);
                    else LeafTop<A, false, T>::tf_load(s, U, t, v[r], rev);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < IT; ++r) {
            const int it = tid + r * NT;
            if (it < K * 1024) {
                const int k = it >> 10, t = it & 1023;
                LeafTop<A, false, T>::tf_store(S + padx(k * L), t, v[r]);
            }
        }
    }
    __syncthreads();
    // 1024-cell warp units on the sub-blocks
    constexpr int NSUB = L / 1024;
    for (int u = warp; u < K * NSUB; u += NW) {
        const int k = u / NSUB, p = u - k * NSUB;
        vec2<T> *ws = S + padx(k * L + 1024 * p);
        if (tks[k].dst) unit_big<1024, 5, T, true>(ws, U, kcu, lane);
        else unit_big<1024, 5, T, false>(ws, U, kcu, lane);
        __syncwarp();
    }
    __syncthreads();
    // TB: every column's outputs held in registers across one barrier, then the
    // natural block spectrum in place, then coalesced stores along the runs
    {
        vec2<T> out[IT][G];
#pragma unroll
        for (int r = 0; r < IT; ++r) {
            const int it = tid + r * NT;
            if (it < K * 1024) {
                const int k = it >> 10, i = it & 1023;
                const vec2<T> *s = S + padx(k * L);
                if (tks[k].dst) LeafTop<A, true, T>::tb(s, i, out[r]);
                else LeafTop<A, false, T>::tb(s, i, out[r]);
            }
        }
        __syncthreads();
        // QFT_LEAF_TMA_STORE: the spectrum is written in W0 memory order (a reversed
        // run's slot e at L-1-e) and leaves by tensor-map TMA stores of the padded rows
        const bool mo = QFT_LEAF_TMA_STORE && use_tma;
#pragma unroll
        for (int r = 0; r < IT; ++r) {
            const int it = tid + r * NT;
            if (it < K * 1024) {
                const int k = it >> 10, i = it & 1023;
                if (QFT_TB_ROT && sizeof(T) == 8 && (G == 8 || G == 4)) {
                    // fp64: column i's G cells are 16-byte lanes of one 128-byte row segment;
                    // stored slot q-th by every lane they hit the same bank group 4 ways
                    // (ncu: 4x the ideal wavefronts).  Lane i starts its G stores at slot
                    // rot instead, rot chosen so the 8 lanes of a quarter-warp hit 8
                    // distinct bank groups (checked exhaustively for every column / layout),
                    // the register array rotated by a select network to match.
                    const bool rv = mo && tks[k].sg < 0;
                    const int ob = padx(k * L) + (rv ? padx(L - G - i * G) : padx(i * G));
                    const int rot = G == 8 ? ((i - ob) & 7) : (((i >> 1) - ob) & 3);
                    vec2<T> v[G];
#pragma unroll
                    for (int q = 0; q < G; ++q) v[q] = out[r][rv ? G - 1 - q : q];
#pragma unroll
                    for (int bsh = 1; bsh < G; bsh <<= 1) {  // v[q] <- v[(q + rot) mod G]
                        const bool take = rot & bsh;
                        vec2<T> t[G];
#pragma unroll
                        for (int q = 0; q < G; ++q) t[q] = take ? v[(q + bsh) & (G - 1)] : v[q];
#pragma unroll
                        for (int q = 0; q < G; ++q) v[q] = t[q];
                    }
                    vec2<T> *o = S + ob;
#pragma unroll
                    for (int q = 0; q < G; ++q) o[(q + rot) & (G - 1)] = v[q];
                } else if (mo && tks[k].sg < 0) {
                    vec2<T> *o = S + padx(k * L) + padx(L - G - i * G);  // slots i*G+q at L-1-(i*G+q)
#pragma unroll
                    for (int q = 0; q < G; ++q) o[G - 1 - q] = out[r][q];
                } else {
                    vec2<T> *o = S + padx(k * L) + padx(i * G);  // G <= 32 slots inside one 32-cell row
#pragma unroll
                    for (int q = 0; q < G; ++q) o[q] = out[r][q];
                }
            }
        }
    }
    __syncthreads();
    if (QFT_LEAF_TMA_STORE && use_tma) {
        // one thread: the generic-proxy writes of S (published by the barrier) before
        // the async-proxy reads, the row boxes to W0 (the 2 pad doubles of every
        // 66-double box row fall outside the tensor and are not written), then wait
        // until the stores have read S -- the caller's barrier follows
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int k = 0; k < K; ++k) {
                const LeafTask tk = tks[k];
                const int lo = tk.sg > 0 ? tk.c : tk.c - (L - 1);
                tma_cells_store(reinterpret_cast<const vec2<double> *>(S + padx(k * L)), tmap, wrow + lo / 32, L);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        return;
    }
    for (int k = 0; k < K; ++k) {
        const LeafTask tk = tks[k];
        const vec2<T> *s = S + padx(k * L);
        vec2<T> *dst = wb + tk.c;
        if constexpr (LIN) {
            const vec2<T> *d = s + padx(tid);
            vec2<T> *q = dst + tk.sg * tid;
            const long long step = (long long)tk.sg * NT;
#pragma unroll 8
            for (int r = 0; r < L / NT; ++r, d += NT + NT / 32, q += step) *q = *d;
        } else {
#pragma unroll 8
            for (int e = tid; e < L; e += NT) dst[tk.sg * e] = s[padx(e)];
        }
    }
}

template <int SUBLOG, typename T>
QFT_DEV void sub_item(const vec2<T> *w0b, int m, vec2<T> *W, const T *U, const T *kcu, vec2<T> *cbuf, vec2<T> *sbuf,
                      int tid, const vec2<T> *xb, const CUtensorMap *tmap = nullptr, long long wrow = 0,
                      uint64_t *bar = nullptr, uint32_t *phase = nullptr) {
    using P = SPlan<SUBLOG>;
    using C = ItemCfg<SUBLOG, T>;
    constexpr int NT = C::NT, NW = C::NW;
    const int warp = tid >> 5, lane = tid & 31;
    if (xb) {
        // no fold pass: the sub-signal s[k] = x[k 2^J0] folded and routed while
        // loading -- the big signal's fold x[n] +- x[N-n] at n = k 2^J0 is the
        // sub-signal's fold s[k] +- s[N'-k] (shared.py:28-35, a0_item)
        const int J0 = __ffs(m) - SUBLOG;  // m = 2^(n-1), m' = 2^(SUBLOG-1)
#pragma unroll 8
        for (int r = 0; r < (P::m + NT - 1) / NT; ++r) {
            const int k = tid + r * NT;
            if (k < P::m) {
                const vec2<T> a = xb[k << J0], b = xb[k ? 2 * m - (k << J0) : m];
                if (k == 0) {
                    W[padx(P::BASE)] = a;      // s(0) = x[0]
                    W[padx(P::BASE + 1)] = b;  // s(m') = x[m]
                } else {
                    const int jj = ctz32((uint32_t)k);
                    const int cell = P::m - (1 << (SUBLOG - 1 - jj)) + (k >> (jj + 1));
                    W[padx(cell)] = vadd(a, b);
                    W[padx(P::S0 + cell)] = sine_cell(a, b, cell);
                }
            }
        }
    } else if (tmap) {
        // fp64: the cosine cells [m - m', m) and the sine cells [N - m', N) (whose
        // last cell is the base s(0)) by TMA into the padded sub-signal layout
        constexpr int MP = P::m;
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_expect(bar, 2u * (uint32_t)(MP / 32 / kTmaRows) * kTmaBoxBytes);
            tma_cells(reinterpret_cast<vec2<double> *>(W), tmap, wrow + (m - MP) / 32, MP, bar);
            tma_cells(reinterpret_cast<vec2<double> *>(W + padx(P::S0)), tmap, wrow + (2 * m - MP) / 32, MP, bar);
        }
        if (tid == 32) W[padx(P::BASE + 1)] = w0b[2 * m];  // s(m')
        mbar_wait(bar, *phase);
        *phase ^= 1u;
    } else {
        // the folded blocks j >= J0 are contiguous in W0: cosine cells [m - m', m-1),
        // sine cells [N - m', N-1), base pair N-1, N  ->  the sub-signal's layout
        constexpr int MP = P::m;
        const vec2<T> *wc = w0b + (m - MP), *ws = w0b + (2 * m - MP);
        if constexpr (MP % NT == 0 && NT % 32 == 0) {
            // cells tid + r NT (the last cosine / sine cell MP-1 is unused or the base)
            vec2<T> *dc = W + padx(tid), *dsn = W + padx(P::S0 + tid);
#pragma unroll 8
            for (int r = 0; r < MP / NT; ++r, dc += NT + NT / 32, dsn += NT + NT / 32) {
                const int c = tid + r * NT;
                if (c < MP - 1) {
                    cp_async_cell<T>(dc, wc + c);
                    cp_async_cell<T>(dsn, ws + c);
                }
            }
        } else {
            for (int c = tid; c < MP - 1; c += NT) {
                cp_async_cell<T>(W + padx(c), wc + c);
                cp_async_cell<T>(W + padx(P::S0 + c), ws + c);
            }
        }
        if (tid < 2) cp_async_cell<T>(W + padx(P::BASE + tid), w0b + 2 * m - 1 + tid);
        cp_async_wait_all();
    }
    __syncthreads();
    if (QFT_SC && !xb) {
        // cells copied from W0 (natural order): the single-pass layout holds the
        // odd sine cells negated (qft_smem.cuh QFT_SC)
        for (int c = 2 * tid + 1; c < P::m - 1; c += 2 * NT) {
            const vec2<T> v = W[padx(P::S0 + c)];
            W[padx(P::S0 + c)] = vec2<T>{-v.x, -v.y};
        }
        __syncthreads();
    }
    if constexpr (P::JH > 0) top_f<SUBLOG, T, 0>(W, U, 1, tid);
    fused_units<SUBLOG, T, 0, 1, NW>(W, U, kcu, 1, warp, lane);
    __syncthreads();
    if constexpr (P::JH > 0) top_b<SUBLOG, T, 0>(W, 1, tid);
    // C_J0[k] = cv, S_J0[k] = sv for k in [0, m'] (S_J0 at 0 and m' unused)
    auto emit = [&](int k, vec2<T> cv, vec2<T> sv) {
        cbuf[k] = cv;
        sbuf[k] = sv;
    };
    for (int t = tid; t < P::DT; t += NT) Chain<SUBLOG, T>::unit_e(W, emit, t);
}

// FX: the instance for plans that fold x on load (fold_x != 0); the other instance
// serves the plans with a fold pass -- each drops the other's paths (the pair gather
// of the fold-on-load leaves cost the shared instance 800 bytes of spills)
template <int SUBLOG, typename T, bool FX>
__global__ void __launch_bounds__(ItemCfg<SUBLOG, T>::NT, 1)
    lg_item_kernel(vec2<T> *W0, long long Ws, int log2n, const Item *__restrict__ items, int ni,
                   const LeafTask *__restrict__ tasks, long long batch, const T *__restrict__ Ug,
                   const __grid_constant__ LeeConstL<T> kc, const vec2<T> *__restrict__ x, int fold_x_arg,
                   const __grid_constant__ CUtensorMap tmap, int use_tma) {
    constexpr int fold_x = FX ? 1 : 0;
    (void)fold_x_arg;
    using C = ItemCfg<SUBLOG, T>;
    constexpr int NT = C::NT, NW = C::NW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    vec2<T> *S = reinterpret_cast<vec2<T> *>(smem_raw);
    T *U = reinterpret_cast<T *>(smem_raw + C::U_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::BAR_OFF);
    uint32_t phase = 0;
    const CUtensorMap *tm = (sizeof(T) == 8 && use_tma && !fold_x) ? &tmap : nullptr;
    const int tid = threadIdx.x;
    const int N = 1 << log2n;
    const int nu = C::UCELLS < N / 4 ? C::UCELLS : N / 4;
    for (int i = tid; i < nu; i += NT) U[i] = Ug[i];
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();
    for (long long g = blockIdx.x; g < batch * ni; g += gridDim.x) {
        const long long b = g / ni;
        const Item it = items[g - b * ni];
        vec2<T> *wb = W0 + b * Ws;
        // pull the next item's cells into L2 while this one runs
        if (tid == 0 && g + gridDim.x < batch * ni) {
            const long long g2 = g + gridDim.x, b2 = g2 / ni;
            if (fold_x) {
                // the items of a signal gather from all of its input: the CTA that
                // starts the signal's first item pulls the whole signal into L2
                if (g2 == b2 * ni) l2_prefetch(x + b2 * N, (uint32_t)(N * sizeof(vec2<T>)));
            } else {
                long long lo[3];
                int cnt[3];
                const int nr = item_runs<SUBLOG>(items[g2 - b2 * ni], tasks, N, lo, cnt);
                for (int r = 0; r < nr; ++r) l2_prefetch(W0 + b2 * Ws + lo[r], (uint32_t)(cnt[r] * sizeof(vec2<T>)));
            }
        }
        const long long wrow = b * (Ws / 32);  // first tensor-map row of signal b
        if (it.kind == 0) {
            vec2<T> *cbuf = wb + (N + 2);
            sub_item<SUBLOG, T>(wb, N / 2, S, U, kc.u, cbuf, cbuf + SPlan<SUBLOG>::m + 1, tid,
                                fold_x ? x + b * N : nullptr, tm, wrow, bar, &phase);
        } else if (it.kind == 1) {
            leaf_item<SUBLOG, T, NT, NW, 1, FX>(tasks + it.k0, 1, S, U, kc.u, wb, tid, x + b * N, N, tm, wrow, bar,
                                                &phase);
        } else {
            leaf_item<SUBLOG - 1, T, NT, NW, 2, FX>(tasks + it.k0, 2, S, U, kc.u, wb, tid, x + b * N, N, tm, wrow, bar,
                                             &phase);
        }
        __syncthreads();
    }
    // the leaves' tensor stores (QFT_LEAF_TMA_STORE) complete before the kernel ends
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename T, int LOG2N, int RC>
__global__ void lg_chain_kernel(const vec2<T> *W0, const vec2<T> *W1, const vec2<T> *__restrict__ x,
                                vec2<T> *__restrict__ y, uint32_t cmask, uint32_t smask, long long batch, long long Ws,
                                int J0, int mj0) {
    constexpr int N = 1 << LOG2N;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > (N >> (RC + 1))) return;
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        GChain<T> g;
        g.n = LOG2N;
        g.N = N;
        g.m = N / 2;
        g.w0 = W0 + b * Ws;
        g.w1 = W1 + b * Ws;
        g.x = x + (long long)b * N;
        g.cmask = cmask;
        g.smask = smask;
        g.J0 = J0;
        g.cb = g.w0 + (N + 2);
        g.sb = g.cb + mj0 + 1;
        g.template unit<RC>(y + b * N, t);
    }
}

template <typename T, int LOG2N, int RC, int MODE>
__global__ void lg_chain_real_kernel(const vec2<T> *W0, const vec2<T> *W1, void *y, uint32_t cmask, uint32_t smask,
                                     long long batch, long long nreal, long long Ws, int J0, int mj0) {
    constexpr int N = 1 << LOG2N, m = N / 2;
    constexpr long long OL = MODE == 3 ? m - 1 : m + 1;  // output row length (complex for rdft)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > (N >> (RC + 1))) return;
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        GChain<T> g;
        g.n = LOG2N;
        g.N = N;
        g.m = m;
        g.w0 = W0 + b * Ws;
        g.w1 = W1 + b * Ws;
        g.x = nullptr;
        g.cmask = cmask;
        g.smask = smask;
        g.J0 = J0;
        g.cb = g.w0 + (N + 2);
        g.sb = g.cb + mj0 + 1;
        const long long ra = 2 * b;
        const bool has_b = ra + 1 < nreal;
        if constexpr (MODE == 1) {
            vec2<T> *yy = static_cast<vec2<T> *>(y);
            g.template unit_real<RC, MODE>(yy + ra * OL, yy + (ra + 1) * OL, has_b, t);
        } else {
            T *yy = static_cast<T *>(y);
            g.template unit_real<RC, MODE>(yy + ra * OL, yy + (ra + 1) * OL, has_b, t);
        }
    }
}

// ------------------------------------------------------------------ host
template <typename K, typename... A>
static cudaError_t launch(K k, dim3 g, dim3 bl, size_t smem, cudaStream_t st, A... a) {
    k<<<g, bl, smem, st>>>(a...);
    return cudaGetLastError();
}

static unsigned ybatch(long long batch) { return (unsigned)std::min<long long>(batch, 65535); }

// Tensor map of W0 (fp64) as rows of 32 cells: dims {64 doubles, rows}, box
// {kTmaBoxCols, kTmaRows} (the 2 columns past each row are out of bounds and
// zero-filled: the padded shared layout).  cuTensorMapEncodeTiled comes from the
// driver through the runtime's entry-point query (no -lcuda).  Returns 0 when
// TMA is unavailable (the item kernel then uses per-thread async copies).
static int tma_map_w0(CUtensorMap *map, void *w0, long long cells) {
#if QFT_LARGE_PREC == 64
#ifdef QFT_NO_TMA
    (void)map; (void)w0; (void)cells;
    return 0;
#else
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return 0;
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[2] = {64, (cuuint64_t)(cells / 32)};
    const cuuint64_t strides[1] = {64 * sizeof(double)};
    const cuuint32_t box[2] = {kTmaBoxCols, kTmaRows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, w0, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 1 : 0;
#endif
#else
    (void)map; (void)w0; (void)cells;
    return 0;
#endif
}

extern "C++" {

int QFT_LG(qft_large_create)(int log2n, int real_modes, void **out) {
    auto *p = new QFT_LG(LargePlan)(log2n, real_modes != 0);
    const Sched &S = p->s;
    int rc = 0;
    p->fset.resize(S.f.size());
    p->bset.resize(S.b.size());
    for (size_t d = 0; d < S.f.size(); ++d) {
        // staged tasks (lg_f_staged_kernel): fp64 first-touch cosine tasks and their sine
        // partner (same R, block j and length), stored as adjacent pairs
        auto partner = [&](int R, const FTask &f) -> const FTask * {
            if (!(QFT_F_STAGED && QFT_LARGE_PREC == 64 && f.j >= 0)) return nullptr;
            for (auto &q : S.f[d].at(R))
                if (q.second == 1 && q.first.j == f.j && q.first.L == f.L) return &q.first;
            return nullptr;
        };
        auto staged_task = [&](int R, const FTask &f, int side) {
            if (side == 0) return partner(R, f) != nullptr;
            for (auto &q : S.f[d].at(R))
                if (q.second == 0 && q.first.j == f.j && q.first.L == f.L && partner(R, q.first)) return true;
            return false;
        };
        for (int staged = 0; staged < 2; ++staged) {
            TaskSet ts;
            ts.staged = staged;
            std::vector<FTask> tk;
            std::vector<int> ds, rs;
            std::vector<Chunk> ch;
            for (auto &kv : S.f[d])
                for (size_t i = 0; i < kv.second.size(); ++i) {
                    const FTask &f = kv.second[i].first;
                    const int side = kv.second[i].second;
                    const bool st = staged_task(kv.first, f, side);
                    if (st != (staged == 1)) continue;
                    if (st && side == 1) continue;  // pushed with its cosine partner
                    const int id = (int)tk.size();
                    tk.push_back(f);
                    ds.push_back(side);
                    rs.push_back(kv.first);
                    if (st) {
                        tk.push_back(*partner(kv.first, f));
                        ds.push_back(1);
                        rs.push_back(kv.first);
                    }
                    const int groups = f.L >> kv.first;
                    // fp64 R = 5: two threads per reflection group
                    const int step = st ? stg_groups(kv.first)
                                        : ((QFT_LARGE_PREC == 64 && kv.first == 5) ? kChunk / 2 : kChunk);
                    for (int t0 = 0; t0 < groups; t0 += step) ch.push_back({id, t0});
                }
            if (tk.empty()) continue;
            ts.ntasks = (int)tk.size();
            ts.nchunks = (int)ch.size();
            rc |= upload(tk, &ts.d_tasks) | upload(ds, &ts.d_dsts) | upload(rs, &ts.d_rs) | upload(ch, &ts.d_chunks);
            p->fset[d].push_back(ts);
        }
        for (auto &kv : S.b[d]) {
            TaskSet ts;
            ts.R = kv.first;
            std::vector<Chunk> ch;
            const int step = (QFT_LARGE_PREC == 64 && kv.first == 5) ? kBChunk / 2 : kBChunk;
            for (size_t i = 0; i < kv.second.size(); ++i) {
                const int cols = kv.second[i].L >> kv.first;
                for (int t0 = 0; t0 < cols; t0 += step) ch.push_back({(int)i, t0});
            }
            ts.ntasks = (int)kv.second.size();
            ts.nchunks = (int)ch.size();
            rc |= upload(kv.second, &ts.d_tasks) | upload(ch, &ts.d_chunks);
            p->bset[d].push_back(ts);
        }
    }
    // work items per signal: the sub-signal, every 2^sublog leaf, pairs of 2^(sublog-1) leaves
    {
        std::vector<Item> items{{0, 0}};
        std::vector<LeafTask> leaves;
        for (auto &kv : S.leaf) {
            if (kv.first != p->sublog && kv.first != p->sublog - 1) return -1;  // schedule invariant
            const bool pair = kv.first == p->sublog - 1;
            if (pair && kv.second.size() % 2) return -1;
            for (size_t i = 0; i < kv.second.size(); i += pair ? 2 : 1) {
                items.push_back({pair ? 2 : 1, (int)leaves.size()});
                leaves.push_back(kv.second[i]);
                if (pair) leaves.push_back(kv.second[i + 1]);
            }
        }
        p->nitems = (int)items.size();
        rc |= upload(items, &p->d_items) | upload(leaves, &p->d_leaves);
    }
    p->launches = S.fold ? 3 : 2;
    for (auto &v : p->fset) p->launches += (int)v.size();
    for (auto &v : p->bset) p->launches += (int)v.size();
    *out = p;
    return rc ? -1 : 0;
}

void QFT_LG(qft_large_destroy)(void *pp) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    if (!p) return;
    for (auto *sets : {&p->fset, &p->bset})
        for (auto &v : *sets)
            for (auto &t : v) {
                cudaFree(t.d_tasks);
                cudaFree(t.d_dsts);
                cudaFree(t.d_chunks);
                cudaFree(t.d_rs);
            }
    cudaFree(p->d_items);
    cudaFree(p->d_leaves);
    delete p;
}

void QFT_LG(qft_large_info)(void *pp, int *passes, int *launches) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    *passes = p->s.passes();
    *launches = p->launches;
}

long long QFT_LG(qft_large_scratch_cells)(void *pp) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    // per signal and buffer: N+2 cells + C_J0 / S_J0 of the sub-signal, rounded
    // up to whole 32-cell rows (the TMA tile view of W0)
    const long long c = (long long)p->s.N + 2 + 2 * ((1ll << (p->sublog - 1)) + 1);
    return (c + 31) / 32 * 32;
}

int QFT_LG(qft_large_exec)(void *pp, int mode, const void *d_in, void *d_out, long long batch, long long nreal,
                           const void *d_U, const void *uhead, void *scratch, cudaStream_t st) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    using T = Real;
    const Sched &S = p->s;
    const long long Ws = QFT_LG(qft_large_scratch_cells)(pp);
    vec2<T> *W0 = (vec2<T> *)scratch, *W1 = W0 + batch * Ws;
    const vec2<T> *x = (const vec2<T> *)d_in;
    vec2<T> *y = (vec2<T> *)d_out;
    const T *U = (const T *)d_U;
    LeeConstL<T> kc;
    memcpy(kc.u, uhead, sizeof(kc.u));
    const unsigned yb = ybatch(batch);
    cudaError_t e;
    // fold pass (real modes; complex plans fold on first touch)
    if (mode != 0 && !S.fold) return (int)cudaErrorInvalidValue;
    if (S.fold) {
        if (mode == 0) {
            const long long work = batch * (((S.m >> S.jfold) + kFoldN - 1) / kFoldN);
            const unsigned grid = (unsigned)std::min<long long>(work, 1 << 20);
            e = launch(lg_fold_kernel<T>, dim3(grid), dim3(kFoldT), 0, st, x, W0, S.n, S.jfold, batch, Ws);
        } else {
            if (S.jfold != 0) return (int)cudaErrorInvalidValue;  // real modes need the full fold pass
            const long long work = batch * ((S.m + 1 + kFoldN - 1) / kFoldN);
            const unsigned grid = (unsigned)std::min<long long>(work, 1 << 20);
            const T *xr = (const T *)d_in;
            switch (mode) {
                case 1: e = launch(lg_fold_real_kernel<T, 1>, dim3(grid), dim3(kFoldT), 0, st, xr, W0, S.n, batch, nreal, Ws); break;
                case 2: e = launch(lg_fold_real_kernel<T, 2>, dim3(grid), dim3(kFoldT), 0, st, xr, W0, S.n, batch, nreal, Ws); break;
                case 3: e = launch(lg_fold_real_kernel<T, 3>, dim3(grid), dim3(kFoldT), 0, st, xr, W0, S.n, batch, nreal, Ws); break;
                default: return (int)cudaErrorInvalidValue;
            }
        }
        if (e) return (int)e;
    }
    // forward passes: one launch per depth
    for (auto &v : p->fset)
        for (auto &ts : v) {
            const long long work = (long long)ts.nchunks * batch;
            const unsigned grid = (unsigned)std::min<long long>(work, 1 << 20);
            if (ts.staged) {
                const int smem = 32 * stg_groups(5) * 2 * (int)sizeof(vec2<T>);  // the largest stage (R = 5, 4)
                e = cudaFuncSetAttribute(lg_f_staged_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (!e)
                    e = launch(lg_f_staged_kernel<T>, dim3(grid), dim3(kStgT), (size_t)smem, st, W0,
                               (const FTask *)ts.d_tasks, (const int *)ts.d_rs, (const Chunk *)ts.d_chunks,
                               ts.nchunks, U, batch, Ws, x, S.N);
            } else {
                e = launch(lg_f_kernel<T>, dim3(grid), dim3(kChunk), 0, st, W0, (const FTask *)ts.d_tasks,
                           (const int *)ts.d_dsts, (const int *)ts.d_rs, (const Chunk *)ts.d_chunks, ts.nchunks, U,
                           batch, Ws, x, S.N);
            }
            if (e) return (int)e;
        }
    // sub-signal + leaves (one persistent launch)
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const long long work = batch * p->nitems;
        const unsigned grid = (unsigned)std::min<long long>(work, sms);
        const Item *it = (const Item *)p->d_items;
        const LeafTask *lv = (const LeafTask *)p->d_leaves;
        CUtensorMap tmap;
        memset(&tmap, 0, sizeof(tmap));
        const int use_tma = QFT_LARGE_PREC == 64 && S.fold && tma_map_w0(&tmap, W0, batch * Ws);
        auto run = [&](auto kern, int nt, int smem) -> cudaError_t {
            cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e2) return e2;
            return launch(kern, dim3(grid), dim3(nt), (size_t)smem, st, W0, Ws, S.n, it, p->nitems, lv, batch, U, kc, x,
                          (int)!S.fold, tmap, use_tma);
        };
        switch (p->sublog) {
#if QFT_LARGE_PREC == 32 || QFT_FOLD64
#define QFT_IT(SL)                                                                                       \
    case SL:                                                                                             \
        e = S.fold ? run(lg_item_kernel<SL, T, false>, ItemCfg<SL, T>::NT, ItemCfg<SL, T>::SMEM)         \
                   : run(lg_item_kernel<SL, T, true>, ItemCfg<SL, T>::NT, ItemCfg<SL, T>::SMEM);         \
        break;
#else
#define QFT_IT(SL) \
    case SL: e = run(lg_item_kernel<SL, T, false>, ItemCfg<SL, T>::NT, ItemCfg<SL, T>::SMEM); break;
#endif
            QFT_IT(12) QFT_IT(13)
#if QFT_LARGE_PREC == 32
            QFT_IT(14)
#endif
#undef QFT_IT
            default: return (int)cudaErrorInvalidValue;
        }
        if (e) return (int)e;
    }
    // backward passes, deepest first (outputs staged in shared memory: G*128 cells)
    auto bsm = [](int R) { const int c = kBChunk << R; return (size_t)(c + c / 32 + 1) * sizeof(vec2<T>); };
    for (int d = (int)p->bset.size() - 1; d >= 0; --d)
        for (auto &ts : p->bset[d]) {
            dim3 g(ts.nchunks, yb);
            const BTask *tk = (const BTask *)ts.d_tasks;
            const Chunk *ch = (const Chunk *)ts.d_chunks;
            switch (ts.R) {
                case 1: e = launch(lg_b_kernel<1, T>, g, dim3(kBChunk), bsm(1), st, W0, W1, tk, ch, batch, Ws); break;
                case 2: e = launch(lg_b_kernel<2, T>, g, dim3(kBChunk), bsm(2), st, W0, W1, tk, ch, batch, Ws); break;
                case 3: e = launch(lg_b_kernel<3, T>, g, dim3(kBChunk), bsm(3), st, W0, W1, tk, ch, batch, Ws); break;
                case 4: e = launch(lg_b_kernel<4, T>, g, dim3(kBChunk), bsm(4), st, W0, W1, tk, ch, batch, Ws); break;
#if QFT_LARGE_PREC == 64
                case 5: e = launch(lg_b_pair_kernel<T>, g, dim3(kBChunk), bsm(4), st, W0, W1, tk, ch, batch, Ws); break;
#endif
#if QFT_LARGE_PREC == 32
                case 5: e = launch(lg_b_kernel<5, T>, g, dim3(kBChunk), bsm(5), st, W0, W1, tk, ch, batch, Ws); break;
#endif
                default: return (int)cudaErrorInvalidValue;
            }
            if (e) return (int)e;
        }
    // chain levels J0-1 .. 0 + recombination
    const int RC = p->J0 < kRC ? p->J0 : kRC;
    const int threads = (S.N >> (RC + 1)) + 1;
    const dim3 cg((threads + 127) / 128, yb), cb(128);
    const vec2<T> *w0 = W0, *w1 = W1;
    const int mj0 = 1 << (p->sublog - 1);
#define QFT_CH(LG, R)                                                                                           \
    case LG * 8 + R:                                                                                            \
        switch (mode) {                                                                                         \
            case 0: e = launch(lg_chain_kernel<T, LG, R>, cg, cb, 0, st, w0, w1, x, y, S.cmask, S.smask, batch,  \
                               Ws, p->J0, mj0); break;                                                          \
            case 1: e = launch(lg_chain_real_kernel<T, LG, R, 1>, cg, cb, 0, st, w0, w1, d_out, S.cmask, S.smask, \
                               batch, nreal, Ws, p->J0, mj0); break;                                            \
            case 2: e = launch(lg_chain_real_kernel<T, LG, R, 2>, cg, cb, 0, st, w0, w1, d_out, S.cmask, S.smask, \
                               batch, nreal, Ws, p->J0, mj0); break;                                            \
            case 3: e = launch(lg_chain_real_kernel<T, LG, R, 3>, cg, cb, 0, st, w0, w1, d_out, S.cmask, S.smask, \
                               batch, nreal, Ws, p->J0, mj0); break;                                            \
        }                                                                                                       \
        break;
#define QFT_CHR(LG) QFT_CH(LG, 1) QFT_CH(LG, 2) QFT_CH(LG, 3) QFT_CH(LG, 4)
    switch (S.n * 8 + RC) {
        QFT_CHR(13) QFT_CHR(14) QFT_CHR(15) QFT_CHR(16) QFT_CHR(17) QFT_CHR(18) QFT_CHR(19) QFT_CHR(20)
        default: return (int)cudaErrorInvalidValue;
    }
#undef QFT_CHR
#undef QFT_CH
    return (int)e;
}

}  // extern "C++"
