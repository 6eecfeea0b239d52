// qft_large.cu -- plan builder and launchers of the multi-pass path (qft_large.cuh).
// Compiled once per precision (-DQFT_LARGE_PREC=32|64).
//
// The plan builder replays the improved recursion at the level of Lee blocks
// (improved.py:49-112: fold, secant-scale the odd child, recurse, neighbour
// sums) and cuts every block larger than the leaf size into passes of at most
// RG fold levels, tracking where each sub-block's cells are (runs) and in which
// scratch buffer each spectrum ends up.  This is the "fixed kernel schedule"
// compiled from the decomposition tree (SURVEY.md §2 plan builder).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "qft_large_api.h"
#include "qft_large_plan.h"

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

constexpr int kLeafLog = QFT_LARGE_PREC == 32 ? 10 : 9;  // warp leaf: L <= 1024 (fp32) / 512 (fp64)
constexpr int kRG = QFT_LARGE_PREC == 32 ? 5 : 4;         // fold levels per F/B pass
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
    void *d_tasks = nullptr, *d_dsts = nullptr, *d_chunks = nullptr, *d_rs = nullptr;
    int ntasks = 0, nchunks = 0;
};

using Sched = LargeSchedule<kLeafLog, kRG>;

}  // namespace

struct QFT_LG(LargePlan) {
    Sched s;
    std::vector<std::vector<TaskSet>> fset, bset;
    std::vector<TaskSet> lset;
    int launches = 0;
    explicit QFT_LG(LargePlan)(int log2n) : s(log2n) {}
};

template <typename TT>
static int upload(const std::vector<TT> &v, void **d) {
    if (v.empty()) return 0;
    if (cudaMalloc(d, v.size() * sizeof(TT)) != cudaSuccess) return -1;
    return cudaMemcpy(*d, v.data(), v.size() * sizeof(TT), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : -1;
}

// ------------------------------------------------------------------ kernels
template <typename T>
__global__ void lg_fold_kernel(const vec2<T> *__restrict__ x, vec2<T> *__restrict__ W0, int N, int log2n,
                               long long batch, long long Ws) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N / 2) return;
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) lg_fold_item<T>(x + b * N, W0 + b * Ws, n, N, log2n);
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

template <int L, typename T>
__global__ void lg_leaf_thread_kernel(vec2<T> *W0, const LeafTask *__restrict__ tasks, int ntasks, long long batch,
                                      long long Ws, const __grid_constant__ LeeConstL<T> kc,
                                      const vec2<T> *__restrict__ x, int N) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ntasks) return;
    const LeafTask tk = tasks[k];
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        if (tk.dst) lg_leaf_thread<L, T, true>(W0 + b * Ws, tk, kc.u, x + b * N, N);
        else lg_leaf_thread<L, T, false>(W0 + b * Ws, tk, kc.u, x + b * N, N);
    }
}

template <int R, typename T>
__global__ void __launch_bounds__(128) lg_leaf_warp_kernel(vec2<T> *W0, const LeafTask *__restrict__ tasks, int ntasks,
                                                           long long batch, long long Ws, const T *__restrict__ U,
                                                           const __grid_constant__ LeeConstL<T> kc,
                                                           const vec2<T> *__restrict__ x, int N) {
    constexpr int L = 32 << R, PADL = L + L / 32 + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    vec2<T> *s = reinterpret_cast<vec2<T> *>(smem_raw) + warp * PADL;
    const int k = blockIdx.x * 4 + warp;
    if (k >= ntasks) return;
    const LeafTask tk = tasks[k];
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        vec2<T> *w = W0 + b * Ws;
        if (tk.j >= 0) {
            const vec2<T> *xb = x + b * N;
#pragma unroll 4
            for (int e = lane; e < L; e += 32)
                s[e + (e >> 5)] = tk.dst ? fold_load<T, true>(xb, N, tk.j, e) : fold_load<T, false>(xb, N, tk.j, e);
        } else {
#pragma unroll 8
            for (int e = lane; e < L; e += 32) s[e + (e >> 5)] = w[tk.c + tk.sg * e];
        }
        __syncwarp();
        if (tk.dst) {
            using WL = WarpLee<R, T, true>;
            typename WL::F f;
            f.load(s, lane, U);
            __syncwarp();
            f.store(s, lane);
            __syncwarp();
            if (lane < (1 << R)) WL::lee32(s, lane, kc.u);
            __syncwarp();
            typename WL::B bb;
            bb.compute(s, lane);
            __syncwarp();
            bb.store(s, lane);
        } else {
            using WL = WarpLee<R, T, false>;
            typename WL::F f;
            f.load(s, lane, U);
            __syncwarp();
            f.store(s, lane);
            __syncwarp();
            if (lane < (1 << R)) WL::lee32(s, lane, kc.u);
            __syncwarp();
            typename WL::B bb;
            bb.compute(s, lane);
            __syncwarp();
            bb.store(s, lane);
        }
        __syncwarp();
        for (int e = lane; e < L; e += 32) w[tk.c + tk.sg * e] = s[e + (e >> 5)];
        __syncwarp();
    }
}

template <typename T, int LOG2N>
__global__ void lg_chain_kernel(const vec2<T> *W0, const vec2<T> *W1, const vec2<T> *__restrict__ x,
                                vec2<T> *__restrict__ y, uint32_t cmask, uint32_t smask, long long batch, long long Ws) {
    constexpr int N = 1 << LOG2N;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > (N >> (kRC + 1))) return;
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
        g.template unit<kRC>(y + b * N, t);
    }
}

// ------------------------------------------------------------------ host
template <typename K, typename... A>
static cudaError_t launch(K k, dim3 g, dim3 bl, size_t smem, cudaStream_t st, A... a) {
    k<<<g, bl, smem, st>>>(a...);
    return cudaGetLastError();
}

static unsigned ybatch(long long batch) { return (unsigned)std::min<long long>(batch, 65535); }

extern "C++" {

int QFT_LG(qft_large_create)(int log2n, void **out) {
    auto *p = new QFT_LG(LargePlan)(log2n);
    const Sched &S = p->s;
    int rc = 0;
    p->fset.resize(S.f.size());
    p->bset.resize(S.b.size());
    for (size_t d = 0; d < S.f.size(); ++d) {
        {
            TaskSet ts;
            std::vector<FTask> tk;
            std::vector<int> ds, rs;
            std::vector<Chunk> ch;
            for (auto &kv : S.f[d])
                for (size_t i = 0; i < kv.second.size(); ++i) {
                    const int id = (int)tk.size();
                    tk.push_back(kv.second[i].first);
                    ds.push_back(kv.second[i].second);
                    rs.push_back(kv.first);
                    const int groups = kv.second[i].first.L >> kv.first;
                    for (int t0 = 0; t0 < groups; t0 += kChunk) ch.push_back({id, t0});
                }
            ts.ntasks = (int)tk.size();
            ts.nchunks = (int)ch.size();
            rc |= upload(tk, &ts.d_tasks) | upload(ds, &ts.d_dsts) | upload(rs, &ts.d_rs) | upload(ch, &ts.d_chunks);
            p->fset[d].push_back(ts);
        }
        for (auto &kv : S.b[d]) {
            TaskSet ts;
            ts.R = kv.first;
            std::vector<Chunk> ch;
            for (size_t i = 0; i < kv.second.size(); ++i) {
                const int cols = kv.second[i].L >> kv.first;
                for (int t0 = 0; t0 < cols; t0 += kBChunk) ch.push_back({(int)i, t0});
            }
            ts.ntasks = (int)kv.second.size();
            ts.nchunks = (int)ch.size();
            rc |= upload(kv.second, &ts.d_tasks) | upload(ch, &ts.d_chunks);
            p->bset[d].push_back(ts);
        }
    }
    for (auto &kv : S.leaf) {
        TaskSet ts;
        ts.R = kv.first;  // log2 L
        ts.ntasks = (int)kv.second.size();
        rc |= upload(kv.second, &ts.d_tasks);
        p->lset.push_back(ts);
    }
    p->launches = 2 + (int)p->lset.size();
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
    for (auto &t : p->lset) cudaFree(t.d_tasks);
    delete p;
}

void QFT_LG(qft_large_info)(void *pp, int *passes, int *launches) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    *passes = p->s.passes();
    *launches = p->launches;
}

long long QFT_LG(qft_large_scratch_cells)(void *pp) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    return (long long)p->s.N + 2;  // per signal and buffer
}

int QFT_LG(qft_large_exec)(void *pp, const void *d_in, void *d_out, long long batch, const void *d_U,
                           const void *uhead, void *scratch, cudaStream_t st) {
    auto *p = (QFT_LG(LargePlan) *)pp;
    using T = Real;
    const Sched &S = p->s;
    const long long Ws = (long long)S.N + 2;
    vec2<T> *W0 = (vec2<T> *)scratch, *W1 = W0 + batch * Ws;
    const vec2<T> *x = (const vec2<T> *)d_in;
    vec2<T> *y = (vec2<T> *)d_out;
    const T *U = (const T *)d_U;
    LeeConstL<T> kc;
    memcpy(kc.u, uhead, sizeof(kc.u));
    const unsigned yb = ybatch(batch);
    cudaError_t e;
    // forward passes: one launch per depth
    for (auto &v : p->fset)
        for (auto &ts : v) {
            const long long work = (long long)ts.nchunks * batch;
            const unsigned grid = (unsigned)std::min<long long>(work, 1 << 20);
            e = launch(lg_f_kernel<T>, dim3(grid), dim3(kChunk), 0, st, W0, (const FTask *)ts.d_tasks,
                       (const int *)ts.d_dsts, (const int *)ts.d_rs, (const Chunk *)ts.d_chunks, ts.nchunks, U, batch,
                       Ws, x, S.N);
            if (e) return (int)e;
        }
    // leaves
    for (auto &ts : p->lset) {
        const LeafTask *tk = (const LeafTask *)ts.d_tasks;
        const int lg = ts.R;
        if (lg <= 5) {
            dim3 g((ts.ntasks + 127) / 128, yb);
            switch (lg) {
                case 0: e = launch(lg_leaf_thread_kernel<1, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
                case 1: e = launch(lg_leaf_thread_kernel<2, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
                case 2: e = launch(lg_leaf_thread_kernel<4, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
                case 3: e = launch(lg_leaf_thread_kernel<8, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
                case 4: e = launch(lg_leaf_thread_kernel<16, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
                case 5: e = launch(lg_leaf_thread_kernel<32, T>, g, dim3(128), 0, st, W0, tk, ts.ntasks, batch, Ws, kc, x, S.N); break;
            }
        } else {
            const int R = lg - 5, L = 32 << R;
            const size_t smem = 4 * (size_t)(L + L / 32 + 1) * sizeof(vec2<T>);
            dim3 g((ts.ntasks + 3) / 4, yb);
            switch (R) {
                case 1: e = launch(lg_leaf_warp_kernel<1, T>, g, dim3(128), smem, st, W0, tk, ts.ntasks, batch, Ws, U, kc, x, S.N); break;
                case 2: e = launch(lg_leaf_warp_kernel<2, T>, g, dim3(128), smem, st, W0, tk, ts.ntasks, batch, Ws, U, kc, x, S.N); break;
                case 3: e = launch(lg_leaf_warp_kernel<3, T>, g, dim3(128), smem, st, W0, tk, ts.ntasks, batch, Ws, U, kc, x, S.N); break;
                case 4: e = launch(lg_leaf_warp_kernel<4, T>, g, dim3(128), smem, st, W0, tk, ts.ntasks, batch, Ws, U, kc, x, S.N); break;
#if QFT_LARGE_PREC == 32
                case 5: e = launch(lg_leaf_warp_kernel<5, T>, g, dim3(128), smem, st, W0, tk, ts.ntasks, batch, Ws, U, kc, x, S.N); break;
#endif
                default: return (int)cudaErrorInvalidValue;
            }
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
#if QFT_LARGE_PREC == 32
                case 5: e = launch(lg_b_kernel<5, T>, g, dim3(kBChunk), bsm(5), st, W0, W1, tk, ch, batch, Ws); break;
#endif
                default: return (int)cudaErrorInvalidValue;
            }
            if (e) return (int)e;
        }
    // chain + recombination
    const int threads = (S.N >> (kRC + 1)) + 1;
    const dim3 cg((threads + 127) / 128, yb), cb(128);
    const vec2<T> *w0 = W0, *w1 = W1;
    switch (S.n) {
#define QFT_CH(LG) case LG: e = launch(lg_chain_kernel<T, LG>, cg, cb, 0, st, w0, w1, x, y, S.cmask, S.smask, batch, Ws); break;
        QFT_CH(13) QFT_CH(14) QFT_CH(15) QFT_CH(16) QFT_CH(17) QFT_CH(18) QFT_CH(19) QFT_CH(20)
#undef QFT_CH
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)e;
}

}  // extern "C++"
