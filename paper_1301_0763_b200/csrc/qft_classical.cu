// qft_classical.cu -- the classical QFT (classical.py:64-167) on the GPU, the
// north star's "classical QFT for comparison" entry point.
//
// The classical recursion splits harmonic parity first and grows storage by one
// cell at every odd-cosine conversion (dc_t1t, tree.py:92-102), so it does not
// fit the in-place Lee-block layout of the improved kernels.  It runs as a
// warp-cooperative recursion: one warp per signal (or per pair of real rows),
// every node's elementwise loop spread over the 32 lanes, __syncwarp between
// dependent steps, temporaries in a per-warp arena in global memory (L1/L2
// resident).  Same arithmetic contract as everywhere: one IEEE rounding per
// op in the reference's operand order, no FMA (explicit .rn intrinsics).
#include <cuda_runtime.h>

#include <cstdlib>

#include "qft_classical_lv.cuh"
#include "qft_common.cuh"

#if !defined(QFT_CL_PREC)
#error "compile with -DQFT_CL_PREC=32|64"
#endif
#if QFT_CL_PREC == 32
using Real = float;
#define QFT_CL(name) name##_f32
#else
using Real = double;
#define QFT_CL(name) name##_f64
#endif

using namespace qft;
using V = vec2<Real>;

namespace {

struct Ctx {
    V *arena;        // this warp's scratch
    size_t used;
    const Real *T;   // natural table of the top periodization NT: T[n * NT / N] = 1/(2cos(2 pi n/N))
    int NT;
    int lane;
};

__device__ __forceinline__ V *alloc(Ctx &c, int n) {
    V *p = c.arena + c.used;
    c.used += (size_t)((n + 1) & ~1);
    return p;
}
__device__ __forceinline__ Real hsec(const Ctx &c, int n, int N) { return c.T[(long long)n * (c.NT / N)]; }

__device__ void cl_dct(Ctx &c, const V *x, int N, V *out);
__device__ void cl_dct_odd(Ctx &c, const V *x, int N, V *out);
__device__ void cl_dst(Ctx &c, const V *x, int N, V *out);
__device__ void cl_dst_odd(Ctx &c, const V *x, int N, V *out);

// classical._dct (classical.py:64-74): harmonic split of dc_tt (elaborations.py:96-101)
__device__ __noinline__ void cl_dct(Ctx &c, const V *x, int N, V *out) {
    const int L = c.lane;
    if (N == 2) {
        if (L == 0) {
            out[0] = vadd(x[0], x[1]);
            out[1] = vsub(x[0], x[1]);
        }
        __syncwarp();
        return;
    }
    const size_t mark = c.used;
    const int q = N / 4, m = N / 2;
    V *even = alloc(c, q + 1), *odd = alloc(c, q);
    for (int i = L; i < q; i += 32) {
        const V a = x[i], b = x[m - i];
        even[i] = vadd(a, b);
        odd[i] = vsub(a, b);
    }
    if (L == 0) even[q] = x[q];
    __syncwarp();
    V *se = alloc(c, q + 1), *so = alloc(c, q);
    cl_dct(c, even, N / 2, se);
    cl_dct_odd(c, odd, N, so);
    for (int i = L; i <= q; i += 32) out[2 * i] = se[i];
    for (int i = L; i < q; i += 32) out[2 * i + 1] = so[i];
    __syncwarp();
    c.used = mark;
}

// classical._dct_odd (classical.py:77-99): half-secant conversion, dc_t1t split
__device__ __noinline__ void cl_dct_odd(Ctx &c, const V *x, int N, V *out) {
    const int L = c.lane;
    if (N == 4) {
        if (L == 0) out[0] = x[0];
        __syncwarp();
        return;
    }
    if (N == 8) {
        if (L == 0) {
            const V t = vmul(x[1], hsec(c, 1, 8));
            out[0] = vadd(x[0], t);
            out[1] = vsub(x[0], t);
        }
        __syncwarp();
        return;
    }
    const size_t mark = c.used;
    const int q = N / 4;
    V *conv = alloc(c, q);
    if (L == 0) conv[0] = vmul(x[0], (Real)0.5);  // table.half (counting.py:109)
    for (int n = 1 + L; n < q; n += 32) conv[n] = vmul(x[n], hsec(c, n, N));
    __syncwarp();
    const int q2 = N / 8, m2 = N / 4;
    V *even = alloc(c, q2 + 1), *odd = alloc(c, q2);
    if (L == 0) {
        even[0] = vadd(conv[0], V{(Real)0, (Real)0});  // the explicit zero pair (elaborations.py:107-108)
        odd[0] = vsub(conv[0], V{(Real)0, (Real)0});
        even[q2] = conv[q2];
    }
    for (int i = 1 + L; i < q2; i += 32) {
        const V a = conv[i], b = conv[m2 - i];
        even[i] = vadd(a, b);
        odd[i] = vsub(a, b);
    }
    __syncwarp();
    V *se = alloc(c, q2 + 1), *so = alloc(c, q2);
    cl_dct(c, even, N / 4, se);
    cl_dct_odd(c, odd, N / 2, so);
    V *half = alloc(c, m2 + 1);
    for (int i = L; i <= q2; i += 32) half[2 * i] = se[i];
    for (int i = L; i < q2; i += 32) half[2 * i + 1] = so[i];
    __syncwarp();
    for (int i = L; i < q; i += 32) out[i] = vadd(half[i], half[i + 1]);
    __syncwarp();
    c.used = mark;
}

// classical._dst (classical.py:102-109): harmonic split of ds_tt (elaborations.py:117-122)
__device__ __noinline__ void cl_dst(Ctx &c, const V *x, int N, V *out) {
    const int L = c.lane;
    if (N == 4) {
        if (L == 0) out[0] = x[0];
        __syncwarp();
        return;
    }
    const size_t mark = c.used;
    const int q = N / 4, m = N / 2;
    V *even = alloc(c, q - 1), *odd = alloc(c, q);
    for (int i = L; i < q - 1; i += 32) {
        const V a = x[i], b = x[m - 2 - i];
        even[i] = vsub(a, b);
        odd[i] = vadd(a, b);
    }
    if (L == 0) odd[q - 1] = x[q - 1];
    __syncwarp();
    V *se = alloc(c, q - 1), *so = alloc(c, q);
    cl_dst(c, even, N / 2, se);
    cl_dst_odd(c, odd, N, so);
    for (int i = L; i < q - 1; i += 32) out[2 * i + 1] = se[i];
    for (int i = L; i < q; i += 32) out[2 * i] = so[i];
    __syncwarp();
    c.used = mark;
}

// classical._dst_odd (classical.py:112-129): centre peel, conversion, partial sums
__device__ __noinline__ void cl_dst_odd(Ctx &c, const V *x, int N, V *out) {
    const int L = c.lane;
    const int q = N / 4;
    if (N == 4) {
        if (L == 0) out[0] = x[0];
        __syncwarp();
        return;
    }
    const size_t mark = c.used;
    const V center = x[q - 1];
    V *conv = alloc(c, q - 1), *spec = alloc(c, q - 1);
    for (int n = 1 + L; n < q; n += 32) conv[n - 1] = vmul(x[n - 1], hsec(c, n, N));
    __syncwarp();
    cl_dst(c, conv, N / 2, spec);
    V *partial = alloc(c, q);
    if (L == 0) {
        partial[0] = spec[0];
        partial[q - 1] = spec[q - 2];
    }
    for (int i = 1 + L; i < q - 1; i += 32) partial[i] = vadd(spec[i - 1], spec[i]);
    __syncwarp();
    for (int i = L; i < q; i += 32) out[i] = (i & 1) ? vsub(partial[i], center) : vadd(partial[i], center);
    __syncwarp();
    c.used = mark;
}

// shared.rdft_packed (shared.py:21-43) on a vec2 stream, returning C[0..m], S[1..m-1]
__device__ void cl_real(Ctx &c, const V *x, int N, V *C, V *S) {
    const int L = c.lane, m = N / 2;
    V *dc = alloc(c, m + 1), *ds = alloc(c, m - 1);
    if (L == 0) {
        dc[0] = x[0];
        dc[m] = x[m];
    }
    for (int n = 1 + L; n < m; n += 32) {
        const V h = x[n], t = x[N - n];
        dc[n] = vadd(h, t);
        ds[n - 1] = vsub(h, t);
    }
    __syncwarp();
    cl_dct(c, dc, N, C);
    cl_dst(c, ds, N, S);
}

// mode 0: complex rows; 1/2/3: rdft / dct0 / dst0 on real row pairs
template <int MODE>
__global__ void __launch_bounds__(128) classical_kernel(const void *in, void *out, long long units, long long nreal,
                                                        int N, const Real *T, V *arena, size_t arena_cells) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    Ctx c{arena + warp * arena_cells, 0, T, N, lane};
    const int m = N / 2;
    for (long long u = warp; u < units; u += nwarps) {
        c.used = 0;
        if constexpr (MODE == 0) {
            const V *x = (const V *)in + u * N;
            V *y = (V *)out + u * N;
            if (N == 2) {
                if (lane == 0) {
                    y[0] = vadd(x[0], x[1]);
                    y[1] = vsub(x[0], x[1]);
                }
                __syncwarp();
                continue;
            }
            V *C = alloc(c, m + 1), *S = alloc(c, m - 1);
            cl_real(c, x, N, C, S);
            // shared.cdft_interleaved recombination (shared.py:58-72)
            for (int k = lane; k <= m; k += 32) {
                if (k == 0 || k == m) {
                    y[k] = C[k];
                } else {
                    const V cv = C[k], sv = S[k - 1], uu = {sv.y, -sv.x};
                    y[k] = vadd(cv, uu);
                    y[N - k] = vsub(cv, uu);
                }
            }
            __syncwarp();
        } else {
            const int RL = MODE == 1 ? N : (MODE == 2 ? m + 1 : m - 1);
            const Real *xr = (const Real *)in;
            const long long ra = 2 * u, rb = ra + 1 < nreal ? ra + 1 : ra;
            const bool has_b = ra + 1 < nreal;
            V *x = alloc(c, RL);
            for (int i = lane; i < RL; i += 32) x[i] = V{xr[ra * RL + i], xr[rb * RL + i]};
            __syncwarp();
            if constexpr (MODE == 1) {
                V *ya = (V *)out + ra * (m + 1);
                if (N == 2) {
                    if (lane == 0) {
                        const V s = vadd(x[0], x[1]), d = vsub(x[0], x[1]);
                        ya[0] = {s.x, (Real)0};
                        ya[1] = {d.x, (Real)0};
                        if (has_b) {
                            ya[2] = {s.y, (Real)0};
                            ya[3] = {d.y, (Real)0};
                        }
                    }
                } else {
                    V *C = alloc(c, m + 1), *S = alloc(c, m - 1);
                    cl_real(c, x, N, C, S);
                    for (int k = lane; k <= m; k += 32) {
                        const bool edge = (k == 0) || (k == m);
                        const V sv = edge ? V{(Real)0, (Real)0} : S[k - 1];
                        ya[k] = {C[k].x, edge ? (Real)0 : -sv.x};
                        if (has_b) ya[m + 1 + k] = {C[k].y, edge ? (Real)0 : -sv.y};
                    }
                }
            } else if constexpr (MODE == 2) {
                V *C = alloc(c, m + 1);
                cl_dct(c, x, N, C);
                Real *ya = (Real *)out + ra * (m + 1);
                for (int k = lane; k <= m; k += 32) {
                    ya[k] = C[k].x;
                    if (has_b) ya[m + 1 + k] = C[k].y;
                }
            } else {
                V *S = alloc(c, m - 1);
                cl_dst(c, x, N, S);
                Real *ya = (Real *)out + ra * (m - 1);
                for (int k = lane; k < m - 1; k += 32) {
                    ya[k] = S[k].x;
                    if (has_b) ya[m - 1 + k] = S[k].y;
                }
            }
            __syncwarp();
        }
    }
}

// high-water mark of the arena (cells), replaying the allocation pattern
long long hwm_dct(int N);
long long hwm_dct_odd(int N);
long long hwm_dst(int N);
long long hwm_dst_odd(int N);
long long r2(long long n) { return (n + 1) & ~1LL; }
long long hwm_dct(int N) {
    if (N == 2) return 0;
    const int q = N / 4;
    const long long base = r2(q + 1) + r2(q) + r2(q + 1) + r2(q);
    const long long a = hwm_dct(N / 2), b = hwm_dct_odd(N);
    return base + (a > b ? a : b);
}
long long hwm_dct_odd(int N) {
    if (N <= 8) return 0;
    const int q = N / 4, q2 = N / 8, m2 = N / 4;
    const long long base = r2(q) + r2(q2 + 1) + r2(q2) + r2(q2 + 1) + r2(q2);
    const long long a = hwm_dct(N / 4), b = hwm_dct_odd(N / 2);
    const long long rec = a > b ? a : b;
    const long long tail = r2(m2 + 1);
    return base + (rec > tail ? rec : tail);
}
long long hwm_dst(int N) {
    if (N == 4) return 0;
    const int q = N / 4;
    const long long base = r2(q - 1) + r2(q) + r2(q - 1) + r2(q);
    const long long a = hwm_dst(N / 2), b = hwm_dst_odd(N);
    return base + (a > b ? a : b);
}
long long hwm_dst_odd(int N) {
    if (N == 4) return 0;
    const int q = N / 4;
    const long long base = r2(q - 1) + r2(q - 1);
    const long long a = hwm_dst(N / 2), tail = r2(q);
    return base + (a > tail ? a : tail);
}

}  // namespace

// cells of arena per warp for periodization N (upper bound incl. the mode's buffers)
long long QFT_CL(qft_classical_arena_cells)(int N) {
    if (N < 4) return 16;
    const int m = N / 2;
    const long long real = r2(m + 1) + r2(m - 1) + hwm_dct(N) + hwm_dst(N) + 2 * r2(m + 1);
    return real + r2(N) + 64;
}

int QFT_CL(qft_classical_exec)(int mode, const void *in, void *out, long long units, long long nreal, int N,
                               const void *T, void *arena, size_t arena_cells, int warps, cudaStream_t st) {
    const int blocks = (warps + 3) / 4;
    V *ar = (V *)arena;
    const Real *t = (const Real *)T;
    switch (mode) {
        case 0: classical_kernel<0><<<blocks, 128, 0, st>>>(in, out, units, nreal, N, t, ar, arena_cells); break;
        case 1: classical_kernel<1><<<blocks, 128, 0, st>>>(in, out, units, nreal, N, t, ar, arena_cells); break;
        case 2: classical_kernel<2><<<blocks, 128, 0, st>>>(in, out, units, nreal, N, t, ar, arena_cells); break;
        case 3: classical_kernel<3><<<blocks, 128, 0, st>>>(in, out, units, nreal, N, t, ar, arena_cells); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

// ===========================================================================
// Level-synchronous classical QFT (qft_classical_lv.cuh): N >= 32.
//   whole-signal kernel   the tree of one signal (or pair of real rows) in two
//                         shared-memory buffers; one CTA per signal, persistent
//   large N               the top d0 levels as global passes over W0/W1, the
//                         sub-trees of periodization 2^sublog in shared memory
//                         (in place in the global buffer), the d0 backward
//                         levels as global passes
// ===========================================================================
namespace {

constexpr int kLvMaxSmem = 227 * 1024;

QFT_HD int lv_smem_bytes(int lognn) { return 2 * cl::buf_cells(lognn) * (int)sizeof(V); }

// the opaque (-0, -0) addend of the packed fp32 multiplies, once per kernel
__device__ __forceinline__ void lv_load_mz(cl::Mul<float> &m) { m.z = __ldg(&::qft_mzero_pair); }
__device__ __forceinline__ void lv_load_mz(cl::Mul<double> &) {}

// shared memory of the whole-signal kernel (one signal per iteration): two buffers + the natural table
QFT_HD int lv_tree_smem_bytes(int lognn) { return lv_smem_bytes(lognn) + (1 << (lognn - 2)) * (int)sizeof(Real); }

// forward levels, register-level bases and backward levels of nt trees (signal s in the
// buffer pair at P + s * 2 * buf): the items of all trees flat over the CTA's threads
// (ONE: nt == 1, the tree index drops out of the item loops)
template <bool ONE>
__device__ __forceinline__ void lv_run_trees(const cl::Tree<Real> &t, V *P, int buf, int nt_arg, int tid, int NT) {
    const int nt = ONE ? 1 : nt_arg;
    const int D = t.depth(), coff = cl::cen_off(t.lognn);
    const int lf = t.lognn - 2, lb = D + 1;  // log2 of the level / base items per tree
    for (int d = 0; d < D; ++d) {
        for (int it = tid; it < (nt << lf); it += NT) {
            V *P0 = ONE ? P : P + (it >> lf) * 2 * buf, *P1 = P0 + buf;
            t.fwd_item((d & 1) ? P1 : P0, (d & 1) ? P0 : P1, P0 + coff, d, it & ((1 << lf) - 1));
        }
        __syncthreads();
    }
    for (int it = tid; it < (nt << lb); it += NT) {
        V *P0 = ONE ? P : P + (it >> lb) * 2 * buf;
        t.base_item((D & 1) ? P0 + buf : P0, it & ((1 << lb) - 1));
    }
    __syncthreads();
    for (int d = D - 1; d >= 0; --d) {
        for (int it = tid; it < (nt << lf); it += NT) {
            V *P0 = ONE ? P : P + (it >> lf) * 2 * buf, *P1 = P0 + buf;
            t.bwd_item(((d + 1) & 1) ? P1 : P0, (d & 1) ? P1 : P0, P0 + coff, d, it & ((1 << lf) - 1));
        }
        __syncthreads();
    }
}

// MINB: resident CTAs per SM the register budget is set for (1: 512 threads, else 256)
template <int MODE, int MINB>
__global__ void __launch_bounds__(MINB == 1 ? 512 : 256, MINB)
    cl_tree_kernel(const void *in, void *out, long long units, long long nreal, int log2n, int tt,
                   const Real *__restrict__ Tt) {
    // tt signals (or pairs of real rows) per CTA iteration: small trees have few items
    // per level, so several share the CTA's threads
    extern __shared__ __align__(16) unsigned char cl_smem[];
    const int buf = cl::buf_cells(log2n);
    V *P = reinterpret_cast<V *>(cl_smem);
    Real *Ts = reinterpret_cast<Real *>(P + 2 * buf * tt);  // the natural table, N/4 entries
    cl::Tree<Real> t{log2n, log2n, cl::cos_cells(log2n), false, MODE != 3, MODE != 2, Ts};
    lv_load_mz(t.mul);
    const int N = 1 << log2n, m = N / 2, lm = log2n - 1, tid = threadIdx.x, NT = blockDim.x;
    for (int i = tid; i < N / 4; i += NT) Ts[i] = Tt[i];  // published by the first barrier below
    for (long long u0 = (long long)blockIdx.x * tt; u0 < units; u0 += (long long)gridDim.x * tt) {
        const int nt = (int)(units - u0 < tt ? units - u0 : tt);
        for (int it = tid; it < (nt << lm); it += NT)
            cl::ingest_item<MODE, Real>(in, u0 + (it >> lm), nreal, N, P + (it >> lm) * 2 * buf, t.CB, it & (m - 1));
        __syncthreads();
        if (tt == 1) lv_run_trees<true>(t, P, buf, 1, tid, NT);
        else lv_run_trees<false>(t, P, buf, nt, tid, NT);
        for (int it = tid; it < nt * (m + 1); it += NT) {
            const int sidx = it / (m + 1), k = it - sidx * (m + 1);
            cl::emit_item<MODE, Real>(out, u0 + sidx, nreal, N, P + sidx * 2 * buf, t.CB, k);
        }
        __syncthreads();
    }
}

template <int MODE, int MINB>
cudaError_t lv_launch_tree(const void *in, void *out, long long units, long long nreal, int log2n, const Real *Tt,
                           int tt, int smem, int num_sms, cudaStream_t st) {
    auto kern = cl_tree_kernel<MODE, MINB>;
    constexpr int NT = MINB == 1 ? 512 : 256;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;  // what the registers and the shared memory really allow
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const long long ctas = (long long)num_sms * per_sm;
    // small batches: fewer signals per CTA iteration so that every SM gets work
    if (units < ctas * tt) tt = (int)((units + ctas - 1) / ctas);
    if (tt < 1) tt = 1;
    long long grid = (units + tt - 1) / tt;
    if (grid > ctas) grid = ctas;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, NT, smem, st>>>(in, out, units, nreal, log2n, tt, Tt);
    return cudaGetLastError();
}

// large N: fold (ingest) of every signal into the roots of W0
template <int MODE>
__global__ void __launch_bounds__(256) cl_gingest_kernel(const void *in, V *W0, long long Ws, long long units,
                                                         long long nreal, int log2n) {
    const int N = 1 << log2n, m = N / 2, CB = cl::cos_cells(log2n);
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= m) return;
    for (long long u = blockIdx.y; u < units; u += gridDim.y)
        cl::ingest_item<MODE, Real>(in, u, nreal, N, W0 + u * Ws, CB, n);
}
template <int MODE>
__global__ void __launch_bounds__(256) cl_gemit_kernel(void *out, const V *W0, long long Ws, long long units,
                                                       long long nreal, int log2n) {
    const int N = 1 << log2n, m = N / 2, CB = cl::cos_cells(log2n);
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > m) return;
    for (long long u = blockIdx.y; u < units; u += gridDim.y)
        cl::emit_item<MODE, Real>(out, u, nreal, N, W0 + u * Ws, CB, k);
}
// one global forward (BWD = false: src = level d, dst = level d+1) or backward
// (BWD = true: src = level d+1 spectra, dst = level d) level of every signal
template <bool BWD>
__global__ void __launch_bounds__(256) cl_glevel_kernel(const V *src, V *dst, V *W0, long long Ws, long long units, int log2n,
                                                        int d, bool do_cos, bool do_sin,
                                                        const Real *__restrict__ Tt) {
    cl::Tree<Real> t{log2n, log2n, cl::cos_cells(log2n), false, do_cos, do_sin, Tt};
    lv_load_mz(t.mul);
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= (BWD ? t.bwd_items() : t.fwd_items())) return;
    for (long long u = blockIdx.y; u < units; u += gridDim.y) {
        V *cen = W0 + u * Ws + cl::cen_off(log2n);  // the centres live in buffer 0
        if (BWD) t.bwd_item(src + u * Ws, dst + u * Ws, cen, d, it);
        else t.fwd_item(src + u * Ws, dst + u * Ws, cen, d, it);
    }
}
// the sub-trees rooted at depth d0 (periodization 2^(log2n - d0)), in place in Wd
__global__ void __launch_bounds__(256, 3) cl_subtree_kernel(V *Wd, long long Ws, long long units, int log2n, int d0,
                                                         bool do_cos, bool do_sin, const Real *__restrict__ Tt) {
    extern __shared__ __align__(16) unsigned char cl_smem[];
    const int sublog = log2n - d0, S0 = 1 << (sublog - 1), CBtop = cl::cos_cells(log2n);
    V *P0 = reinterpret_cast<V *>(cl_smem);
    const int tid = threadIdx.x, NT = blockDim.x;
    for (long long g = blockIdx.x; g < (units << d0); g += gridDim.x) {
        const long long u = g >> d0;
        const int b = (int)(g & ((1LL << d0) - 1));
        cl::Tree<Real> t{sublog, log2n, cl::cos_cells(sublog), (b & 1) != 0, do_cos, do_sin, Tt};
        lv_load_mz(t.mul);
        V *wc = Wd + u * Ws + cl::cos_off(S0, b), *ws = Wd + u * Ws + CBtop + (long long)b * cl::sin_stride_of(log2n, d0);
        const int nc = S0 + ((b & 1) ? 0 : 1);
        if (do_cos)
            for (int i = tid; i < nc; i += NT) P0[i] = wc[i];
        if (do_sin)
            for (int i = tid; i < S0 - 1; i += NT) P0[t.CB + i] = ws[i];
        __syncthreads();
        lv_run_trees<true>(t, P0, cl::buf_cells(sublog), 1, tid, NT);
        if (do_cos)
            for (int i = tid; i < nc; i += NT) wc[i] = P0[i];
        if (do_sin)
            for (int i = tid; i < S0 - 1; i += NT) ws[i] = P0[t.CB + i];
        __syncthreads();
    }
}

template <int MODE>
cudaError_t lv_launch_mode(const void *in, void *out, long long units, long long nreal, int log2n, const Real *Tt,
                           V *arena, size_t arena_bytes, int num_sms, cudaStream_t st) {
    if (lv_tree_smem_bytes(log2n) <= kLvMaxSmem) {
        static const int minb_env = [] {  // QFT_CL_MINB=1|2|3: force the register budget (A/B)
            const char *v = getenv("QFT_CL_MINB");
            return v ? atoi(v) : 0;
        }();
        // signals per CTA iteration: enough trees that the register-level bases
        // (N/16 per tree) cover the CTA's 256 threads, within a third of the shared memory
        const int pair = lv_smem_bytes(log2n), tab = (1 << (log2n - 2)) * (int)sizeof(Real);
        int tt = 256 / (1 << (log2n - 4));
        if (tt < 1) tt = 1;
        while (tt > 1 && tt * pair + tab > 72 * 1024) tt >>= 1;
        const int smem = tt * pair + tab;
        const int fit = kLvMaxSmem / (smem + 1024);
        int minb = fit >= 3 ? 3 : (fit >= 2 ? 2 : 1);
        if (minb_env >= 1 && minb_env <= 3 && minb_env <= (fit > 1 ? fit : 1)) minb = minb_env;
        switch (minb) {
            case 1: return lv_launch_tree<MODE, 1>(in, out, units, nreal, log2n, Tt, tt, smem, num_sms, st);
            case 2: return lv_launch_tree<MODE, 2>(in, out, units, nreal, log2n, Tt, tt, smem, num_sms, st);
            default: return lv_launch_tree<MODE, 3>(in, out, units, nreal, log2n, Tt, tt, smem, num_sms, st);
        }
    }
    // large N: global levels down to sub-trees of 2^sublog
    const int sublog = sizeof(Real) == 4 ? 12 : 11, d0 = log2n - sublog;
    const long long Ws = cl::buf_cells(log2n);
    const int N = 1 << log2n, m = N / 2;
    const bool do_cos = MODE != 3, do_sin = MODE != 2;
    long long chunk = (long long)(arena_bytes / (2 * (size_t)Ws * sizeof(V)));
    if (chunk < 1) return cudaErrorMemoryAllocation;
    const int ssm = lv_smem_bytes(sublog);
    cudaError_t e = cudaFuncSetAttribute(cl_subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
    if (e != cudaSuccess) return e;
    const size_t in_row = MODE == 0 ? (size_t)N * sizeof(V) : 2 * (size_t)(MODE == 1 ? N : (MODE == 2 ? m + 1 : m - 1)) * sizeof(Real);
    const size_t out_row = MODE == 0 ? (size_t)N * sizeof(V) : (MODE == 1 ? 2 * (size_t)(m + 1) * sizeof(V) : 2 * (size_t)(MODE == 2 ? m + 1 : m - 1) * sizeof(Real));
    for (long long u0 = 0; u0 < units; u0 += chunk) {
        const long long nu = units - u0 < chunk ? units - u0 : chunk;
        V *W[2] = {arena, arena + nu * Ws};
        const unsigned gy = (unsigned)(nu < 65535 ? nu : 65535);
        const char *cin = (const char *)in + (size_t)u0 * in_row;
        char *cout = (char *)out + (size_t)u0 * out_row;
        const long long nr = nreal - 2 * u0;  // real rows left (real modes)
        cl_gingest_kernel<MODE><<<dim3((m + 255) / 256, gy), 256, 0, st>>>(cin, W[0], Ws, nu, nr, log2n);
        for (int d = 0; d < d0; ++d)
            cl_glevel_kernel<false><<<dim3(((N / 4) + 255) / 256, gy), 256, 0, st>>>(W[d & 1], W[(d + 1) & 1], W[0], Ws, nu,
                                                                                   log2n, d, do_cos, do_sin, Tt);
        {
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cl_subtree_kernel, 256, ssm);
            if (e != cudaSuccess) return e;
            long long grid = (long long)num_sms * (per_sm > 0 ? per_sm : 1);
            if (grid > (nu << d0)) grid = nu << d0;
            cl_subtree_kernel<<<(unsigned)grid, 256, ssm, st>>>(W[d0 & 1], Ws, nu, log2n, d0, do_cos, do_sin, Tt);
        }
        for (int d = d0 - 1; d >= 0; --d)
            cl_glevel_kernel<true><<<dim3(((N / 4) + 255) / 256, gy), 256, 0, st>>>(W[(d + 1) & 1], W[d & 1], W[0], Ws, nu,
                                                                                  log2n, d, do_cos, do_sin, Tt);
        cl_gemit_kernel<MODE><<<dim3((m + 1 + 255) / 256, gy), 256, 0, st>>>(cout, W[0], Ws, nu, nr, log2n);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

// bytes of global scratch the level-synchronous path wants for `units` signals
// (0: the whole tree fits shared memory); any amount >= one signal's works (chunked)
long long QFT_CL(qft_classical_lv_arena_bytes)(int log2n, long long units) {
    if (log2n < cl::kBaseLog || lv_tree_smem_bytes(log2n) <= kLvMaxSmem) return 0;
    const long long per = 2 * (long long)cl::buf_cells(log2n) * (long long)sizeof(V);
    // QFT_CL_ARENA_MB: scratch budget (tests use a small one to exercise the chunking)
    long long budget = 4LL << 30;
    if (const char *v = getenv("QFT_CL_ARENA_MB")) {
        const long long mb = atoll(v);
        if (mb > 0) budget = mb << 20;
    }
    const long long cap = budget / per > 0 ? budget / per : 1;
    return per * (units < cap ? units : cap);
}

// mode 0: complex rows; 1/2/3: rdft / dct0 / dst0 on real row pairs.  N >= 32.
int QFT_CL(qft_classical_lv_exec)(int mode, const void *in, void *out, long long units, long long nreal, int log2n,
                                  const void *T, void *arena, size_t arena_bytes, int num_sms, cudaStream_t st) {
    if (log2n < cl::kBaseLog) return (int)cudaErrorInvalidValue;
    const Real *t = (const Real *)T;
    V *ar = (V *)arena;
    cudaError_t e;
    switch (mode) {
        case 0: e = lv_launch_mode<0>(in, out, units, nreal, log2n, t, ar, arena_bytes, num_sms, st); break;
        case 1: e = lv_launch_mode<1>(in, out, units, nreal, log2n, t, ar, arena_bytes, num_sms, st); break;
        case 2: e = lv_launch_mode<2>(in, out, units, nreal, log2n, t, ar, arena_bytes, num_sms, st); break;
        case 3: e = lv_launch_mode<3>(in, out, units, nreal, log2n, t, ar, arena_bytes, num_sms, st); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)e;
}
