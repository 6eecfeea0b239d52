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
