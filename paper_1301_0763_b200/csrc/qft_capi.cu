// qft_capi.cu -- the C ABI declared in include/qft_b200.h: plans (constant
// tables built with the reference's two-tier recipe), dispatch to the
// per-size transform kernels (qft_inst.cu), layout conversion for the
// reference's (N, batch) layout, the pipelined host path, and the seeded
// device input generator used by the benchmarks.
#include <cuda_runtime.h>
#include <cstdint>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qft_b200.h"
#include "qft_launch.cuh"
#include "qft_large_api.h"

// classical QFT (qft_classical.cu, one translation unit per precision)
long long qft_classical_arena_cells_f32(int N);
long long qft_classical_arena_cells_f64(int N);
long long qft_classical_lv_arena_bytes_f32(int log2n, long long units);
long long qft_classical_lv_arena_bytes_f64(int log2n, long long units);
int qft_classical_lv_exec_f32(int mode, const void *in, void *out, long long units, long long nreal, int log2n,
                              const void *T, void *arena, size_t arena_bytes, int num_sms, cudaStream_t st);
int qft_classical_lv_exec_f64(int mode, const void *in, void *out, long long units, long long nreal, int log2n,
                              const void *T, void *arena, size_t arena_bytes, int num_sms, cudaStream_t st);
int qft_classical_exec_f32(int mode, const void *in, void *out, long long units, long long nreal, int N, const void *T,
                           void *arena, size_t arena_cells, int warps, cudaStream_t st);
int qft_classical_exec_f64(int mode, const void *in, void *out, long long units, long long nreal, int N, const void *T,
                           void *arena, size_t arena_cells, int warps, cudaStream_t st);

using namespace qft;

// ============================================================== errors
static thread_local std::string g_last_error;
static int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}
#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(QFT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// ============================================================== constants
// Two-tier recipe of counting.py:116-140.  float64: cos in x87 long double with
// a 50-digit pi, 1/(2c) in long double, rounded once.  float32: in double,
// rounded once.  Depends only on the reduced fraction m/N (exact here).
static const long double kWidePi = 3.14159265358979323846264338327950288419716939937510L;

static void natural_table_f64(int N, std::vector<double> &T) {
    T.assign(N / 4, 0.0);
    T[0] = (double)cosl(2.0L * kWidePi * (1.0L / 8.0L));
    for (int m = 1; m < N / 4; ++m) {
        long double c = cosl(2.0L * kWidePi * ((long double)m / (long double)N));
        T[m] = (double)(1.0L / (2.0L * c));
    }
}
static void natural_table_f32(int N, std::vector<float> &T) {
    T.assign(N / 4, 0.0f);
    T[0] = (float)cos(2.0 * M_PI * (1.0 / 8.0));
    for (int m = 1; m < N / 4; ++m) {
        double c = cos(2.0 * M_PI * ((double)m / (double)N));
        T[m] = (float)(1.0 / (2.0 * c));
    }
}
// level table U (qft_lee.cuh): U[0] = cos8, U[S/2+i] = T[(2i+1) N/(4S)]
template <typename T>
static void level_table(int N, const std::vector<T> &Tn, std::vector<T> &U) {
    U.assign(N / 4 >= 2 ? N / 4 : 2, (T)0);
    if (N < 8) return;
    U[0] = Tn[0];
    for (int S = 2; S <= N / 4; S *= 2)
        for (int i = 0; i < S / 2; ++i) U[S / 2 + i] = Tn[(size_t)(2 * i + 1) * (N / (4 * S))];
}

// (N, batch) <-> (batch, N) for complex elements: tiled transpose through smem.
// dst[b*N + n] = src[n*B + b]  (to_batch_major)   /   dst[n*B + b] = src[b*N + n]
template <typename T>
__global__ void qft_transpose(const vec2<T> *__restrict__ src, vec2<T> *__restrict__ dst, long long rows,
                              long long cols) {
    // src is rows x cols (row-major), dst is cols x rows
    // grid.x walks the column tiles, grid.y (capped at 65535) strides over the row tiles
    __shared__ vec2<T> tile[32][33];
    const long long c0 = (long long)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (long long r0 = (long long)blockIdx.y * 32; r0 < rows; r0 += (long long)gridDim.y * 32) {
        for (int i = ty; i < 32; i += 8) {
            long long r = r0 + i, c = c0 + tx;
            if (r < rows && c < cols) tile[i][tx] = src[r * cols + c];
        }
        __syncthreads();
        for (int i = ty; i < 32; i += 8) {
            long long c = c0 + i, r = r0 + tx;
            if (r < rows && c < cols) dst[c * rows + r] = tile[tx][i];
        }
        __syncthreads();
    }
}
static dim3 transpose_grid(long long rows, long long cols) {
    const long long gy = (rows + 31) / 32;
    return dim3((unsigned)((cols + 31) / 32), (unsigned)(gy < 65535 ? gy : 65535));
}

// general strided gather / scatter (rare layouts)
template <typename T>
__global__ void qft_strided_copy(const vec2<T> *__restrict__ src, vec2<T> *__restrict__ dst, long long batch,
                                 int N, long long sbs, long long ses, long long dbs, long long des) {
    long long total = batch * N;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        long long b = idx / N, n = idx % N;
        dst[b * dbs + n * des] = src[b * sbs + n * ses];
    }
}

// ---------------------------------------------------------------- input generator
// Counter-based N(0,1) generator of the benchmark inputs, keyed on (seed, global
// transform index, n) so a shard equals the same rows of a 1-GPU run.  Box-Muller
// with ln / sin / cos evaluated by fixed polynomials in explicitly rounded IEEE
// double ops (no library transcendentals, no FMA): the numpy twin
// paper_1301_0763_b200/workloads.py:keyed_normal_rows performs the same op
// sequence and reproduces every value bit for bit on the host.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// 1/(2k+1); (-1)^k/(2k+1)!; (-1)^k/(2k)!  (hex literals shared with the twin)
__constant__ double kGenLn[12] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                                  0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                                  0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                                  0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
__constant__ double kGenSin[12] = {0x1.0000000000000p+0,  -0x1.5555555555555p-3, 0x1.1111111111111p-7,
                                   -0x1.a01a01a01a01ap-13, 0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26,
                                   0x1.6124613a86d09p-33,  -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49,
                                   -0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66, -0x1.761b41316381ap-75};
__constant__ double kGenCos[12] = {0x1.0000000000000p+0,  -0x1.0000000000000p-1, 0x1.5555555555555p-5,
                                   -0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22,
                                   0x1.1eed8eff8d898p-29,  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45,
                                   -0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62, -0x1.0ce396db7f853p-70};
__device__ __forceinline__ double gen_ln(double u) {  // u in (0, 1]
    const unsigned long long b = (unsigned long long)__double_as_longlong(u);
    long long e = (long long)((b >> 52) & 0x7ff) - 1023;
    double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    if (m > 0x1.6a09e667f3bcdp+0) {  // sqrt(2)
        m = __dmul_rn(m, 0.5);
        e += 1;
    }
    const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0)), s2 = __dmul_rn(s, s);
    double p = kGenLn[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), kGenLn[k]);
    return __dadd_rn(__dmul_rn((double)e, 0x1.62e42fefa39efp-1), __dmul_rn(__dmul_rn(s, p), 2.0));
}
__device__ __forceinline__ void gen_sincos2pi(double u, double &sn, double &cs) {  // u in [0, 1)
    const double t = __dmul_rn(u, 4.0), qd = floor(t), f = __dsub_rn(t, qd);
    const double x = __dmul_rn(f, 0x1.921fb54442d18p+0), x2 = __dmul_rn(x, x);  // f * pi/2
    double ps = kGenSin[11], pc = kGenCos[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) {
        ps = __dadd_rn(__dmul_rn(ps, x2), kGenSin[k]);
        pc = __dadd_rn(__dmul_rn(pc, x2), kGenCos[k]);
    }
    const double s = __dmul_rn(ps, x), c = pc;
    const int q = (int)qd;
    sn = q == 0 ? s : (q == 1 ? c : (q == 2 ? -s : -c));
    cs = q == 0 ? c : (q == 1 ? -s : (q == 2 ? -c : s));
}
template <typename T>
__global__ void qft_fill_normal_kernel(vec2<T> *out, long long batch, int N, long long first, uint64_t seed) {
    long long total = batch * N;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        long long b = idx / N, n = idx % N;
        uint64_t key = splitmix64(seed ^ splitmix64((uint64_t)(first + b) * 0x100000001B3ull + (uint64_t)n));
        uint64_t k2 = splitmix64(key);
        const double u1 = __dmul_rn((double)((key >> 11) + 1), 0x1p-53);  // (0, 1]
        const double u2 = __dmul_rn((double)(k2 >> 11), 0x1p-53);         // [0, 1)
        const double r = __dsqrt_rn(__dmul_rn(-2.0, gen_ln(u1)));
        double s, c;
        gen_sincos2pi(u2, s, c);
        if constexpr (sizeof(T) == 4)
            out[idx] = {__double2float_rn(__dmul_rn(r, c)), __double2float_rn(__dmul_rn(r, s))};
        else
            out[idx] = {__dmul_rn(r, c), __dmul_rn(r, s)};
    }
}

// ============================================================== plan
struct qft_plan {
    int log2n = 0, N = 0, prec = 0, algo = 0, device = 0;
    int num_sms = 0;
    void *d_U = nullptr;
    size_t u_bytes = 0;
    double uhead64[32] = {0};  // host copy of U[0..32) (kernel-parameter constants)
    float uhead32[32] = {0};
    std::vector<double> t64;
    std::vector<float> t32;
    // scratch for layout conversion / host path
    void *d_scratch = nullptr;
    size_t scratch_bytes = 0;
    static constexpr int kHostStreams = 3;
    static constexpr int kHostSlots = 4;  // host path: chunks in flight
    cudaStream_t streams[kHostStreams] = {nullptr, nullptr, nullptr};
    void *d_host = nullptr;     // host path device buffers (per slot: in, out, 2x layout scratch)
    size_t host_bytes = 0;
    void *h_pin = nullptr;      // host path pinned staging ring for pageable buffers (per slot: in, out)
    size_t pin_bytes = 0;
    std::mutex mu;
    void *large = nullptr;      // multi-pass schedule
    void *large_real = nullptr; // its real-mode variant (fold pass over every block), built on first use
    bool multipass = false;     // served by the multi-pass schedule
    void *d_T = nullptr;        // natural table T[0..N/4) on the device (classical recursion)
    void *d_arena = nullptr;    // classical: per-warp scratch
    size_t arena_bytes = 0;
    void *d_lscratch = nullptr; // its scratch (two buffers of N+2 cells per signal of a chunk)
    size_t lscratch_bytes = 0;
    // Recorded on the exec stream after the last kernel of every call; the next
    // call's stream waits on it before its first kernel.  Calls on one plan from
    // different streams therefore never overlap on the plan-owned scratch
    // (d_scratch, d_lscratch, d_arena, d_host), and qft_plan_set_table waits on it
    // before it overwrites the constants that earlier kernels may still read.
    cudaEvent_t ev_use = nullptr;
};

// Switch to the plan's device for one ABI call and restore the caller's device
// on every return path.
struct DevGuard {
    int prev = -1;
    bool switched = false;
    cudaError_t err = cudaSuccess;
    explicit DevGuard(int dev) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) {
            err = cudaSetDevice(dev);
            switched = err == cudaSuccess;
        }
    }
    ~DevGuard() {
        if (switched) cudaSetDevice(prev);
    }
};
#define DEV_GUARD(p)                                                                     \
    DevGuard _dg((p)->device);                                                           \
    if (_dg.err != cudaSuccess)                                                          \
        return fail(QFT_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_dg.err))

// stream-order one call on the plan: wait for the previous call before, mark after.
// While the stream is being captured into a CUDA graph the call is recorded as
// plain graph nodes (an event recorded outside the capture cannot be waited on
// inside it): ordering a replayed graph against other streams' calls on the same
// plan is then the caller's, as for any captured work.
static bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}
static int use_begin(qft_plan *p, cudaStream_t st) {
    if (capturing(st)) return 0;
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_use, 0));
    return 0;
}
static int use_end(qft_plan *p, cudaStream_t st) {
    if (capturing(st)) return 0;
    CUDA_TRY(cudaEventRecord(p->ev_use, st));
    return 0;
}

// per-instance launchers, one translation unit each (qft_inst.cu)
#define QFT_DECL(P, L) int qft_inst_launch_##P##_##L(const LaunchArgs *, int); void qft_inst_cfg_##P##_##L(int *);
#define QFT_DECL_ALL(P) \
    QFT_DECL(P, 1) QFT_DECL(P, 2) QFT_DECL(P, 3) QFT_DECL(P, 4) QFT_DECL(P, 5) QFT_DECL(P, 6) QFT_DECL(P, 7) \
    QFT_DECL(P, 8) QFT_DECL(P, 9) QFT_DECL(P, 10) QFT_DECL(P, 11) QFT_DECL(P, 12) QFT_DECL(P, 13) QFT_DECL(P, 14)
QFT_DECL_ALL(32)
QFT_DECL_ALL(64)
typedef int (*launch_fn)(const LaunchArgs *, int);
#define QFT_ROW(P)                                                                                              \
    {nullptr, qft_inst_launch_##P##_1, qft_inst_launch_##P##_2, qft_inst_launch_##P##_3, qft_inst_launch_##P##_4, \
     qft_inst_launch_##P##_5, qft_inst_launch_##P##_6, qft_inst_launch_##P##_7, qft_inst_launch_##P##_8,         \
     qft_inst_launch_##P##_9, qft_inst_launch_##P##_10, qft_inst_launch_##P##_11, qft_inst_launch_##P##_12,     \
     qft_inst_launch_##P##_13, qft_inst_launch_##P##_14}
static const launch_fn kLaunch[2][15] = {QFT_ROW(32), QFT_ROW(64)};
typedef void (*cfg_fn)(int *);
#define QFT_CROW(P)                                                                                   \
    {nullptr, qft_inst_cfg_##P##_1, qft_inst_cfg_##P##_2, qft_inst_cfg_##P##_3, qft_inst_cfg_##P##_4,   \
     qft_inst_cfg_##P##_5, qft_inst_cfg_##P##_6, qft_inst_cfg_##P##_7, qft_inst_cfg_##P##_8,             \
     qft_inst_cfg_##P##_9, qft_inst_cfg_##P##_10, qft_inst_cfg_##P##_11, qft_inst_cfg_##P##_12,         \
     qft_inst_cfg_##P##_13, qft_inst_cfg_##P##_14}
static const cfg_fn kCfg[2][15] = {QFT_CROW(32), QFT_CROW(64)};
static constexpr int kMaxLog2N = 14;  // largest single-pass instance (fp32; fp64 up to 13)

static constexpr int kMaxLargeLog2N = 20;
// single-pass shared-memory kernel built for (log2n, prec)
static bool smem_available(int log2n, int prec) {
    if (log2n < 1 || log2n > kMaxLog2N) return false;
    if (log2n <= 12) return true;
    int cfg[3] = {0, 0, 0};
    kCfg[prec == QFT_PREC_F32 ? 0 : 1][log2n](cfg);
    return cfg[0] > 0;
}
// multi-pass path: N beyond the single-pass kernels, or forced for N >= 2^13
// by QFT_MULTIPASS=1 at plan creation (A/B comparisons and tests)
static bool is_large(const qft_plan *p) { return p->multipass; }

// mode 0: batch complex signals; modes 1-3 (rdft / dct0 / dst0): nreal real rows,
// batch = row pairs (one vec2 signal per pair)
static int launch_large(qft_plan *p, int mode, const void *in, void *out, long long batch, long long nreal,
                        cudaStream_t st) {
    void *lp = p->large;
    if (mode != 0) {  // real modes: a schedule whose fold pass covers every block
        if (!p->large_real) {
            int e = p->prec == QFT_PREC_F32 ? qft_large_create_f32(p->log2n, 1, &p->large_real)
                                            : qft_large_create_f64(p->log2n, 1, &p->large_real);
            if (e) return fail(QFT_ECUDA, "multi-pass schedule upload failed");
        }
        lp = p->large_real;
    }
    // bound the scratch (two buffers per signal) to ~6 GiB: chunk the batch
    const size_t esz = p->prec == QFT_PREC_F32 ? 8 : 16, rsz = esz / 2;
    const long long cells = p->prec == QFT_PREC_F32 ? qft_large_scratch_cells_f32(lp) : qft_large_scratch_cells_f64(lp);
    const size_t per = 2 * (size_t)cells * esz;
    long long chunk = (long long)(((size_t)6 << 30) / per);
#ifdef QFT_LARGE_L2_MB
    // experiment: sub-batches whose scratch stays L2-resident across the passes
    {
        const long long l2c = (long long)(((size_t)QFT_LARGE_L2_MB << 20) / per);
        if (l2c < chunk) chunk = l2c;
    }
#endif
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    if (p->lscratch_bytes < per * (size_t)chunk) {
        if (p->d_lscratch) {  // grown: earlier calls may still use the old buffer
            cudaEventSynchronize(p->ev_use);
            cudaFree(p->d_lscratch);
        }
        p->d_lscratch = nullptr;
        p->lscratch_bytes = 0;
        CUDA_TRY(cudaMalloc(&p->d_lscratch, per * (size_t)chunk));
        p->lscratch_bytes = per * (size_t)chunk;
    }
    const void *uh = p->prec == QFT_PREC_F32 ? (const void *)p->uhead32 : (const void *)p->uhead64;
    const long long m = p->N / 2;
    // bytes per input / output unit (a signal, or a real row)
    const size_t ib = mode == 0 ? (size_t)p->N * esz : (size_t)(mode == 1 ? p->N : (mode == 2 ? m + 1 : m - 1)) * rsz;
    const size_t ob = mode == 0 ? (size_t)p->N * esz : (mode == 1 ? (size_t)(m + 1) * esz : (size_t)(mode == 2 ? m + 1 : m - 1) * rsz);
    for (long long b0 = 0; b0 < batch; b0 += chunk) {
        const long long nb = batch - b0 < chunk ? batch - b0 : chunk;
        const long long u0 = mode == 0 ? b0 : 2 * b0;  // first unit of the chunk
        const long long nr = mode == 0 ? 0 : (nreal - u0 < 2 * nb ? nreal - u0 : 2 * nb);
        const char *ci = (const char *)in + (size_t)u0 * ib;
        char *co = (char *)out + (size_t)u0 * ob;
        int e = p->prec == QFT_PREC_F32
                    ? qft_large_exec_f32(lp, mode, ci, co, nb, nr, p->d_U, uh, p->d_lscratch, st)
                    : qft_large_exec_f64(lp, mode, ci, co, nb, nr, p->d_U, uh, p->d_lscratch, st);
        if (e) return fail(QFT_ECUDA, std::string("multi-pass launch: ") + cudaGetErrorString((cudaError_t)e));
    }
    return 0;
}

static int launch_classical(qft_plan *p, int mode, const void *in, void *out, long long units, long long nreal,
                            cudaStream_t st) {
    const bool f32 = p->prec == QFT_PREC_F32;
    if (p->d_T == nullptr) return fail(QFT_EINVAL, "plan was not created for the classical algorithm");
    static const bool recursive = [] {  // QFT_CLASSICAL_RECURSIVE=1: the warp-recursive kernel at every N (A/B, tests)
        const char *v = getenv("QFT_CLASSICAL_RECURSIVE");
        return v && v[0] == '1';
    }();
    if (p->log2n >= 5 && !recursive) {
        // level-synchronous schedule (qft_classical_lv.cuh): whole tree in shared
        // memory, or global levels + shared-memory sub-trees with W0/W1 in the arena
        const size_t need = (size_t)(f32 ? qft_classical_lv_arena_bytes_f32(p->log2n, units)
                                         : qft_classical_lv_arena_bytes_f64(p->log2n, units));
        if (p->arena_bytes < need) {
            if (p->d_arena) {  // grown: earlier calls may still use the old buffer
                cudaEventSynchronize(p->ev_use);
                cudaFree(p->d_arena);
            }
            p->d_arena = nullptr;
            p->arena_bytes = 0;
            CUDA_TRY(cudaMalloc(&p->d_arena, need));
            p->arena_bytes = need;
        }
        int e = f32 ? qft_classical_lv_exec_f32(mode, in, out, units, nreal, p->log2n, p->d_T, p->d_arena,
                                                need, p->num_sms, st)
                    : qft_classical_lv_exec_f64(mode, in, out, units, nreal, p->log2n, p->d_T, p->d_arena,
                                                need, p->num_sms, st);
        if (e) return fail(QFT_ECUDA, std::string("classical launch: ") + cudaGetErrorString((cudaError_t)e));
        return 0;
    }
    const long long cells = f32 ? qft_classical_arena_cells_f32(p->N) : qft_classical_arena_cells_f64(p->N);
    const size_t vb = f32 ? 8 : 16;
    long long warps = units < (long long)p->num_sms * 16 ? units : (long long)p->num_sms * 16;
    // keep the arena below ~8 GiB
    const long long cap = (long long)(((size_t)8 << 30) / ((size_t)cells * vb));
    if (warps > cap) warps = cap;
    if (warps < 1) warps = 1;
    const size_t need = (size_t)warps * (size_t)cells * vb;
    if (p->arena_bytes < need) {
        if (p->d_arena) {  // grown: earlier calls may still use the old buffer
            cudaEventSynchronize(p->ev_use);
            cudaFree(p->d_arena);
        }
        p->d_arena = nullptr;
        p->arena_bytes = 0;
        CUDA_TRY(cudaMalloc(&p->d_arena, need));
        p->arena_bytes = need;
    }
    // the recursion is ~2 lg N calls deep with ~128-byte frames: raise the
    // per-thread stack once (the default 1 KB overflows from N = 64)
    {
        size_t cur = 0;
        const size_t need = (size_t)(2 * p->log2n + 16) * 192;
        CUDA_TRY(cudaDeviceGetLimit(&cur, cudaLimitStackSize));
        if (cur < need) CUDA_TRY(cudaDeviceSetLimit(cudaLimitStackSize, need));
    }
    int e = f32 ? qft_classical_exec_f32(mode, in, out, units, nreal, p->N, p->d_T, p->d_arena, cells, (int)warps, st)
                : qft_classical_exec_f64(mode, in, out, units, nreal, p->N, p->d_T, p->d_arena, cells, (int)warps, st);
    if (e) return fail(QFT_ECUDA, std::string("classical launch: ") + cudaGetErrorString((cudaError_t)e));
    return 0;
}

static int launch_contig(qft_plan *p, const void *in, void *out, long long batch, cudaStream_t st) {
    if (p->algo == QFT_ALGO_CLASSICAL) return launch_classical(p, 0, in, out, batch, 0, st);
    if (is_large(p)) return launch_large(p, 0, in, out, batch, 0, st);
    if (!smem_available(p->log2n, p->prec))
        return fail(QFT_EUNSUPPORTED, "periodization 2^" + std::to_string(p->log2n) + " not built yet");
    LaunchArgs a{in, out, batch, p->d_U, p->prec == QFT_PREC_F32 ? (const void *)p->uhead32 : (const void *)p->uhead64,
                 p->num_sms, st};
    int e = kLaunch[p->prec == QFT_PREC_F32 ? 0 : 1][p->log2n](&a, 0);
    if (e != 0) return fail(QFT_ECUDA, std::string("kernel launch: ") + cudaGetErrorString((cudaError_t)e));
    return 0;
}

static bool size_supported(int log2n) { return log2n >= 1 && log2n <= kMaxLargeLog2N; }

// Exported functions inherit C linkage from their extern "C" declarations in qft_b200.h.

int qft_version(void) { return 100; }

const char *qft_last_error(void) { return g_last_error.c_str(); }

int qft_plan_create(qft_plan **out, int log2n, int prec, int algo, int device) {
    if (!out) return fail(QFT_EINVAL, "plan pointer is NULL");
    *out = nullptr;
    if (log2n < 1 || log2n > 30) return fail(QFT_EINVAL, "periodization must be a power of two >= 2");
    if (prec != QFT_PREC_F32 && prec != QFT_PREC_F64) return fail(QFT_EINVAL, "prec must be 32 or 64");
    if (algo != QFT_ALGO_IMPROVED && algo != QFT_ALGO_CLASSICAL) return fail(QFT_EINVAL, "unknown algorithm");
    if (!size_supported(log2n))
        return fail(QFT_EUNSUPPORTED, "periodization 2^" + std::to_string(log2n) + " not built yet");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(QFT_EINVAL, "bad device ordinal");
    DevGuard _dg(device);
    if (_dg.err != cudaSuccess) return fail(QFT_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_dg.err));
    qft_plan *p = new qft_plan();
    p->log2n = log2n;
    p->N = 1 << log2n;
    p->prec = prec;
    p->algo = algo;
    p->device = device;
    if (algo == QFT_ALGO_IMPROVED) {
        const char *fm = getenv("QFT_MULTIPASS");
        const bool force = fm && fm[0] == '1' && log2n >= 13;
        p->multipass = force || !smem_available(log2n, prec);
    }
    cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
    int rc = 0;
    if (cudaEventCreateWithFlags(&p->ev_use, cudaEventDisableTiming) != cudaSuccess)
        rc = fail(QFT_ECUDA, "event creation failed");
    if (prec == QFT_PREC_F64) {
        std::vector<double> U;
        if (p->N >= 8) natural_table_f64(p->N, p->t64);
        level_table(p->N, p->t64, U);
        for (size_t i = 0; i < 32 && i < U.size(); ++i) p->uhead64[i] = U[i];
        p->u_bytes = U.size() * sizeof(double);
        if (cudaMalloc(&p->d_U, p->u_bytes) != cudaSuccess ||
            cudaMemcpy(p->d_U, U.data(), p->u_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
            rc = fail(QFT_ECUDA, "table upload failed");
    } else {
        std::vector<float> U;
        if (p->N >= 8) natural_table_f32(p->N, p->t32);
        level_table(p->N, p->t32, U);
        for (size_t i = 0; i < 32 && i < U.size(); ++i) p->uhead32[i] = U[i];
        p->u_bytes = U.size() * sizeof(float);
        if (cudaMalloc(&p->d_U, p->u_bytes) != cudaSuccess ||
            cudaMemcpy(p->d_U, U.data(), p->u_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
            rc = fail(QFT_ECUDA, "table upload failed");
    }
    if (!rc && algo == QFT_ALGO_CLASSICAL) {
        const size_t tb = (size_t)(p->N >= 8 ? p->N / 4 : 1) * (prec == QFT_PREC_F32 ? 4 : 8);
        const void *src = prec == QFT_PREC_F32 ? (const void *)p->t32.data() : (const void *)p->t64.data();
        double zero[1] = {0};
        if (cudaMalloc(&p->d_T, tb) != cudaSuccess ||
            cudaMemcpy(p->d_T, p->N >= 8 ? src : (const void *)zero, p->N >= 8 ? tb : 1, cudaMemcpyHostToDevice) !=
                cudaSuccess)
            rc = fail(QFT_ECUDA, "table upload failed");
    } else if (!rc && is_large(p)) {
        int e = prec == QFT_PREC_F32 ? qft_large_create_f32(log2n, 0, &p->large)
                                     : qft_large_create_f64(log2n, 0, &p->large);
        if (e) rc = fail(QFT_ECUDA, "multi-pass schedule upload failed");
    }
    if (rc) {
        qft_plan_destroy(p);
        return rc;
    }
    *out = p;
    return 0;
}

int qft_plan_destroy(qft_plan *p) {
    if (!p) return 0;
    DevGuard _dg(p->device);
    if (p->ev_use) {
        cudaEventSynchronize(p->ev_use);
        cudaEventDestroy(p->ev_use);
    }
    if (p->d_U) cudaFree(p->d_U);
    if (p->d_scratch) cudaFree(p->d_scratch);
    if (p->d_lscratch) cudaFree(p->d_lscratch);
    if (p->d_T) cudaFree(p->d_T);
    if (p->d_arena) cudaFree(p->d_arena);
    if (p->d_host) cudaFree(p->d_host);
    if (p->h_pin) cudaFreeHost(p->h_pin);
    for (void *lp : {p->large, p->large_real}) {
        if (!lp) continue;
        if (p->prec == QFT_PREC_F32) qft_large_destroy_f32(lp);
        else qft_large_destroy_f64(lp);
    }
    for (auto &s : p->streams)
        if (s) cudaStreamDestroy(s);
    delete p;
    return 0;
}

int qft_plan_get_info(const qft_plan *p, qft_plan_info_t *info) {
    if (!p || !info) return fail(QFT_EINVAL, "NULL argument");
    memset(info, 0, sizeof(*info));
    info->log2n = p->log2n;
    info->prec = p->prec;
    info->algo = p->algo;
    info->passes = 1;
    info->kernel_launches = 1;
    int cfg[3] = {0, 0, 0};
    if (smem_available(p->log2n, p->prec)) kCfg[p->prec == QFT_PREC_F32 ? 0 : 1][p->log2n](cfg);
    if (p->algo == QFT_ALGO_CLASSICAL) {
        info->passes = 0;  // recursion in a per-warp arena (L1/L2 resident), not HBM passes
        info->kernel_launches = 1;
        info->threads_per_cta = 128;
        info->scratch_bytes = (int64_t)p->arena_bytes;
        return 0;
    }
    if (is_large(p)) {
        int passes = 0, launches = 0;
        if (p->prec == QFT_PREC_F32) qft_large_info_f32(p->large, &passes, &launches);
        else qft_large_info_f64(p->large, &passes, &launches);
        info->passes = passes;
        info->kernel_launches = launches;
        info->smem_bytes = 0;
        info->threads_per_cta = 256;
        info->ctas_per_sm = 0;
        info->signals_per_cta = 0;
        info->scratch_bytes = (int64_t)(p->scratch_bytes + p->lscratch_bytes);
        return 0;
    }
    info->smem_bytes = cfg[0];
    info->threads_per_cta = cfg[1];
    info->ctas_per_sm = p->log2n >= 6 ? 1 : 0;
    info->signals_per_cta = cfg[2];
    info->scratch_bytes = (int64_t)p->scratch_bytes;
    return 0;
}

int qft_plan_table(const qft_plan *p, void *h_out) {
    if (!p || !h_out) return fail(QFT_EINVAL, "NULL argument");
    if (p->N < 8) return 0;
    if (p->prec == QFT_PREC_F64) memcpy(h_out, p->t64.data(), p->t64.size() * sizeof(double));
    else memcpy(h_out, p->t32.data(), p->t32.size() * sizeof(float));
    return 0;
}

int qft_plan_set_table(qft_plan *p, const void *h_table) {
    if (!p || !h_table) return fail(QFT_EINVAL, "NULL argument");
    if (p->N < 8) return 0;
    std::lock_guard<std::mutex> lk(p->mu);
    DEV_GUARD(p);
    // kernels enqueued by earlier calls (on any stream) may still read d_U / d_T
    CUDA_TRY(cudaEventSynchronize(p->ev_use));
    if (p->prec == QFT_PREC_F64) {
        const double *t = (const double *)h_table;
        p->t64.assign(t, t + p->N / 4);
        std::vector<double> U;
        level_table(p->N, p->t64, U);
        for (size_t i = 0; i < 32 && i < U.size(); ++i) p->uhead64[i] = U[i];
        CUDA_TRY(cudaMemcpy(p->d_U, U.data(), U.size() * sizeof(double), cudaMemcpyHostToDevice));
        if (p->d_T) CUDA_TRY(cudaMemcpy(p->d_T, p->t64.data(), p->t64.size() * sizeof(double), cudaMemcpyHostToDevice));
    } else {
        const float *t = (const float *)h_table;
        p->t32.assign(t, t + p->N / 4);
        std::vector<float> U;
        level_table(p->N, p->t32, U);
        for (size_t i = 0; i < 32 && i < U.size(); ++i) p->uhead32[i] = U[i];
        CUDA_TRY(cudaMemcpy(p->d_U, U.data(), U.size() * sizeof(float), cudaMemcpyHostToDevice));
        if (p->d_T) CUDA_TRY(cudaMemcpy(p->d_T, p->t32.data(), p->t32.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    return 0;
}

static int ensure_scratch(qft_plan *p, size_t bytes) {
    if (p->scratch_bytes >= bytes) return 0;
    if (p->d_scratch) {  // grown: earlier calls may still use the old buffer
        cudaEventSynchronize(p->ev_use);
        cudaFree(p->d_scratch);
    }
    p->d_scratch = nullptr;
    p->scratch_bytes = 0;
    CUDA_TRY(cudaMalloc(&p->d_scratch, bytes));
    p->scratch_bytes = bytes;
    return 0;
}

template <typename T>
static int layout_copy(const void *src, void *dst, long long batch, int N, long long sbs, long long ses,
                       long long dbs, long long des, cudaStream_t st, int num_sms) {
    if (sbs == N && ses == 1 && dbs == N && des == 1) {
        CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)batch * N * sizeof(vec2<T>), cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    if (ses == batch && sbs == 1 && dbs == N && des == 1) {  // (N, B) -> (B, N)
        qft_transpose<T><<<transpose_grid(N, batch), dim3(32, 8), 0, st>>>((const vec2<T> *)src, (vec2<T> *)dst, N,
                                                                           batch);
    } else if (sbs == N && ses == 1 && des == batch && dbs == 1) {  // (B, N) -> (N, B)
        qft_transpose<T><<<transpose_grid(batch, N), dim3(32, 8), 0, st>>>((const vec2<T> *)src, (vec2<T> *)dst, batch,
                                                                           N);
    } else {
        qft_strided_copy<T><<<num_sms * 8, 256, 0, st>>>((const vec2<T> *)src, (vec2<T> *)dst, batch, N, sbs, ses,
                                                          dbs, des);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
}

// scratch: NULL -> the plan's own (grown on demand); else >= 2*batch*N elements
static int exec_impl(qft_plan *p, const void *d_in, void *d_out, int64_t batch, int64_t ibs, int64_t ies,
                     int64_t obs, int64_t oes, cudaStream_t st, void *scratch = nullptr) {
    if (batch == 0) return 0;
    const int N = p->N;
    // the kernels read the input with 16-byte vector loads and TMA bulk copies
    // (and prefetch it by 16-byte-aligned bulk prefetches): a batch-major input
    // that is not 16-byte aligned (an fp32 view at an odd element offset) goes
    // through the aligned scratch copy like any other layout
    const bool in_c = (ibs == N && ies == 1) && ((uintptr_t)d_in % 16 == 0), out_c = (obs == N && oes == 1);
    const size_t esz = p->prec == QFT_PREC_F32 ? 8 : 16;
    const size_t bytes = (size_t)batch * N * esz;
    const void *src = d_in;
    void *dst = d_out;
    if ((!in_c || !out_c) && !scratch) {
        int rc = ensure_scratch(p, (in_c ? 0 : bytes) + (out_c ? 0 : bytes));
        if (rc) return rc;
        scratch = p->d_scratch;
    }
    char *scr = (char *)scratch;
    if (!in_c) {
        int rc = p->prec == QFT_PREC_F32
                     ? layout_copy<float>(d_in, scr, batch, N, ibs, ies, N, 1, st, p->num_sms)
                     : layout_copy<double>(d_in, scr, batch, N, ibs, ies, N, 1, st, p->num_sms);
        if (rc) return rc;
        src = scr;
        scr += bytes;
    }
    if (!out_c) dst = scr;
    int rc = launch_contig(p, src, dst, batch, st);
    if (rc) return rc;
    if (!out_c) {
        rc = p->prec == QFT_PREC_F32 ? layout_copy<float>(dst, d_out, batch, N, N, 1, obs, oes, st, p->num_sms)
                                     : layout_copy<double>(dst, d_out, batch, N, N, 1, obs, oes, st, p->num_sms);
        if (rc) return rc;
    }
    return 0;
}

int qft_exec_cdft(const qft_plan *cp, const void *d_in, void *d_out, int64_t batch, int64_t ibs, int64_t ies,
                  int64_t obs, int64_t oes, void *stream) {
    qft_plan *p = const_cast<qft_plan *>(cp);
    if (!p || (!d_in && batch) || (!d_out && batch)) return fail(QFT_EINVAL, "NULL argument");
    if (batch < 0) return fail(QFT_EINVAL, "negative batch");
    if (d_in == d_out && batch) return fail(QFT_EINVAL, "transform is out-of-place: d_in must differ from d_out");
    DEV_GUARD(p);
    std::lock_guard<std::mutex> lk(p->mu);
    cudaStream_t st = (cudaStream_t)stream;
    int rc = use_begin(p, st);
    if (!rc) rc = exec_impl(p, d_in, d_out, batch, ibs, ies, obs, oes, st);
    const int rc2 = use_end(p, st);
    return rc ? rc : rc2;
}

int qft_exec_real(const qft_plan *cp, int kind, const void *d_in, void *d_out, int64_t nrows, void *stream) {
    qft_plan *p = const_cast<qft_plan *>(cp);
    if (!p || (nrows && (!d_in || !d_out))) return fail(QFT_EINVAL, "NULL argument");
    if (kind < QFT_KIND_RDFT || kind > QFT_KIND_DST0) return fail(QFT_EINVAL, "kind must be rdft, dct0 or dst0");
    if (nrows < 0) return fail(QFT_EINVAL, "negative row count");
    if (kind == QFT_KIND_DST0 && p->log2n < 2) return fail(QFT_EINVAL, "the sine transform needs N >= 4");
    if (nrows == 0) return 0;
    if (d_in == d_out) return fail(QFT_EINVAL, "transform is out-of-place: d_in must differ from d_out");
    DEV_GUARD(p);
    std::lock_guard<std::mutex> lk(p->mu);
    cudaStream_t st = (cudaStream_t)stream;
    int rc = use_begin(p, st);
    if (rc) return rc;
    if (p->algo == QFT_ALGO_CLASSICAL) {
        rc = launch_classical(p, kind, d_in, d_out, (nrows + 1) / 2, nrows, st);
    } else if (p->multipass) {
        rc = launch_large(p, kind, d_in, d_out, (nrows + 1) / 2, nrows, st);
    } else {
        LaunchArgs a{d_in, d_out, (nrows + 1) / 2, p->d_U,
                     p->prec == QFT_PREC_F32 ? (const void *)p->uhead32 : (const void *)p->uhead64, p->num_sms, st,
                     nrows};
        int e = kLaunch[p->prec == QFT_PREC_F32 ? 0 : 1][p->log2n](&a, kind);
        if (e != 0) rc = fail(QFT_ECUDA, std::string("kernel launch: ") + cudaGetErrorString((cudaError_t)e));
    }
    const int rc2 = use_end(p, st);
    return rc ? rc : rc2;
}

// ============================================================== host path
// Host worker pool for the pageable-memory host path: the calling thread plus
// up to 15 workers run one parallel_for at a time (the copies between ordinary
// pageable host memory and the plan's pinned staging ring).
class HostPool {
  public:
    static HostPool &get() {
        static HostPool pool;
        return pool;
    }
    int size() const { return (int)th_.size() + 1; }
    // f(part, nparts) on every thread of the pool (part 0 on the caller)
    void run(const std::function<void(int, int)> &f) {
        std::lock_guard<std::mutex> one(run_mu_);
        const int n = size();
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0, n);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }

  private:
    HostPool() {
        int hw = (int)std::thread::hardware_concurrency();
        int n = hw < 2 ? 1 : (hw > 16 ? 16 : hw);
        for (int i = 1; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    void loop(int idx) {
        int seen = 0;
        for (;;) {
            const std::function<void(int, int)> *job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
            }
            (*job)(idx, size());
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)> *job_ = nullptr;
    int gen_ = 0, pending_ = 0;
    bool stop_ = false;
};

// rows x width bytes: dst[r*dpitch ..] <- src[r*spitch ..], split over the pool
static void parallel_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t rows) {
    if (rows == 1) {  // one contiguous run: split it by bytes
        HostPool::get().run([&](int part, int n) {
            const size_t lo = width * part / n, hi = width * (part + 1) / n;
            if (hi > lo) memcpy((char *)dst + lo, (const char *)src + lo, hi - lo);
        });
        return;
    }
    HostPool::get().run([&](int part, int n) {
        const size_t lo = rows * part / n, hi = rows * (part + 1) / n;
        for (size_t r = lo; r < hi; ++r) memcpy((char *)dst + r * dpitch, (const char *)src + r * spitch, width);
    });
}

static bool is_pinned(const void *h) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();  // clear: an unknown host pointer is pageable memory
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

int qft_exec_cdft_host(qft_plan *p, const void *h_in, void *h_out, int64_t batch, int64_t ibs, int64_t ies,
                       int64_t obs, int64_t oes) {
    if (!p || (batch && (!h_in || !h_out))) return fail(QFT_EINVAL, "NULL argument");
    if (batch <= 0) return batch == 0 ? 0 : fail(QFT_EINVAL, "negative batch");
    DEV_GUARD(p);
    std::lock_guard<std::mutex> lk(p->mu);
    const int N = p->N;
    const size_t esz = p->prec == QFT_PREC_F32 ? 8 : 16;
    const bool batch_major_in = (ibs == N && ies == 1), batch_major_out = (obs == N && oes == 1);
    const bool ref_in = (ies == batch && ibs == 1), ref_out = (oes == batch && obs == 1);
    if (!(batch_major_in || ref_in) || !(batch_major_out || ref_out))
        return fail(QFT_EINVAL, "host path supports batch-major or (N, batch) layouts only");
    // pageable host buffers are staged through the plan's pinned ring by the
    // host worker pool (a driver-staged pageable DMA runs at ~1/5 of PCIe)
    const bool stage_in = !is_pinned(h_in), stage_out = !is_pinned(h_out);
    for (auto &s : p->streams)
        if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    // chunk the batch over NS buffer slots: the host copies, H2D copy, transform
    // and D2H copy of different chunks overlap (both copy directions run concurrently)
    constexpr int NS = qft_plan::kHostSlots;
    const size_t target = (size_t)32 << 20;  // bytes per chunk
    long long chunk = (long long)(target / ((size_t)N * esz));
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    const size_t cbytes = (size_t)chunk * N * esz;
    // per slot: in, out, 2x layout scratch; kept in the plan across calls
    if (p->host_bytes < cbytes * 4 * NS) {
        if (p->d_host) {  // grown: earlier calls may still use the old buffer
            cudaEventSynchronize(p->ev_use);
            cudaFree(p->d_host);
        }
        p->d_host = nullptr;
        p->host_bytes = 0;
        CUDA_TRY(cudaMalloc(&p->d_host, cbytes * 4 * NS));
        p->host_bytes = cbytes * 4 * NS;
    }
    if ((stage_in || stage_out) && p->pin_bytes < cbytes * 2 * NS) {
        if (p->h_pin) cudaFreeHost(p->h_pin);  // the previous call synchronised before returning
        p->h_pin = nullptr;
        p->pin_bytes = 0;
        CUDA_TRY(cudaHostAlloc(&p->h_pin, cbytes * 2 * NS, cudaHostAllocPortable));
        p->pin_bytes = cbytes * 2 * NS;
    }
    char *bufs = (char *)p->d_host;
    // streams: H2D copies, transforms (serialised: the plan's scratch is shared),
    // D2H copies; chunk k uses buffer slot k % NS, events chain the stages
    cudaStream_t sin = p->streams[0], scomp = p->streams[1], sout = p->streams[2];
    // earlier device-path calls on other streams may still use the plan's scratch
    CUDA_TRY(cudaStreamWaitEvent(sin, p->ev_use, 0));
    CUDA_TRY(cudaStreamWaitEvent(scomp, p->ev_use, 0));
    cudaEvent_t ev_in[NS], ev_out[NS], ev_free[NS];
    for (int i = 0; i < NS; ++i) {
        CUDA_TRY(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
    }
    const long long nchunks = (batch + chunk - 1) / chunk;
    auto cols = [&](long long k) { return (batch - k * chunk) < chunk ? (batch - k * chunk) : chunk; };
    // host side of chunk k's output: pinned staging slot -> the caller's buffer
    auto copy_out = [&](long long k) -> int {
        const int slot = (int)(k % NS);
        const long long b0 = k * chunk, nb = cols(k);
        CUDA_TRY(cudaEventSynchronize(ev_free[slot]));
        const char *src = (const char *)p->h_pin + (2 * slot + 1) * cbytes;
        if (batch_major_out)
            parallel_copy2d((char *)h_out + (size_t)b0 * N * esz, 0, src, 0, (size_t)nb * N * esz, 1);
        else
            parallel_copy2d((char *)h_out + (size_t)b0 * esz, (size_t)batch * esz, src, (size_t)nb * esz,
                            (size_t)nb * esz, (size_t)N);
        return 0;
    };
    constexpr int LAG = NS - 1;  // chunks in flight between the host copy-in and copy-out
    int rc = 0;
    for (long long it = 0; it < nchunks && !rc; ++it) {
        const long long b0 = it * chunk, nb = cols(it);
        const int slot = (int)(it % NS);
        char *din = bufs + slot * 4 * cbytes, *dout = din + cbytes, *dscr = din + 2 * cbytes;
        cudaError_t e = cudaSuccess;
        if (it >= NS) e = cudaStreamWaitEvent(sin, ev_free[slot], 0);  // slot's previous D2H done
        if (e == cudaSuccess) {
            const char *hsrc = (const char *)h_in + (batch_major_in ? (size_t)b0 * N * esz : (size_t)b0 * esz);
            if (stage_in) {
                // the staging slot's previous H2D copy must be done before the host rewrites it
                char *pin = (char *)p->h_pin + 2 * slot * cbytes;
                if (it >= NS) e = cudaEventSynchronize(ev_in[slot]);
                if (batch_major_in)
                    parallel_copy2d(pin, 0, hsrc, 0, (size_t)nb * N * esz, 1);
                else  // columns [b0, b0+nb) of the (N, batch) array -> (N, nb) contiguous
                    parallel_copy2d(pin, (size_t)nb * esz, hsrc, (size_t)batch * esz, (size_t)nb * esz, (size_t)N);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(din, pin, (size_t)nb * N * esz, cudaMemcpyHostToDevice, sin);
            } else if (batch_major_in) {
                e = cudaMemcpyAsync(din, hsrc, (size_t)nb * N * esz, cudaMemcpyHostToDevice, sin);
            } else {  // columns [b0, b0+nb) of the (N, batch) array -> (N, nb) pitched
                e = cudaMemcpy2DAsync(din, (size_t)nb * esz, hsrc, (size_t)batch * esz, (size_t)nb * esz, (size_t)N,
                                      cudaMemcpyHostToDevice, sin);
            }
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_in[slot], sin);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(scomp, ev_in[slot], 0);
        if (e != cudaSuccess) {
            rc = fail(QFT_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
            break;
        }
        // device layout of the chunk: batch-major (nb, N) or (N, nb)
        rc = exec_impl(p, din, dout, nb, batch_major_in ? N : 1, batch_major_in ? 1 : nb, batch_major_out ? N : 1,
                       batch_major_out ? 1 : nb, scomp, dscr);
        if (rc) break;
        e = cudaEventRecord(ev_out[slot], scomp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev_out[slot], 0);
        if (e == cudaSuccess) {
            if (stage_out)  // contiguous into the pinned slot; copy_out scatters it later
                e = cudaMemcpyAsync((char *)p->h_pin + (2 * slot + 1) * cbytes, dout, (size_t)nb * N * esz,
                                    cudaMemcpyDeviceToHost, sout);
            else if (batch_major_out)
                e = cudaMemcpyAsync((char *)h_out + (size_t)b0 * N * esz, dout, (size_t)nb * N * esz,
                                    cudaMemcpyDeviceToHost, sout);
            else
                e = cudaMemcpy2DAsync((char *)h_out + (size_t)b0 * esz, (size_t)batch * esz, dout, (size_t)nb * esz,
                                      (size_t)nb * esz, (size_t)N, cudaMemcpyDeviceToHost, sout);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_free[slot], sout);
        if (e != cudaSuccess) {
            rc = fail(QFT_ECUDA, std::string("D2H: ") + cudaGetErrorString(e));
            break;
        }
        // the output slot of chunk it-LAG+NS ... is reused NS chunks later: drain chunk it-LAG now
        if (stage_out && it >= LAG) rc = copy_out(it - LAG);
    }
    if (stage_out && !rc)
        for (long long k = nchunks > LAG ? nchunks - LAG : 0; k < nchunks && !rc; ++k) rc = copy_out(k);
    if (cudaEventRecord(p->ev_use, sout) != cudaSuccess && !rc) rc = fail(QFT_ECUDA, "event record failed");
    for (auto &st : p->streams) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess && !rc) rc = fail(QFT_ECUDA, std::string("sync: ") + cudaGetErrorString(e));
    }
    for (int i = 0; i < NS; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_out[i]);
        cudaEventDestroy(ev_free[i]);
    }
    return rc;
}

int qft_fill_normal(const qft_plan *p, void *d_out, int64_t batch, int64_t first_index, uint64_t seed, void *stream) {
    if (!p || (!d_out && batch)) return fail(QFT_EINVAL, "NULL argument");
    if (batch <= 0) return 0;
    DEV_GUARD(p);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->prec == QFT_PREC_F32)
        qft_fill_normal_kernel<float><<<p->num_sms * 16, 256, 0, st>>>((vec2<float> *)d_out, batch, p->N, first_index,
                                                                        seed);
    else
        qft_fill_normal_kernel<double><<<p->num_sms * 16, 256, 0, st>>>((vec2<double> *)d_out, batch, p->N,
                                                                         first_index, seed);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

