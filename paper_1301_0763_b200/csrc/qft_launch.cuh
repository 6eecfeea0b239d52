// qft_launch.cuh -- the batched transform kernels and their launchers.
//   qft_cdft_reg   N <= 32     : one thread per signal, whole transform in registers
//   qft_cdft_smem  N = 64..4096: one signal per CTA iteration, persistent grid,
//                                shared-memory working set, phases of qft_smem.cuh
// Each (precision, N) instance is compiled in its own translation unit
// (qft_inst.cu) so the build parallelises.
#pragma once
#include <cuda_runtime.h>

#include "qft_smem.cuh"

namespace qft {

struct LaunchArgs {
    const void *in;
    void *out;
    long long batch;
    const void *U;  // level table (device)
    int num_sms;
    cudaStream_t stream;
};

template <int NN, typename T>
__global__ void __launch_bounds__(128) qft_cdft_reg(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out,
                                                    long long batch, const T *__restrict__ U) {
    __shared__ T sU[NN / 4 >= 2 ? NN / 4 : 2];
    for (int i = threadIdx.x; i < (NN / 4 >= 2 ? NN / 4 : 2); i += blockDim.x) sU[i] = U[i];
    __syncthreads();
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < batch;
         b += (long long)gridDim.x * blockDim.x) {
        vec2<T> x[NN], y[NN];
#pragma unroll
        for (int n = 0; n < NN; ++n) x[n] = in[b * NN + n];
        cdft_reg<NN, T>(x, y, sU);
#pragma unroll
        for (int n = 0; n < NN; ++n) out[b * NN + n] = y[n];
    }
}

template <int LOG2N, typename T, int J>
__device__ __forceinline__ void run_phase_a(vec2<T> *w, const T *U, int unit, int lane) {
    if constexpr (J < SPlan<LOG2N>::JF) {
        if (unit == 2 * J) f_unit<LOG2N, J, false, T>(w, U, lane);
        else if (unit == 2 * J + 1) f_unit<LOG2N, J, true, T>(w, U, lane);
        else run_phase_a<LOG2N, T, J + 1>(w, U, unit, lane);
    }
}

template <int LOG2N, typename T, int J, bool DST>
__device__ __forceinline__ void run_c_side(vec2<T> *w, int lane) {
    BUnit<LOG2N, J, DST, T> b;
    b.load(w, lane);
    __syncwarp();
    b.store(w, lane);
}

template <int LOG2N, typename T, int J>
__device__ __forceinline__ void run_phase_c(vec2<T> *w, int unit, int lane) {
    if constexpr (J < SPlan<LOG2N>::JF) {
        if (unit == 2 * J) run_c_side<LOG2N, T, J, false>(w, lane);
        else if (unit == 2 * J + 1) run_c_side<LOG2N, T, J, true>(w, lane);
        else run_phase_c<LOG2N, T, J + 1>(w, unit, lane);
    }
}

template <int LOG2N, typename T, int NW>
__global__ void __launch_bounds__(NW * 32) qft_cdft_smem(const vec2<T> *__restrict__ in, vec2<T> *__restrict__ out,
                                                         long long batch, const T *__restrict__ Ug) {
    using P = SPlan<LOG2N>;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    vec2<T> *w = reinterpret_cast<vec2<T> *>(smem_raw);
    T *U = reinterpret_cast<T *>(smem_raw + sizeof(vec2<T>) * P::W_PADDED);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int i = tid; i < P::UCELLS; i += NT) U[i] = Ug[i];
    __syncthreads();

    for (long long b = blockIdx.x; b < batch; b += gridDim.x) {
        const vec2<T> *x = in + b * P::N;
        vec2<T> *y = out + b * P::N;
        // A0: fold + route
        for (int n = tid; n <= P::m; n += NT) a0_item<LOG2N, T>(x, w, n);
        __syncthreads();
        // A: forward levels of the big blocks (one warp per block side)
        if constexpr (P::JF > 0) {
            for (int u = warp; u < 2 * P::JF; u += NW) run_phase_a<LOG2N, T, 0>(w, U, u, lane);
            __syncthreads();
        }
        // B: full sub-transforms + tail
        for (int u = tid; u < P::NB_UNITS; u += NT) b_unit<LOG2N, T>(w, U, u);
        __syncthreads();
        // C: backward levels of the big blocks
        if constexpr (P::JF > 0) {
            for (int u = warp; u < 2 * P::JF; u += NW) run_phase_c<LOG2N, T, 0>(w, u, lane);
            __syncthreads();
        }
        // D: chain top + recombination -> global
        for (int t = tid; t <= P::MRC; t += NT) Chain<LOG2N, T>::unit(w, y, t);
        __syncthreads();
    }
}

constexpr int kSmemWarps = 4;

inline int smem_bytes_for(int log2n, int prec) {
    if (log2n < 6) return 0;
    const int N = 1 << log2n;
    const int cells = N + 32;
    const int padded = cells + cells / 32 + 1;
    const int vb = prec == 32 ? 8 : 16, sb = prec == 32 ? 4 : 8;
    return padded * vb + (N / 4) * sb;
}


template <int LOG2N, typename T>
cudaError_t launch_smem(const LaunchArgs &a) {
    auto kern = qft_cdft_smem<LOG2N, T, kSmemWarps>;
    const int smem = smem_bytes_for(LOG2N, sizeof(T) == 4 ? 32 : 64);
    cudaError_t e;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSmemWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long long grid = (long long)a.num_sms * per_sm;
    if (grid > a.batch) grid = a.batch;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kSmemWarps * 32, smem, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch,
                                                          (const T *)a.U);
    return cudaGetLastError();
}

template <int NN, typename T>
cudaError_t launch_reg(const LaunchArgs &a) {
    long long blocks = (a.batch + 127) / 128;
    long long cap = (long long)a.num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    qft_cdft_reg<NN, T><<<(unsigned)blocks, 128, 0, a.stream>>>((const vec2<T> *)a.in, (vec2<T> *)a.out, a.batch,
                                                            (const T *)a.U);
    return cudaGetLastError();
}

}  // namespace qft
