// Micro-benchmarks of the instruction rates the transform kernels depend on
// (tools only): packed fp32 add throughput/latency vs scalar, one warp per SM
// sub-partition (4 warps per CTA, 1 CTA).
#include <cstdio>
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
template <int ACC>
__global__ void k_fadd2(unsigned long long *out, long long *cyc, int iters) {
    unsigned long long a[ACC];
    for (int i = 0; i < ACC; ++i) a[i] = threadIdx.x * 7 + i;
    unsigned long long b = 0x3f8000003f800000ull;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ACC; ++i) a[i] = fadd2(a[i], b);
    long long t1 = clock64();
    unsigned long long s = 0;
    for (int i = 0; i < ACC; ++i) s ^= a[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int ACC>
__global__ void k_fadd(float *out, long long *cyc, int iters) {
    float a[ACC];
    for (int i = 0; i < ACC; ++i) a[i] = threadIdx.x * 7 + i;
    float b = 1.0f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ACC; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < ACC; ++i) s += a[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// LDS.64 throughput: each lane loads ACC independent 8-byte words per iteration
template <int ACC>
__global__ void k_lds(unsigned long long *out, long long *cyc, int iters, int mask = -1) {
    __shared__ unsigned long long sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    if (!((mask >> (threadIdx.x >> 5)) & 1)) return;
    unsigned long long s = 0;
    int base = threadIdx.x & 31;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        unsigned long long v[ACC];
#pragma unroll
        for (int i = 0; i < ACC; ++i) asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v[i]) : "r"((unsigned)__cvta_generic_to_shared(&sm[(base + 32 * i + it) & 4095])));
#pragma unroll
        for (int i = 0; i < ACC; ++i) s += v[i];
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// LDS.128 / LDS.32 / STS.64 throughput
template <int ACC, int W>
__global__ void k_ldsw(unsigned long long *out, long long *cyc, int iters) {
    __shared__ __align__(16) unsigned long long sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    unsigned long long s = 0;
    int base = threadIdx.x & 31;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        unsigned long long v[ACC];
#pragma unroll
        for (int i = 0; i < ACC; ++i) {
            const unsigned a = (unsigned)__cvta_generic_to_shared(&sm[((base + 32 * i + it) * 2) & 4095]);
            if (W == 16) {
                unsigned long long b;
                asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v[i]), "=l"(b) : "r"(a));
                v[i] ^= b;
            } else if (W == 4) {
                unsigned b;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(b) : "r"(a));
                v[i] = b;
            } else if (W == -8) {
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"((unsigned long long)it));
                v[i] = 0;
            } else if (W == -16) {
                asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"((unsigned long long)it), "l"((unsigned long long)i));
                v[i] = 0;
            } else {
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v[i]) : "r"(a));
            }
        }
#pragma unroll
        for (int i = 0; i < ACC; ++i) s += v[i];
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    unsigned long long *o;
    long long *c, h;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&c, 64);
    const int it = 4096;
    for (int w : {1, 2, 4, 8, 12, 16}) {
        int nt = 32 * w;
        k_fadd2<8><<<1, nt>>>(o, c, it);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double f2 = (double)h / (it * 8.0);
        k_fadd2<1><<<1, nt>>>(o, c, it);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double f2l = (double)h / it;
        k_fadd<16><<<1, nt>>>((float *)o, c, it);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double f1 = (double)h / (it * 16.0);
        k_lds<8><<<1, nt>>>(o, c, it);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double l = (double)h / (it * 8.0);
        printf("warps/CTA %2d: FADD2 %.2f cyc/inst/warp (dep chain %.2f), FADD %.2f, LDS.64 %.2f cyc/inst/warp\n", w, f2, f2l, f1, l);
    }
    for (int w : {1, 4, 16}) {
        double r[5];
        int k = 0;
        for (int W : {4, 8, 16, -8, -16}) {
            switch (W) {
                case 4: k_ldsw<8, 4><<<1, 32 * w>>>(o, c, it); break;
                case 8: k_ldsw<8, 8><<<1, 32 * w>>>(o, c, it); break;
                case 16: k_ldsw<8, 16><<<1, 32 * w>>>(o, c, it); break;
                case -8: k_ldsw<8, -8><<<1, 32 * w>>>(o, c, it); break;
                case -16: k_ldsw<8, -16><<<1, 32 * w>>>(o, c, it); break;
            }
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            r[k++] = (double)h / (it * 8.0);
        }
        printf("warps %2d: cyc/inst/warp LDS.32 %.2f LDS.64 %.2f LDS.128 %.2f STS.64 %.2f STS.128 %.2f\n", w, r[0], r[1], r[2], r[3], r[4]);
    }
    // which warps share an SM sub-partition: run only warps {0, w} of an 8-warp CTA
    for (int w = 1; w < 8; ++w) {
        k_lds<8><<<1, 256>>>(o, c, it, 1 | (1 << w));
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("LDS.64 warps {0,%d} active: %.2f cyc/inst/warp\n", w, (double)h / (it * 8.0));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
