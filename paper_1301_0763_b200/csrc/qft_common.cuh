// qft_common.cuh -- arithmetic contract and small helpers shared by every
// improved-QFT kernel.
//
// The arithmetic contract is the reference's counted primitives
// (/root/reference/pkg/src/quickfourier/counting.py:40-81): every value is one
// IEEE round-to-nearest add, sub or mul of two operands.  On the device we use
// the explicit __fadd_rn/__fmul_rn/__dadd_rn/__dmul_rn intrinsics, which the
// compiler never contracts into FMA (the build also passes -fmad=false).
// Functions are __host__ __device__ so the test-only host emulator
// (tests/emu/) can execute the exact same index logic on the CPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define QFT_HD __host__ __device__ __forceinline__
#define QFT_DEV __device__ __forceinline__
// a real call on the device: one copy of a large body shared by its callers
// (instruction-cache footprint), inlined on the host
#define QFT_HD_CALL __host__ __device__ __noinline__
#else
#define QFT_HD inline
#define QFT_DEV inline
#define QFT_HD_CALL inline
#endif

#if defined(__CUDACC__)
// (-0, -0) as a packed fp32 pair in a mutable device global (see vmul<float>);
// declared for both compilation passes so the host stub can register it.
static __device__ unsigned long long qft_mzero_pair = 0x8000000080000000ull;
#endif

namespace qft {

// One complex sample, or -- inside the real-factor recursion -- the pair
// (value of the Re-part signal, value of the Im-part signal).  Both halves
// follow the identical operation DAG (shared.py:56-57), so the kernels run
// them as one 2-vector stream.
template <typename T>
struct alignas(2 * sizeof(T)) vec2 {
    T x, y;
};

QFT_HD float radd(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
QFT_HD float rsub(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fsub_rn(a, b);
#else
    return a - b;
#endif
}
QFT_HD float rmul(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}
QFT_HD double radd(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
QFT_HD double rsub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
QFT_HD double rmul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}

template <typename T>
QFT_HD vec2<T> vadd(vec2<T> a, vec2<T> b) { return {radd(a.x, b.x), radd(a.y, b.y)}; }
template <typename T>
QFT_HD vec2<T> vsub(vec2<T> a, vec2<T> b) { return {rsub(a.x, b.x), rsub(a.y, b.y)}; }
template <typename T>
QFT_HD vec2<T> vmul(vec2<T> a, T c) { return {rmul(a.x, c), rmul(a.y, c)}; }

#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(QFT_NO_F32X2)
// sm_100a packed fp32 adds: one FADD2 per (Re-part, Im-part) pair.  .rn is the
// IEEE round-to-nearest single-precision op on each lane (denormals preserved),
// i.e. bit-identical to two scalar __fadd_rn.  Multiplies stay scalar
// (mul.rn.f32): ptxas 12.9 contracts mul.rn.f32x2 (and fma.rn.f32x2 with a -0
// addend) followed by add.rn.f32x2 into FFMA2 even under --fmad=false, which
// would change the rounding; scalar .rn multiplies are never contracted.
// tests/test_sass.py checks the built kernels contain no FFMA/FFMA2/DFMA.
QFT_DEV unsigned long long pk(vec2<float> a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
QFT_DEV vec2<float> upk(unsigned long long r) {
    vec2<float> a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
template <>
QFT_DEV vec2<float> vadd<float>(vec2<float> a, vec2<float> b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
template <>
QFT_DEV vec2<float> vsub<float>(vec2<float> a, vec2<float> b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
#if !defined(QFT_SCALAR_MUL)
// Packed multiply without contraction: x*c + z with z = (-0, -0) read from a
// mutable device global, so ptxas cannot fold a following add into it.
// x*c + (-0) == x*c bit for bit (x*c = +0 gives +0 + -0 = +0, -0 stays -0).
template <>
QFT_DEV vec2<float> vmul<float>(vec2<float> a, float c) {
    unsigned long long r;
    const unsigned long long z = __ldg(&::qft_mzero_pair);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(vec2<float>{c, c})), "l"(z));
    return upk(r);
}
#endif

#endif
template <typename T>
QFT_HD vec2<T> vsel(bool p, vec2<T> a, vec2<T> b) { return p ? a : b; }

QFT_HD int ctz32(uint32_t v) {
#if defined(__CUDA_ARCH__)
    return __ffs((int)v) - 1;
#else
    return __builtin_ctz(v);
#endif
}

// Position of element `t` of input slot `s` of an r-level reflection group
// of a Lee block of size L is c + sg*t.  Restates the fold pairing of
// elaborations.py:113-126 (element i with L-1-i) applied r times; every slot
// is a contiguous (possibly reversed) run, and the runs tile the block.
QFT_HD void run_of(int r, int L, int s, int &c, int &sg) {
    int A = 0, B = 1;
    while (r > 0) {
        int H = 1 << (r - 1);
        if (s >= H) {
            s = (1 << r) - 1 - s;
            A += B * (L - 1);
            B = -B;
        }
        L >>= 1;
        --r;
    }
    c = A;
    sg = B;
}

}  // namespace qft
