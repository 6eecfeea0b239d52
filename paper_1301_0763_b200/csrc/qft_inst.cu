// qft_inst.cu -- one (precision, N) instance of the transform kernels.
// Compiled once per instance with -DQFT_INST_PREC={32,64} -DQFT_INST_LOG2N={1..14}.
// An instance whose working area does not fit in shared memory (fp64 N = 2^14)
// reports cfg[0] = 0 and is served by the multi-pass path.
#include "qft_pipe.cuh"

#if !defined(QFT_INST_PREC) || !defined(QFT_INST_LOG2N)
#error "compile with -DQFT_INST_PREC=<32|64> -DQFT_INST_LOG2N=<1..14>"
#endif

#ifndef QFT_REG64
#define QFT_REG64 1  // complex fp32 N = 64: one thread per signal in registers behind the shared-memory staging (146 registers; fp64 would spill)
#endif

#define QFT_CAT3(a, b, c) a##_##b##_##c
#define QFT_NAME(P, L) QFT_CAT3(qft_inst_launch, P, L)

namespace {
#if QFT_INST_PREC == 32
using Real = float;
#else
using Real = double;
#endif
}  // namespace

#define QFT_CFGNAME(P, L) QFT_CAT3(qft_inst_cfg, P, L)

namespace {
// templates, so that the branch of an instance that does not fit is discarded
template <int L, typename R>
void smem_cfg(int *cfg) {
    if constexpr (qft::smem_fits<L, R>()) {
        using K = qft::KCfg<L, R>;
        cfg[0] = K::SMEM;
        cfg[1] = K::NT;
        cfg[2] = K::TT;
        if constexpr (qft::use_pipe<L, R>()) {  // the cdft path
            using C = qft::PCfg<L, R>;
            cfg[0] = C::SMEM;
            cfg[1] = C::NT;
            cfg[2] = C::TT;
            if constexpr (QFT_PIPE == 3 && qft::GCfg<L, R>::FITS) {
                cfg[0] = qft::GCfg<L, R>::SMEM;
                cfg[1] = qft::GCfg<L, R>::NT;
                cfg[2] = qft::GCfg<L, R>::NG;
            }
        }
    } else {
        cfg[0] = cfg[1] = cfg[2] = 0;
    }
}
template <int L, typename R>
int smem_launch(const qft::LaunchArgs *a, int mode) {
    if constexpr (qft::smem_fits<L, R>()) {
        switch (mode) {
            case 0:
                if constexpr (qft::use_pipe<L, R>()) return (int)qft::launch_pipe<L, R>(*a);
                else if constexpr (QFT_REG64 && L == 6 && sizeof(R) == 4) return (int)qft::launch_reg<64, R, 0>(*a);
                else return (int)qft::launch_smem<L, R, 0>(*a);
            case 1: return (int)qft::launch_smem<L, R, 1>(*a);
            case 2: return (int)qft::launch_smem<L, R, 2>(*a);
            case 3: return (int)qft::launch_smem<L, R, 3>(*a);
        }
    }
    return (int)cudaErrorInvalidValue;
}
}  // namespace

// cfg[0] dynamic smem bytes, cfg[1] threads per CTA, cfg[2] signals per CTA iteration
void QFT_CFGNAME(QFT_INST_PREC, QFT_INST_LOG2N)(int *cfg) {
#if QFT_INST_LOG2N <= 5
    cfg[0] = 0;
    cfg[1] = 128;
    cfg[2] = 1;
#else
    smem_cfg<QFT_INST_LOG2N, Real>(cfg);
#endif
}

// mode: 0 cdft, 1 rdft, 2 dct0, 3 dst0 (real modes: a->batch = row pairs, a->nreal = rows)
int QFT_NAME(QFT_INST_PREC, QFT_INST_LOG2N)(const qft::LaunchArgs *a, int mode) {
    constexpr int L = QFT_INST_LOG2N;
#if QFT_INST_LOG2N <= 5
    switch (mode) {
        case 0: return (int)qft::launch_reg<(1 << L), Real, 0>(*a);
        case 1: return (int)qft::launch_reg<(1 << L), Real, 1>(*a);
        case 2: return (int)qft::launch_reg<(1 << L), Real, 2>(*a);
        case 3:
            if constexpr (L >= 2) return (int)qft::launch_reg<(1 << L), Real, 3>(*a);
            return (int)cudaErrorInvalidValue;
    }
#else
    return smem_launch<L, Real>(a, mode);
#endif
    return (int)cudaErrorInvalidValue;
}
