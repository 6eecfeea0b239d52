// qft_inst.cu -- one (precision, N) instance of the transform kernels.
// Compiled once per instance with -DQFT_INST_PREC={32,64} -DQFT_INST_LOG2N={1..12}.
#include "qft_launch.cuh"

#if !defined(QFT_INST_PREC) || !defined(QFT_INST_LOG2N)
#error "compile with -DQFT_INST_PREC=<32|64> -DQFT_INST_LOG2N=<1..12>"
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

// cfg[0] dynamic smem bytes, cfg[1] threads per CTA, cfg[2] signals per CTA iteration
void QFT_CFGNAME(QFT_INST_PREC, QFT_INST_LOG2N)(int *cfg) {
#if QFT_INST_LOG2N <= 5
    cfg[0] = 0;
    cfg[1] = 128;
    cfg[2] = 1;
#else
    using K = qft::KCfg<QFT_INST_LOG2N, Real>;
    cfg[0] = K::SMEM;
    cfg[1] = K::NT;
    cfg[2] = K::TT;
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
    switch (mode) {
        case 0: return (int)qft::launch_smem<L, Real, 0>(*a);
        case 1: return (int)qft::launch_smem<L, Real, 1>(*a);
        case 2: return (int)qft::launch_smem<L, Real, 2>(*a);
        case 3: return (int)qft::launch_smem<L, Real, 3>(*a);
    }
#endif
    return (int)cudaErrorInvalidValue;
}
