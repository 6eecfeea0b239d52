// classical_emu.cpp -- test-only host emulation of the level-synchronous
// classical QFT (paper_1301_0763_b200/csrc/qft_classical_lv.cuh): runs the very
// item functions the CUDA kernels run, with the kernels' schedule (whole tree, or
// global levels + sub-trees cut at depth d0) as plain loops.  Checked bit for bit
// against the oracle's classical restatement by tests/test_emulator.py.
#include <cstring>
#include <vector>

#include "../../paper_1301_0763_b200/csrc/qft_classical_lv.cuh"

using namespace qft;

namespace {

template <typename T>
void run_tree(const cl::Tree<T> &t, vec2<T> *P0, vec2<T> *P1) {
    const int D = t.depth();
    vec2<T> *cen = P0 + cl::cen_off(t.lognn);
    for (int d = 0; d < D; ++d)
        for (int it = 0; it < t.fwd_items(); ++it) t.fwd_item((d & 1) ? P1 : P0, (d & 1) ? P0 : P1, cen, d, it);
    for (int it = 0; it < t.base_items(); ++it) t.base_item((D & 1) ? P1 : P0, it);
    for (int d = D - 1; d >= 0; --d)
        for (int it = 0; it < t.bwd_items(); ++it) t.bwd_item(((d + 1) & 1) ? P1 : P0, (d & 1) ? P1 : P0, cen, d, it);
}

template <int MODE, typename T>
int run_mode(int lg, int sublog, const void *in, void *out, long units, long nreal, const T *Tt) {
    const int N = 1 << lg, m = N / 2;
    const bool do_cos = MODE != 3, do_sin = MODE != 2;
    const int Ws = cl::buf_cells(lg), CB = cl::cos_cells(lg);
    std::vector<vec2<T>> W0(Ws), W1(Ws);
    for (long u = 0; u < units; ++u) {
        // poison: a cell read before it is written shows up as a mismatch
        std::memset(W0.data(), 0x7f, sizeof(vec2<T>) * Ws);
        std::memset(W1.data(), 0x7f, sizeof(vec2<T>) * Ws);
        for (int n = 0; n < m; ++n) cl::ingest_item<MODE, T>(in, u, nreal, N, W0.data(), CB, n);
        const cl::Tree<T> top{lg, lg, CB, false, do_cos, do_sin, Tt};
        if (sublog <= 0 || sublog >= lg) {
            run_tree(top, W0.data(), W1.data());
        } else {
            const int d0 = lg - sublog, S0 = 1 << (sublog - 1);
            vec2<T> *W[2] = {W0.data(), W1.data()};
            for (int d = 0; d < d0; ++d)
                for (int it = 0; it < top.fwd_items(); ++it) top.fwd_item(W[d & 1], W[(d + 1) & 1], W0.data() + cl::cen_off(lg), d, it);
            std::vector<vec2<T>> P0(cl::buf_cells(sublog)), P1(cl::buf_cells(sublog));
            for (int b = 0; b < (1 << d0); ++b) {
                const cl::Tree<T> t{sublog, lg, cl::cos_cells(sublog), (b & 1) != 0, do_cos, do_sin, Tt};
                vec2<T> *wc = W[d0 & 1] + cl::cos_off(S0, b), *ws = W[d0 & 1] + CB + b * cl::sin_stride_of(lg, d0);
                const int nc = S0 + ((b & 1) ? 0 : 1);
                std::memset(P0.data(), 0x7f, sizeof(vec2<T>) * P0.size());
                std::memset(P1.data(), 0x7f, sizeof(vec2<T>) * P1.size());
                if (do_cos) std::memcpy(P0.data(), wc, sizeof(vec2<T>) * nc);
                if (do_sin) std::memcpy(P0.data() + t.CB, ws, sizeof(vec2<T>) * (S0 - 1));
                run_tree(t, P0.data(), P1.data());
                if (do_cos) std::memcpy(wc, P0.data(), sizeof(vec2<T>) * nc);
                if (do_sin) std::memcpy(ws, P0.data() + t.CB, sizeof(vec2<T>) * (S0 - 1));
            }
            for (int d = d0 - 1; d >= 0; --d)
                for (int it = 0; it < top.bwd_items(); ++it) top.bwd_item(W[(d + 1) & 1], W[d & 1], W0.data() + cl::cen_off(lg), d, it);
        }
        for (int k = 0; k <= m; ++k) cl::emit_item<MODE, T>(out, u, nreal, N, W0.data(), CB, k);
    }
    return 0;
}

template <typename T>
int run(int lg, int mode, int sublog, const void *in, void *out, long units, long nreal, const T *Tt) {
    if (lg < cl::kBaseLog) return -1;
    switch (mode) {
        case 0: return run_mode<0, T>(lg, sublog, in, out, units, nreal, Tt);
        case 1: return run_mode<1, T>(lg, sublog, in, out, units, nreal, Tt);
        case 2: return run_mode<2, T>(lg, sublog, in, out, units, nreal, Tt);
        case 3: return run_mode<3, T>(lg, sublog, in, out, units, nreal, Tt);
    }
    return -1;
}

}  // namespace

// units: complex rows (mode 0) or pairs of real rows (modes 1-3, nreal rows in all);
// sublog > 0: cut the tree into sub-trees of periodization 2^sublog (the large-N schedule)
extern "C" int emu_classical_f32(int lg, int mode, int sublog, const void *in, void *out, long units, long nreal,
                                 const void *T) {
    return run<float>(lg, mode, sublog, in, out, units, nreal, (const float *)T);
}
extern "C" int emu_classical_f64(int lg, int mode, int sublog, const void *in, void *out, long units, long nreal,
                                 const void *T) {
    return run<double>(lg, mode, sublog, in, out, units, nreal, (const double *)T);
}
