// tests/emu/kernel_emu.cpp -- TEST-ONLY host emulation of the device phase
// functions in paper_1301_0763_b200/csrc/qft_smem.cuh.
//
// It runs the exact index/arithmetic code of the shared-memory kernel on the
// CPU (one "thread" at a time, the B-phase split into load / __syncwarp /
// store exactly like the kernel) so that the layout logic can be checked
// bit-for-bit against the oracle without a GPU.  It is never used by the
// product path, which fails loudly without its CUDA extension.
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../paper_1301_0763_b200/csrc/qft_smem.cuh"
#include "../../paper_1301_0763_b200/csrc/qft_large_plan.h"
#include "../../paper_1301_0763_b200/csrc/qft_leaf.cuh"

using namespace qft;

template <typename T>
static void build_U(int N, const T *Tnat, std::vector<T> &U) {
    // Tnat = natural table T[m] = halfsec(m/N), T[0] = cos8; U[S/2+i] = T[(2i+1) N/(4S)]
    U.assign(N / 4 > 1 ? N / 4 : 2, (T)0);
    U[0] = Tnat[0];
    for (int S = 2; S <= N / 4; S *= 2)
        for (int i = 0; i < S / 2; ++i) U[S / 2 + i] = Tnat[(2 * i + 1) * (N / (4 * S))];
}

// big warp unit (unit_big in qft_launch.cuh) on the block at padded pointer wb
template <int L, int R, typename T, bool DST, bool REV = false>
static void emu_unit_big(vec2<T> *wb, const T *U, int ub = DST ? 1 : 0) {
    std::vector<FBlockP<L, R, DST, T>> f(32);
    for (int t = 0; t < 32; ++t) f[t].template load<REV>(wb, U, t);   // all lanes load ...
    for (int t = 0; t < 32; ++t) f[t].store(wb, t);     // ... __syncwarp ... store
    for (int p = 0; p < (1 << R); ++p) b_l32p<DST, T>(wb + 33 * p, U, ub, p & 1);
    using CB = CBlockP<R, DST, T>;
    std::vector<CB> c(32);
    std::vector<std::vector<vec2<T>>> outs(32, std::vector<vec2<T>>(CB::G));
    for (int i = 0; i < 32; ++i) c[i].load(wb, i);
    for (int i = 0; i < 32; ++i) {
        const vec2<T> *hc = CB::halo_colp(wb, i);  // the device reads the halo column before any store
        auto halo = [&](int p) { return hc[33 * p]; };
        c[i].compute(i, halo, outs[i].data());
    }
    for (int i = 0; i < 32; ++i) CB::storep(wb, i, outs[i].data());
}

template <int LOG2N, typename T, int J, bool DST>
static void emu_f_side(vec2<T> *w, const T *U) {
    std::vector<FBlock<LOG2N, J, DST, T>> lanes(32);
    for (int t = 0; t < 32; ++t) lanes[t].load(w, U, t);
    for (int t = 0; t < 32; ++t) lanes[t].store(w, t);
}
template <int LOG2N, typename T, int J, bool DST>
static void emu_c_side(vec2<T> *w) {
    using P = SPlan<LOG2N>;
    using CB = CBlockP<P::RF(J), DST, T>;
    vec2<T> *wb = w + padx((DST ? P::S0 : 0) + P::off(J));
    std::vector<CB> lanes(32);
    std::vector<std::vector<vec2<T>>> outs(32, std::vector<vec2<T>>(CB::G));
    for (int i = 0; i < 32; ++i) lanes[i].load(wb, i);
    for (int i = 0; i < 32; ++i) {
        const vec2<T> *hc = CB::halo_colp(wb, i);
        auto halo = [&](int p) { return hc[33 * p]; };
        lanes[i].compute(i, halo, outs[i].data());
    }
    for (int i = 0; i < 32; ++i) CB::storep(wb, i, outs[i].data());
}
// rest unit (unit_rest): blocks JR..JF-1, Lee-32 chunks from K0, small blocks
template <int LOG2N, typename T, int J, bool DST>
static void emu_rest_f(vec2<T> *w, const T *U) {
    if constexpr (J < SPlan<LOG2N>::JF) {
        emu_f_side<LOG2N, T, J, DST>(w, U);
        emu_rest_f<LOG2N, T, J + 1, DST>(w, U);
    }
}
template <int LOG2N, typename T, int J, bool DST>
static void emu_rest_c(vec2<T> *w) {
    if constexpr (J < SPlan<LOG2N>::JF) {
        emu_c_side<LOG2N, T, J, DST>(w);
        emu_rest_c<LOG2N, T, J + 1, DST>(w);
    }
}
template <int LOG2N, typename T, bool DST>
static void emu_unit_rest(vec2<T> *w, const T *U, int ub = DST ? 1 : 0) {
    using P = SPlan<LOG2N>;
    emu_rest_f<LOG2N, T, P::JR, DST>(w, U);
    for (int k = P::K0; k < P::NL32; ++k) b_l32<DST, T>(w, (DST ? P::S0 : 0) + 32 * k, U, ub, k & 1);
    b_small<LOG2N, DST, T>(w, U, ub);
    emu_rest_c<LOG2N, T, P::JR, DST>(w);
}
// top levels (top_f / top_b): every item loads before any store
template <int LOG2N, typename T, int J, bool DST>
static void emu_top_f(vec2<T> *w, const T *U) {
    if constexpr (J < SPlan<LOG2N>::JH) {
        using TP = Top<LOG2N, J, DST, T>;
        std::vector<vec2<T>> v(1024 * TP::G);
        for (int t = 0; t < 1024; ++t) TP::f_load(w, U, t, &v[t * TP::G]);
        for (int t = 0; t < 1024; ++t) TP::f_store(w, t, &v[t * TP::G]);
        emu_top_f<LOG2N, T, J + 1, DST>(w, U);
    }
}
template <int LOG2N, typename T, int J, bool DST>
static void emu_top_b(vec2<T> *w) {
    if constexpr (J < SPlan<LOG2N>::JH) {
        using TP = Top<LOG2N, J, DST, T>;
        std::vector<vec2<T>> o(1024 * TP::G);
        for (int i = 0; i < 1024; ++i) TP::b_compute(w, i, &o[i * TP::G]);
        for (int i = 0; i < 1024; ++i) TP::b_store(w, i, &o[i * TP::G]);
        emu_top_b<LOG2N, T, J + 1, DST>(w);
    }
}
// TF -> fused units -> TB of one side, in the kernel's order
template <int LOG2N, typename T, bool DST>
static void emu_side_impl(vec2<T> *w, const T *U, int ub) {
    using P = SPlan<LOG2N>;
    emu_top_f<LOG2N, T, 0, DST>(w, U);
    for (int bu = 0; bu < P::NU1; ++bu)
        emu_unit_big<P::LB, P::RB, T, DST>(w + padx((DST ? P::S0 : 0) + P::big_cell(bu)), U, ub);
    emu_unit_rest<LOG2N, T, DST>(w, U, ub);
    emu_top_b<LOG2N, T, 0, DST>(w);
}
// QFT_SC: the sine side is the cosine code on the sine region (qft_launch.cuh run_unit)
template <int LOG2N, typename T, bool DST>
static void emu_side(vec2<T> *w, const T *U) {
    if (QFT_SC && DST) emu_side_impl<LOG2N, T, false>(w + padx(SPlan<LOG2N>::S0), U, 1);
    else emu_side_impl<LOG2N, T, DST>(w, U, DST ? 1 : 0);
}

template <int LOG2N, typename T>
static void emu_one(const vec2<T> *x, vec2<T> *y, const T *U) {
    using P = SPlan<LOG2N>;
    std::vector<vec2<T>> Wv(P::PADDED);
    vec2<T> *w = Wv.data();
    if (P::m < 64)
        for (int n = 0; n < P::m; ++n) a0_item<LOG2N, T>(x, w, n);
    for (int c = 0; c < P::m / 64; ++c) {
        // the device shuffles lane l-1's first mirror element up; emulate with the same loads
        for (int l = 0; l < 32; ++l) {
            auto shfl_up = [&](vec2<T> v) {
                (void)v;
                const int lp = l > 0 ? l - 1 : l;
                return x[P::N - 64 * c - 2 * lp - 2];
            };
            a0_chunk64<LOG2N, T>(x, w, c, l, a0_lane64<LOG2N>(l), shfl_up);
        }
        if (!QFT_A0_LANE0) a0_item<LOG2N, T>(x, w, 64 * c);  // else lane 0 of the chunk did n = 64c
    }
    emu_side<LOG2N, T, false>(w, U);
    emu_side<LOG2N, T, true>(w, U);
    for (int t = 0; t < P::DT; ++t) Chain<LOG2N, T>::unit(w, y, t);
}

// real modes (1 rdft, 2 dct0, 3 dst0) on one pair of rows (xa, xb)
template <int LOG2N, typename T, int MODE>
static void emu_real_one(const T *xa, const T *xb, T *ya, T *yb, const T *U) {
    using P = SPlan<LOG2N>;
    std::vector<vec2<T>> Wv(P::PADDED);
    vec2<T> *w = Wv.data();
    for (int n = 0; n <= P::m; ++n) a0_item_real<LOG2N, T, MODE>(xa, xb, w, n);
    if (MODE != 3) emu_side<LOG2N, T, false>(w, U);
    if (MODE != 2) emu_side<LOG2N, T, true>(w, U);
    auto emit = [&](int k, vec2<T> cv, vec2<T> sv) {
        if constexpr (MODE == 1) {
            const bool edge = (k == 0) || (k == P::m);
            ya[2 * k] = cv.x;
            ya[2 * k + 1] = edge ? (T)0 : -sv.x;
            yb[2 * k] = cv.y;
            yb[2 * k + 1] = edge ? (T)0 : -sv.y;
        } else if constexpr (MODE == 2) {
            ya[k] = cv.x;
            yb[k] = cv.y;
        } else {
            if (k == 0 || k == P::m) return;
            ya[k - 1] = sv.x;
            yb[k - 1] = sv.y;
        }
    };
    for (int t = 0; t < P::DT; ++t) Chain<LOG2N, T>::unit_e(w, emit, t);
}

template <typename T, int SUBLOG, int MODE>
static int emu_large_real(int log2n, const T *xa, const T *xb, T *ya, T *yb, const T *U);

template <typename T, int MODE>
static int emu_real_dispatch(int log2n, const T *xa, const T *xb, T *ya, T *yb, const T *U) {
    const int cap = sizeof(T) == 4 ? 14 : 13;
    if (log2n > cap) {
        const int sl = log2n - 1 < cap ? log2n - 1 : cap;
        if (sl == 13) return emu_large_real<T, 13, MODE>(log2n, xa, xb, ya, yb, U);
        if (sl == 14) return emu_large_real<T, 14, MODE>(log2n, xa, xb, ya, yb, U);
        return -1;
    }
    switch (log2n) {
        case 6: emu_real_one<6, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 7: emu_real_one<7, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 8: emu_real_one<8, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 9: emu_real_one<9, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 10: emu_real_one<10, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 11: emu_real_one<11, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 12: emu_real_one<12, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 13: emu_real_one<13, T, MODE>(xa, xb, ya, yb, U); return 0;
        case 14: emu_real_one<14, T, MODE>(xa, xb, ya, yb, U); return 0;
    }
    return -1;
}

template <int NN, typename T>
static void emu_reg(const vec2<T> *x, vec2<T> *y, const T *U) {
    cdft_reg<NN, T>(x, y, U);
}

// ---------------------------------------------------------------- large N
// the multi-pass path of qft_large.cu: F passes (blocks j < J0 above the leaf
// size), the sub-signal transform of x[k 2^J0], CTA leaves, B passes, chain
template <int R, typename T>
static void emu_f_task(vec2<T> *w, const FTask &tk, int dst, const T *U, const vec2<T> *x, int N) {
    for (int t = 0; t < (tk.L >> R); ++t) {
        if (dst) lg_f_group<R, T, true>(w, tk, t, U, x, N);
        else lg_f_group<R, T, false>(w, tk, t, U, x, N);
    }
}
template <int R, typename T>
static void emu_b_task(vec2<T> **W, const BTask &tk) {
    for (int i = 0; i < (tk.L >> R); ++i) {
        if (tk.dst) lg_b_column<R, T, true>(W, tk, i);
        else lg_b_column<R, T, false>(W, tk, i);
    }
}
template <int A, typename T, bool DST>
static void emu_leaf_dst(vec2<T> *w, const LeafTask &tk, const T *U, const vec2<T> *x, int N) {
    using LT = LeafTop<A, DST, T>;
    constexpr int L = 1 << A;
    std::vector<vec2<T>> sv(L + L / 32 + 1);
    vec2<T> *s = sv.data();
    for (int e = 0; e < L; ++e) s[padx(e)] = tk.j >= 0 ? fold_load<T, DST>(x, N, tk.j, e) : w[tk.c + tk.sg * e];
    {  // TF: every item loads before any store (CTA barrier)
        std::vector<vec2<T>> v(1024 * LT::G);
        for (int t = 0; t < 1024; ++t) LT::tf_load(s, U, t, &v[t * LT::G]);
        for (int t = 0; t < 1024; ++t) LT::tf_store(s, t, &v[t * LT::G]);
    }
    for (int p = 0; p < L / 1024; ++p) emu_unit_big<1024, 5, T, DST>(s + padx(1024 * p), U);
    for (int i = 0; i < 1024; ++i) {  // TB reads shared memory only, writes the run
        vec2<T> out[LT::G];
        LT::tb(s, i, out);
        for (int q = 0; q < LT::G; ++q) w[tk.c + tk.sg * (i * LT::G + q)] = out[q];
    }
}
template <int A, typename T>
static void emu_leaf(vec2<T> *w, const LeafTask &tk, const T *U, const vec2<T> *x, int N) {
    if (tk.dst) emu_leaf_dst<A, T, true>(w, tk, U, x, N);
    else emu_leaf_dst<A, T, false>(w, tk, U, x, N);
}
template <int SUBLOG, typename T>
static void emu_sub(const vec2<T> *w0, int m, vec2<T> *cb, vec2<T> *sb, const T *U, const vec2<T> *x = nullptr) {
    using P = SPlan<SUBLOG>;
    std::vector<vec2<T>> Wv(P::PADDED);
    vec2<T> *w = Wv.data();
    if (x) {  // no fold pass: fold the sub-signal x[k 2^J0] while loading (sub_item)
        int J0 = 0;
        while ((P::m << J0) < m) ++J0;
        for (int k = 0; k < P::m; ++k) {
            const vec2<T> a = x[k << J0], b = x[k ? 2 * m - (k << J0) : m];
            if (k == 0) {
                w[padx(P::BASE)] = a;
                w[padx(P::BASE + 1)] = b;
            } else {
                const int jj = ctz32((uint32_t)k);
                const int cell = P::m - (1 << (SUBLOG - 1 - jj)) + (k >> (jj + 1));
                w[padx(cell)] = vadd(a, b);
                w[padx(P::S0 + cell)] = sine_cell(a, b, cell);
            }
        }
    } else {
    // the folded blocks j >= J0 of W0 are the sub-signal's blocks (sub_item)
    for (int c = 0; c < P::m - 1; ++c) {
        w[padx(c)] = w0[m - P::m + c];
        w[padx(P::S0 + c)] = w0[2 * m - P::m + c];
    }
    w[padx(P::BASE)] = w0[2 * m - 1];
    w[padx(P::BASE + 1)] = w0[2 * m];
    if (QFT_SC)  // the single-pass layout holds the odd sine cells negated (sub_item)
        for (int c = 1; c < P::m - 1; c += 2) w[padx(P::S0 + c)] = vec2<T>{-w[padx(P::S0 + c)].x, -w[padx(P::S0 + c)].y};
    }
    emu_side<SUBLOG, T, false>(w, U);
    emu_side<SUBLOG, T, true>(w, U);
    auto emit = [&](int k, vec2<T> cv, vec2<T> sv) {
        cb[k] = cv;
        sb[k] = sv;
    };
    for (int t = 0; t < P::DT; ++t) Chain<SUBLOG, T>::unit_e(w, emit, t);
}

template <typename T, int SUBLOG>
static int emu_large(int log2n, const vec2<T> *x, vec2<T> *y, const T *U) {
    const int J0 = log2n - SUBLOG, RG = 5;
    // complex plans fold on load (no fold pass) for fp32 with J0 <= 2 (qft_large.cu fold_on_load)
    LargeSchedule S(log2n, SUBLOG, RG, J0, !(sizeof(T) == 4 && J0 <= 2));
    const int N = S.N, mj0 = 1 << (SUBLOG - 1);
    const long long Ws = N + 2 + 2 * (mj0 + 1);
    std::vector<vec2<T>> W0(Ws), W1(Ws);
    vec2<T> *W[2] = {W0.data(), W1.data()};
    if (S.fold)
        for (int n = 0; n < N / 2; n += 1 << S.jfold) lg_fold_item<T>(x, W[0], n, N, log2n);  // fold pass (blocks j >= jfold)
    for (auto &lvl : S.f)
        for (auto &kv : lvl)
            for (auto &td : kv.second) {
                switch (kv.first) {
                    case 1: emu_f_task<1, T>(W[0], td.first, td.second, U, x, N); break;
                    case 2: emu_f_task<2, T>(W[0], td.first, td.second, U, x, N); break;
                    case 3: emu_f_task<3, T>(W[0], td.first, td.second, U, x, N); break;
                    case 4: emu_f_task<4, T>(W[0], td.first, td.second, U, x, N); break;
                    case 5: emu_f_task<5, T>(W[0], td.first, td.second, U, x, N); break;
                }
            }
    vec2<T> *cb = W[0] + (N + 2), *sb = cb + mj0 + 1;
    emu_sub<SUBLOG, T>(W[0], N / 2, cb, sb, U, S.fold ? nullptr : x);
    for (auto &kv : S.leaf) {
        if (kv.first != SUBLOG && kv.first != SUBLOG - 1) return -2;
        for (auto &tk : kv.second) {
            if (kv.first == SUBLOG) emu_leaf<SUBLOG, T>(W[0], tk, U, x, N);
            else emu_leaf<SUBLOG - 1, T>(W[0], tk, U, x, N);
        }
    }
    for (int d = (int)S.b.size() - 1; d >= 0; --d)
        for (auto &kv : S.b[d])
            for (auto &tk : kv.second) {
                switch (kv.first) {
                    case 1: emu_b_task<1, T>(W, tk); break;
                    case 2: emu_b_task<2, T>(W, tk); break;
                    case 3: emu_b_task<3, T>(W, tk); break;
                    case 4: emu_b_task<4, T>(W, tk); break;
                    case 5: emu_b_task<5, T>(W, tk); break;
                }
            }
    GChain<T> g;
    g.n = log2n;
    g.N = N;
    g.m = N / 2;
    g.w0 = W[0];
    g.w1 = W[1];
    g.x = x;
    g.cmask = S.cmask;
    g.smask = S.smask;
    g.J0 = J0;
    g.cb = cb;
    g.sb = sb;
    const int RC = J0 < 4 ? J0 : 4;
    for (int t = 0; t <= (N >> (RC + 1)); ++t) {
        switch (RC) {
            case 1: g.template unit<1>(y, t); break;
            case 2: g.template unit<2>(y, t); break;
            case 3: g.template unit<3>(y, t); break;
            case 4: g.template unit<4>(y, t); break;
        }
    }
    return 0;
}
// real modes through the multi-pass path: fold pass over every block (no
// first touch), same items / B passes, real-mode chain emit
template <typename T, int SUBLOG, int MODE>
static int emu_large_real(int log2n, const T *xa, const T *xb, T *ya, T *yb, const T *U) {
    const int J0 = log2n - SUBLOG, RG = 5;
    LargeSchedule S(log2n, SUBLOG, RG, J0, true, false);
    const int N = S.N, mj0 = 1 << (SUBLOG - 1);
    const long long Ws = N + 2 + 2 * (mj0 + 1);
    std::vector<vec2<T>> W0(Ws), W1(Ws);
    vec2<T> *W[2] = {W0.data(), W1.data()};
    for (int n = 0; n < N / 2; ++n) lg_fold_real_item<T, MODE>(xa, xb, W[0], n, N, log2n);
    for (auto &lvl : S.f)
        for (auto &kv : lvl)
            for (auto &td : kv.second) {
                switch (kv.first) {
                    case 1: emu_f_task<1, T>(W[0], td.first, td.second, U, nullptr, N); break;
                    case 2: emu_f_task<2, T>(W[0], td.first, td.second, U, nullptr, N); break;
                    case 3: emu_f_task<3, T>(W[0], td.first, td.second, U, nullptr, N); break;
                    case 4: emu_f_task<4, T>(W[0], td.first, td.second, U, nullptr, N); break;
                    case 5: emu_f_task<5, T>(W[0], td.first, td.second, U, nullptr, N); break;
                }
            }
    vec2<T> *cb = W[0] + (N + 2), *sb = cb + mj0 + 1;
    emu_sub<SUBLOG, T>(W[0], N / 2, cb, sb, U);
    for (auto &kv : S.leaf)
        for (auto &tk : kv.second) {
            if (kv.first == SUBLOG) emu_leaf<SUBLOG, T>(W[0], tk, U, nullptr, N);
            else emu_leaf<SUBLOG - 1, T>(W[0], tk, U, nullptr, N);
        }
    for (int d = (int)S.b.size() - 1; d >= 0; --d)
        for (auto &kv : S.b[d])
            for (auto &tk : kv.second) {
                switch (kv.first) {
                    case 1: emu_b_task<1, T>(W, tk); break;
                    case 2: emu_b_task<2, T>(W, tk); break;
                    case 3: emu_b_task<3, T>(W, tk); break;
                    case 4: emu_b_task<4, T>(W, tk); break;
                    case 5: emu_b_task<5, T>(W, tk); break;
                }
            }
    GChain<T> g;
    g.n = log2n;
    g.N = N;
    g.m = N / 2;
    g.w0 = W[0];
    g.w1 = W[1];
    g.x = nullptr;
    g.cmask = S.cmask;
    g.smask = S.smask;
    g.J0 = J0;
    g.cb = cb;
    g.sb = sb;
    const int RC = J0 < 4 ? J0 : 4;
    // the emulator's output rows: rdft as interleaved (re, im) pairs
    for (int t = 0; t <= (N >> (RC + 1)); ++t) {
        switch (RC) {
            case 1: g.template unit_real<1, MODE>(ya, yb, true, t); break;
            case 2: g.template unit_real<2, MODE>(ya, yb, true, t); break;
            case 3: g.template unit_real<3, MODE>(ya, yb, true, t); break;
            case 4: g.template unit_real<4, MODE>(ya, yb, true, t); break;
        }
    }
    return 0;
}

// sub-signal size of the device plan (qft_large.cu sublog_for)
template <typename T>
static int emu_large_any(int log2n, const vec2<T> *x, vec2<T> *y, const T *U) {
    const int cap = sizeof(T) == 4 ? 14 : 13;
    const int sl = log2n - 1 < cap ? log2n - 1 : cap;
    switch (sl) {
        case 12: return emu_large<T, 12>(log2n, x, y, U);
        case 13: return emu_large<T, 13>(log2n, x, y, U);
        case 14: return emu_large<T, 14>(log2n, x, y, U);
    }
    return -1;
}

template <typename T>
static int emu_dispatch(int log2n, const vec2<T> *x, vec2<T> *y, const T *U) {
    switch (log2n) {
        case 1: emu_reg<2, T>(x, y, U); return 0;
        case 2: emu_reg<4, T>(x, y, U); return 0;
        case 3: emu_reg<8, T>(x, y, U); return 0;
        case 4: emu_reg<16, T>(x, y, U); return 0;
        case 5: emu_reg<32, T>(x, y, U); return 0;
        case 6: emu_one<6, T>(x, y, U); return 0;
        case 7: emu_one<7, T>(x, y, U); return 0;
        case 8: emu_one<8, T>(x, y, U); return 0;
        case 9: emu_one<9, T>(x, y, U); return 0;
        case 10: emu_one<10, T>(x, y, U); return 0;
        case 11: emu_one<11, T>(x, y, U); return 0;
        case 12: emu_one<12, T>(x, y, U); return 0;
        case 13: emu_one<13, T>(x, y, U); return 0;
        case 14: emu_one<14, T>(x, y, U); return 0;
        default:
            if (log2n < 13 || log2n > 20) return -1;
            return emu_large_any<T>(log2n, x, y, U);
    }
}

template <typename T>
static int emu_real(int mode, int log2n, const T *x, T *y, long nrows, const T *Tnat) {
    const int N = 1 << log2n, m = N / 2;
    const int rl = mode == 1 ? N : (mode == 2 ? m + 1 : m - 1);
    const int ol = mode == 1 ? 2 * (m + 1) : rl;
    std::vector<T> U;
    build_U(N, Tnat, U);
    for (long r = 0; r + 1 < nrows; r += 2) {
        const T *xa = x + r * rl, *xb = xa + rl;
        T *ya = y + r * ol, *yb = ya + ol;
        int rc = mode == 1 ? emu_real_dispatch<T, 1>(log2n, xa, xb, ya, yb, U.data())
               : mode == 2 ? emu_real_dispatch<T, 2>(log2n, xa, xb, ya, yb, U.data())
                           : emu_real_dispatch<T, 3>(log2n, xa, xb, ya, yb, U.data());
        if (rc) return rc;
    }
    return 0;
}

extern "C" {
// multi-pass schedule emulation for any N = 2^13 .. 2^20
int emu_large_f64(int log2n, const double *x, double *y, long batch, const double *Tnat) {
    std::vector<double> U;
    build_U(1 << log2n, Tnat, U);
    for (long b = 0; b < batch; ++b) {
        const long o = 2L * (1L << log2n) * b;
        int rc = emu_large_any<double>(log2n, (const vec2<double> *)(x + o), (vec2<double> *)(y + o), U.data());
        if (rc) return rc;
    }
    return 0;
}
int emu_large_f32(int log2n, const float *x, float *y, long batch, const float *Tnat) {
    std::vector<float> U;
    build_U(1 << log2n, Tnat, U);
    for (long b = 0; b < batch; ++b) {
        const long o = 2L * (1L << log2n) * b;
        int rc = emu_large_any<float>(log2n, (const vec2<float> *)(x + o), (vec2<float> *)(y + o), U.data());
        if (rc) return rc;
    }
    return 0;
}
int emu_real_f32(int mode, int log2n, const float *x, float *y, long nrows, const float *T) {
    return emu_real<float>(mode, log2n, x, y, nrows, T);
}
int emu_real_f64(int mode, int log2n, const double *x, double *y, long nrows, const double *T) {
    return emu_real<double>(mode, log2n, x, y, nrows, T);
}
// x, y: batch-major interleaved complex; Tnat: natural table for N (N >= 8)
int emu_cdft_f64(int log2n, const double *x, double *y, long batch, const double *Tnat) {
    const int N = 1 << log2n;
    std::vector<double> U;
    double dummy[2] = {0, 0};
    if (N >= 8) build_U(N, Tnat, U); else U.assign(dummy, dummy + 2);
    for (long b = 0; b < batch; ++b) {
        int rc = emu_dispatch<double>(log2n, (const vec2<double> *)(x + 2L * N * b),
                                      (vec2<double> *)(y + 2L * N * b), U.data());
        if (rc) return rc;
    }
    return 0;
}
int emu_cdft_f32(int log2n, const float *x, float *y, long batch, const float *Tnat) {
    const int N = 1 << log2n;
    std::vector<float> U;
    float dummy[2] = {0, 0};
    if (N >= 8) build_U(N, Tnat, U); else U.assign(dummy, dummy + 2);
    for (long b = 0; b < batch; ++b) {
        int rc = emu_dispatch<float>(log2n, (const vec2<float> *)(x + 2L * N * b),
                                     (vec2<float> *)(y + 2L * N * b), U.data());
        if (rc) return rc;
    }
    return 0;
}
}
