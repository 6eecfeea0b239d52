// qft_large.cuh -- device phases of the multi-pass path (N > 2^14 fp32 / 2^13 fp64).
//
// Signals larger than one SM's shared memory are cut along the improved
// recursion itself (qft_large.cu): the Lee blocks j >= J0 are the blocks of the
// sub-signal transform of x[k 2^J0] (single-pass machinery, qft_launch.cuh),
// blocks of 2^SUBLOG cells or less are CTA-resident leaves (qft_leaf.cuh), and
// only blocks larger than that are cut in HBM by the passes here:
//   fold   x -> W0: x[n] +- x[N-n] routed to Lee block j = ctz(n) (shared.py:28-35)
//   F(d)   in-place forward fold levels (r <= 5 per pass; fp64 r = 5 on lane pairs) of every
//          block larger than the leaf size; the first touch folds x on load;
//          each pass leaves 2^r sub-blocks as contiguous (possibly reversed)
//          runs of the same cells
//   B(d)   backward levels (neighbour sums + interleave), deepest first,
//          ping-pong W0 <-> W1, output in natural spectrum order
//   chain  time-split chain levels J0-1 .. 0 + complex recombination -> y
//          (elaborations.py:78-89, shared.py:58-72)
// The host plan builder (qft_large_plan.h) compiles the decomposition tree of
// the reference recursion into these task lists.
#pragma once
#include "qft_lee.cuh"

namespace qft {

// ----------------------------------------------------------------- tasks
struct FTask {        // r forward levels of one run (in place)
    int c, sg, L;     // run: element e at cell c + sg*e
    int j;            // >= 0: the run is all of Lee block j -> fold x on load (no fold pass)
};
struct LeafTask {     // full Lee of one run (in place, spectrum along the run)
    int c, sg, L, dst;
    int j;            // >= 0: all of Lee block j, folded on first touch (-1: a run already in W0)
};

// element i of Lee block j read straight from the input: sample n = 2^j (2i+1),
// dc = x[n] + x[N-n], ds = x[n] - x[N-n] (shared.py:28-35)
template <typename T, bool DST>
QFT_HD vec2<T> fold_load(const vec2<T> *x, int N, int j, int i) {
    const int n = (2 * i + 1) << j;
    const vec2<T> a = x[n], b = x[N - n];
    return DST ? vsub(a, b) : vadd(a, b);
}
struct BTask {        // r backward levels: 2^r sub-block spectra -> natural block spectrum
    int c, sg, L;     // parent run (its sub-blocks are the runs of run_of(r, L, p))
    int in_buf, leaf; // sub-block spectra in W[in_buf]; leaf: along each run, else forward at its min cell
    int out_buf, out0;  // block spectrum written to W[out_buf] cells [out0, out0 + L)
    int dst;
};

// runtime-L forward levels (lee_fwd with a runtime block size)
template <int R, typename T, bool DST>
QFT_HD void lee_fwd_rt(vec2<T> *v, int t, int L, const T *U) {
    if constexpr (R > 0) {
        constexpr int G = 1 << R, H = G / 2;
        vec2<T> nv[G];
#pragma unroll
        for (int s = 0; s < H; ++s) {
            int c, sg;
            run_of(R - 1, L / 2, s, c, sg);
            const int i = c + sg * t;
            vec2<T> a = v[s], b = v[G - 1 - s];
            const T k = U[L / 2 + i];
            if constexpr (!DST) {
                nv[s] = vadd(a, b);
                nv[H + s] = vmul(vsub(a, b), k);
            } else {
                nv[s] = vsub(a, b);
                nv[H + s] = vmul(vadd(a, b), k);
            }
        }
        lee_fwd_rt<R - 1, T, DST>(nv, t, L / 2, U);
        lee_fwd_rt<R - 1, T, DST>(nv + H, t, L / 2, U);
#pragma unroll
        for (int s = 0; s < G; ++s) v[s] = nv[s];
    }
}

// ----------------------------------------------------------------- fold
// cells: cosine block j at m - 2^(n-1-j) + i, sine at m + same, s(0) at N-1, s(m) at N
template <typename T>
QFT_HD void lg_fold_item(const vec2<T> *x, vec2<T> *w, int n, int N, int log2n) {
    const int m = N / 2;
    if (n == 0) {
        w[N - 1] = x[0];
        w[N] = x[m];
    } else {
        vec2<T> a = x[n], b = x[N - n];
        const int j = ctz32((uint32_t)n);
        const int cell = m - (1 << (log2n - 1 - j)) + (n >> (j + 1));
        w[cell] = vadd(a, b);
        w[m + cell] = vsub(a, b);
    }
}

// ----------------------------------------------------------------- F pass
// ld(s, e): the value of slot s (element e of the block) before the first level
template <int R, typename T, bool DST, class Ld>
QFT_HD void lg_f_group_ld(vec2<T> *w, const FTask &tk, int t, const T *U, Ld &&ld) {
    constexpr int G = 1 << R;
    vec2<T> v[G];
#pragma unroll
    for (int s = 0; s < G; ++s) {
        int c, sg;
        run_of(R, tk.L, s, c, sg);
        v[s] = ld(s, c + sg * t);
    }
    lee_fwd_rt<R, T, DST>(v, t, tk.L, U);
#pragma unroll
    for (int s = 0; s < G; ++s) {  // slot s keeps its cells (in place)
        int c, sg;
        run_of(R, tk.L, s, c, sg);
        w[tk.c + tk.sg * (c + sg * t)] = v[s];
    }
}
template <int R, typename T, bool DST>
QFT_HD void lg_f_group(vec2<T> *w, const FTask &tk, int t, const T *U, const vec2<T> *x = nullptr, int N = 0) {
    constexpr int G = 1 << R;
    vec2<T> v[G];
#pragma unroll
    for (int s = 0; s < G; ++s) {
        int c, sg;
        run_of(R, tk.L, s, c, sg);
        v[s] = tk.j >= 0 ? fold_load<T, DST>(x, N, tk.j, c + sg * t) : w[tk.c + tk.sg * (c + sg * t)];
    }
    lee_fwd_rt<R, T, DST>(v, t, tk.L, U);
#pragma unroll
    for (int s = 0; s < G; ++s) {  // slot s keeps its cells (in place)
        int c, sg;
        run_of(R, tk.L, s, c, sg);
        w[tk.c + tk.sg * (c + sg * t)] = v[s];
    }
}

#if defined(__CUDACC__)
// Five forward levels split over a lane pair (fp64: 32 cells of one thread would
// not fit its registers).  lee_fwd_rt<5> is the top fold of every slot pair
// (s, 31-s) followed by two independent 4-level problems on the even child
// (slots 0..15) and the odd child (slots 16..31); thread h of the pair forms
// child h of the top fold and runs its four levels -- the same operations on
// the same operands as lg_f_group<5>.  Both lanes of a pair must be in one warp.
// ld(s, e): the value of slot s (element e of the block) before the first level
template <typename T, bool DST, class Ld>
QFT_DEV void lg_f_pair5_ld(vec2<T> *w, const FTask &tk, int t, int h, const T *U, Ld &&ld) {
    constexpr int R = 5, G = 32, H = 16;
    const int L = tk.L;
    auto at = [&](int s) {
        int c, sg;
        run_of(R, L, s, c, sg);
        return c + sg * t;
    };
    vec2<T> nv[H];
#pragma unroll
    for (int s = 0; s < H; ++s) {
        const int ea = at(s), eb = at(G - 1 - s);
        const vec2<T> a = ld(s, ea);
        const vec2<T> b = ld(G - 1 - s, eb);
        int c, sg;
        run_of(R - 1, L / 2, s, c, sg);
        const T k = U[L / 2 + c + sg * t];
        const vec2<T> sum = vadd(a, b), dif = vsub(a, b);
        if constexpr (!DST) nv[s] = h ? vmul(dif, k) : sum;
        else nv[s] = h ? vmul(sum, k) : dif;
    }
    lee_fwd_rt<R - 1, T, DST>(nv, t, L / 2, U);
    __syncwarp();  // every lane's loads of the run precede the in-place stores
#pragma unroll
    for (int s = 0; s < H; ++s) w[tk.c + tk.sg * at(h * H + s)] = nv[s];
}
template <typename T, bool DST>
QFT_DEV void lg_f_pair5(vec2<T> *w, const FTask &tk, int t, int h, const T *U, const vec2<T> *x, int N) {
    lg_f_pair5_ld<T, DST>(w, tk, t, h, U, [&](int, int e) {
        return tk.j >= 0 ? fold_load<T, DST>(x, N, tk.j, e) : w[tk.c + tk.sg * e];
    });
}

#endif  // __CUDACC__

// ----------------------------------------------------------------- B pass
template <int R, typename T, bool DST>
QFT_HD void lg_b_column_out(vec2<T> *const *W, const BTask &tk, int i, vec2<T> *out) {
    constexpr int G = 1 << R;
    const int S = tk.L >> R;
    const vec2<T> *src = W[tk.in_buf];
    vec2<T> own[G], hal[G];
    const int ih = DST ? (i > 0 ? i - 1 : i) : (i < S - 1 ? i + 1 : i);
#pragma unroll
    for (int p = 0; p < G; ++p) {
        int c, sg;
        run_of(R, tk.L, p, c, sg);
        const int rc = tk.c + tk.sg * c, rs = tk.sg * sg;  // sub-block run
        int st, dir;
        if (tk.leaf) {
            st = rc;
            dir = rs;
        } else {
            st = rs > 0 ? rc : rc - (S - 1);
            dir = 1;
        }
        own[p] = src[st + dir * i];
        hal[p] = src[st + dir * ih];
    }
    auto halo = [&](int p) { return hal[p]; };
    const bool edge = DST ? (i == 0) : (i == S - 1);
    lee_bwd_fn<R, DST, T>(own, 0, halo, edge, out);
}
#if defined(__CUDACC__)
// Five backward levels of column i split over a lane pair (the inverse of
// lg_f_pair5): thread h runs the four levels of child h (sub-blocks 16h..16h+15),
// the pair swaps the halves the top level's interleave needs (shfl_xor 16), and
// thread h emits the block spectrum slots [16h, 16h+16) of the column -- the
// same operations on the same operands as lg_b_column_out<5>.
template <typename T, bool DST>
QFT_DEV void lg_b_pair5_out(vec2<T> *const *W, const BTask &tk, int i, int h, vec2<T> *out) {
    constexpr int R = 5, H = 16;
    const int S = tk.L >> R;
    const vec2<T> *src = W[tk.in_buf];
    const int ih = DST ? (i > 0 ? i - 1 : i) : (i < S - 1 ? i + 1 : i);
    auto addr = [&](int p, int col) {
        int c, sg;
        run_of(R, tk.L, p, c, sg);
        const int rc = tk.c + tk.sg * c, rs = tk.sg * sg;
        return tk.leaf ? rc + rs * col : (rs > 0 ? rc : rc - (S - 1)) + col;
    };
    vec2<T> own[H], hal[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
        own[q] = src[addr(h * H + q, i)];
        hal[q] = src[addr(h * H + q, ih)];
    }
    // the top level's halo: the leftmost leaf of the odd child (thread 1 has it)
    const vec2<T> hv = DST ? src[addr(H, ih)] : hal[0];
    auto halo = [&](int p) { return hal[p - h * H]; };
    const bool edge = DST ? (i == 0) : (i == S - 1);
    vec2<T> r[H];  // child h: e (h = 0) or o (h = 1)
    lee_bwd_fn<R - 1, DST, T>(own, h * H, halo, edge, r);
    // swap: thread 0 gets o[0..8], thread 1 gets e[8..16)
    vec2<T> rcv[H / 2 + 1];
#pragma unroll
    for (int q = 0; q <= H / 2; ++q) {
        const vec2<T> snd = h ? r[q] : r[q < H / 2 ? H / 2 + q : H - 1];
        rcv[q].x = __shfl_xor_sync(0xffffffffu, snd.x, 16);
        rcv[q].y = __shfl_xor_sync(0xffffffffu, snd.y, 16);
    }
    if constexpr (!DST) {
        // out[2t] = e[t], out[2t+1] = o[t] + o[t+1], out[31] = o[15] (+ halo)
        if (h == 0) {
#pragma unroll
            for (int t = 0; t < H / 2; ++t) {
                out[2 * t] = r[t];
                out[2 * t + 1] = vadd(rcv[t], rcv[t + 1]);
            }
        } else {
#pragma unroll
            for (int t = 0; t < H / 2; ++t) {
                out[2 * t] = rcv[t];
                out[2 * t + 1] = t < H / 2 - 1 ? vadd(r[H / 2 + t], r[H / 2 + t + 1]) : (edge ? r[H - 1] : vadd(r[H - 1], hv));
            }
        }
    } else {
        // out[2t+1] = e[t], out[2t] = o[t-1] + o[t], out[0] = (halo +) o[0]
        if (h == 0) {
            out[0] = edge ? rcv[0] : vadd(hv, rcv[0]);
#pragma unroll
            for (int t = 1; t < H / 2; ++t) out[2 * t] = vadd(rcv[t - 1], rcv[t]);
#pragma unroll
            for (int t = 0; t < H / 2; ++t) out[2 * t + 1] = r[t];
        } else {
#pragma unroll
            for (int t = 0; t < H / 2; ++t) {
                out[2 * t] = vadd(r[H / 2 + t - 1], r[H / 2 + t]);
                out[2 * t + 1] = rcv[t];
            }
        }
    }
}

#endif  // __CUDACC__

template <int R, typename T, bool DST>
QFT_HD void lg_b_column(vec2<T> *const *W, const BTask &tk, int i) {
    constexpr int G = 1 << R;
    vec2<T> out[G];
    lg_b_column_out<R, T, DST>(W, tk, i, out);
    vec2<T> *dst = W[tk.out_buf] + tk.out0 + i * G;
#pragma unroll
    for (int s = 0; s < G; ++s) dst[s] = out[s];
}

// ----------------------------------------------------------------- chain
// Each thread t in [0, m_RC] (m_RC = N >> (RC+1)) descends the chain from the
// DCT base to level RC (index at level J: the distance of t to the nearest
// multiple of m_{J-1}), then unfolds RC levels and writes 2^(RC+1) outputs.
// Duplicate slots (self-paired indices) write identical values twice.
template <typename T>
struct GChain {
    const vec2<T> *w0, *w1;  // scratch buffers
    const vec2<T> *x;        // the input signal: base pair s(0) = x[0], s(m) = x[m]
    uint32_t cmask, smask;   // bit j: the cosine / sine spectrum of block j is in W1
    int n, N, m;
    // J0 > 0: C_J0[k], S_J0[k] (k in [0, m_J0]) come from the sub-signal
    // transform (cb, sb) instead of the descent from the DCT base
    int J0 = 0;
    const vec2<T> *cb = nullptr, *sb = nullptr;

    QFT_HD int off(int j) const { return m - (1 << (n - 1 - j)); }
    QFT_HD vec2<T> OC(int j, int k) const { return ((cmask >> j) & 1 ? w1 : w0)[off(j) + k]; }
    QFT_HD vec2<T> OS(int j, int h) const { return ((smask >> j) & 1 ? w1 : w0)[m + off(j) + h - 1]; }
    QFT_HD int qj(int j) const { return 1 << (n - 2 - j); }

    // C_RC[t], S_RC[t]
    template <int RC>
    QFT_HD void descend(int t, vec2<T> &cv, vec2<T> &sv) const {
        // level n-1: [s0 + sm, s0 - sm] at index kk_{n-1} in {0, 1}
        auto kk = [&](int J) -> int {  // index at level J
            if (J == RC) return t;
            const int P = 2 << (n - 1 - J);  // m_{J-1}
            const int r = t & (P - 1);
            return r < P - r ? r : P - r;
        };
        int Jtop = n - 2;
        if (J0 > 0) {
            const int k0 = kk(J0);
            cv = cb[k0];
            sv = sb[k0];
            Jtop = J0 - 1;
        } else {
            const vec2<T> s0 = x[0], sm = x[m];
            cv = kk(n - 1) == 0 ? vadd(s0, sm) : vsub(s0, sm);
            sv = vec2<T>{(T)0, (T)0};
        }
#pragma unroll 20
        for (int J = Jtop; J >= RC; --J) {
            const int k = kk(J), q = qj(J);
            const int k1 = k < q ? k : 2 * q - k;  // index at level J+1
            if (k != q) {
                const vec2<T> o = OC(J, k1);
                cv = k < q ? vadd(cv, o) : vsub(cv, o);
                const vec2<T> os = OS(J, k1 > 0 ? k1 : 1);
                sv = k < q ? vadd(os, sv) : vsub(os, sv);
            } else {
                sv = OS(J, q);  // leaf; C copies
            }
        }
    }

    QFT_HD void emit(vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) const {
        if (k == 0 || k == m) {
            y[k] = cv;
        } else {
            const vec2<T> u = {sv.y, -sv.x};
            y[k] = vadd(cv, u);
            y[N - k] = vsub(cv, u);
        }
    }

    // unfold RC levels; emit(k, C_0[k], S_0[k]) for every harmonic k of the group
    template <int J, class Emit>
    QFT_HD void up_e(Emit &emit_fn, int k, vec2<T> cv, vec2<T> sv) const {
        if constexpr (J == 0) {
            emit_fn(k, cv, sv);
        } else {
            const int q = qj(J - 1), mm = 2 * q;
            const bool self = (k == q);
            const vec2<T> o = OC(J - 1, self ? 0 : k);
            const vec2<T> os = OS(J - 1, k > 0 ? k : 1);
            const vec2<T> clo = self ? cv : vadd(cv, o), chi = self ? cv : vsub(cv, o);
            const vec2<T> slo = self ? os : vadd(os, sv), shi = self ? os : vsub(os, sv);
            up_e<J - 1>(emit_fn, k, clo, slo);
            up_e<J - 1>(emit_fn, self ? q : mm - k, chi, shi);
        }
    }

    template <int RC>
    QFT_HD void unit(vec2<T> *y, int t) const {
        vec2<T> cv, sv;
        descend<RC>(t, cv, sv);
        auto e = [&](int k, vec2<T> c, vec2<T> s) { emit(y, k, c, s); };
        up_e<RC>(e, t, cv, sv);
    }
    // real modes (MODE 1 rdft, 2 dct0, 3 dst0): the two lanes are two real rows
    // a, b (b absent when has_b is false); outputs as qft_cdft_smem's real modes
    template <int RC, int MODE>
    QFT_HD void unit_real(void *ya, void *yb, bool has_b, int t) const {
        vec2<T> cv, sv;
        descend<RC>(t, cv, sv);
        auto e = [&](int k, vec2<T> c, vec2<T> s) {
            if constexpr (MODE == 1) {  // packed half spectrum -> complex (shared.py:38-43, 94-101)
                const bool edge = (k == 0) || (k == m);
                static_cast<vec2<T> *>(ya)[k] = {c.x, edge ? (T)0 : -s.x};
                if (has_b) static_cast<vec2<T> *>(yb)[k] = {c.y, edge ? (T)0 : -s.y};
            } else if constexpr (MODE == 2) {
                static_cast<T *>(ya)[k] = c.x;
                if (has_b) static_cast<T *>(yb)[k] = c.y;
            } else {
                if (k == 0 || k == m) return;
                static_cast<T *>(ya)[k - 1] = s.x;
                if (has_b) static_cast<T *>(yb)[k - 1] = s.y;
            }
        };
        up_e<RC>(e, t, cv, sv);
    }
};

// ----------------------------------------------------------------- fold (real modes)
// Two real rows a, b of the mode's stored length as one vec2 signal, written
// into the Lee-block cell layout (the a0_item_real routing of qft_smem.cuh):
// rdft folds x[n] +- x[N-n]; dct0 / dst0 place s(n) on the cosine / sine side.
template <typename T, int MODE>
QFT_HD void lg_fold_real_item(const T *xa, const T *xb, vec2<T> *w, int n, int N, int log2n) {
    const int m = N / 2;
    auto at = [&](int i) { return vec2<T>{xa[i], xb[i]}; };
    auto cell_of = [&](int nn) {
        const int j = ctz32((uint32_t)nn);
        return m - (1 << (log2n - 1 - j)) + (nn >> (j + 1));
    };
    if constexpr (MODE == 1) {
        if (n == 0) {
            w[N - 1] = at(0);
            w[N] = at(m);
        } else {
            const vec2<T> a = at(n), b = at(N - n);
            const int c = cell_of(n);
            w[c] = vadd(a, b);
            w[m + c] = vsub(a, b);
        }
    } else if constexpr (MODE == 2) {
        if (n == 0) {
            w[N - 1] = at(0);
            w[N] = at(m);
        } else {
            w[cell_of(n)] = at(n);
        }
    } else {
        if (n > 0) w[m + cell_of(n)] = at(n - 1);
    }
}

}  // namespace qft
