// qft_smem.cuh -- single-CTA improved-QFT of one length-N complex signal held
// in shared memory (N = 2^6 .. 2^12 fp32, 2^6 .. 2^11 fp64).
//
// Working layout W (vec2 cells, padded address p + p/32 to break bank
// conflicts of stride-32 accesses):
//   C region [0, m]     : Lee block j (cosine, L_j = N/2^(j+2)) at off_j = m - 2L_j,
//                         base pair s(0), s(m) at m-1, m
//   S region [m+1, N)   : Lee block j (sine) at m+1+off_j
//   tail     [N, N+32)  : C_JC (17 cells) and S_JC (15 cells), the cosine/sine
//                         spectra of the 32-point sub-problem (JC = LOG2N-5)
// Sample n = 2^j (2i+1) of the folded signal is element i of Lee block j: this
// is the time-parity chain of improved._dct / _dst (improved.py:43, :81)
// unrolled, with no arithmetic.
//
// Phases (one __syncthreads between phases):
//   A0  fold x[n] +- x[N-n] and route (shared.py:28-35)            global -> W
//   A   RF forward levels of each big block (L > 32), in place        W -> W
//   B   full Lee DCT-II/DST-II of every 32-cell sub-block and of the
//       small blocks; the 32-point tail (improved.py:36-112)          W -> W
//   C   RF backward levels of each big block (one warp per block)     W -> W
//   D   time-split chain (elaborations.py:329-340) for the top RC levels,
//       complex recombination (shared.py:58-72)                     W -> global
#pragma once
#include "qft_lee.cuh"

namespace qft {

QFT_HD int padx(int p) { return p + (p >> 5); }

template <int LOG2N>
struct SPlan {
    static constexpr int N = 1 << LOG2N, m = N / 2, q = N / 4;
    static constexpr int JC = LOG2N - 5;                    // tail level (N_JC = 32)
    static constexpr int JF = LOG2N > 7 ? LOG2N - 7 : 0;    // blocks j < JF are big (L > 32)
    static constexpr int RC = JC < 4 ? JC : 4;              // chain levels unfolded in phase D
    static constexpr int L(int j) { return 1 << (LOG2N - 2 - j); }
    static constexpr int off(int j) { return m - 2 * L(j); }
    static constexpr int RF(int j) { return LOG2N - 7 - j; }  // big block: L = 32 << RF
    static constexpr int TAIL = N;                          // tail cells
    static constexpr int W_CELLS = N + 32;
    static constexpr int W_PADDED = W_CELLS + W_CELLS / 32 + 1;
    // phase B units: big sub-blocks (both sides), small blocks (both sides), tail
    static constexpr int NSUB = JF > 0 ? (1 << (LOG2N - 6)) - 2 : 0;  // per side: sum 2^RF(j)
    static constexpr int NSMALL = JC - JF;                  // per side
    static constexpr int NB_UNITS = 2 * NSUB + 2 * NSMALL + 1;
    static constexpr int MRC = N >> (RC + 1);               // phase D threads: t in [0, MRC]
    static constexpr int UCELLS = N / 4;                    // level-table entries
};

// ---------------------------------------------------------------- phase A0
template <int LOG2N, typename T>
QFT_HD void a0_item(const vec2<T> *x, vec2<T> *w, int n) {
    using P = SPlan<LOG2N>;
    if (n == 0) {
        w[padx(P::m - 1)] = x[0];  // dc[0] = x[0]
    } else if (n == P::m) {
        w[padx(P::m)] = x[P::m];   // dc[m] = x[m]
    } else {
        vec2<T> a = x[n], b = x[P::N - n];
        const int j = ctz32((uint32_t)n);
        const int i = n >> (j + 1);
        const int off = P::m - 2 * (1 << (LOG2N - 2 - j));
        w[padx(off + i)] = vadd(a, b);              // dc[n]   = x[n] + x[N-n]
        w[padx(P::m + 1 + off + i)] = vsub(a, b);   // ds[n-1] = x[n] - x[N-n]
    }
}

// ---------------------------------------------------------------- phase A
template <int LOG2N, int J, bool DST, typename T>
QFT_HD void f_unit(vec2<T> *w, const T *U, int t) {
    using P = SPlan<LOG2N>;
    constexpr int L = P::L(J), R = P::RF(J), G = 1 << R;
    constexpr int base = (DST ? P::m + 1 : 0) + P::off(J);
    vec2<T> v[G];
#pragma unroll
    for (int s = 0; s < G; ++s) {
        int c, sg;
        run_of(R, L, s, c, sg);
        v[s] = w[padx(base + c + sg * t)];
    }
    lee_fwd<R, L, DST, T>(v, t, U);
#pragma unroll
    for (int s = 0; s < G; ++s) {
        int c, sg;
        run_of(R, L, s, c, sg);
        w[padx(base + c + sg * t)] = v[s];
    }
}

// ---------------------------------------------------------------- phase B
template <int L, bool DST, typename T>
QFT_HD void full_run(vec2<T> *w, int base, int c, int sg, const T *U) {
    vec2<T> v[L];
#pragma unroll
    for (int e = 0; e < L; ++e) v[e] = w[padx(base + c + sg * e)];
    lee_full<L, DST, T>(v, U);
#pragma unroll
    for (int e = 0; e < L; ++e) w[padx(base + c + sg * e)] = v[e];
}

// cell of dc sample n (0 <= n <= m) / ds sample n (1 <= n < m) in W
template <int LOG2N>
QFT_HD int dc_cell(int n) {
    using P = SPlan<LOG2N>;
    if (n == 0) return P::m - 1;
    if (n == P::m) return P::m;
    const int j = ctz32((uint32_t)n);
    return P::m - 2 * (1 << (LOG2N - 2 - j)) + (n >> (j + 1));
}
template <int LOG2N>
QFT_HD int ds_cell(int n) {
    using P = SPlan<LOG2N>;
    const int j = ctz32((uint32_t)n);
    return P::m + 1 + P::m - 2 * (1 << (LOG2N - 2 - j)) + (n >> (j + 1));
}

template <int LOG2N, typename T>
QFT_HD void tail_unit(vec2<T> *w, const T *U) {
    using P = SPlan<LOG2N>;
    constexpr int ST = 1 << P::JC;  // sample stride of the 32-point sub-problem
    vec2<T> xc[17], xs[15], oc[17], os[15];
#pragma unroll
    for (int k = 0; k <= 16; ++k) xc[k] = w[padx(dc_cell<LOG2N>(k * ST))];
#pragma unroll
    for (int k = 1; k <= 15; ++k) xs[k - 1] = w[padx(ds_cell<LOG2N>(k * ST))];
    dct0_reg<32, T>(xc, oc, U);
    dst0_reg<32, T>(xs, os, U);
#pragma unroll
    for (int k = 0; k <= 16; ++k) w[padx(P::TAIL + k)] = oc[k];
#pragma unroll
    for (int k = 0; k < 15; ++k) w[padx(P::TAIL + 17 + k)] = os[k];
}

template <int LOG2N, int J, typename T>
QFT_HD void b_big_dispatch(vec2<T> *w, const T *U, int pp, bool dst) {
    using P = SPlan<LOG2N>;
    if constexpr (J < P::JF) {
        constexpr int G = 1 << P::RF(J);
        if (pp < G) {
            // after phase A, sub-block pp is the run c0 + sg0*e, e in [0, 32)
            int c0, sg0;
            run_of(P::RF(J), P::L(J), pp, c0, sg0);
            if (dst) full_run<32, true, T>(w, P::m + 1 + P::off(J), c0, sg0, U);
            else full_run<32, false, T>(w, P::off(J), c0, sg0, U);
        } else {
            b_big_dispatch<LOG2N, J + 1, T>(w, U, pp - G, dst);
        }
    }
}

template <int LOG2N, int J, typename T>
QFT_HD void b_small_dispatch(vec2<T> *w, const T *U, int jj, bool dst) {
    using P = SPlan<LOG2N>;
    if constexpr (J < P::JC) {
        if (jj == J) {
            constexpr int L = P::L(J);
            if (dst) full_run<L, true, T>(w, P::m + 1 + P::off(J), 0, 1, U);
            else full_run<L, false, T>(w, P::off(J), 0, 1, U);
        } else {
            b_small_dispatch<LOG2N, J + 1, T>(w, U, jj, dst);
        }
    }
}

template <int LOG2N, typename T>
QFT_HD void b_unit(vec2<T> *w, const T *U, int u) {
    using P = SPlan<LOG2N>;
    if (u < 2 * P::NSUB) {
        const bool dst = u >= P::NSUB;
        b_big_dispatch<LOG2N, 0, T>(w, U, dst ? u - P::NSUB : u, dst);
    } else if (u < 2 * P::NSUB + 2 * P::NSMALL) {
        const int v = u - 2 * P::NSUB;
        const bool dst = v >= P::NSMALL;
        b_small_dispatch<LOG2N, P::JF, T>(w, U, P::JF + (dst ? v - P::NSMALL : v), dst);
    } else {
        tail_unit<LOG2N, T>(w, U);
    }
}

// ---------------------------------------------------------------- phase C
template <int LOG2N, int J, bool DST, typename T>
struct BUnit {
    using P = SPlan<LOG2N>;
    static constexpr int L = P::L(J), R = P::RF(J), G = 1 << R;
    static constexpr int base = (DST ? P::m + 1 : 0) + P::off(J);
    vec2<T> own[G], halo[G];

    QFT_HD void load(const vec2<T> *w, int i) {
        const int ih = DST ? i - 1 : i + 1;
        const bool has_halo = ih >= 0 && ih < 32;
#pragma unroll
        for (int p = 0; p < G; ++p) {
            int c, sg;
            run_of(R, L, p, c, sg);
            own[p] = w[padx(base + c + sg * i)];
            if (p > 0) halo[p] = has_halo ? w[padx(base + c + sg * ih)] : own[p];
        }
        halo[0] = own[0];
    }
    QFT_HD void store(vec2<T> *w, int i) const {
        vec2<T> out[G];
        const bool edge = DST ? (i == 0) : (i == 31);
        lee_bwd<R, DST, T>(own, halo, edge, out);
#pragma unroll
        for (int s = 0; s < G; ++s) w[padx(base + i * G + s)] = out[s];
    }
};

// ---------------------------------------------------------------- phase D
template <int LOG2N, typename T>
struct Chain {
    using P = SPlan<LOG2N>;
    static QFT_HD vec2<T> OC(const vec2<T> *w, int j, int k) { return w[padx(P::m - 2 * (1 << (LOG2N - 2 - j)) + k)]; }
    // sine spectrum of block j at harmonic h (slot h-1)
    static QFT_HD vec2<T> OS(const vec2<T> *w, int j, int h) {
        return w[padx(P::m + 1 + P::m - 2 * (1 << (LOG2N - 2 - j)) + h - 1)];
    }

    // C_J[k] for 0 <= k <= m_J, descending the chain to the tail
    template <int J>
    static QFT_HD vec2<T> descC(const vec2<T> *w, int k) {
        if constexpr (J == P::JC) {
            return w[padx(P::TAIL + k)];
        } else {
            constexpr int qj = 1 << (LOG2N - 2 - J), mj = 2 * qj;
            const int kk = k <= qj ? k : mj - k;
            vec2<T> e = descC<J + 1>(w, kk);
            if (k == qj) return e;                   // out[q] = E[q]
            vec2<T> o = OC(w, J, kk);
            return k < qj ? vadd(e, o) : vsub(e, o);  // E+O / E-O
        }
    }
    // S_J[k] for 1 <= k <= m_J - 1 (other k: unused garbage, in-bounds reads)
    template <int J>
    static QFT_HD vec2<T> descS(const vec2<T> *w, int k) {
        if constexpr (J == P::JC) {
            return w[padx(P::TAIL + 17 + (k > 0 ? k - 1 : 0))];
        } else {
            constexpr int qj = 1 << (LOG2N - 2 - J), mj = 2 * qj;
            if (k == qj) return OS(w, J, qj);          // out[q-1] = O[q-1]
            const int kk = k < qj ? k : mj - k;
            vec2<T> e = descS<J + 1>(w, kk);
            vec2<T> o = OS(w, J, kk);
            return k < qj ? vadd(o, e) : vsub(o, e);  // O+E / O-E
        }
    }

    static QFT_HD void emit(vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) {
        if (k == 0 || k == P::m) {
            y[k] = cv;
        } else {
            vec2<T> lo, hi;
            recombine(cv, sv, lo, hi);
            y[k] = lo;
            y[P::N - k] = hi;
        }
    }

    template <int J>
    static QFT_HD void up(const vec2<T> *w, vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) {
        if constexpr (J == 0) {
            emit(y, k, cv, sv);
        } else {
            constexpr int qj = 1 << (LOG2N - 2 - (J - 1)), mj = 2 * qj;
            const bool self = (k == qj);
            vec2<T> o = OC(w, J - 1, self ? 0 : k);
            vec2<T> os = OS(w, J - 1, k);
            vec2<T> clo = self ? cv : vadd(cv, o);
            vec2<T> chi = self ? cv : vsub(cv, o);
            vec2<T> slo = self ? os : vadd(os, sv);
            vec2<T> shi = self ? os : vsub(os, sv);
            up<J - 1>(w, y, k, clo, slo);
            up<J - 1>(w, y, self ? qj : mj - k, chi, shi);
        }
    }

    static QFT_HD void unit(const vec2<T> *w, vec2<T> *y, int t) {
        vec2<T> cv = descC<P::RC>(w, t);
        vec2<T> sv = descS<P::RC>(w, t);
        up<P::RC>(w, y, t, cv, sv);
    }
};

}  // namespace qft
