// qft_smem.cuh -- improved-QFT of length-N complex signals (N = 2^6 .. 2^12)
// held in shared memory; a CTA works on T signals at a time.
//
// Working layout W of one signal (vec2 cells, padded address p + p/32 so that
// the stride-32 accesses of phases B/C are bank-conflict free):
//   [0, m-1)      cosine Lee blocks j = 0..n-2 (L_j = N/2^(j+2)) at off_j = m - 2L_j
//   [m, N-1)      sine   Lee blocks at m + off_j
//   N-1, N        the DCT base pair s(0), s(m)
// Sample n = 2^j (2i+1) of the folded signal is element i of Lee block j: the
// time-parity chain of improved._dct / _dst (improved.py:43, :81) unrolled.
//
// Phases (one __syncthreads between phases, all warps of the CTA run the same
// phase so the instruction stream is shared):
//   A0  fold x[n] +- x[N-n] and route (shared.py:28-35)           staging -> W
//   A   forward fold levels of the big blocks (L > 32); sub-blocks of 32
//       are written sub-block-major                                 W -> W
//   B   full Lee DCT-II/DST-II of every 32-cell chunk; small blocks  W -> W
//   C   backward levels of the big blocks (halo = neighbour lane)   W -> W
//   D   time-split chain (elaborations.py:329-340) + complex
//       recombination (shared.py:58-72)                          W -> global
#pragma once
#include "qft_lee.cuh"

// QFT_CHAIN_MID = k > 0: the bottom k chain levels are computed once by one warp
// in phase C (the rest by each phase-D thread's descent); 0: all by descent
#ifndef QFT_CHAIN_MID
#define QFT_CHAIN_MID 0
#endif

namespace qft {

QFT_HD constexpr int padx(int p) { return p + (p >> 5); }

template <int LOG2N>
struct SPlan {
    static constexpr int n = LOG2N, N = 1 << LOG2N, m = N / 2, q = N / 4;
    static constexpr int JF = n > 7 ? n - 7 : 0;     // big blocks j < JF (L > 32)
    static constexpr int JS = n - 6;                 // first small block (L = 16)
    static constexpr int RC = n - 2 < 4 ? n - 2 : 4; // chain levels unfolded in phase D
    static constexpr int L(int j) { return 1 << (n - 2 - j); }
    static constexpr int off(int j) { return m - 2 * L(j); }
    static constexpr int RF(int j) { return n - 7 - j; }  // big block: L = 32 << RF
    static constexpr int S0 = m;                     // sine region
    static constexpr int BASE = N - 1;               // s(0) at N-1, s(m) at N
    static constexpr int JM0 = n - 1 - QFT_CHAIN_MID;
    static constexpr int JM = QFT_CHAIN_MID ? (JM0 > RC + 1 ? JM0 : RC + 1) : n - 1;  // chain-mid level
    static constexpr int MJM = N >> (JM + 1);        // m_JM: C_JM has MJM+1 cells, S_JM MJM-1
    static constexpr int CHC = N + 1;                // C_JM cells [CHC, CHC + MJM]
    static constexpr int CHS = CHC + MJM + 1;        // S_JM harmonic h at CHS + h - 1
    static constexpr int CELLS = CHS + MJM;
    static_assert(JM > n - 2 || (1 << (n - 2 - JM)) <= 32, "chain-mid blocks must be finished by phase B");
    static constexpr int PADDED = CELLS + CELLS / 32 + 1;
    static constexpr int NL32 = n >= 7 ? m / 32 - 1 : 0;  // Lee-32 chunks per side
    static constexpr int NWU = 2 * ((JF >= 1) + (JF >= 2)); // phase A/C warp units
    static constexpr int MRC = N >> (RC + 1);        // m_RC: phase-D thread t in [0, MRC]
    static constexpr int DT = MRC + 1;               // phase D threads per signal
    static constexpr int UCELLS = N / 4;             // level-table entries
};

// ---------------------------------------------------------------- phase A0
// Unit k in [0, m/8) folds the pairs (n, N-n) for n = 8k+1 .. 8k+8 and routes
// them (shared.py:28-35); unit 0 also routes s(0), and n = m is the base s(m).
template <typename T>
QFT_HD void ld2(const vec2<T> *p, vec2<T> &a, vec2<T> &b) {  // p 16-byte aligned
#if defined(__CUDA_ARCH__)
    if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        a = {v.x, v.y};
        b = {v.z, v.w};
        return;
    }
#endif
    a = p[0];
    b = p[1];
}

// item n in [0, m): n = 0 routes s(0) and s(m); else folds the pair (n, N-n)
template <int LOG2N, typename T>
QFT_HD void a0_item(const vec2<T> *x, vec2<T> *w, int n) {
    using P = SPlan<LOG2N>;
    if (n == 0) {
        w[padx(P::BASE)] = x[0];
        w[padx(P::BASE + 1)] = x[P::m];
    } else {
        vec2<T> a = x[n], b = x[P::N - n];
        const int j = ctz32((uint32_t)n);
        const int cell = P::m - (1 << (LOG2N - 1 - j)) + (n >> (j + 1));  // off_j + i
        w[padx(cell)] = vadd(a, b);              // dc[n]   = x[n] + x[N-n]
        w[padx(P::S0 + cell)] = vsub(a, b);      // ds[n-1] = x[n] - x[N-n]
    }
}

// A0 by chunks of 32 consecutive n: lane l (1..31) handles n = 32c + l, whose
// class j = ctz(l) and cell off_j + (n >> (j+1)) = A_l + c * B_l do not depend
// on c except through B_l; lane 0's n = 32c (c >= 1) are done by a0_item.
struct A0Lane {
    int A, B, sh;  // padded cosine cell of chunk c: A + c*B + (c >> sh)
};
template <int LOG2N>
QFT_HD A0Lane a0_lane(int l) {
    using P = SPlan<LOG2N>;
    A0Lane r;
    const int j = ctz32((uint32_t)(l | 32));
    // cell = off_j + (n >> (j+1)) with off_j a multiple of 32 and (l >> (j+1)) + c*B mod 32 < 32,
    // so padx(cell) = off_j + off_j/32 + (l >> (j+1)) + c*B + (c >> (j+1))
    const int off = P::m - (1 << (LOG2N - 1 - j));
    r.A = off + (off >> 5) + (l >> (j + 1));
    r.B = 32 >> (j + 1);
    r.sh = j + 1;
    return r;
}
template <int LOG2N, typename T>
QFT_HD void a0_chunk(const vec2<T> *x, vec2<T> *w, int c, int l, A0Lane a) {
    using P = SPlan<LOG2N>;
    const int n = 32 * c + l;
    vec2<T> u = x[n], v = x[P::N - n];
    const int pc = a.A + c * a.B + (c >> a.sh);
    w[pc] = vadd(u, v);                      // dc[n]   = x[n] + x[N-n]
    w[pc + padx(P::S0)] = vsub(u, v);        // ds[n-1] = x[n] - x[N-n]  (S0 is a multiple of 32)
}

// A0 by chunks of 64 consecutive n (n = 64c + 2l and 64c + 2l + 1 for lane l):
// one aligned pair load per side, the odd samples (Lee block 0) go to 32
// consecutive cells, the even ones to block 1 + ctz(l); lane l's even mirror
// x[N - 64c - 2l] is the first element of lane l-1's mirror pair.
struct A0Lane64 {
    int A, B, sh;  // padded cosine cell of the even sample of chunk c: A + c*B + (c >> sh)
};
template <int LOG2N>
QFT_HD A0Lane64 a0_lane64(int l) {
    using P = SPlan<LOG2N>;
    A0Lane64 r;
    const int j = 1 + ctz32((uint32_t)(l | 32));  // block of n = 64c + 2l (l != 0)
    const int off = P::m - (1 << (LOG2N - 1 - j));
    r.A = off + (off >> 5) + (l >> j);
    r.B = 32 >> j;
    r.sh = j;
    return r;
}
template <int LOG2N, typename T, class ShflUp>
QFT_HD void a0_chunk64(const vec2<T> *x, vec2<T> *w, int c, int l, A0Lane64 a, ShflUp &&shfl_up) {
    using P = SPlan<LOG2N>;
    vec2<T> xe, xo, mn, mo;
    ld2(x + 64 * c + 2 * l, xe, xo);                // x[n_e], x[n_o]
    ld2(x + P::N - 64 * c - 2 * l - 2, mn, mo);     // x[N - n_e - 2], x[N - n_o]
    const vec2<T> me = shfl_up(mn);                  // x[N - n_e] from lane l-1
    const int po = 33 * c + l;                       // block 0 cell 32c + l, padded
    w[po] = vadd(xo, mo);
    w[po + padx(P::S0)] = vsub(xo, mo);
    if (l) {
        const int pe = a.A + c * a.B + (c >> a.sh);
        w[pe] = vadd(xe, me);
        w[pe + padx(P::S0)] = vsub(xe, me);
    }
}

// ---------------------------------------------------------------- modes
// MODE 0 cdft (complex signals), 1 rdft, 2 dct0, 3 dst0.  For the real modes two
// real signals a, b ride in one vec2 (both follow the identical DAG).
// A0 item n in [0, m] of a real pair (rows xa, xb of the mode's stored length).
template <int LOG2N, typename T, int MODE>
QFT_HD void a0_item_real(const T *xa, const T *xb, vec2<T> *w, int n) {
    using P = SPlan<LOG2N>;
    auto at = [&](int i) { return vec2<T>{xa[i], xb[i]}; };
    auto cell_of = [&](int nn) {
        const int j = ctz32((uint32_t)nn);
        return P::m - (1 << (LOG2N - 1 - j)) + (nn >> (j + 1));
    };
    if constexpr (MODE == 1) {  // rdft: fold x[n] +- x[N-n] (shared.py:28-35)
        if (n == 0) {
            w[padx(P::BASE)] = at(0);
            w[padx(P::BASE + 1)] = at(P::m);
        } else if (n < P::m) {
            const vec2<T> a = at(n), b = at(P::N - n);
            const int c = cell_of(n);
            w[padx(c)] = vadd(a, b);
            w[padx(P::S0 + c)] = vsub(a, b);
        }
    } else if constexpr (MODE == 2) {  // dct0: values s(0..m) are the cosine signal
        if (n == 0) w[padx(P::BASE)] = at(0);
        else if (n == P::m) w[padx(P::BASE + 1)] = at(P::m);
        else w[padx(cell_of(n))] = at(n);
    } else {  // dst0: values s(1..m-1) are the sine signal (slot n-1)
        if (n > 0 && n < P::m) w[padx(P::S0 + cell_of(n))] = at(n - 1);
    }
}

template <int LOG2N, typename T>
QFT_HD void a0_unit8(const vec2<T> *x, vec2<T> *w, int k) {
    using P = SPlan<LOG2N>;
    vec2<T> f[9], r[8];
#pragma unroll
    for (int e = 0; e < 8; e += 2) ld2(x + 8 * k + e, f[e], f[e + 1]);
    f[8] = x[8 * k + 8];
#pragma unroll
    for (int e = 0; e < 8; e += 2) ld2(x + P::N - 8 * k - 8 + e, r[e], r[e + 1]);
    // r[e] = x[N - n] for n = 8k + 8 - e
    constexpr int off0 = P::off(0), off1 = P::off(1), off2 = P::off(2);
    vec2<T> *c0 = w + padx(off0 + 4 * k), *s0 = w + padx(P::S0 + off0 + 4 * k);
#pragma unroll
    for (int d = 1; d < 8; d += 2) {  // odd n: block 0, i = 4k + (d-1)/2
        c0[(d - 1) / 2] = vadd(f[d], r[8 - d]);
        s0[(d - 1) / 2] = vsub(f[d], r[8 - d]);
    }
    vec2<T> *c1 = w + padx(off1 + 2 * k), *s1 = w + padx(P::S0 + off1 + 2 * k);
    c1[0] = vadd(f[2], r[6]);  // n = 8k+2: block 1, i = 2k
    s1[0] = vsub(f[2], r[6]);
    c1[1] = vadd(f[6], r[2]);  // n = 8k+6: i = 2k+1
    s1[1] = vsub(f[6], r[2]);
    w[padx(off2 + k)] = vadd(f[4], r[4]);  // n = 8k+4: block 2, i = k
    w[padx(P::S0 + off2 + k)] = vsub(f[4], r[4]);
    const int n8 = 8 * k + 8;
    if (n8 == P::m) {
        w[padx(P::BASE + 1)] = f[8];  // dc[m] = x[m]
    } else {
        const int j = ctz32((uint32_t)n8);
        const int cell = P::m - (1 << (LOG2N - 1 - j)) + (n8 >> (j + 1));
        w[padx(cell)] = vadd(f[8], r[0]);
        w[padx(P::S0 + cell)] = vsub(f[8], r[0]);
    }
    if (k == 0) w[padx(P::BASE)] = f[0];  // dc[0] = x[0]
}

// ---------------------------------------------------------------- phase A
// Lane t of the warp owning big block J of one side: loads its reflection group,
// folds RF levels, and (after __syncwarp) writes element t of sub-block p to
// cell 32p + t of the block.
template <int LOG2N, int J, bool DST, typename T>
struct FBlock {
    using P = SPlan<LOG2N>;
    static constexpr int L = P::L(J), R = P::RF(J), G = 1 << R;
    static constexpr int base = (DST ? P::S0 : 0) + P::off(J);  // multiple of 32
    vec2<T> v[G];
    QFT_HD void load(const vec2<T> *w, const T *U, int t) {
        const vec2<T> *bf = w + padx(base) + t;       // forward runs
        const vec2<T> *br = w + padx(base) + 31 - t;  // reversed runs
#pragma unroll
        for (int s = 0; s < G; ++s) {
            int c, sg;
            run_of(R, L, s, c, sg);  // compile-time after unrolling
            const int u = c >> 5;    // the run is the 32-aligned chunk u
            v[s] = sg > 0 ? bf[33 * u] : br[33 * u];
        }
        lee_fwd<R, L, DST, T>(v, t, U);
    }
    QFT_HD void store(vec2<T> *w, int t) const {
        vec2<T> *o = w + padx(base) + t;
#pragma unroll
        for (int p = 0; p < G; ++p) o[33 * p] = v[p];
    }
};

// ---------------------------------------------------------------- phase B
// Lee-32 on the 32-cell chunk starting at (padded) cell p0; in place.
template <bool DST, typename T>
QFT_HD void b_l32(vec2<T> *w, int chunk_base, const T *U) {
    vec2<T> *c = w + padx(chunk_base);
    vec2<T> v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = c[e];
    lee_full<32, DST, T>(v, U);
#pragma unroll
    for (int e = 0; e < 32; ++e) c[e] = v[e];
}

template <int LOG2N, bool DST, typename T, int J>
QFT_HD void b_small_rec(vec2<T> *w, const T *U) {
    using P = SPlan<LOG2N>;
    if constexpr (J <= LOG2N - 2) {
        constexpr int L = P::L(J);
        vec2<T> v[L];
        constexpr int b0 = (DST ? P::S0 : 0) + P::off(J);
#pragma unroll
        for (int e = 0; e < L; ++e) v[e] = w[padx(b0 + e)];
        lee_full<L, DST, T>(v, U);
#pragma unroll
        for (int e = 0; e < L; ++e) w[padx(b0 + e)] = v[e];
        b_small_rec<LOG2N, DST, T, J + 1>(w, U);
    }
}
// all blocks with L <= 16 of one side
template <int LOG2N, bool DST, typename T>
QFT_HD void b_small(vec2<T> *w, const T *U) {
    constexpr int J0 = SPlan<LOG2N>::JS > 0 ? SPlan<LOG2N>::JS : 0;
    b_small_rec<LOG2N, DST, T, J0>(w, U);
}

// ---------------------------------------------------------------- phase C
// Lane i of the warp owning big block J of one side: column i of the 2^R
// sub-block spectra -> block spectrum slots [i*2^R, (i+1)*2^R), natural order.
// The halo Z_p[i+1] (DCT) / Z_p[i-1] (DST) is the neighbour lane's own value.
template <int LOG2N, int J, bool DST, typename T>
struct CBlock {
    using P = SPlan<LOG2N>;
    static constexpr int R = P::RF(J), G = 1 << R;
    static constexpr int base = (DST ? P::S0 : 0) + P::off(J);
    vec2<T> own[G];
    QFT_HD void load(const vec2<T> *w, int i) {
        const vec2<T> *c = w + padx(base) + i;
#pragma unroll
        for (int p = 0; p < G; ++p) own[p] = c[33 * p];
    }
    // halo column (i+1 for DCT, i-1 for DST; the edge lane re-reads its own column)
    QFT_HD static const vec2<T> *halo_col(const vec2<T> *w, int i) {
        const int ih = DST ? (i > 0 ? i - 1 : i) : (i < 31 ? i + 1 : i);
        return w + padx(base) + ih;
    }
    // halo(p) must return the neighbour lane's own[p]
    template <class Halo>
    QFT_HD void compute(int i, Halo &&halo, vec2<T> *out) const {
        const bool edge = DST ? (i == 0) : (i == 31);
        lee_bwd_fn<R, DST, T>(own, 0, halo, edge, out);
    }
    QFT_HD static void store(vec2<T> *w, int i, const vec2<T> *out) {
        // slots i*G .. i*G+G-1 lie inside one 32-cell chunk: contiguous when padded
        vec2<T> *o = w + padx(base + i * G);
#pragma unroll
        for (int s = 0; s < G; ++s) o[s] = out[s];
    }
};

// ---------------------------------------------------------------- phase D
template <int LOG2N, typename T>
struct Chain {
    using P = SPlan<LOG2N>;
    static constexpr int n = LOG2N;
    static QFT_HD constexpr int qj(int j) { return 1 << (n - 2 - j); }
    // cosine spectrum of Lee block j, slot k
    static QFT_HD vec2<T> OC(const vec2<T> *w, int j, int k) { return w[padx(P::off(j) + k)]; }
    // sine spectrum of Lee block j, harmonic h (slot h-1)
    static QFT_HD vec2<T> OS(const vec2<T> *w, int j, int h) { return w[padx(P::S0 + P::off(j) + h - 1)]; }

    // ---- chain-mid (phase C, one warp per signal): C_j, S_j for j = n-1 .. JM,
    // bottom-up, in place in the chain cells (elaborations.py:329-340).
    // C_j[k] = E[k]+O[k], C_j[m_j-k] = E[k]-O[k] (k < q_j), C_j[q_j] = E[q_j];
    // S_j[h] = O[h]+E[h], S_j[m_j-h] = O[h]-E[h] (h < q_j), S_j[q_j] = O[q_j].
    static QFT_HD void mid_level_load(const vec2<T> *w, int j, int k, vec2<T> &c, vec2<T> &s) {
        const int q = qj(j), mm = 2 * q;
        if (k <= mm) {  // C_j[k]
            const int kk = k <= q ? k : mm - k;
            vec2<T> e = w[padx(P::CHC + kk)];
            if (k == q) c = e;
            else {
                vec2<T> o = OC(w, j, kk);
                c = k < q ? vadd(e, o) : vsub(e, o);
            }
        }
        if (k >= 1 && k < mm) {  // S_j[k]
            if (k == q) s = OS(w, j, q);
            else {
                const int kk = k < q ? k : mm - k;
                vec2<T> o = OS(w, j, kk);
                vec2<T> e = w[padx(P::CHS + kk - 1)];
                s = k < q ? vadd(o, e) : vsub(o, e);
            }
        }
    }
    static QFT_HD void mid_level_store(vec2<T> *w, int j, int k, vec2<T> c, vec2<T> s) {
        const int mm = 2 * qj(j);
        if (k <= mm) w[padx(P::CHC + k)] = c;
        if (k >= 1 && k < mm) w[padx(P::CHS + k - 1)] = s;
    }
    static QFT_HD void mid_base(vec2<T> *w) {  // C_{n-1} = DCT-0 of two points
        vec2<T> s0 = w[padx(P::BASE)], sm = w[padx(P::BASE + 1)];
        w[padx(P::CHC)] = vadd(s0, sm);
        w[padx(P::CHC + 1)] = vsub(s0, sm);
    }

    // C_J[k], 0 <= k <= m_J: descend the time-split chain to the DCT base (or to
    // the chain-mid level JM computed in phase C)
    template <int J>
    static QFT_HD vec2<T> descCJ(const vec2<T> *w, int k) {
        if constexpr (QFT_CHAIN_MID && J == P::JM) {
            return w[padx(P::CHC + k)];
        } else if constexpr (J == n - 1) {  // DCT-0 of two points: [s0 + sm, s0 - sm]
            vec2<T> s0 = w[padx(P::BASE)], sm = w[padx(P::BASE + 1)];
            return k == 0 ? vadd(s0, sm) : vsub(s0, sm);
        } else {
            constexpr int q = qj(J), mm = 2 * q;
            const int kk = k <= q ? k : mm - k;
            vec2<T> e = descCJ<J + 1>(w, kk);
            if (k == q) return e;                       // out[q] = E[q]
            vec2<T> o = OC(w, J, kk);
            return k < q ? vadd(e, o) : vsub(e, o);     // E+O / E-O
        }
    }
    // S_J[k], 1 <= k <= m_J - 1 (k = 0, m_J: unused value, in-bounds reads)
    template <int J>
    static QFT_HD vec2<T> descSJ(const vec2<T> *w, int k) {
        constexpr int q = qj(J), mm = 2 * q;
        if constexpr (QFT_CHAIN_MID && J == P::JM) {
            return w[padx(P::CHS + (k > 0 ? k - 1 : 0))];
        } else if constexpr (J == n - 2) {
            return OS(w, J, 1);                         // _dst base: copy
        } else {
            if (k == q) return OS(w, J, q);             // out[q-1] = O[q-1]
            const int kk = k < q ? k : mm - k;
            vec2<T> e = descSJ<J + 1>(w, kk);
            vec2<T> o = OS(w, J, kk);
            return k < q ? vadd(o, e) : vsub(o, e);     // O+E / O-E
        }
    }
    static QFT_HD vec2<T> descC(const vec2<T> *w, int k) { return descCJ<P::RC>(w, k); }
    static QFT_HD vec2<T> descS(const vec2<T> *w, int k) { return descSJ<P::RC>(w, k); }

    static QFT_HD void emit(vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) {
        // S(k) = (C1 + S2, C2 - S1), S(N-k) = (C1 - S2, C2 + S1) (shared.py:218-221):
        // with u = (S2, -S1): S(k) = cv + u, S(N-k) = cv - u, bit for bit
        // (x - (-y) == x + y and x + (-y) == x - y in IEEE arithmetic).
        const vec2<T> u = {sv.y, -sv.x};
        y[k] = vadd(cv, u);
        y[P::N - k] = vsub(cv, u);
    }

    // regular thread: every index stays strictly inside (0, q_j) at every level
    template <int J>
    static QFT_HD void up(const vec2<T> *w, vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) {
        if constexpr (J == 0) {
            emit(y, k, cv, sv);
        } else {
            constexpr int mm = 2 * qj(J - 1);
            vec2<T> o = OC(w, J - 1, k), os = OS(w, J - 1, k);
            up<J - 1>(w, y, k, vadd(cv, o), vadd(os, sv));
            up<J - 1>(w, y, mm - k, vsub(cv, o), vsub(os, sv));
        }
    }

    // special thread: groups of t = 0 and t = m_RC; every index is compile-time
    template <int J, int K>
    static QFT_HD void up_s(const vec2<T> *w, vec2<T> *y, vec2<T> cv, vec2<T> sv) {
        if constexpr (J == 0) {
            if constexpr (K == 0 || K == P::m) y[K] = cv;  // harmonics 0, N/2: copies
            else emit(y, K, cv, sv);
        } else {
            constexpr int q = qj(J - 1), mm = 2 * q;
            if constexpr (K == q) {                        // C copy, S leaf
                up_s<J - 1, q>(w, y, cv, OS(w, J - 1, q));
            } else {
                vec2<T> o = OC(w, J - 1, K);
                if constexpr (K == 0) {                    // no sine harmonic 0
                    up_s<J - 1, 0>(w, y, vadd(cv, o), sv);
                    up_s<J - 1, mm>(w, y, vsub(cv, o), sv);
                } else {
                    vec2<T> os = OS(w, J - 1, K);
                    up_s<J - 1, K>(w, y, vadd(cv, o), vadd(os, sv));
                    up_s<J - 1, mm - K>(w, y, vsub(cv, o), vsub(os, sv));
                }
            }
        }
    }

    // t in [0, MRC): t = 0 is the special thread (groups 0 and MRC)
    // ---- uniform phase-D thread (t in [0, MRC], no special path) ----------
    // index of thread t's chain value at level J > RC: the distance of t to the
    // nearest multiple of m_{J-1} (composition of the folds k -> min(k, m_j - k))
    template <int J>
    static QFT_HD int kk(int t) {
        if constexpr (J == P::RC) {
            return t;
        } else {
            constexpr int Pm = 2 << (n - 1 - J);  // m_{J-1}
            const int r = t & (Pm - 1);
            return r < Pm - r ? r : Pm - r;
        }
    }
    // C_J / S_J at index kk<J>(t), bottom-up; every load address depends on t
    // only, so all loads issue before the dependent add chain
    template <int J>
    static QFT_HD void desc2(const vec2<T> *w, int t, vec2<T> &cv, vec2<T> &sv) {
        if constexpr (J == n - 1) {
            const vec2<T> s0 = w[padx(P::BASE)], sm = w[padx(P::BASE + 1)];
            cv = kk<J>(t) == 0 ? vadd(s0, sm) : vsub(s0, sm);  // DCT-0 of two points
            sv = s0;                                             // (unused)
        } else {
            desc2<J + 1>(w, t, cv, sv);
            constexpr int q = qj(J);
            const int k = kk<J>(t), k1 = kk<J + 1>(t);  // k1 = min(k, 2q - k)
            const vec2<T> o = OC(w, J, k1);
            const vec2<T> os = OS(w, J, k1 > 0 ? k1 : 1);
            const bool self = (k == q), lo = (k < q);
            cv = self ? cv : (lo ? vadd(cv, o) : vsub(cv, o));   // E+O / E-O / E[q]
            sv = self ? os : (lo ? vadd(os, sv) : vsub(os, sv)); // O+E / O-E / O[q]
        }
    }

    static QFT_HD void emit_u(vec2<T> *y, int k, vec2<T> cv, vec2<T> sv) {
        const vec2<T> u = {sv.y, -sv.x};
        const bool edge = (k == 0) || (k == P::m);  // harmonics 0, N/2: copies
        y[k] = edge ? cv : vadd(cv, u);
        if (!edge) y[P::N - k] = vsub(cv, u);
    }
    // unfold with self-paired indices (k == q_j) duplicated: both children get
    // the C copy / S leaf and write identical values.  emit(k, C_0[k], S_0[k]).
    template <int J, class Emit>
    static QFT_HD void up_e(const vec2<T> *w, Emit &emit, int k, vec2<T> cv, vec2<T> sv) {
        if constexpr (J == 0) {
            emit(k, cv, sv);
        } else {
            constexpr int q = qj(J - 1), mm = 2 * q;
            const bool self = (k == q);
            const vec2<T> o = OC(w, J - 1, k < q ? k : 0);
            const vec2<T> os = OS(w, J - 1, k > 0 ? k : 1);
            up_e<J - 1>(w, emit, k, self ? cv : vadd(cv, o), self ? os : vadd(os, sv));
            up_e<J - 1>(w, emit, self ? q : mm - k, self ? cv : vsub(cv, o), self ? os : vsub(os, sv));
        }
    }

    template <class Emit>
    static QFT_HD void unit_e(const vec2<T> *w, Emit &emit, int t) {
        vec2<T> cv, sv;
        if constexpr (P::RC < n - 1) desc2<P::RC>(w, t, cv, sv);
        up_e<P::RC>(w, emit, t, cv, sv);
    }
    static QFT_HD void unit(const vec2<T> *w, vec2<T> *y, int t) {
        auto emit = [&](int k, vec2<T> cv, vec2<T> sv) { emit_u(y, k, cv, sv); };
        unit_e(w, emit, t);
    }
};

}  // namespace qft
