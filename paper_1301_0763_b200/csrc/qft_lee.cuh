// qft_lee.cuh -- register-level building blocks of the improved QFT.
//
// Constant table layout used by every kernel ("level table" U):
//   U[0]         = cos(2 pi/8)                       (counting.py:176-178)
//   U[S/2 + i]   = 1/(2 cos(2 pi (2i+1)/(4S)))        for S = 2,4,8,...; i < S/2
// i.e. the half-secants a Lee block of size S (the reference's _dct_oo/_dst_oo
// at periodization 4S, improved.py:66 and :105) multiplies its odd child by,
// stored contiguously per level so that neighbouring lanes read neighbouring
// words.  Values are bit-identical to the reference's TrigTable entries: a
// half-secant depends only on the reduced fraction (counting.py:152-158).
#pragma once
#include "qft_common.cuh"

namespace qft {

// ---------------------------------------------------------------------------
// Full Lee DCT-II / DST-II of size L held in registers.
//   DCT: restates improved._dct_ot (improved.py:49-56) + _dct_oo (:59-74)
//   DST: restates improved._dst_ot (improved.py:87-94) + _dst_oo (:97-112)
// In: v[i] = x_i (odd-time samples in slot order).  Out: v[k] = spectrum slot k
// (DCT: harmonic k; DST: harmonic k+1).
// ---------------------------------------------------------------------------
// ub: index of the L == 2 base constant -- 0 for the DCT, 1 for the DST; the
// DCT code run on a sine block stored "as cosine" (QFT_SC, qft_smem.cuh) passes 1.
template <int L, bool DST, typename T>
QFT_HD void lee_full(vec2<T> *v, const T *U, int ub = DST ? 1 : 0) {
    if constexpr (L > 1) {
        constexpr int H = L / 2;
        vec2<T> e[H], o[H];
#pragma unroll
        for (int i = 0; i < H; ++i) {
            vec2<T> a = v[i], b = v[L - 1 - i];
            // L == 2 is the eight-point base: DCT uses the named cos(2pi/8)
            // (improved.py:63), DST the half-secant at 1/8 (improved.py:102).
            T c = (L == 2) ? U[ub] : U[H + i];
            if constexpr (!DST) {
                e[i] = vadd(a, b);
                o[i] = vmul(vsub(a, b), c);
            } else {
                e[i] = vsub(a, b);
                o[i] = vmul(vadd(a, b), c);
            }
        }
        lee_full<H, DST, T>(e, U, ub);
        lee_full<H, DST, T>(o, U, ub);
        if constexpr (!DST) {
#pragma unroll
            for (int i = 0; i < H; ++i) v[2 * i] = e[i];
#pragma unroll
            for (int i = 0; i < H - 1; ++i) v[2 * i + 1] = vadd(o[i], o[i + 1]);
            v[L - 1] = o[H - 1];
        } else {
#pragma unroll
            for (int i = 0; i < H; ++i) v[2 * i + 1] = e[i];
            v[0] = o[0];
#pragma unroll
            for (int i = 1; i < H; ++i) v[2 * i] = vadd(o[i - 1], o[i]);
        }
    }
}

// ---------------------------------------------------------------------------
// R forward fold levels of a Lee block of size L for reflection group t.
// Slot s of v holds element run_of(R, L, s)(t) of the block; afterwards slot p
// holds element t of sub-block p (sub-blocks in [even | odd] recursive order,
// size L >> R).  Same fold + secant scaling as lee_full, first R levels only.
// ---------------------------------------------------------------------------
template <int R, int L, bool DST, typename T>
QFT_HD void lee_fwd(vec2<T> *v, int t, const T *U) {
    if constexpr (R > 0) {
        constexpr int G = 1 << R, H = G / 2;
        vec2<T> nv[G];
#pragma unroll
        for (int s = 0; s < H; ++s) {
            int c, sg;
            run_of(R - 1, L / 2, s, c, sg);
            const int i = c + sg * t;  // element index of slot s within this block
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
        lee_fwd<R - 1, L / 2, DST, T>(nv, t, U);
        lee_fwd<R - 1, L / 2, DST, T>(nv + H, t, U);
#pragma unroll
        for (int s = 0; s < G; ++s) v[s] = nv[s];
    }
}

// ---------------------------------------------------------------------------
// R backward levels for column i of 2^R sub-block spectra (the neighbour sums
// of improved.py:72-73 / :110-111 and the free interleaves of
// elaborations.py:137-148).  v[p] = Z_p[i] (p relative to absolute index pofs);
// halo(p) returns Z_p[i+1] (DCT) or Z_p[i-1] (DST) for absolute p -- the halo is
// always a raw sub-block value because the first element of the next column's
// range is reached through copies only.  edge: i is the last (DCT) / first
// (DST) column, where the reference copies instead of adding.
// Out: block spectrum slots [i*2^R, (i+1)*2^R).
// ---------------------------------------------------------------------------
// PRE: the odd sub-blocks (odd p) arrive with their deepest neighbour sum already
// formed -- Z_p[i] + Z_p[i+1] (DCT; Z_p[i-1] + Z_p[i] for the DST; the edge column
// a copy) -- by the Lee-32 step that produced them (b_l32p, qft_smem.cuh), which
// held both operands in one lane: the deepest level is then a pure interleave and
// reads no halo (16 of the 31 halo reads of a 32-sub-block column).
template <int R, bool DST, typename T, class Halo, bool PRE = false>
QFT_HD void lee_bwd_fn(const vec2<T> *v, int pofs, Halo &halo, bool edge, vec2<T> *out) {
    if constexpr (R == 0) {
        out[0] = v[0];
    } else if constexpr (PRE && R == 1) {
        out[DST ? 1 : 0] = v[0];
        out[DST ? 0 : 1] = v[1];
    } else {
        constexpr int H = 1 << (R - 1);
        vec2<T> e[H], o[H];
        lee_bwd_fn<R - 1, DST, T, Halo, PRE>(v, pofs, halo, edge, e);
        lee_bwd_fn<R - 1, DST, T, Halo, PRE>(v + H, pofs + H, halo, edge, o);
        const vec2<T> hv = halo(pofs + H);  // leftmost leaf of the odd child
        if constexpr (!DST) {
#pragma unroll
            for (int t = 0; t < H; ++t) out[2 * t] = e[t];
#pragma unroll
            for (int t = 0; t < H - 1; ++t) out[2 * t + 1] = vadd(o[t], o[t + 1]);
            out[2 * H - 1] = edge ? o[H - 1] : vadd(o[H - 1], hv);
        } else {
#pragma unroll
            for (int t = 0; t < H; ++t) out[2 * t + 1] = e[t];
#pragma unroll
            for (int t = 1; t < H; ++t) out[2 * t] = vadd(o[t - 1], o[t]);
            out[0] = edge ? o[0] : vadd(hv, o[0]);
        }
    }
}

// ---------------------------------------------------------------------------
// Whole cosine / sine transforms in registers (small periodization NN).
//   dct0_reg: improved._dct (improved.py:36-46), x = [s(0)..s(NN/2)]
//   dst0_reg: improved._dst (improved.py:77-84), x = [s(1)..s(NN/2-1)]
// ---------------------------------------------------------------------------
template <int NN, typename T>
QFT_HD void dct0_reg(const vec2<T> *x, vec2<T> *out, const T *U) {
    if constexpr (NN == 2) {
        out[0] = vadd(x[0], x[1]);
        out[1] = vsub(x[0], x[1]);
    } else {
        constexpr int q = NN / 4, m = NN / 2;
        vec2<T> even[q + 1], se[q + 1], odd[q];
#pragma unroll
        for (int i = 0; i <= q; ++i) even[i] = x[2 * i];
#pragma unroll
        for (int i = 0; i < q; ++i) odd[i] = x[2 * i + 1];
        dct0_reg<NN / 2, T>(even, se, U);
        lee_full<q, false, T>(odd, U);
#pragma unroll
        for (int k = 0; k < q; ++k) {
            out[k] = vadd(se[k], odd[k]);
            out[m - k] = vsub(se[k], odd[k]);
        }
        out[q] = se[q];
    }
}

template <int NN, typename T>
QFT_HD void dst0_reg(const vec2<T> *x, vec2<T> *out, const T *U) {
    if constexpr (NN == 4) {
        out[0] = x[0];
    } else {
        constexpr int q = NN / 4, m = NN / 2;
        vec2<T> even[q - 1], se[q - 1], odd[q];
#pragma unroll
        for (int i = 0; i < q - 1; ++i) even[i] = x[2 * i + 1];
#pragma unroll
        for (int i = 0; i < q; ++i) odd[i] = x[2 * i];
        dst0_reg<NN / 2, T>(even, se, U);
        lee_full<q, true, T>(odd, U);
#pragma unroll
        for (int k = 0; k < q - 1; ++k) {
            out[k] = vadd(odd[k], se[k]);
            out[m - 2 - k] = vsub(odd[k], se[k]);
        }
        out[q - 1] = odd[q - 1];
    }
}

// Complex recombination of one harmonic pair (shared.py:64-71):
// cv = (C1(k), C2(k)) cosine spectra of the Re/Im parts, sv = (S1(k), S2(k))
// sine spectra.  The reference forms Re S(k) = C1 - (-S2) etc.; x - (-y) is
// x + y bit for bit in IEEE arithmetic.
template <typename T>
QFT_HD void recombine(vec2<T> cv, vec2<T> sv, vec2<T> &lo, vec2<T> &hi) {
    lo = {radd(cv.x, sv.y), rsub(cv.y, sv.x)};  // S(k)
    hi = {rsub(cv.x, sv.y), radd(cv.y, sv.x)};  // S(N-k)
}

// Whole complex transform of a small periodization in registers:
// shared.cdft_interleaved (shared.py:46-72) over rdft_packed (:21-43).
template <int NN, typename T>
QFT_HD void cdft_reg(const vec2<T> *x, vec2<T> *y, const T *U) {
    if constexpr (NN == 2) {
        y[0] = vadd(x[0], x[1]);
        y[1] = vsub(x[0], x[1]);
    } else {
        constexpr int m = NN / 2;
        vec2<T> dc[m + 1], ds[m - 1 > 0 ? m - 1 : 1], C[m + 1], S[m - 1 > 0 ? m - 1 : 1];
        dc[0] = x[0];
        dc[m] = x[m];
#pragma unroll
        for (int n = 1; n < m; ++n) {
            dc[n] = vadd(x[n], x[NN - n]);
            ds[n - 1] = vsub(x[n], x[NN - n]);
        }
        dct0_reg<NN, T>(dc, C, U);
        dst0_reg<NN, T>(ds, S, U);
        y[0] = C[0];
        y[m] = C[m];
#pragma unroll
        for (int k = 1; k < m; ++k) recombine(C[k], S[k - 1], y[k], y[NN - k]);
    }
}

}  // namespace qft
