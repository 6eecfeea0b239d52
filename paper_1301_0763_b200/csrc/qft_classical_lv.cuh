// qft_classical_lv.cuh -- the classical QFT (classical.py:64-129) as a level-
// synchronous schedule: the building blocks shared by the CUDA kernels
// (qft_classical.cu) and the test-only host emulator (tests/emu/).
//
// The classical recursion is a regular binary tree once the odd-harmonic
// conversion is attached to the node it belongs to:
//
//   cosine side   node (d, b), S = Nn >> (d+1), q = S/2
//     b even: dct node   D(Nn >> d)      S+1 cells   classical._dct     (:64-74)
//     b odd : odd node   O(Nn >> (d-1))  S   cells   classical._dct_odd (:77-99)
//     both have the children (d+1, 2b) = D with q+1 cells (even harmonics) and
//     (d+1, 2b+1) = O with q cells (odd harmonics): D folds x[i] +- x[S-i]
//     (elaborations.py:96-101), O first multiplies by the half-secants and folds
//     the converted signal as dc_t1t (elaborations.py:102-112, the cell S absent).
//     Backward: D interleaves its children's spectra, O adds neighbours of the
//     interleave (classical.py:98-99).
//   sine side     node (d, b) = S(Nn >> d), S-1 cells (stride S)
//     children (d+1, 2b) = the even-harmonic fold x[i] - x[S-2-i] and
//     (d+1, 2b+1) = the odd-harmonic fold x[i] + x[S-2-i] scaled by the
//     half-secants (classical._dst_odd :112-129 attached to its mother); the
//     centre x[q-1] is parked in a side array (cell 2^d + b: it must survive the
//     deeper levels, which reuse both buffers).
//     Backward: partial sums of child 2b+1's spectrum +- the centre, interleaved
//     with child 2b's spectrum (classical.py:119-128, elaborations.py:145-148).
//
// Layout of depth d of one (sub-)tree in a buffer: cosine node b at
// cos_off(S, b) = b S + ceil(b/2) (the D nodes carry the one extra cell of the
// dc_t1t growth, tree.py:92-102), sine node b at CB + b S (S + 1 at the base
// depth).  Depth d lives in
// buffer d & 1; a node's spectrum replaces its input cells.  Nodes of
// periodization 32 (S = 16) are finished by one thread each in registers with the
// reference recursion instantiated at compile time (dct_r / dct_odd_r / dst_r /
// dst_odd_r below).  Every value is the same single IEEE operation on the same
// operands as in the reference (counting.py:40-81).
#pragma once
#include "qft_common.cuh"

namespace qft {
namespace cl {

constexpr int kBaseLog = 5;  // nodes of periodization 2^5 are register-level bases

QFT_HD int cos_off(int S, int b) { return b * S + ((b + 1) >> 1); }
// depth of the register-level bases of a (sub-)tree of periodization 2^lognn
QFT_HD int base_depth(int lognn) { return lognn - kBaseLog; }
// cells of the cosine area (the deepest level is the largest: Nn/2 + 2^(D-1))
QFT_HD int cos_cells(int lognn) {
    const int D = base_depth(lognn);
    return (1 << (lognn - 1)) + (D >= 1 ? (1 << (D - 1)) : 1) + 1;
}
// cells of one buffer: cosine area, sine area, centres (used in buffer 0 only)
// (the sine area holds one pad cell per base node, Tree::sin_stride)
QFT_HD int cen_off(int lognn) { return cos_cells(lognn) + (1 << (lognn - 1)) + (1 << (lognn > kBaseLog ? lognn - kBaseLog : 0)); }
QFT_HD int buf_cells(int lognn) { return cen_off(lognn) + (1 << (base_depth(lognn) > 0 ? base_depth(lognn) : 0)); }

// stride of the sine nodes of depth d of a tree of periodization 2^lognn: S, plus
// one pad cell at the base depth (Tree::sin_stride)
QFT_HD int sin_stride_of(int lognn, int d) { return (1 << (lognn - 1 - d)) + (d == base_depth(lognn) ? 1 : 0); }

// vec2 * constant.  fp32 on the device: the packed multiply x*c + z with the opaque
// (-0, -0) addend of vmul<float> (qft_common.cuh), z loaded once per kernel instead
// of once per multiply
template <typename T>
struct Mul {
    QFT_HD vec2<T> operator()(vec2<T> a, T c) const { return vmul(a, c); }
};
template <>
struct Mul<float> {
    unsigned long long z = 0x8000000080000000ull;  // the kernels overwrite it with the global's value
    QFT_HD vec2<float> operator()(vec2<float> a, float c) const {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(QFT_NO_F32X2) && !defined(QFT_SCALAR_MUL)
        unsigned long long r;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(vec2<float>{c, c})), "l"(z));
        return upk(r);
#else
        return vmul(a, c);
#endif
    }
};

// half-secant 1/(2cos(2 pi n / 2^lognode)) from the natural table of the top
// periodization 2^logtop (counting.py:152-158: a constant depends only on the
// reduced fraction)
template <typename T>
struct HS {
    const T *Tt;
    int logtop;
    QFT_HD T operator()(int n, int lognode) const { return Tt[n << (logtop - lognode)]; }
};

// ---------------------------------------------------------------- register-level bases
template <int Nn, typename T>
QFT_HD void dct_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs);
template <int No, typename T>
QFT_HD void dct_odd_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs);
template <int Nn, typename T>
QFT_HD void dst_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs);
template <int No, typename T>
QFT_HD void dst_odd_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs);

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }

// classical._dct (classical.py:64-74): x = s(0..Nn/2) -> S(0..Nn/2)
template <int Nn, typename T>
QFT_HD void dct_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs) {
    if constexpr (Nn == 2) {
        out[0] = vadd(x[0], x[1]);
        out[1] = vsub(x[0], x[1]);
    } else {
        constexpr int q = Nn / 4, m = Nn / 2;
        vec2<T> even[q + 1], odd[q], se[q + 1], so[q];
#pragma unroll
        for (int i = 0; i < q; ++i) {
            even[i] = vadd(x[i], x[m - i]);
            odd[i] = vsub(x[i], x[m - i]);
        }
        even[q] = x[q];
        dct_r<Nn / 2, T>(even, se, hs);
        dct_odd_r<Nn, T>(odd, so, hs);
#pragma unroll
        for (int i = 0; i <= q; ++i) out[2 * i] = se[i];
#pragma unroll
        for (int i = 0; i < q; ++i) out[2 * i + 1] = so[i];
    }
}

// classical._dct_odd (classical.py:77-99): x = s(0..No/4-1) -> odd harmonics
template <int No, typename T>
QFT_HD void dct_odd_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs) {
    if constexpr (No == 4) {
        out[0] = x[0];
    } else if constexpr (No == 8) {
        const vec2<T> t = vmul(x[1], hs(1, 3));
        out[0] = vadd(x[0], t);
        out[1] = vsub(x[0], t);
    } else {
        constexpr int q = No / 4, q2 = No / 8, m2 = No / 4, lg = ilog2(No);
        const vec2<T> zero = {(T)0, (T)0};
        vec2<T> conv[q], even[q2 + 1], odd[q2], se[q2 + 1], so[q2], half[m2 + 1];
        conv[0] = vmul(x[0], (T)0.5);  // table.half (counting.py:109)
#pragma unroll
        for (int n = 1; n < q; ++n) conv[n] = vmul(x[n], hs(n, lg));
        even[0] = vadd(conv[0], zero);  // the explicit zero pair (elaborations.py:107-108)
        odd[0] = vsub(conv[0], zero);
#pragma unroll
        for (int i = 1; i < q2; ++i) {
            even[i] = vadd(conv[i], conv[m2 - i]);
            odd[i] = vsub(conv[i], conv[m2 - i]);
        }
        even[q2] = conv[q2];
        dct_r<No / 4, T>(even, se, hs);
        dct_odd_r<No / 2, T>(odd, so, hs);
#pragma unroll
        for (int i = 0; i <= q2; ++i) half[2 * i] = se[i];
#pragma unroll
        for (int i = 0; i < q2; ++i) half[2 * i + 1] = so[i];
#pragma unroll
        for (int i = 0; i < q; ++i) out[i] = vadd(half[i], half[i + 1]);
    }
}

// classical._dst (classical.py:102-109): x = s(1..Nn/2-1) -> S(1..Nn/2-1)
template <int Nn, typename T>
QFT_HD void dst_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs) {
    if constexpr (Nn == 4) {
        out[0] = x[0];
    } else {
        constexpr int q = Nn / 4, m = Nn / 2;
        vec2<T> even[q - 1 > 0 ? q - 1 : 1], odd[q], se[q - 1 > 0 ? q - 1 : 1], so[q];
#pragma unroll
        for (int i = 0; i < q - 1; ++i) {
            even[i] = vsub(x[i], x[m - 2 - i]);
            odd[i] = vadd(x[i], x[m - 2 - i]);
        }
        odd[q - 1] = x[q - 1];
        dst_r<Nn / 2, T>(even, se, hs);
        dst_odd_r<Nn, T>(odd, so, hs);
#pragma unroll
        for (int i = 0; i < q - 1; ++i) out[2 * i + 1] = se[i];
#pragma unroll
        for (int i = 0; i < q; ++i) out[2 * i] = so[i];
    }
}

// classical._dst_odd (classical.py:112-129): x = s(1..No/4) -> odd harmonics
template <int No, typename T>
QFT_HD void dst_odd_r(const vec2<T> *x, vec2<T> *out, const HS<T> &hs) {
    if constexpr (No == 4) {
        out[0] = x[0];
    } else {
        constexpr int q = No / 4, lg = ilog2(No);
        const vec2<T> center = x[q - 1];
        vec2<T> conv[q - 1], spec[q - 1], partial[q];
#pragma unroll
        for (int n = 1; n < q; ++n) conv[n - 1] = vmul(x[n - 1], hs(n, lg));
        dst_r<No / 2, T>(conv, spec, hs);
        partial[0] = spec[0];
        partial[q - 1] = spec[q - 2];
#pragma unroll
        for (int i = 1; i < q - 1; ++i) partial[i] = vadd(spec[i - 1], spec[i]);
#pragma unroll
        for (int i = 0; i < q; ++i) out[i] = (i & 1) ? vsub(partial[i], center) : vadd(partial[i], center);
    }
}

// ---------------------------------------------------------------- one tree, level by level
// A (sub-)tree of periodization 2^lognn whose half-secants come from the table
// of the top periodization 2^logtop; root_odd: the cosine root is an O node
// (only sub-trees cut out of a larger transform: its periodization is 2^(lognn+1)).
template <typename T>
struct Tree {
    int lognn, logtop, CB;
    bool root_odd, do_cos, do_sin;
    const T *Tt;
    Mul<T> mul = {};
    QFT_HD int depth() const { return base_depth(lognn); }
    QFT_HD bool odd_type(int d, int b) const { return d ? (b & 1) : root_odd; }

    // forward level d -> d+1, item in [0, Nn/4): (node b, element i < q)
    // cen: the tree's centre array (2^D cells)
    QFT_HD void fwd_item(const vec2<T> *src, vec2<T> *dst, vec2<T> *cen, int d, int item) const {
        const int lq = lognn - 2 - d, q = 1 << lq, S = 2 * q;
        const int b = item >> lq, i = item & (q - 1);
        if (do_cos) {
            const vec2<T> *x = src + cos_off(S, b);
            vec2<T> *ev = dst + cos_off(q, 2 * b), *od = dst + cos_off(q, 2 * b + 1);
            if (!odd_type(d, b)) {  // elaborations.py:96-101
                if (i == 0) ev[q] = x[q];
                const vec2<T> a = x[i], c = x[S - i];
                ev[i] = vadd(a, c);
                od[i] = vsub(a, c);
            } else {  // classical.py:86-92, elaborations.py:102-112
                const int sh = logtop - (lognn + 1 - d);  // node periodization 4S
                if (i == 0) {
                    ev[q] = mul(x[q], Tt[q << sh]);
                    const vec2<T> c0 = mul(x[0], (T)0.5), zero = {(T)0, (T)0};
                    ev[0] = vadd(c0, zero);
                    od[0] = vsub(c0, zero);
                } else {
                    const vec2<T> a = mul(x[i], Tt[i << sh]);
                    const vec2<T> c = mul(x[S - i], Tt[(S - i) << sh]);
                    ev[i] = vadd(a, c);
                    od[i] = vsub(a, c);
                }
            }
        }
        if (do_sin) {  // elaborations.py:117-122 + classical.py:118-119
            const vec2<T> *x = src + CB + b * S;
            const int cs = sin_stride(d + 1);
            vec2<T> *ev = dst + CB + (2 * b) * cs, *oc = dst + CB + (2 * b + 1) * cs;
            if (i < q - 1) {
                const int sh = logtop - (lognn - d);  // node periodization 2S
                const vec2<T> a = x[i], c = x[S - 2 - i];
                ev[i] = vsub(a, c);
                oc[i] = mul(vadd(a, c), Tt[(i + 1) << sh]);
            } else {
                cen[(1 << d) + b] = x[q - 1];  // the centre s(N/4)
            }
        }
    }

    // stride of the sine nodes of depth d: S, except at the base depth, where one
    // pad cell per node makes the per-thread base accesses (thread = node) bank-conflict free
    QFT_HD int sin_stride(int d) const { return sin_stride_of(lognn, d); }

    // backward level d+1 -> d, item in [0, Nn/4): (node b, slot pair 2i, 2i+1 with i < q)
    QFT_HD void bwd_item(const vec2<T> *chi, vec2<T> *dst, const vec2<T> *cen, int d, int item) const {
        const int lq = lognn - 2 - d, q = 1 << lq, S = 2 * q;
        const int b = item >> lq, i = item & (q - 1);
        if (do_cos) {
            const vec2<T> *se = chi + cos_off(q, 2 * b), *so = chi + cos_off(q, 2 * b + 1);
            vec2<T> *out = dst + cos_off(S, b) + 2 * i;
            const vec2<T> e0 = se[i], o0 = so[i];
            if (!odd_type(d, b)) {  // interleave (elaborations.py:137-140)
                out[0] = e0;
                out[1] = o0;
                if (i == 0) out[S] = se[q];
            } else {  // neighbour sums of the interleave (classical.py:98-99)
                out[0] = vadd(e0, o0);
                out[1] = vadd(o0, se[i + 1]);
            }
        }
        if (do_sin) {  // classical.py:120-128, elaborations.py:145-148
            const int cs = sin_stride(d + 1);
            const vec2<T> *se = chi + CB + (2 * b) * cs, *sp = chi + CB + (2 * b + 1) * cs;
            vec2<T> *out = dst + CB + b * S + 2 * i;
            const vec2<T> center = cen[(1 << d) + b];
            const vec2<T> partial = i == 0 ? sp[0] : (i == q - 1 ? sp[q - 2] : vadd(sp[i - 1], sp[i]));
            out[0] = (i & 1) ? vsub(partial, center) : vadd(partial, center);
            if (i < q - 1) out[1] = se[i];
        }
    }

    // register-level bases at depth D, item in [0, 2^(D+1)): cosine nodes (D nodes
    // first, then O nodes, so warps stay uniform), then sine nodes
    QFT_HD void base_item(vec2<T> *buf, int item) const {
        constexpr int NB = 1 << kBaseLog, SB = NB / 2;
        const int D = depth(), nn = 1 << D;
        const HS<T> hs{Tt, logtop};
        if (item < nn) {
            if (!do_cos) return;
            const int b = D ? (item < nn / 2 ? 2 * item : 2 * (item - nn / 2) + 1) : 0;
            vec2<T> *x = buf + cos_off(SB, b);
            if (!odd_type(D, b)) {
                vec2<T> v[SB + 1], o[SB + 1];
#pragma unroll
                for (int e = 0; e <= SB; ++e) v[e] = x[e];
                dct_r<NB, T>(v, o, hs);
#pragma unroll
                for (int e = 0; e <= SB; ++e) x[e] = o[e];
            } else {
                vec2<T> v[SB], o[SB];
#pragma unroll
                for (int e = 0; e < SB; ++e) v[e] = x[e];
                dct_odd_r<2 * NB, T>(v, o, hs);
#pragma unroll
                for (int e = 0; e < SB; ++e) x[e] = o[e];
            }
        } else {
            if (!do_sin) return;
            vec2<T> *x = buf + CB + (item - nn) * (D ? SB + 1 : SB);
            vec2<T> v[SB - 1], o[SB - 1];
#pragma unroll
            for (int e = 0; e < SB - 1; ++e) v[e] = x[e];
            dst_r<NB, T>(v, o, hs);
#pragma unroll
            for (int e = 0; e < SB - 1; ++e) x[e] = o[e];
        }
    }
    QFT_HD int fwd_items() const { return 1 << (lognn - 2); }
    QFT_HD int bwd_items() const { return 1 << (lognn - 2); }
    QFT_HD int base_items() const { return 2 << depth(); }
};

// ---------------------------------------------------------------- ingest / emit of a whole signal
// MODE 0 cdft, 1 rdft, 2 dct0, 3 dst0 (two real rows a, b ride in one vec2).
// ingest item n in [0, m): shared.rdft_packed fold (shared.py:28-35) into the
// roots (cosine root at 0, sine root at CB)
template <int MODE, typename T>
QFT_HD void ingest_item(const void *in, long long unit, long long nreal, int N, vec2<T> *buf, int CB, int n) {
    const int m = N / 2;
    if constexpr (MODE == 0) {
        const vec2<T> *x = (const vec2<T> *)in + unit * N;
        if (n == 0) {
            buf[0] = x[0];
            buf[m] = x[m];
        } else {
            const vec2<T> h = x[n], t = x[N - n];
            buf[n] = vadd(h, t);
            buf[CB + n - 1] = vsub(h, t);
        }
    } else {
        const T *xr = (const T *)in;
        const long long RL = MODE == 1 ? N : (MODE == 2 ? m + 1 : m - 1);
        const long long ra = 2 * unit, rb = ra + 1 < nreal ? ra + 1 : ra;
        auto at = [&](int i) { return vec2<T>{xr[ra * RL + i], xr[rb * RL + i]}; };
        if constexpr (MODE == 1) {
            if (n == 0) {
                buf[0] = at(0);
                buf[m] = at(m);
            } else {
                const vec2<T> h = at(n), t = at(N - n);
                buf[n] = vadd(h, t);
                buf[CB + n - 1] = vsub(h, t);
            }
        } else if constexpr (MODE == 2) {
            buf[n] = at(n);
            if (n == 0) buf[m] = at(m);
        } else {
            if (n < m - 1) buf[CB + n] = at(n);
        }
    }
}

// emit item k in [0, m]: shared.cdft_interleaved recombination (shared.py:58-72)
// or the real modes' outputs
template <int MODE, typename T>
QFT_HD void emit_item(void *out, long long unit, long long nreal, int N, const vec2<T> *buf, int CB, int k) {
    const int m = N / 2;
    const bool edge = (k == 0) || (k == m);
    if constexpr (MODE == 0) {
        vec2<T> *y = (vec2<T> *)out + unit * N;
        if (edge) {
            y[k] = buf[k];
        } else {
            const vec2<T> cv = buf[k], sv = buf[CB + k - 1], uu = {sv.y, -sv.x};
            y[k] = vadd(cv, uu);
            y[N - k] = vsub(cv, uu);
        }
    } else {
        const long long ra = 2 * unit;
        const bool has_b = ra + 1 < nreal;
        if constexpr (MODE == 1) {
            vec2<T> *ya = (vec2<T> *)out + ra * (m + 1);
            const vec2<T> cv = buf[k];
            const vec2<T> sv = edge ? vec2<T>{(T)0, (T)0} : buf[CB + k - 1];
            ya[k] = {cv.x, edge ? (T)0 : -sv.x};
            if (has_b) ya[m + 1 + k] = {cv.y, edge ? (T)0 : -sv.y};
        } else if constexpr (MODE == 2) {
            T *ya = (T *)out + ra * (m + 1);
            ya[k] = buf[k].x;
            if (has_b) ya[m + 1 + k] = buf[k].y;
        } else {
            if (k < m - 1) {
                T *ya = (T *)out + ra * (m - 1);
                ya[k] = buf[CB + k].x;
                if (has_b) ya[m - 1 + k] = buf[CB + k].y;
            }
        }
    }
}

}  // namespace cl
}  // namespace qft
