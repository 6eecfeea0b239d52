// qft_leaf.cuh -- one CTA-resident Lee block ("leaf") of the multi-pass path.
//
// A leaf of L = 2^A cells (A > 10) is held in shared memory in natural element
// order (padded address p + p/32).  Its Lee DCT-II / DST-II (improved._dct_ii /
// _dst_ii, improved.py:49-112) runs as
//   TF  RT = A-10 forward fold levels per reflection group, results held in
//       registers across one CTA barrier, then stored sub-block-major
//   U   every 1024-cell sub-block is a warp unit (qft_launch.cuh unit_big)
//       -> natural sub-block spectrum in place
//   TB  RT backward levels (neighbour sums + interleave) per column i of the
//       sub-block spectra -> block spectrum slots [i 2^RT, (i+1) 2^RT)
// Same fold / secant / neighbour-sum operations as the reference recursion, in
// the same order, so the spectrum is bit-identical.
#pragma once
#include "qft_smem.cuh"
#include "qft_large.cuh"

namespace qft {

template <int A, bool DST, typename T>
struct LeafTop {
    static constexpr int L = 1 << A, RT = A - 10, G = 1 << RT, S = 1024;
    static_assert(A > 10, "leaves above one warp unit");
    // TF item t in [0, 1024): reflection group t, RT levels (slot p = element t
    // of sub-block p); the caller holds v across a CTA barrier, then stores
    // sub-block-major (sub-block p at cells [1024p, 1024p + 1024))
    // rev: the run was loaded in memory order and is reversed (element e at L-1-e)
    QFT_HD static void tf_load(const vec2<T> *s, const T *U, int t, vec2<T> *v, bool rev = false) {
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int c, sg;
            run_of(RT, L, q, c, sg);
            const int e = c + sg * t;
            v[q] = s[padx(rev ? L - 1 - e : e)];
        }
        lee_fwd<RT, L, DST, T>(v, t, U);
    }
    // the same, with the leaf being all of Lee block j read straight from the
    // input signal x (first touch folds x[n] +- x[N-n], shared.py:28-35)
    QFT_HD static void tf_load_x(const vec2<T> *x, int N, int j, const T *U, int t, vec2<T> *v) {
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int c, sg;
            run_of(RT, L, q, c, sg);
            v[q] = fold_load<T, DST>(x, N, j, c + sg * t);
        }
        lee_fwd<RT, L, DST, T>(v, t, U);
    }
    QFT_HD static void tf_store(vec2<T> *s, int t, const vec2<T> *v) {
#pragma unroll
        for (int p = 0; p < G; ++p) s[padx(S * p + t)] = v[p];
    }
    // TB column i in [0, 1024): reads the natural sub-block spectra (+ halo
    // column), outputs block spectrum slots [i 2^RT, (i+1) 2^RT)
    QFT_HD static void tb(const vec2<T> *s, int i, vec2<T> *out) {
        const int ih = DST ? (i > 0 ? i - 1 : i) : (i < S - 1 ? i + 1 : i);
        vec2<T> own[G];
#pragma unroll
        for (int p = 0; p < G; ++p) own[p] = s[padx(S * p + i)];
        auto halo = [&](int p) { return s[padx(S * p + ih)]; };
        const bool edge = DST ? (i == 0) : (i == S - 1);
        lee_bwd_fn<RT, DST, T>(own, 0, halo, edge, out);
    }
};

// The cosine and the sine leaf of one Lee block read straight from x: one gather
// of x[n], x[N-n] feeds both folds (dc = a + b, ds = a - b, shared.py:28-35), then
// each side runs its own RT levels -- the operations of two tf_load_x calls.
template <int A, typename T>
QFT_HD void tf_load_x_pair(const vec2<T> *x, int N, int j, const T *U, int t, vec2<T> *vc, vec2<T> *vs) {
    using LC = LeafTop<A, false, T>;
#pragma unroll
    for (int q = 0; q < LC::G; ++q) {
        int c, sg;
        run_of(LC::RT, LC::L, q, c, sg);
        const int n = (2 * (c + sg * t) + 1) << j;
        const vec2<T> a = x[n], b = x[N - n];
        vc[q] = vadd(a, b);
        vs[q] = vsub(a, b);
    }
    lee_fwd<LC::RT, LC::L, false, T>(vc, t, U);
    lee_fwd<LC::RT, LC::L, true, T>(vs, t, U);
}

}  // namespace qft
