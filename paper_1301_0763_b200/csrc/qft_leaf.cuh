// qft_leaf.cuh -- one CTA-resident Lee block ("leaf") of the multi-pass path.
//
// A leaf of L = 2^A cells (A > 10) is held in shared memory in natural element
// order (padded address p + p/32).  Its Lee DCT-II / DST-II (improved._dct_ii /
// _dst_ii, improved.py:49-112) runs as
//   TF  RT = A-10 forward fold levels, in place: reflection group t keeps its
//       cells, so sub-block p is the (possibly reversed) run run_of(RT, L, p)
//   U   every 1024-cell sub-block is a warp unit (qft_launch.cuh unit_big,
//       reading a reversed run with REV) -> natural sub-block spectrum at the
//       run's lowest cell
//   TB  RT backward levels (neighbour sums + interleave) per column i of the
//       sub-block spectra -> block spectrum slots [i 2^RT, (i+1) 2^RT)
// Same fold / secant / neighbour-sum operations as the reference recursion, in
// the same order, so the spectrum is bit-identical.
#pragma once
#include "qft_smem.cuh"

namespace qft {

template <int A, bool DST, typename T>
struct LeafTop {
    static constexpr int L = 1 << A, RT = A - 10, G = 1 << RT, S = 1024;
    static_assert(A > 10, "leaves above one warp unit");
    // TF item t in [0, 1024): in place
    QFT_HD static void tf(vec2<T> *s, const T *U, int t) {
        vec2<T> v[G];
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int c, sg;
            run_of(RT, L, q, c, sg);
            v[q] = s[padx(c + sg * t)];
        }
        lee_fwd<RT, L, DST, T>(v, t, U);
#pragma unroll
        for (int q = 0; q < G; ++q) {
            int c, sg;
            run_of(RT, L, q, c, sg);
            s[padx(c + sg * t)] = v[q];
        }
    }
    // sub-block p: lowest cell and direction
    QFT_HD static void sub(int p, int &lo, bool &rev) {
        int c, sg;
        run_of(RT, L, p, c, sg);
        rev = sg < 0;
        lo = rev ? c - (S - 1) : c;
    }
    // TB column i in [0, 1024): reads the natural sub-block spectra (+ halo column)
    QFT_HD static void tb(const vec2<T> *s, int i, vec2<T> *out) {
        const int ih = DST ? (i > 0 ? i - 1 : i) : (i < S - 1 ? i + 1 : i);
        vec2<T> own[G];
        int lo[G];
#pragma unroll
        for (int p = 0; p < G; ++p) {
            int c, sg;
            run_of(RT, L, p, c, sg);
            lo[p] = sg > 0 ? c : c - (S - 1);
            own[p] = s[padx(lo[p] + i)];
        }
        auto halo = [&](int p) { return s[padx(lo[p] + ih)]; };
        const bool edge = DST ? (i == 0) : (i == S - 1);
        lee_bwd_fn<RT, DST, T>(own, 0, halo, edge, out);
    }
};

}  // namespace qft
