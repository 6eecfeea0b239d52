// qft_large_plan.h -- host-side schedule of the multi-pass path (pure C++, also
// used by the test-only CPU emulator).
//
// Replays the improved recursion at the level of Lee blocks (improved.py:49-112:
// fold, secant-scale the odd child, recurse, neighbour sums): every block of the
// time-parity chain (improved.py:43, :81) larger than the leaf size 2^LEAFLOG is
// cut by forward passes of at most RG fold levels.  A pass keeps every slot of a
// reflection group on its own cells, so each sub-block is a contiguous
// (possibly reversed) run; the schedule records the runs, the backward tasks
// that undo each cut (deepest first) and which scratch buffer (W0/W1) finally
// holds each block's spectrum.  This is the kernel schedule compiled from the
// signal-type decomposition tree (dc_tt -> dc_ot -> dc_oo ..., taxonomy.py).
#pragma once
#include <map>
#include <utility>
#include <vector>

#include "qft_large.cuh"

namespace qft {

struct LargeSchedule {
    int n = 0, N = 0, m = 0;
    int LEAFLOG = 10, RG = 5;  // leaf size 2^LEAFLOG, fold levels per F/B pass
    std::vector<std::map<int, std::vector<std::pair<FTask, int>>>> f;  // [depth][R] -> (task, dst)
    std::vector<std::map<int, std::vector<BTask>>> b;                  // [depth][R]
    std::map<int, std::vector<LeafTask>> leaf;                         // [log2 L]
    uint32_t cmask = 0, smask = 0;  // bit j: block j's final spectrum is in W1

    struct Loc {
        int buf, leaf;
    };

    Loc decompose(int c, int sg, int L, int dst, int depth, int j = -1) {
        int lg = 0;
        while ((1 << lg) < L) ++lg;
        if (lg <= LEAFLOG) {
            leaf[lg].push_back({c, sg, L, dst, j});
            return {0, 1};
        }
        const int r = RG < lg - LEAFLOG ? RG : lg - LEAFLOG;
        if ((int)f.size() <= depth) {
            f.resize(depth + 1);
            b.resize(depth + 1);
        }
        f[depth][r].push_back({FTask{c, sg, L, j}, dst});
        const int S = L >> r;
        Loc sub{0, 1};
        for (int p = 0; p < (1 << r); ++p) {
            int cp, sp;
            run_of(r, L, p, cp, sp);
            sub = decompose(c + sg * cp, sg * sp, S, dst, depth + 1);
        }
        b[depth][r].push_back(BTask{c, sg, L, sub.buf, sub.leaf, 1 - sub.buf, sg > 0 ? c : c - (L - 1), dst});
        return {1 - sub.buf, 0};
    }

    // jmax > 0: only the blocks j < jmax (the rest belong to the sub-signal
    // transform of x[2^jmax k], see qft_large.cu)
    // fold_pass: a separate pass folds x into W0 first (no fold on first touch)
    // first_touch = false: the fold pass covers every block (real modes, whose
    // input is not the complex fold)
    LargeSchedule(int log2n, int leaflog, int rg, int jmax = -1, bool fold_pass = false, bool first_touch = true)
        : n(log2n), N(1 << log2n), m(1 << (log2n - 1)), LEAFLOG(leaflog), RG(rg) {
        fold = fold_pass;
        const int jend = jmax > 0 ? jmax : n - 1;
        // blocks j < jfold are cut by F passes whose first touch folds x; with a
        // fold pass, it folds only the samples of blocks j >= jfold
        jfold = 0;
        while (first_touch && jfold < jend && (1 << (n - 2 - jfold)) > (1 << LEAFLOG)) ++jfold;
        for (int side = 0; side < 2; ++side)
            for (int j = 0; j < jend; ++j) {
                const int L = 1 << (n - 2 - j);
                Loc l = decompose(side * m + m - 2 * L, 1, L, side, 0, (fold_pass && j >= jfold) ? -1 : j);
                if (l.buf) (side ? smask : cmask) |= 1u << j;
            }
    }
    bool fold = false;  // a separate fold pass precedes the F passes
    int jfold = 0;      // the fold pass covers the samples n with ctz(n) >= jfold (and n = 0)
    int passes() const { return (fold ? 3 : 2) + 2 * (int)f.size(); }  // [fold], F..., leaves, B..., chain
};

}  // namespace qft
