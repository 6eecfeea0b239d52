// qft_smem.cuh -- improved-QFT of length-N complex signals (N = 2^6 .. 2^14)
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
//   D   time-split chain (elaborations.py:78-89) + complex
//       recombination (shared.py:58-72)                          W -> global
// N > 4096: the "huge" Lee blocks (L > 1024) first get RT = n-12-j top fold
// levels from the whole CTA (TF, W -> W, 1024-cell sub-blocks written
// sub-block-major), then every 1024-cell sub-block is a warp unit exactly like
// block 0 of N = 4096, then the whole CTA runs the RT top backward levels (TB).
#pragma once
#include "qft_lee.cuh"

#ifndef QFT_A0_SPLIT
#define QFT_A0_SPLIT 0  // A0 even-sample stores in two groups (block 1 / blocks >= 2)
#endif
#ifndef QFT_A0_LANE0
#define QFT_A0_LANE0 0  // A0 chunk lane 0 also folds n = 64c (else a separate pass)
#endif
#ifndef QFT_CHAIN_LIN
#define QFT_CHAIN_LIN 0  // phase-D unfold with linear addresses (Chain::up_l); measured neutral (58.3 vs 58.5M, config 2)
#endif
#ifndef QFT_RC_SMALL
#define QFT_RC_SMALL 5  // phase-D unfold depth for N = 2^12
#endif
#ifndef QFT_RC_MID
// N = 512 .. 2048 and N <= 256: the small CTAs of these sizes (several resident per SM,
// qft_launch.cuh cps_for) want more, shorter phase-D items.  Measured depth 5 / 4 / 3
// (GB/s, tools/size_sweep.py): fp32 2^7 2882 / 3436 / 3807, 2^8 2968 / 3464 / 3533,
// 2^9 3375 / 3736 / 3680, 2^10 3646 / 3796 / 3630, 2^11 3364 / 3363 / 3241;
// fp64 2^7 3239 / 4007 / 4135, 2^9 3447 / 3644 / 3624, 2^11 3338 / 3455 / 3410
#define QFT_RC_MID 4
#endif
#ifndef QFT_RC_TINY
#define QFT_RC_TINY 3
#endif
#ifndef QFT_RC_BIG
#define QFT_RC_BIG 5  // phase-D unfold depth for N >= 2^13 (257 items at 2^14)
#endif

#ifndef QFT_SC
// Sine side stored "as cosine": the sine cell of odd index (its element index
// within the Lee block has the same parity) holds -ds instead of ds, the
// cosine-side code runs on it (with the DST's L = 2 base constant), and each
// sine block's spectrum lands reversed (slot k at L-1-k).  Exact: negation
// commutes with IEEE rounding, the DCT fold of (a, -b) is the DST fold of
// (a, b) (x - y == x + (-y)), and the DCT-II of ((-1)^i x_i) is the reversed
// DST-II of x operation for operation (tests/emu checks it bit for bit).  One
// code path for both sides halves the warp-unit code the instruction cache
// must hold (ncu: no_instruction was the top stall of the unit phase).
#define QFT_SC 1
#endif

namespace qft {

QFT_HD constexpr int padx(int p) { return p + (p >> 5); }

// the sine cell with index `cell` (relative to the sine region) of the fold
// a = x[n], b = x[N-n]: ds = a - b, negated on odd cells when QFT_SC
template <typename T>
QFT_HD vec2<T> sine_cell(vec2<T> a, vec2<T> b, int cell) {
    return (QFT_SC && (cell & 1)) ? vsub(b, a) : vsub(a, b);
}
// a value placed on the sine side as is (dst0 input), negated on odd cells when QFT_SC
template <typename T>
QFT_HD vec2<T> sine_val(vec2<T> v, int cell) {
    return (QFT_SC && (cell & 1)) ? vec2<T>{-v.x, -v.y} : v;
}

template <int LOG2N>
struct SPlan {
    static constexpr int n = LOG2N, N = 1 << LOG2N, m = N / 2, q = N / 4;
    static constexpr int JF = n > 7 ? n - 7 : 0;     // big blocks j < JF (L > 32)
    static constexpr int JS = n - 6;                 // first small block (L = 16)
    static constexpr int RC0 = n >= 13 ? QFT_RC_BIG : (n >= 12 ? QFT_RC_SMALL : (n >= 9 ? QFT_RC_MID : QFT_RC_TINY));
    static constexpr int RC = n - 2 < RC0 ? n - 2 : RC0;  // chain levels unfolded in phase D
    static constexpr int L(int j) { return 1 << (n - 2 - j); }
    static constexpr int off(int j) { return m - 2 * L(j); }
    static constexpr int RF(int j) { return n - 7 - j; }  // big block: L = 32 << RF
    static constexpr int S0 = m;                     // sine region
    static constexpr int BASE = N - 1;               // s(0) at N-1, s(m) at N
    static constexpr int CELLS = N + 1;
    static constexpr int PADDED = CELLS + CELLS / 32 + 1;
    static constexpr int NL32 = n >= 7 ? m / 32 - 1 : 0;  // Lee-32 chunks per side
    static constexpr int MRC = N >> (RC + 1);        // m_RC: phase-D thread t in [0, MRC]
    static constexpr int DT = MRC + 1;               // phase D threads per signal
    static constexpr int UCELLS = N / 4;             // level-table entries
    // huge blocks (L > 1024): j < JH, RT(j) top levels leave 1024-cell sub-blocks
    static constexpr int JH = n > 12 ? n - 12 : 0;
    static constexpr int RT(int j) { return n - 12 - j; }
    // "big" warp units per side: block 0 (n <= 12), or every 1024-cell
    // (sub-)block of the blocks j <= n-12 (n > 12); the "rest" unit does the
    // blocks j >= JR, the L = 32 block and the small blocks
    static constexpr int NU1 = n <= 12 ? (JF >= 1 ? 1 : 0) : (1 << (n - 11)) - 1;
    static constexpr int JR = n <= 12 ? 1 : n - 11;
    static constexpr int K0 = JF >= 1 ? off(JR) / 32 : 0;  // first Lee-32 chunk of the rest unit
    static constexpr int LB = n <= 12 ? (JF >= 1 ? L(0) : 32) : 1024;  // big unit length
    static constexpr int RB = n <= 12 ? (JF >= 1 ? RF(0) : 0) : 5;
    // first cell of big unit u (one side)
    static QFT_HD int big_cell(int u) {
        if (n <= 12) return 0;
        int j = 0;
        while (u >= (1 << RT(j))) {
            u -= 1 << RT(j);
            ++j;
        }
        return off(j) + 1024 * u;
    }
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
        w[padx(cell)] = vadd(a, b);                       // dc[n]   = x[n] + x[N-n]
        w[padx(P::S0 + cell)] = sine_cell(a, b, cell);    // ds[n-1] = x[n] - x[N-n]
    }
}

// A0 by chunks of 64 consecutive n (n = 64c + 2l and 64c + 2l + 1 for lane l):
// one aligned pair load per side, the odd samples (Lee block 0) go to 32
// consecutive cells, the even ones to block 1 + ctz(l); lane l's even mirror
// x[N - 64c - 2l] is the first element of lane l-1's mirror pair.
struct A0Lane64 {
    int A, B, sh;  // padded cosine cell of the even sample of chunk c: A + c*B + (c >> sh)
    int lj;        // its unpadded cell is off + c*B + lj (parity: (c*B + lj) & 1)
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
    r.lj = l >> j;
    return r;
}
template <typename T>
struct A0Chunk64 {
    vec2<T> xe, xo, mn, mo, m0;
    // lane 0 also loads the mirror x[N - 64c] of its even sample n = 64c
    // (x[m] for c = 0: the base pair s(0), s(m))
    template <int LOG2N>
    QFT_HD void load(const vec2<T> *x, int c, int l) {
        constexpr int N = 1 << LOG2N;
        ld2(x + 64 * c + 2 * l, xe, xo);             // x[n_e], x[n_o]
        ld2(x + N - 64 * c - 2 * l - 2, mn, mo);     // x[N - n_e - 2], x[N - n_o]
        if (QFT_A0_LANE0 && l == 0) m0 = x[c ? N - 64 * c : N / 2];
    }
    // Stores: the odd samples (block 0, 32 consecutive cells), then the even
    // samples in two groups -- block 1 (odd lanes, 16 consecutive cells) and
    // blocks >= 2 (with lane 0's n = 64c) -- so no store instruction mixes the
    // block-1 run with the other blocks (bank conflicts).
    template <int LOG2N, class ShflUp>
    QFT_HD void store(vec2<T> *w, int c, int l, const A0Lane64 &a, ShflUp &&shfl_up) const {
        using P = SPlan<LOG2N>;
        constexpr int PS = padx(P::S0);
        const vec2<T> me = shfl_up(mn);                  // x[N - n_e] from lane l-1
        const int po = 33 * c + l;                       // block 0 cell 32c + l, padded
        w[po] = vadd(xo, mo);
        w[po + PS] = sine_cell(xo, mo, l);  // cell 32c + l
        const int pe = a.A + c * a.B + (c >> a.sh);
        const int pc = c * a.B + a.lj;      // parity of the even sample's cell
#if QFT_A0_SPLIT
        if (l & 1) {
            w[pe] = vadd(xe, me);
            w[pe + PS] = sine_cell(xe, me, pc);
        }
#if defined(__CUDA_ARCH__)
        __syncwarp();
#endif
        if (l > 0 && !(l & 1)) {
#else
        if (l > 0) {
#endif
            w[pe] = vadd(xe, me);
            w[pe + PS] = sine_cell(xe, me, pc);
        } else if (QFT_A0_LANE0 && l == 0) {
            if (c == 0) {
                w[padx(P::BASE)] = xe;      // dc[0] = x[0]
                w[padx(P::BASE + 1)] = m0;  // dc[m] = x[m]
            } else {
                const int n = 64 * c, j = ctz32((uint32_t)n);
                const int cell = P::m - (1 << (LOG2N - 1 - j)) + (n >> (j + 1));
                w[padx(cell)] = vadd(xe, m0);
                w[padx(P::S0 + cell)] = sine_cell(xe, m0, cell);
            }
        }
    }
};
template <int LOG2N, typename T, class ShflUp>
QFT_HD void a0_chunk64(const vec2<T> *x, vec2<T> *w, int c, int l, A0Lane64 a, ShflUp &&shfl_up) {
    A0Chunk64<T> ch;
    ch.template load<LOG2N>(x, c, l);
    ch.template store<LOG2N>(w, c, l, a, shfl_up);
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
            w[padx(P::S0 + c)] = sine_cell(a, b, c);
        }
    } else if constexpr (MODE == 2) {  // dct0: values s(0..m) are the cosine signal
        if (n == 0) w[padx(P::BASE)] = at(0);
        else if (n == P::m) w[padx(P::BASE + 1)] = at(P::m);
        else w[padx(cell_of(n))] = at(n);
    } else {  // dst0: values s(1..m-1) are the sine signal (slot n-1)
        if (n > 0 && n < P::m) w[padx(P::S0 + cell_of(n))] = sine_val(at(n - 1), cell_of(n));
    }
}

// ---------------------------------------------------------------- phase A
// Lane t of the warp owning a big block of L = 32 << R cells (padded pointer wb
// to its first cell, a multiple of 32): loads its reflection group, folds R
// levels, and (after __syncwarp) writes element t of sub-block p to cell 32p + t.
template <int L, int R, bool DST, typename T>
struct FBlockP {
    static constexpr int G = 1 << R, NCH = L / 32;
    vec2<T> v[G];
    // REV: the block's element e is stored at cell L-1-e (a reversed run)
    template <bool REV = false>
    QFT_HD void load(const vec2<T> *wb, const T *U, int t) {
        const vec2<T> *bf = wb + t;       // forward runs
        const vec2<T> *br = wb + 31 - t;  // reversed runs
#pragma unroll
        for (int s = 0; s < G; ++s) {
            int c, sg;
            run_of(R, L, s, c, sg);  // compile-time after unrolling
            const int u = c >> 5;    // the run is the 32-aligned chunk u
            if constexpr (REV)       // chunk u is stored as chunk NCH-1-u, direction flipped
                v[s] = sg > 0 ? br[33 * (NCH - 1 - u)] : bf[33 * (NCH - 1 - u)];
            else
                v[s] = sg > 0 ? bf[33 * u] : br[33 * u];
        }
        lee_fwd<R, L, DST, T>(v, t, U);
    }
    QFT_HD void store(vec2<T> *wb, int t) const {
        vec2<T> *o = wb + t;
#pragma unroll
        for (int p = 0; p < G; ++p) o[33 * p] = v[p];
    }
};
// Lee block J of one side of a signal at w
template <int LOG2N, int J, bool DST, typename T>
struct FBlock : FBlockP<SPlan<LOG2N>::L(J), SPlan<LOG2N>::RF(J), DST, T> {
    using P = SPlan<LOG2N>;
    using Base = FBlockP<P::L(J), P::RF(J), DST, T>;
    static constexpr int base = (DST ? P::S0 : 0) + P::off(J);  // multiple of 32
    QFT_HD void load(const vec2<T> *w, const T *U, int t) { Base::load(w + padx(base), U, t); }
    QFT_HD void store(vec2<T> *w, int t) const { Base::store(w + padx(base), t); }
};

// ---------------------------------------------------------------- top levels (N > 4096)
// Huge block J of one side (L > 1024, RT = n-12-J top levels).  TF item t in
// [0, 1024): the reflection group t, RT forward levels, element t of sub-block p
// -> cell 1024p + t.  TB item i in [0, 1024): column i of the 2^RT sub-block
// spectra (+ halo column) -> block spectrum slots [i 2^RT, (i+1) 2^RT).
template <int LOG2N, int J, bool DST, typename T>
struct Top {
    using P = SPlan<LOG2N>;
    static constexpr int L = P::L(J), R = P::RT(J), G = 1 << R;
    static constexpr int base = (DST ? P::S0 : 0) + P::off(J);
    static_assert(L >> R == 1024, "top levels leave 1024-cell sub-blocks");
    QFT_HD static void f_load(const vec2<T> *w, const T *U, int t, vec2<T> *v) {
#pragma unroll
        for (int s = 0; s < G; ++s) {
            int c, sg;
            run_of(R, L, s, c, sg);
            v[s] = w[padx(base + c + sg * t)];
        }
        lee_fwd<R, L, DST, T>(v, t, U);
    }
    QFT_HD static void f_store(vec2<T> *w, int t, const vec2<T> *v) {
#pragma unroll
        for (int p = 0; p < G; ++p) w[padx(base + 1024 * p + t)] = v[p];
    }
    QFT_HD static void b_compute(const vec2<T> *w, int i, vec2<T> *out) {
        const int ih = DST ? (i > 0 ? i - 1 : i) : (i < 1023 ? i + 1 : i);
        vec2<T> own[G];
#pragma unroll
        for (int p = 0; p < G; ++p) own[p] = w[padx(base + 1024 * p + i)];
        auto halo = [&](int p) { return w[padx(base + 1024 * p + ih)]; };
        const bool edge = DST ? (i == 0) : (i == 1023);
        lee_bwd_fn<R, DST, T>(own, 0, halo, edge, out);
    }
    QFT_HD static void b_store(vec2<T> *w, int i, const vec2<T> *out) {
        vec2<T> *o = w + padx(base + i * G);  // G <= 32 slots inside one 32-cell chunk
#pragma unroll
        for (int s = 0; s < G; ++s) o[s] = out[s];
    }
};

// ---------------------------------------------------------------- phase B
// Lee-32 on the 32-cell chunk at padded pointer c; in place.
// ub: the L = 2 base constant index (lee_full).  QFT_L32_CALL: one copy of the
// Lee-32 body for the big and the rest units (instruction-cache footprint)
#ifndef QFT_L32_CALL
#define QFT_L32_CALL 0  // measured slower (54.0 vs 58.3M tr/s, config 2): the call boundary costs more than the saved instruction fetch
#endif
#if QFT_L32_CALL
#define QFT_L32_ATTR QFT_HD_CALL
#else
#define QFT_L32_ATTR QFT_HD
#endif
#ifndef QFT_PRESUM
// The Lee-32 step of an odd sub-block (odd chunk index: every block cut into
// sub-blocks starts at an even chunk and has an even number of them, and the
// uncut L = 32 block sits at an even chunk) also forms the first backward level's
// neighbour sums Z[i] + Z[i+1] -- the same operation on the same operands the C
// step would do with a halo read of the next column -- so phase C reads 15 halo
// cells per column instead of 31 (lee_bwd_fn PRE, qft_lee.cuh).
#define QFT_PRESUM 1
#endif
// pre: this chunk is an odd sub-block of a cut block (QFT_PRESUM)
template <bool DST, typename T>
QFT_L32_ATTR void b_l32p(vec2<T> *c, const T *U, int ub = DST ? 1 : 0, bool pre = false) {
    vec2<T> v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = c[e];
    lee_full<32, DST, T>(v, U, ub);
    if (QFT_PRESUM && pre) {
        if constexpr (!DST) {
#pragma unroll
            for (int e = 0; e < 31; ++e) v[e] = vadd(v[e], v[e + 1]);  // column 31: the edge copy
        } else {
#pragma unroll
            for (int e = 31; e > 0; --e) v[e] = vadd(v[e - 1], v[e]);  // column 0: the edge copy
        }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) c[e] = v[e];
}
template <bool DST, typename T>
QFT_HD void b_l32(vec2<T> *w, int chunk_base, const T *U, int ub = DST ? 1 : 0, bool pre = false) {
    b_l32p<DST, T>(w + padx(chunk_base), U, ub, pre);
}

template <int LOG2N, bool DST, typename T, int J>
QFT_HD void b_small_rec(vec2<T> *w, const T *U, int ub) {
    using P = SPlan<LOG2N>;
    if constexpr (J <= LOG2N - 2) {
        constexpr int L = P::L(J);
        vec2<T> v[L];
        constexpr int b0 = (DST ? P::S0 : 0) + P::off(J);
#pragma unroll
        for (int e = 0; e < L; ++e) v[e] = w[padx(b0 + e)];
        lee_full<L, DST, T>(v, U, ub);
#pragma unroll
        for (int e = 0; e < L; ++e) w[padx(b0 + e)] = v[e];
        b_small_rec<LOG2N, DST, T, J + 1>(w, U, ub);
    }
}
// all blocks with L <= 16 of one side
template <int LOG2N, bool DST, typename T>
QFT_HD void b_small(vec2<T> *w, const T *U, int ub = DST ? 1 : 0) {
    constexpr int J0 = SPlan<LOG2N>::JS > 0 ? SPlan<LOG2N>::JS : 0;
    b_small_rec<LOG2N, DST, T, J0>(w, U, ub);
}

// ---------------------------------------------------------------- phase C
// Lane i of the warp owning a big block (2^R sub-blocks of 32, padded pointer
// wb): column i of the sub-block spectra -> block spectrum slots
// [i*2^R, (i+1)*2^R), natural order.  The halo Z_p[i+1] (DCT) / Z_p[i-1] (DST)
// is the neighbour lane's own value.
template <int R, bool DST, typename T>
struct CBlockP {
    static constexpr int G = 1 << R;
    vec2<T> own[G];
    QFT_HD void load(const vec2<T> *wb, int i) {
        const vec2<T> *c = wb + i;
#pragma unroll
        for (int p = 0; p < G; ++p) own[p] = c[33 * p];
    }
    // halo column (i+1 for DCT, i-1 for DST; the edge lane re-reads its own column)
    QFT_HD static const vec2<T> *halo_colp(const vec2<T> *wb, int i) {
        const int ih = DST ? (i > 0 ? i - 1 : i) : (i < 31 ? i + 1 : i);
        return wb + ih;
    }
    // halo(p) must return the neighbour lane's own[p]
    template <class Halo>
    QFT_HD void compute(int i, Halo &&halo, vec2<T> *out) const {
        const bool edge = DST ? (i == 0) : (i == 31);
        lee_bwd_fn<R, DST, T, Halo, QFT_PRESUM != 0>(own, 0, halo, edge, out);
    }
    QFT_HD static void storep(vec2<T> *wb, int i, const vec2<T> *out) {
        // slots i*G .. i*G+G-1 lie inside one 32-cell chunk: contiguous when padded
        vec2<T> *o = wb + i * G + ((i * G) >> 5);
#pragma unroll
        for (int s = 0; s < G; ++s) o[s] = out[s];
    }
};
template <int LOG2N, int J, bool DST, typename T>
struct CBlock : CBlockP<SPlan<LOG2N>::RF(J), DST, T> {
    using P = SPlan<LOG2N>;
    using Base = CBlockP<P::RF(J), DST, T>;
    static constexpr int base = (DST ? P::S0 : 0) + P::off(J);
    QFT_HD void load(const vec2<T> *w, int i) { Base::load(w + padx(base), i); }
    QFT_HD static const vec2<T> *halo_col(const vec2<T> *w, int i) { return Base::halo_colp(w + padx(base), i); }
    QFT_HD static void store(vec2<T> *w, int i, const vec2<T> *out) { Base::storep(w + padx(base), i, out); }
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
    // (QFT_SC: the block spectrum is stored reversed, slot h-1 at L_j - h)
    static QFT_HD vec2<T> OS(const vec2<T> *w, int j, int h) {
        return w[padx(P::S0 + P::off(j) + (QFT_SC ? P::L(j) - h : h - 1))];
    }

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
#ifdef QFT_DIAG_NOSTORE  // diagnostic only (tools/probe): keep the math, drop the stores
        const vec2<T> a = edge ? cv : vadd(cv, u), b = vsub(cv, u);
        if (a.x == (T)1.2345e-30 && b.y == (T)1.2345e-30) y[k] = a;
#else
        y[k] = edge ? cv : vadd(cv, u);
        if (!edge) y[P::N - k] = vsub(cv, u);
#endif
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

    // ---- the same unfold with linear addresses (QFT_SC, L_{RC-1} >= 32) ----------
    // Every index the unfold reads at level J is k = K + S*t with K a compile-time
    // multiple of 32 (0, m_J - K, ...) and S = +-1, and every block it reads is
    // 32-aligned, so the padded address is padx(cell(K)) + (S > 0 ? fwd : rev) with
    // the per-thread constants fwd = padx(K0 + t) - padx(K0) = t + t/32 and
    // rev = padx(K0 - t) - padx(K0) = -t - ceil(t/32) (any K0 = 0 mod 32): one
    // shared load with an immediate offset per value instead of index arithmetic.
    // Reads of a self-paired / harmonic-0 slot fall on a neighbouring cell of the
    // working area and are discarded by the same selects as in up_e.
    static constexpr bool LIN = QFT_CHAIN_LIN && QFT_SC && P::RC >= 1 && P::RC < n - 1 && (P::N >> (P::RC + 1)) >= 32;
    template <int J, int K, int S, class Emit>
    static QFT_HD void up_l(const vec2<T> *w, Emit &emit, int k, vec2<T> cv, vec2<T> sv, int fwd, int rev) {
        if constexpr (J == 0) {
            emit(k, cv, sv);
        } else {
            constexpr int q = qj(J - 1), mm = 2 * q;
            constexpr int CB = P::off(J - 1) + K;                  // OC(J-1, K) cell
            constexpr int SB = P::S0 + P::off(J - 1) + P::L(J - 1) - K;  // OS(J-1, K) cell (reversed)
            static_assert(CB % 32 == 0 && SB % 32 == 0, "linear unfold needs 32-aligned cells");
            const bool self = (k == q);
            const vec2<T> o = w[padx(CB) + (S > 0 ? fwd : rev)];
            const vec2<T> os = w[padx(SB) + (S > 0 ? rev : fwd)];
            up_l<J - 1, K, S>(w, emit, k, self ? cv : vadd(cv, o), self ? os : vadd(os, sv), fwd, rev);
            up_l<J - 1, mm - K, -S>(w, emit, self ? q : mm - k, self ? cv : vsub(cv, o), self ? os : vsub(os, sv),
                                    fwd, rev);
        }
    }

    template <class Emit>
    static QFT_HD void unit_e(const vec2<T> *w, Emit &emit, int t) {
        vec2<T> cv, sv;
        if constexpr (P::RC < n - 1) desc2<P::RC>(w, t, cv, sv);
        if constexpr (LIN) up_l<P::RC, 0, 1>(w, emit, t, cv, sv, t + (t >> 5), -t - ((t + 31) >> 5));
        else up_e<P::RC>(w, emit, t, cv, sv);
    }
    static QFT_HD void unit(const vec2<T> *w, vec2<T> *y, int t) {
        auto emit = [&](int k, vec2<T> cv, vec2<T> sv) { emit_u(y, k, cv, sv); };
        unit_e(w, emit, t);
    }
    // half of a phase-D item: the descent, then the low (h = 0) or high (h = 1)
    // child of the first unfold level (selected branch-free), then RC-1 levels
    template <class Emit>
    static QFT_HD void unit_e_half(const vec2<T> *w, Emit &emit, int t, int h) {
        static_assert(P::RC >= 1, "half items need one unfold level");
        vec2<T> cv, sv;
        if constexpr (P::RC < n - 1) desc2<P::RC>(w, t, cv, sv);
        constexpr int q = qj(P::RC - 1), mm = 2 * q;
        const bool self = (t == q);
        const vec2<T> o = OC(w, P::RC - 1, t < q ? t : 0);
        const vec2<T> os = OS(w, P::RC - 1, t > 0 ? t : 1);
        const vec2<T> c_lo = vadd(cv, o), c_hi = vsub(cv, o), s_lo = vadd(os, sv), s_hi = vsub(os, sv);
        const int k = h ? (self ? q : mm - t) : t;
        const vec2<T> c1 = self ? cv : (h ? c_hi : c_lo), s1 = self ? os : (h ? s_hi : s_lo);
        up_e<P::RC - 1>(w, emit, k, c1, s1);
    }
    static QFT_HD void unit_half(const vec2<T> *w, vec2<T> *y, int t, int h) {
        auto emit = [&](int k, vec2<T> cv, vec2<T> sv) { emit_u(y, k, cv, sv); };
        unit_e_half(w, emit, t, h);
    }
};

}  // namespace qft
