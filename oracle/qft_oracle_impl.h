/*
 * oracle/qft_oracle_impl.h -- TEST INFRASTRUCTURE ONLY; included twice by
 * qft_oracle.c with QFT_REAL = double / float.  A scalar restatement of
 *   /root/reference/pkg/src/quickfourier/improved.py   (improved recursion)
 *   /root/reference/pkg/src/quickfourier/classical.py  (classical recursion)
 *   /root/reference/pkg/src/quickfourier/shared.py     (real/complex drivers)
 *   /root/reference/pkg/src/quickfourier/elaborations.py (split kernels)
 * Each function names the reference lines it restates.  `T` is the natural
 * constant table of the top-level periodization NT (see oracle_table_*):
 * a half-secant at local periodization N and time index n is T[n*NT/N].
 */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, QFT_SUF)

typedef QFT_REAL FN(real_t);
#define R FN(real_t)

typedef struct {
    const R *T;   /* natural table T[0..NT/4) */
    int NT;       /* top-level periodization */
    arena_t *ar;
} FN(ctx_t);
#define CTX FN(ctx_t)

static R *FN(rows)(CTX *c, int n) { return (R *)arena_alloc(c->ar, sizeof(R) * (size_t)(n > 0 ? n : 1)); }
static R FN(hsec)(CTX *c, int n, int N) { return c->T[(long)n * (c->NT / N)]; }

/* ================= improved recursion (improved.py:36-112) ================= */
static void FN(imp_dct)(CTX *c, const R *x, int N, R *out);
static void FN(imp_dct_ot)(CTX *c, const R *x, int N, R *out);
static void FN(imp_dct_oo)(CTX *c, const R *x, int N, R *out);
static void FN(imp_dst)(CTX *c, const R *x, int N, R *out);
static void FN(imp_dst_ot)(CTX *c, const R *x, int N, R *out);
static void FN(imp_dst_oo)(CTX *c, const R *x, int N, R *out);

/* improved.py:36-46 with elaborations.py:58-59 (forward) and :78-83 (backward) */
static void FN(imp_dct)(CTX *c, const R *x, int N, R *out) {
    if (N == 2) {
        out[0] = x[0] + x[1];
        out[1] = x[0] - x[1];
        return;
    }
    size_t mark = c->ar->used;
    int q = N / 4, m = N / 2;
    R *even = FN(rows)(c, q + 1), *odd = FN(rows)(c, q);
    for (int i = 0; i <= q; ++i) even[i] = x[2 * i];
    for (int i = 0; i < q; ++i) odd[i] = x[2 * i + 1];
    R *se = FN(rows)(c, q + 1), *so = FN(rows)(c, q);
    FN(imp_dct)(c, even, N / 2, se);
    FN(imp_dct_ot)(c, odd, N, so);
    for (int k = 0; k < q; ++k) out[k] = se[k] + so[k];
    for (int k = 0; k < q; ++k) out[m - k] = se[k] - so[k];
    out[q] = se[q];
    c->ar->used = mark;
}

/* improved.py:49-56 with elaborations.py:113-116 (fold) and :137-140 (interleave) */
static void FN(imp_dct_ot)(CTX *c, const R *x, int N, R *out) {
    int q = N / 4;
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    size_t mark = c->ar->used;
    int h = N / 8;
    R *ev = FN(rows)(c, h), *od = FN(rows)(c, h);
    for (int i = 0; i < h; ++i) {
        R a = x[i], b = x[q - 1 - i];
        ev[i] = a + b;
        od[i] = a - b;
    }
    R *se = FN(rows)(c, h), *so = FN(rows)(c, h);
    FN(imp_dct_ot)(c, ev, N / 2, se);
    FN(imp_dct_oo)(c, od, N, so);
    for (int i = 0; i < h; ++i) {
        out[2 * i] = se[i];
        out[2 * i + 1] = so[i];
    }
    c->ar->used = mark;
}

/* improved.py:59-74 */
static void FN(imp_dct_oo)(CTX *c, const R *x, int N, R *out) {
    if (N == 8) {
        out[0] = x[0] * c->T[0]; /* eighth_cos, improved.py:63 */
        return;
    }
    size_t mark = c->ar->used;
    int h = N / 8;
    R *conv = FN(rows)(c, h), *spec = FN(rows)(c, h);
    for (int i = 0; i < h; ++i) conv[i] = x[i] * FN(hsec)(c, 2 * i + 1, N);
    FN(imp_dct_ot)(c, conv, N / 2, spec);
    for (int j = 0; j < h - 1; ++j) out[j] = spec[j] + spec[j + 1];
    out[h - 1] = spec[h - 1];
    c->ar->used = mark;
}

/* improved.py:77-84 with elaborations.py:60-62 (forward) and :84-89 (backward) */
static void FN(imp_dst)(CTX *c, const R *x, int N, R *out) {
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    size_t mark = c->ar->used;
    int q = N / 4, m = N / 2;
    /* slots are n-1: even samples sit in the odd slots */
    R *even = FN(rows)(c, q - 1), *odd = FN(rows)(c, q);
    for (int i = 0; i < q - 1; ++i) even[i] = x[2 * i + 1];
    for (int i = 0; i < q; ++i) odd[i] = x[2 * i];
    R *se = FN(rows)(c, q - 1), *so = FN(rows)(c, q);
    FN(imp_dst)(c, even, N / 2, se);
    FN(imp_dst_ot)(c, odd, N, so);
    for (int k = 0; k < q - 1; ++k) out[k] = so[k] + se[k];
    for (int k = 0; k < q - 1; ++k) out[m - 2 - k] = so[k] - se[k];
    out[q - 1] = so[q - 1];
    c->ar->used = mark;
}

/* improved.py:87-94 with elaborations.py:123-126 and :145-148 */
static void FN(imp_dst_ot)(CTX *c, const R *x, int N, R *out) {
    int q = N / 4;
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    size_t mark = c->ar->used;
    int h = N / 8;
    R *ev = FN(rows)(c, h), *od = FN(rows)(c, h);
    for (int i = 0; i < h; ++i) {
        R a = x[i], b = x[q - 1 - i];
        ev[i] = a - b;
        od[i] = a + b;
    }
    R *se = FN(rows)(c, h), *so = FN(rows)(c, h);
    FN(imp_dst_ot)(c, ev, N / 2, se);
    FN(imp_dst_oo)(c, od, N, so);
    for (int i = 0; i < h; ++i) {
        out[2 * i + 1] = se[i];
        out[2 * i] = so[i];
    }
    c->ar->used = mark;
}

/* improved.py:97-112 */
static void FN(imp_dst_oo)(CTX *c, const R *x, int N, R *out) {
    if (N == 8) {
        out[0] = x[0] * FN(hsec)(c, 1, 8); /* half_secant(1, 8), improved.py:102 */
        return;
    }
    size_t mark = c->ar->used;
    int h = N / 8;
    R *conv = FN(rows)(c, h), *spec = FN(rows)(c, h);
    for (int i = 0; i < h; ++i) conv[i] = x[i] * FN(hsec)(c, 2 * i + 1, N);
    FN(imp_dst_ot)(c, conv, N / 2, spec);
    out[0] = spec[0];
    for (int j = 1; j < h; ++j) out[j] = spec[j - 1] + spec[j];
    c->ar->used = mark;
}

/* ================= classical recursion (classical.py:64-129) ================= */
static void FN(cla_dct)(CTX *c, const R *x, int N, R *out);
static void FN(cla_dct_odd)(CTX *c, const R *x, int N, R *out);
static void FN(cla_dst)(CTX *c, const R *x, int N, R *out);
static void FN(cla_dst_odd)(CTX *c, const R *x, int N, R *out);

/* classical.py:64-74 with elaborations.py:96-101 and :133-136 */
static void FN(cla_dct)(CTX *c, const R *x, int N, R *out) {
    if (N == 2) {
        out[0] = x[0] + x[1];
        out[1] = x[0] - x[1];
        return;
    }
    size_t mark = c->ar->used;
    int q = N / 4, m = N / 2;
    R *even = FN(rows)(c, q + 1), *odd = FN(rows)(c, q);
    for (int i = 0; i < q; ++i) {
        R a = x[i], b = x[m - i];
        even[i] = a + b;
        odd[i] = a - b;
    }
    even[q] = x[q];
    R *se = FN(rows)(c, q + 1), *so = FN(rows)(c, q);
    FN(cla_dct)(c, even, N / 2, se);
    FN(cla_dct_odd)(c, odd, N, so);
    for (int i = 0; i <= q; ++i) out[2 * i] = se[i];
    for (int i = 0; i < q; ++i) out[2 * i + 1] = so[i];
    c->ar->used = mark;
}

/* classical.py:77-99 with elaborations.py:102-112 (dc_t1t fold) */
static void FN(cla_dct_odd)(CTX *c, const R *x, int N, R *out) {
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    if (N == 8) {
        R t = x[1] * FN(hsec)(c, 1, 8);
        out[0] = x[0] + t;
        out[1] = x[0] - t;
        return;
    }
    size_t mark = c->ar->used;
    int q = N / 4;
    R *conv = FN(rows)(c, q);
    conv[0] = x[0] * (R)0.5; /* table.half, counting.py:109 */
    for (int n = 1; n < q; ++n) conv[n] = x[n] * FN(hsec)(c, n, N);
    /* split_harmonic_parity_forward("dc_t1t", N/2, conv) */
    int q2 = N / 8, m2 = N / 4;
    R *even = FN(rows)(c, q2 + 1), *odd = FN(rows)(c, q2);
    even[0] = conv[0] + (R)0.0;
    odd[0] = conv[0] - (R)0.0;
    for (int i = 1; i < q2; ++i) {
        R a = conv[i], b = conv[m2 - i];
        even[i] = a + b;
        odd[i] = a - b;
    }
    even[q2] = conv[q2];
    R *se = FN(rows)(c, q2 + 1), *so = FN(rows)(c, q2);
    FN(cla_dct)(c, even, N / 4, se);
    FN(cla_dct_odd)(c, odd, N / 2, so);
    R *half = FN(rows)(c, m2 + 1);
    for (int i = 0; i <= q2; ++i) half[2 * i] = se[i];
    for (int i = 0; i < q2; ++i) half[2 * i + 1] = so[i];
    for (int i = 0; i < q; ++i) out[i] = half[i] + half[i + 1];
    c->ar->used = mark;
}

/* classical.py:102-109 with elaborations.py:117-122 and :141-144 */
static void FN(cla_dst)(CTX *c, const R *x, int N, R *out) {
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    size_t mark = c->ar->used;
    int q = N / 4, m = N / 2;
    R *even = FN(rows)(c, q - 1), *odd = FN(rows)(c, q);
    for (int i = 0; i < q - 1; ++i) {
        R a = x[i], b = x[m - 2 - i];
        even[i] = a - b;
        odd[i] = a + b;
    }
    odd[q - 1] = x[q - 1];
    R *se = FN(rows)(c, q - 1), *so = FN(rows)(c, q);
    FN(cla_dst)(c, even, N / 2, se);
    FN(cla_dst_odd)(c, odd, N, so);
    for (int i = 0; i < q - 1; ++i) out[2 * i + 1] = se[i];
    for (int i = 0; i < q; ++i) out[2 * i] = so[i];
    c->ar->used = mark;
}

/* classical.py:112-129 */
static void FN(cla_dst_odd)(CTX *c, const R *x, int N, R *out) {
    int q = N / 4;
    if (N == 4) {
        out[0] = x[0];
        return;
    }
    size_t mark = c->ar->used;
    R center = x[q - 1];
    R *conv = FN(rows)(c, q - 1), *spec = FN(rows)(c, q - 1);
    for (int n = 1; n < q; ++n) conv[n - 1] = x[n - 1] * FN(hsec)(c, n, N);
    FN(cla_dst)(c, conv, N / 2, spec);
    R *partial = FN(rows)(c, q);
    partial[0] = spec[0];
    partial[q - 1] = spec[q - 2];
    for (int i = 1; i < q - 1; ++i) partial[i] = spec[i - 1] + spec[i];
    for (int i = 0; i < q; i += 2) out[i] = partial[i] + center;
    for (int i = 1; i < q; i += 2) out[i] = partial[i] - center;
    c->ar->used = mark;
}

/* ================= shared drivers (shared.py:21-72) ================= */
typedef void (*FN(tf_t))(CTX *, const R *, int, R *);

/* shared.py:21-43: packed [C0, C1, -S1, C2, -S2, ..., C(N/2)] */
static void FN(rdft_packed)(CTX *c, const R *x, int N, FN(tf_t) dct, FN(tf_t) dst, R *out) {
    if (N == 2) {
        out[0] = x[0] + x[1];
        out[1] = x[0] - x[1];
        return;
    }
    size_t mark = c->ar->used;
    int m = N / 2;
    R *dc = FN(rows)(c, m + 1), *ds = FN(rows)(c, m - 1);
    dc[0] = x[0];
    dc[m] = x[m];
    for (int n = 1; n < m; ++n) {
        R head = x[n], tail = x[N - n];
        dc[n] = head + tail;
        ds[n - 1] = head - tail;
    }
    R *sc = FN(rows)(c, m + 1), *ss = FN(rows)(c, m - 1);
    dct(c, dc, N, sc);
    dst(c, ds, N, ss);
    out[0] = sc[0];
    out[N - 1] = sc[m];
    for (int k = 1; k < m; ++k) {
        out[2 * k - 1] = sc[k];
        out[2 * k] = -ss[k - 1];
    }
    c->ar->used = mark;
}

/* shared.py:46-72 on one interleaved signal x[2N] -> out[2N] */
static void FN(cdft_interleaved)(CTX *c, const R *x, int N, FN(tf_t) dct, FN(tf_t) dst, R *out) {
    if (N == 2) {
        out[0] = x[0] + x[2];
        out[1] = x[1] + x[3];
        out[2] = x[0] - x[2];
        out[3] = x[1] - x[3];
        return;
    }
    size_t mark = c->ar->used;
    R *re = FN(rows)(c, N), *im = FN(rows)(c, N);
    for (int n = 0; n < N; ++n) {
        re[n] = x[2 * n];
        im[n] = x[2 * n + 1];
    }
    R *r1 = FN(rows)(c, N), *r2 = FN(rows)(c, N);
    FN(rdft_packed)(c, re, N, dct, dst, r1);
    FN(rdft_packed)(c, im, N, dct, dst, r2);
    out[0] = r1[0];
    out[1] = r2[0];
    out[N] = r1[N - 1];
    out[N + 1] = r2[N - 1];
    for (int k = 1; k < N / 2; ++k) {
        R a = r1[2 * k - 1], b = r1[2 * k], cc = r2[2 * k - 1], d = r2[2 * k];
        out[2 * k] = a - d;                  /* Re S(k)   */
        out[2 * (N - k)] = a + d;            /* Re S(N-k) */
        out[2 * k + 1] = b + cc;             /* Im S(k)   */
        out[2 * (N - k) + 1] = cc - b;       /* Im S(N-k) */
    }
    c->ar->used = mark;
}

/* ================= batched C-ABI entry points ================= */
static size_t FN(arena_bytes)(int N) { return (size_t)16 * sizeof(R) * (size_t)N + ((size_t)1 << 16); }

static int FN(table_for)(int N, R **T) {
    int tn = N >= 8 ? N / 4 : 1;
    *T = (R *)malloc(sizeof(R) * (size_t)tn);
    if (!*T) return -1;
    if (N >= 8) {
        return (sizeof(R) == sizeof(double)) ? oracle_table_f64(N, 0, (double *)*T)
                                             : oracle_table_f32(N, (float *)*T);
    }
    (*T)[0] = 0;
    return 0;
}

/* kind: 0 cdft, 1 rdft(packed), 2 dct0, 3 dst0.  algo: 0 improved, 1 classical.
 * in/out are batch-major; per-signal lengths: cdft 2N -> 2N, rdft N -> N
 * (packed), dct0 N/2+1 -> N/2+1, dst0 N/2-1 -> N/2-1.  `T` may be NULL to use
 * the default two-tier table; otherwise the caller's natural table. */
int FN(oracle_run)(int algo, int kind, int N, const R *in, R *out, long batch, const R *Tin, int nthreads) {
    if (N < 2 || (N & (N - 1))) return -1;
    if (kind == 3 && N < 4) return -1;
    R *T = NULL;
    if (Tin == NULL) {
        if (FN(table_for)(N, &T)) return -2;
    }
    FN(tf_t) dct = algo == 0 ? FN(imp_dct) : FN(cla_dct);
    FN(tf_t) dst = algo == 0 ? FN(imp_dst) : FN(cla_dst);
    long lin = kind == 0 ? 2L * N : kind == 1 ? N : kind == 2 ? N / 2 + 1 : N / 2 - 1;
    int rc = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads) reduction(| : rc)
#endif
    {
        arena_t ar;
        ar.cap = FN(arena_bytes)(N);
        ar.used = 0;
        ar.base = (char *)malloc(ar.cap);
        if (!ar.base) {
            rc |= 1;
        } else {
            CTX c = {Tin ? Tin : T, N, &ar};
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
            for (long b = 0; b < batch; ++b) {
                const R *x = in + b * lin;
                R *y = out + b * lin;
                ar.used = 0;
                if (kind == 0) FN(cdft_interleaved)(&c, x, N, dct, dst, y);
                else if (kind == 1) FN(rdft_packed)(&c, x, N, dct, dst, y);
                else if (kind == 2) dct(&c, x, N, y);
                else dst(&c, x, N, y);
            }
            free(ar.base);
        }
    }
    free(T);
    return rc ? -3 : 0;
}

#undef R
#undef CTX
#undef FN
#undef CAT
#undef CAT2
