/*
 * qft_b200.h -- C ABI of the B200-native improved-QFT library (libqftb200.so).
 *
 * Replaces the body of the reference's transform entry points:
 *   quickfourier.improved.cdft(values, table=None, counter=None)
 *       /root/reference/pkg/src/quickfourier/improved.py:139-150
 *   (and, per plan algo, quickfourier.classical.cdft, classical.py:156-167)
 * with plain pointers and sizes (no torch types).  The Python drop-in
 * (paper_1301_0763_b200.improved) binds these with ctypes; INTEGRATION.md shows
 * the binding a maintainer of the reference would add.
 *
 * Data: interleaved complex (Re, Im) of the plan's precision -- exactly the
 * memory order of numpy complex64 / complex128.  Out-of-place; the input is
 * never written.  Arithmetic reproduces the reference's operation DAG with one
 * IEEE rounding per op, so results are bit-identical to the reference.
 *
 * Every function returns 0 on success or a negative QFT_E* code; the message
 * of the last failure on the calling thread is available from qft_last_error().
 *
 * Sizes: N = 2 .. 2^20 in both precisions.  N <= 2^14 (fp32) / 2^13 (fp64) runs
 * one single-pass kernel; larger N the multi-pass schedule (qft_plan_info_t
 * passes / kernel_launches).  Concurrency: a plan owns scratch memory (multi-
 * pass, classical and layout conversion), so one plan serves one stream at a
 * time, like a cuFFT plan; create one plan per concurrent stream.
 */
#ifndef QFT_B200_H
#define QFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QFT_OK 0
#define QFT_EINVAL -1       /* bad argument (reference raises ValueError)       */
#define QFT_EUNSUPPORTED -2 /* size / precision / algorithm not built            */
#define QFT_ECUDA -3        /* CUDA runtime error (no device, launch failure...) */
#define QFT_ENOMEM -4

#define QFT_PREC_F32 32 /* complex64 input  -> float32 working dtype (improved.py:142) */
#define QFT_PREC_F64 64 /* anything else    -> float64 working dtype                  */

#define QFT_ALGO_IMPROVED 0
#define QFT_ALGO_CLASSICAL 1

#define QFT_KIND_RDFT 1 /* improved.rdft (improved.py:131-136) */
#define QFT_KIND_DCT0 2 /* improved.dct0 (improved.py:117-121) */
#define QFT_KIND_DST0 3 /* improved.dst0 (improved.py:124-128) */

typedef struct qft_plan qft_plan;

typedef struct {
    int32_t log2n;
    int32_t prec;
    int32_t algo;
    int32_t passes;          /* passes over HBM per transform (1 = single-pass) */
    int32_t kernel_launches; /* kernel launches per qft_exec_cdft call          */
    int32_t smem_bytes;      /* dynamic shared memory per CTA of the main kernel */
    int32_t threads_per_cta;
    int32_t ctas_per_sm;     /* resident CTAs per SM of the main kernel          */
    int32_t signals_per_cta; /* signals a CTA transforms per iteration           */
    int64_t scratch_bytes;   /* device scratch owned by the plan                 */
} qft_plan_info_t;

/* Version of this ABI (major*100 + minor). */
int qft_version(void);

/* Create an immutable plan for periodization N = 2^log2n on a CUDA device.
 * Builds the half-secant table with the reference's two-tier recipe
 * (counting.py:116-140) and uploads it.  Replaces classical._resolve's lazy
 * module-global table (classical.py:31-45). */
int qft_plan_create(qft_plan **plan, int log2n, int prec, int algo, int device);
int qft_plan_destroy(qft_plan *plan);
int qft_plan_get_info(const qft_plan *plan, qft_plan_info_t *info);

/* Natural constant table, N/4 entries of the plan precision:
 * T[0] = cos(2 pi/8), T[m] = 1/(2 cos(2 pi m/N)) (TrigTable.half_secant,
 * counting.py:152-178).  For the bit-parity test of the table. */
int qft_plan_table(const qft_plan *plan, void *h_out);
/* Replace the constants with a caller's table (same layout as above), e.g. the
 * values of a user-supplied TrigTable (the reference's `table=` argument). */
int qft_plan_set_table(qft_plan *plan, const void *h_table);

/* Forward DFT S(k) = sum_n s(n) e^{-2 pi i n k/N} of `batch` signals that are
 * already in device memory.  Element n of signal b sits at
 * base + (b*batch_stride + n*elem_stride) complex elements.  The fast path is
 * batch-major contiguous (batch_stride = N, elem_stride = 1); the reference's
 * own layout (N, batch) is elem_stride = batch, batch_stride = 1.
 * Stream-ordered on `stream` (a cudaStream_t, NULL = legacy default stream). */
int qft_exec_cdft(const qft_plan *plan, const void *d_in, void *d_out, int64_t batch,
                  int64_t in_batch_stride, int64_t in_elem_stride,
                  int64_t out_batch_stride, int64_t out_elem_stride, void *stream);

/* Real-input transforms of the same plan (periodization N = 2^log2n) on
 * device rows, batch-major contiguous:
 *   QFT_KIND_RDFT: rows of N reals -> rows of N/2+1 complex (k = 0..N/2; the
 *                  reference's packed half spectrum, complex_from_packed, shared.py:94-101)
 *   QFT_KIND_DCT0: rows of N/2+1 reals s(0..N/2) -> N/2+1 reals
 *   QFT_KIND_DST0: rows of N/2-1 reals s(1..N/2-1) -> N/2-1 reals
 * Precision = the plan's (real float32 for QFT_PREC_F32).  Two rows share one
 * complex-typed lane of the kernels; every row is bit-identical to the reference.
 * On a QFT_ALGO_CLASSICAL plan: classical.rdft / dct0 / dst0 (classical.py:134-153). */
int qft_exec_real(const qft_plan *plan, int kind, const void *d_in, void *d_out, int64_t nrows, void *stream);

/* Same transform on HOST buffers: chunked host->device copy, transform and
 * device->host copy, pipelined over the plan's streams.  Synchronous.  Pinned
 * host memory gives full PCIe bandwidth; pageable memory works but is slower.
 * This is the call behind the reference-facing drop-in on numpy arrays. */
int qft_exec_cdft_host(qft_plan *plan, const void *h_in, void *h_out, int64_t batch,
                       int64_t in_batch_stride, int64_t in_elem_stride,
                       int64_t out_batch_stride, int64_t out_elem_stride);

/* Device-side seeded input generator of the benchmark inputs (configs 2, 5):
 * re, im ~ N(0,1) by Box-Muller from a counter-based hash (splitmix64) of
 * (seed, global transform index first_index + b, n), with ln / sin / cos as fixed
 * polynomials in explicitly rounded double ops.  Its numpy twin
 * paper_1301_0763_b200/workloads.py:keyed_normal_rows reproduces every value bit
 * for bit on the host, so any shard or sampled row regenerates there. */
int qft_fill_normal(const qft_plan *plan, void *d_out, int64_t batch, int64_t first_index,
                    uint64_t seed, void *stream);

/* Message of the last error on this thread ("" if none). */
const char *qft_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* QFT_B200_H */
