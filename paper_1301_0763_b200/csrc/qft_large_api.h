// qft_large_api.h -- internal interface between the C ABI (qft_capi.cu) and the
// per-precision multi-pass translation units (qft_large.cu).
#pragma once
#include <cuda_runtime.h>

#define QFT_LARGE_DECL(SUF)                                                                             \
    int qft_large_create_##SUF(int log2n, int real_modes, void **out);                                  \
    void qft_large_destroy_##SUF(void *p);                                                              \
    void qft_large_info_##SUF(void *p, int *passes, int *launches);                                     \
    long long qft_large_scratch_cells_##SUF(void *p);                                                   \
    int qft_large_exec_##SUF(void *p, int mode, const void *d_in, void *d_out, long long batch,         \
                             long long nreal, const void *d_U, const void *uhead, void *scratch, cudaStream_t st);
QFT_LARGE_DECL(f32)
QFT_LARGE_DECL(f64)
#undef QFT_LARGE_DECL
