/*
 * tn_debug.h -- diagnostic entry points of the same library (unit tests and benchmarks only).
 * Not part of the method's call sequence (see tn.h).
 */
#ifndef TN_B200_DEBUG_H
#define TN_B200_DEBUG_H

#include "tn.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[M][N] = A[M][K] * B[K][N] for complex64 row-major DEVICE buffers through the tensor-core path of
 * tn_contract (3xTF32 split pre-passes + the tcgen05 GEMM).  embed_a selects which
 * operand gets the complex-as-real embedding (0: B, needs N >= 64; 1: A, needs N >= 128).  N and K >= 16
 * must be powers of two; M is arbitrary (ragged last tile).  Synchronises cuda_stream.  EINVAL on bad
 * shapes, ECUDA on a CUDA failure. */
tn_status tn_debug_gemm_tf32x3(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                               int32_t embed_a, void* cuda_stream);

/* Size of the simplified network built by tn_build: alive tensors, all edges, internal
 * (sliceable) edges. */
tn_status tn_debug_network(const tn_ctx* ctx, int64_t* n_tensors, int64_t* n_edges, int64_t* n_internal);

/* Kernel launches of the bound executor: per_slice = kernels in one slice's graph (after tiny-step fusion);
 * per_contract = kernels tn_contract issues once (slice-invariant prologue + the final pipeline sum).
 * A call with n slice ids launches n * per_slice + per_contract kernels.  EINVAL before tn_bind_device. */
tn_status tn_debug_launch_counts(const tn_ctx* ctx, int64_t* per_slice, int64_t* per_contract);

#ifdef __cplusplus
}
#endif
#endif
