// qdot_kernels.h -- internal launchers (C++ linkage), used by qdot_capi.cu.
#pragma once

#include <cuda_runtime.h>

#include "qdot_common.cuh"

namespace qd {

size_t pass1_smem_bytes();
size_t score_smem_bytes();
size_t pass2_smem_bytes();

cudaError_t launch_pass1(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                         const P1Params& prm, cudaStream_t st);
cudaError_t launch_score(const int64_t* A, const int64_t* B, int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta,
                         qdot_result* res, qdot_bin* bins, int64_t n_total, const qdot_config& cfg,
                         bool fuse_finalize, cudaStream_t st);
// fin.A != nullptr: the last pass-2 CTA also finalizes (one GPU: no exchange
// of region B between pass 2 and finalize)
struct P2Fin {
    const int64_t* A = nullptr;
    qdot_result* res = nullptr;
    qdot_bin* bins = nullptr;
};
cudaError_t launch_pass2(const double* x, const double* y, int64_t n, bool norm, const uint32_t* lut_p2,
                         const ScoreMeta* meta, int64_t* B, const double2* list, const uint32_t* list_fill,
                         const P2Fin& fin, cudaStream_t st);
// a whole single-device qdot of n <= small_max() elements (exact strategy) in one
// cluster launch (qdot_small.cuh); score / pass 2 launched after it return at once
// unless it handed the call over (A[A_SMALL] == 2)
cudaError_t launch_small(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                         int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta, qdot_result* res, qdot_bin* bins,
                         const qdot_config& cfg, cudaStream_t st);
int64_t small_max();
// zero `bytes` (a multiple of 16, 16-byte aligned) at region: regions A, B, local
cudaError_t launch_begin(void* region, size_t bytes, cudaStream_t st);
cudaError_t launch_finalize(const int64_t* A, const int64_t* B, const uint32_t* lut_p2, const ScoreMeta* meta,
                            qdot_result* res, qdot_bin* bins, cudaStream_t st);
cudaError_t launch_publish(const void* block, int nbytes, void* host_dev, uint32_t* dev_seq, uint32_t* host_seq_dev,
                           cudaStream_t st);
cudaError_t launch_batched(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, bool norm,
                           const qdot_config& cfg, double* values, int64_t* counts, int32_t* info, qdot_bin* bins,
                           cudaStream_t st);
cudaError_t launch_bin_ids(const double* x, const double* y, int64_t n, bool norm, const int32_t* lut_bin,
                           int32_t* out, cudaStream_t st);

}  // namespace qd
