#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace pars_b200 {

#ifndef PARS_SGD_CLUSTER_CTAS
#define PARS_SGD_CLUSTER_CTAS 8
#endif
constexpr int kSgdCluster = PARS_SGD_CLUSTER_CTAS;  // CTAs (SMs) per epoch cluster (> 8: non-portable)
constexpr uint32_t kSgdRowCap = 10240;  // staged row entries per CTA per step
constexpr uint32_t kSgdCscCap = 10240;  // staged CSC entries per CTA per step
constexpr uint32_t kSgdRunCap = 1024;   // staged runs per CTA per step

size_t sgd_cluster_smem(uint32_t dim, int32_t B);
size_t sgd_cluster_scratch_bytes(int64_t nbatches, uint32_t dim, int64_t total_entries,
                                 int64_t npairs);
int build_compact_rows(pars_ctx* ctx, const int64_t* d_rp, const uint32_t* d_idx,
                       const int32_t* d_cnt, int64_t rows, const uint32_t* d_off, uint32_t* d_cpk,
                       int32_t* d_bad, cudaStream_t st);
int launch_sgd_cluster(pars_ctx* ctx, const int64_t* rp, const uint32_t* cpk,
                       const uint32_t* cpk_off, const double* inv_row, uint32_t dim,
                       const uint32_t* a, const uint32_t* b, const int32_t* y, int64_t npairs,
                       int32_t B, double lr, double margin, double bias, double* w,
                       double* loss_out, unsigned long long* active_out, int64_t total,
                       void* scratch, cudaStream_t st);

}  // namespace pars_b200
