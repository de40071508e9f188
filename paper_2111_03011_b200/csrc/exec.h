// exec.h -- host interface of the device executor (executor.cu).
#pragma once

#include <string>

#include "tnb.h"

namespace tnb {

struct Device;

int dev_bind(Device** out, const Program& prog, int device, void* workspace, size_t bytes, void* stream, int64_t M,
             int max_pipes, std::string& err);
int dev_pipes(const Device* d);
void dev_launch_counts(const Device* d, int64_t* per_slice, int64_t* per_contract);
int dev_contract(Device* d, const uint64_t* ids_sorted, int64_t n, void* amps_out, bool out_dev, double* secs,
                 std::string& err);
int dev_segment_runs(Device* d, const uint64_t* ids_sorted, int64_t n, int64_t* runs);
int dev_profile(Device* d, uint64_t slice_id, tn_launch_stat* stats, int max_stats, int* n_stats, std::string& err);
void dev_destroy(Device* d);
int debug_gemm(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K, int ea, void* stream,
               std::string& err);

}  // namespace tnb
