// group.h -- launch descriptors for K4 / K6.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

struct BqArgs {
    const float4* xyz;          // [B][N] (naive)
    const int64_t* indptr;      // [B][N+1] (rf)
    const int32_t* nbr;         // (rf)
    const double* d2;           // (rf)
    int64_t cap_entries;
    const int32_t* counts;      // [B][L][N] (rf)
    int L, level;
    const int64_t* centroids;   // [B][cent_ld]
    int64_t cent_ld;
    int64_t B, N, n;
    int k;
    double r2;                  // (naive)
    int32_t* idx_out;           // [B][n][k]
    double* dist_out;           // [B][n][k]
    int32_t* cnt_out;           // [B][n]
    const int32_t* status;      // [B] exclusion-build status (rf; nullable): nonzero -> error outputs
};

struct KnnArgs {
    const float4* xyz;
    const int64_t* queries;     // [B][q_ld] or nullptr (= all points)
    int64_t q_ld, nq;
    const int64_t* pool;        // [B][pool_ld] point indices of the downsampled set
    int64_t pool_ld, npool;
    const uint8_t* sampled;     // [B][N] membership (rf)
    const int64_t* indptr;
    const int32_t* nbr;
    const double* d2;
    int64_t cap_entries;
    const int32_t* lvl1_counts;
    int64_t counts_stride;
    int64_t B, N;
    int k;
    int32_t* idx_out;           // [B][nq][k]
    double* dist_out;
    int32_t* cnt_out;
    int32_t* fallback_count;    // [B] (rf)
    const int32_t* status;      // [B] exclusion-build status (rf; nullable)
};

struct SpacingArgs {
    const float4* xyz;
    const int64_t* samples;     // [B][ld]
    int64_t ld, n, B, N;
    double* out_d2;             // [B][n]
};

cudaError_t launch_bq_rf(const BqArgs& a, cudaStream_t s);
cudaError_t launch_bq_naive(const BqArgs& a, cudaStream_t s);
cudaError_t launch_knn_naive(const KnnArgs& a, cudaStream_t s);
cudaError_t launch_knn_rf(const KnnArgs& a, cudaStream_t s);
cudaError_t launch_min_spacing(const SpacingArgs& a, cudaStream_t s);

}  // namespace ps
