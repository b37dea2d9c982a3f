// sampler.h -- launch descriptors for K2 / K3c / K3d.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

constexpr int kMaxSeg = 16;
constexpr int kMaxExtra = 8;

struct ThreshArgs {
    const double* prefix_curve;  // [B][curve_ld], first k0 entries measured
    int64_t curve_ld;
    const double* pow_tab;       // [n] i**e (mode 0)
    const double* given_curve;   // [B][given_ld] (mode 1)
    int64_t given_ld;
    int mode;                    // 0 power, 1 given curve, 2 MLP
    const double* mlp;           // mode 2: packed W1 b1 W2 b2 W3 b3 (float64, row-major)
    int64_t k0, n;
    int nseg;
    int64_t d[kMaxSeg];          // min(floor(n s / nseg), n-1)
    int n_extra;
    double extra_r2[kMaxExtra];
    double* R_out;               // [B][nseg]
    double* r2_levels;           // [B][levels_ld]: nseg segment levels then extras
    int64_t levels_ld;
};

struct SampArgs {
    const int64_t* indptr;       // [B][N+1]
    const int32_t* nbr;          // [B][cap_entries]
    int64_t cap_entries;
    const int32_t* counts;       // [B][L][N]
    int L;
    int nseg;
    int seg_level_rows[kMaxSeg];
    int64_t boundaries[kMaxSeg]; // segment ends, last == n_total
    int64_t k0, n_total, N, B;
    int64_t* out_idx;            // [B][ld_out]; [0, k0) = prefix on entry
    int64_t ld_out;
    uint64_t* state_io;          // [B]
    int pick_lowest;
    int64_t* reached;            // [B]
    int32_t* exhausted;          // [B]
    int32_t* entered;            // [B]
    unsigned char* gws;          // global workspace (per-cloud tables that do not fit in shared memory)
    int64_t gws_stride;
    long long* dbg;              // development timing (PS_SAMPLER_TIMING)
    int tiny;                    // v4, one CTA per cloud: the per-cloud arrays live in shared memory
    int rounds;                  // v4: 1 = MIS in barrier-separated rounds, 0 = dataflow (default)
    int poll_ns;                 // v4 dataflow: poll back-off after the first polls (0: spin)
    int push_grouped;            // v4 P1 push: lane groups per row instead of flattened rows (A/B knob)
    const int32_t* excl_status;  // [B] nullable: nonzero -> the cloud's rows are incomplete (error outputs)
    int grid_c;                  // v4 grid mode: CTAs per cloud (0: cluster mode)
};

struct EtArgs {
    const int64_t* indptr;
    const int32_t* nbr;
    const double* d2;
    int64_t cap_entries;
    const int32_t* lvl1_counts;  // row of the R_1 level: [B] stride counts_stride
    int64_t counts_stride;
    uint8_t* taken;              // [B][N]
    double* md;                  // [B][N]
    const int64_t* out_idx;      // [B][ld_out]
    int64_t ld_out;
    const int64_t* reached;      // [B]
    int64_t n_total, B, N;
    int64_t md_lo, md_hi;        // md reset range (md_hi == 0: all points)
};

struct EtScanArgs {
    const int64_t* indptr;
    const int32_t* nbr;
    const double* d2;
    int64_t cap_entries;
    const int32_t* lvl1_counts;
    int64_t counts_stride;
    const uint8_t* taken;
    double* md;
    const int64_t* reached;      // nullable
    int64_t n_total, B, N, lo, hi;
};

size_t sampler_global_ws_bytes(int64_t B, int64_t N, bool big);  // global workspace
cudaError_t launch_thresholds(const ThreshArgs& a, int64_t B, cudaStream_t s);
cudaError_t launch_sampler(SampArgs a, int64_t B, cudaStream_t s);     // v4 (sampler_v4.cu)
cudaError_t launch_sampler_v4(SampArgs a, int64_t B, cudaStream_t s);
size_t sampler_v4_ws_bytes(int64_t B, int64_t N);
cudaError_t launch_et(const EtArgs& a, cudaStream_t s);
int et_launches();
cudaError_t launch_et_scan(const EtScanArgs& a, cudaStream_t s);
cudaError_t launch_et_shard(const EtArgs& a, int64_t lo, int64_t hi, cudaStream_t s);

}  // namespace ps
