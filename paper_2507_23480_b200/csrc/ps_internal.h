// ps_internal.h -- host-side launch descriptors shared by the .cu files.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace ps {

struct FpsArgs {
    const float4* xyz;          // [B][N]
    double* md;                 // [B][N]
    uint8_t* taken;             // [B][N]
    int64_t* out_idx;           // [B][ld_out]
    double* curve;              // [B][ld_out]
    const int64_t* k_start_dev; // [B] or nullptr -> k_start
    const int64_t* seed_dev;    // [B] or nullptr -> seed
    int64_t N, ld_out, k_start, k_stop, seed;
    int fresh;                  // 1: md=+inf, taken={seed}, out[0]=seed, curve[0]=+inf
    int64_t points_per_cta;     // set by the launcher
    long long* dbg;             // development timing buffer (PS_FPS_TIMING)
    int64_t dbg_t0;             // first recorded iteration offset (PS_FPS_T0)
    double spec_target;         // fps_spec: candidates aimed for per exchange (0: default, < 0: no speculation)
    int poll_ns;                // fps_spec: worker poll back-off in ns (0: default)
};

// Clouds split over G ranks (point-split FPS): rank g owns original indices
// [g*ceil(N/G), (g+1)*ceil(N/G)).  A launch runs Gl ranks per cloud starting
// at g_base (Gl == G: virtual ranks on one GPU; Gl == 1: one rank per GPU).
// mbox: device array of G pointers to each rank's mailbox
// (uint4[B][3][G][kRecU4 * kMbRecs], initialised to 0xff); the tag of every
// (launch, iteration) is unique: seq_base, or -- when seq_dev is set -- the
// word seq_dev[0] written by mbox_epoch_kernel in the same stream (so CUDA
// graph replays never meet a previous replay's records).  A mailbox wait
// longer than timeout_ns (globaltimer) records the failing iteration in
// err[0] (nullable) and traps: a dead or late peer becomes a launch error,
// not a hang.
struct FpsRanks {
    int G, Gl, g_base, all_write;
    int spatial;                // 1: spatial (Morton-cell) partition of the shard over the cluster's CTAs
    uint32_t seq_base;
    uint4* const* mbox;
    const uint32_t* seq_dev;    // nullable: device-side tag base
    unsigned long long timeout_ns;
    unsigned int* err;          // nullable
};

// records per (cloud, set, rank) mailbox slot: meta + header + 32 candidates;
// a record is six 64-bit words {payload u32, tag u32} (kRecU4 uint4s)
constexpr int kMbRecs = 34;
constexpr int kRecU4 = 3;
constexpr int kMaxRanks = 32;   // one warp lane per rank in every exchange
constexpr unsigned long long kMboxTimeoutNs = 10ull * 1000 * 1000 * 1000;

cudaError_t launch_fps(FpsArgs a, int64_t B, cudaStream_t s);          // resident kernel, else legacy
cudaError_t launch_fps_legacy(FpsArgs a, int64_t B, cudaStream_t s);   // register / streaming kernel
cudaError_t launch_fps_spec(FpsArgs a, int64_t B, cudaStream_t s);     // register kernel, speculation
cudaError_t launch_fps_small(FpsArgs a, int64_t B, cudaStream_t s);    // one CTA per small cloud, points in registers
bool fps_res_plan(int64_t N, int64_t nclusters, int G, int* C_out, int* P_out);
unsigned long long split_timeout_ns();
int64_t fps_set_inflight(int64_t clouds);  // throughput hint for the FPS cluster width
size_t csr_fill_ws_bytes(int64_t M, int64_t N);
cudaError_t launch_csr_fill(const int32_t* ei, const int32_t* ej, const double* ed, int64_t M, const int64_t* indptr,
                            int64_t N, int64_t* out_idx, double* out_d2, void* work, size_t work_bytes,
                            cudaStream_t s);  // PS_SPLIT_TIMEOUT_MS, default kMboxTimeoutNs
cudaError_t launch_fps_res(FpsArgs a, const FpsRanks& rk, int64_t B, int C, int P, cudaStream_t s);
int fps_choose_cluster(int64_t N, int64_t B, int* C_out, int* P_out, int* T_out);

// Exclusion-list CSR (one cloud = rows [b][0..N); entries at b*cap_entries).
struct CsrView {
    int64_t* indptr;    // [B][N+1], per-cloud relative offsets
    int32_t* nbr;       // [B][cap_entries]
    double* d2;         // [B][cap_entries]
    int32_t* counts;    // [B][L][N]
    int64_t cap_entries;
    int64_t N;
    int L;
    // method 2, row-sharded build (one rank of a point split): only rows
    // [row_lo, row_hi) are written (indptr, entries, counts) and long rows take
    // spill entries [spill_lo, spill_hi) of the arena.  row_hi == 0 / spill_hi
    // == 0: every row / the whole arena (launch_excl_build normalises).
    int64_t row_lo, row_hi, spill_lo, spill_hi;
};

struct ExclWork {
    uint32_t* edge_i;     // [B][cap_edges]
    uint32_t* edge_j;     // [B][cap_edges]
    double* edge_d2;      // [B][cap_edges]
    int64_t cap_edges;
    unsigned long long* edge_count;  // [B]
    int32_t* deg;         // [B][N] (doubles as the fill cursor)
    int32_t* long_rows;   // [B*N] rows too long for the warp sort (b*N + i)
    unsigned int* long_count;  // [1]
    int32_t* status;      // [B] bit0: edge overflow, bit1: entry overflow
    unsigned long long* spill;  // [B] method 2: entries taken from the spill arena (rows longer than the stride)
};

// Method 2 (fixed-stride rows): row i at i * stride; the entries beyond
// N * stride are the spill arena, from which rows longer than the stride take
// a 16-byte aligned run of their own (indptr[i] then points there).  About
// 1/9 of the capacity is spill.
inline int64_t ell_row_stride(int64_t cap_entries, int64_t N) {
    const int64_t s = (cap_entries / N) * 8 / 9;
    return s >= 4 ? (s & ~int64_t(3)) : s;
}

struct GridParams {
    double ox, oy, oz, inv_h;
    int nx, ny, nz, ncells;
    double h;       // cell width (>= R_max / reach)
    int reach;      // neighbour cells per axis and side that can hold a point within R_max
};

struct GridWork {
    GridParams* params;           // [B]
    int* cell_start;              // [B][max_cells + 1]
    int* cursor;                  // [B][max_cells]
    int32_t* cell_of;             // [B][N]
    int32_t* sorted_idx;          // [B][N]
    float4* sorted_xyz;           // [B][N]
    unsigned long long* evals;    // [B] candidate pairs evaluated
    int max_cells;
};

// method 0: brute-force i<j triangle (every pair evaluated once)
// method 1: uniform grid of cell width >= R_max (identical CSR)
int excl_build_launches(int64_t N, int method);
cudaError_t launch_excl_build(const float4* xyz, int64_t B, int64_t N, const double* r2_levels,
                              int L, int64_t levels_ld, CsrView csr, ExclWork w, GridWork g, int method,
                              cudaStream_t s);
cudaError_t launch_sort_rows(CsrView csr, int64_t B, ExclWork w, cudaStream_t s);
cudaError_t launch_level_counts(CsrView csr, int64_t B, const double* r2_levels, int64_t levels_ld,
                                cudaStream_t s);

}  // namespace ps
