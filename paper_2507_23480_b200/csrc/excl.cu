// excl.cu -- K3a/K3b: fused exclusion-list construction (B200 / sm_100a).
//
// Replaces excl_collect + csr_fill + csr_sort_rows + csr_level_counts
// (/root/reference/pkg/src/pointsample/_kernels.py:111-234).
//
//   excl_pairs     tiled i<j triangle over 128x128 point tiles staged in
//                  shared memory; a conservative float32 pre-filter rejects
//                  almost every pair and survivors are decided exactly in
//                  float64 (no FMA).  Each unordered pair is evaluated once.
//                  Hits are staged in shared memory and flushed to a per-cloud
//                  edge list with one global atomic per flush.
//   excl_degree    per-row degrees from the edge list.
//   excl_scan      per-cloud exclusive scan -> indptr (self included).
//   excl_fill      scatter self + both directions of every edge.
//   excl_sort      rows ordered by (d2, index): warp bitonic in shared memory
//                  for rows <= 256, CTA bitonic for longer rows; the strict
//                  "d2 < r2" level counts are fused into the epilogue.
//
// Row order after the sort is a total order, so the scatter order of the
// fill pass (atomics) never leaks into the output: the CSR is
// byte-identical to the reference's for any schedule.

#include <cfloat>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

namespace {

constexpr int kTile = 128;
constexpr int kPairThreads = 256;
constexpr int kStageCap = 2048;

__device__ __forceinline__ void tile_pair_from_linear(int64_t t, int64_t nt, int64_t* I, int64_t* J) {
    // enumerate (I, J) with I <= J row by row: row I has nt - I entries
    // solve for I via the closed form, then fix rounding
    double a = (double)(2 * nt + 1);
    int64_t i = (int64_t)floor((a - sqrt(a * a - 8.0 * (double)t)) * 0.5);
    if (i < 0) i = 0;
    auto start = [&](int64_t r) { return r * nt - r * (r - 1) / 2; };
    while (i > 0 && start(i) > t) --i;
    while (i + 1 < nt && start(i + 1) <= t) ++i;
    *I = i;
    *J = i + (t - start(i));
}

__global__ void __launch_bounds__(kPairThreads) excl_pairs_kernel(
    const float4* __restrict__ xyz, int64_t N, const double* __restrict__ r2_levels, int L,
    int64_t levels_ld, ExclWork w) {
    __shared__ float4 ti[kTile];
    __shared__ float4 tj[kTile];
    __shared__ uint32_t s_i[kStageCap];
    __shared__ uint32_t s_j[kStageCap];
    __shared__ double s_d[kStageCap];
    __shared__ int s_n;
    __shared__ unsigned long long s_base;

    const int64_t b = blockIdx.y;
    const int64_t nt = (N + kTile - 1) / kTile;
    int64_t I, J;
    tile_pair_from_linear(blockIdx.x, nt, &I, &J);
    const float4* cx = xyz + b * N;
    const int tid = threadIdx.x;

    double r2 = 0.0;
    for (int l = 0; l < L; ++l) r2 = fmax(r2, r2_levels[b * levels_ld + l]);
    const float thr = prefilter_threshold(r2);
    const bool no_filter = !(thr <= FLT_MAX);

    if (tid < kTile) {
        const int64_t i = I * kTile + tid;
        ti[tid] = i < N ? cx[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
        const int64_t j = J * kTile + (tid - kTile);
        tj[tid - kTile] = j < N ? cx[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid == 0) s_n = 0;
    __syncthreads();

    const int li = tid & (kTile - 1);
    const int half = tid >> 7;
    const int64_t gi = I * kTile + li;
    const float4 pi = ti[li];
    const int64_t jlo = J * kTile + half * (kTile / 2);
    const int jbeg = half * (kTile / 2);
    unsigned long long* ecount = w.edge_count + b;
    if (gi < N) {
#pragma unroll 8
        for (int t = 0; t < kTile / 2; ++t) {
            const int64_t gj = jlo + t;
            const float4 pj = tj[jbeg + t];
            const float df = sqdist_f32(pi, pj);
            if ((df < thr || no_filter) && gj < N && gj > gi) {
                const double d = sqdist4(pi, pj);
                if (d < r2) {
                    const int slot = atomicAdd(&s_n, 1);
                    if (slot < kStageCap) {
                        s_i[slot] = (uint32_t)gi;
                        s_j[slot] = (uint32_t)gj;
                        s_d[slot] = d;
                    } else {  // dense pathological tile: direct global append
                        const unsigned long long p = atomicAdd(ecount, 1ull);
                        if (p < (unsigned long long)w.cap_edges) {
                            w.edge_i[b * w.cap_edges + p] = (uint32_t)gi;
                            w.edge_j[b * w.cap_edges + p] = (uint32_t)gj;
                            w.edge_d2[b * w.cap_edges + p] = d;
                        } else {
                            atomicOr(&w.status[b], 1);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    const int n = min(s_n, kStageCap);
    if (n == 0) return;
    if (tid == 0) s_base = atomicAdd(ecount, (unsigned long long)n);
    __syncthreads();
    const unsigned long long base = s_base;
    for (int k = tid; k < n; k += kPairThreads) {
        const unsigned long long p = base + k;
        if (p < (unsigned long long)w.cap_edges) {
            w.edge_i[b * w.cap_edges + p] = s_i[k];
            w.edge_j[b * w.cap_edges + p] = s_j[k];
            w.edge_d2[b * w.cap_edges + p] = s_d[k];
        } else {
            atomicOr(&w.status[b], 1);
        }
    }
}

__global__ void excl_degree_kernel(int64_t N, ExclWork w) {
    const int64_t b = blockIdx.y;
    const int64_t m = min((int64_t)w.edge_count[b], w.cap_edges);
    int32_t* deg = w.deg + b * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        atomicAdd(&deg[w.edge_i[b * w.cap_edges + e]], 1);
        atomicAdd(&deg[w.edge_j[b * w.cap_edges + e]], 1);
    }
}

// One CTA per cloud: indptr = exclusive scan of (deg + 1); deg <- indptr (cursor).
__global__ void __launch_bounds__(1024) excl_scan_kernel(int64_t N, ExclWork w, CsrView csr, int add_self) {
    __shared__ int64_t warp_sums[32];
    __shared__ int64_t carry;
    const int64_t b = blockIdx.x;
    int32_t* deg = w.deg + b * N;
    int64_t* indptr = csr.indptr + b * (N + 1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < N; base += 1024) {
        const int64_t i = base + tid;
        const int64_t v = i < N ? (int64_t)deg[i] + add_self : 0;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int64_t s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(kFull, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const int64_t excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
        if (i < N) {
            indptr[i] = excl;
            deg[i] = (int32_t)excl;  // cursor (cap_entries < 2^31 enforced by host)
        }
        __syncthreads();
        if (tid == 0) carry += warp_sums[31];
        __syncthreads();
    }
    if (tid == 0) {
        indptr[N] = carry;
        if (carry > csr.cap_entries) atomicOr(&w.status[b], 2);
    }
}

__global__ void excl_fill_kernel(int64_t N, ExclWork w, CsrView csr) {
    const int64_t b = blockIdx.y;
    const int64_t m = min((int64_t)w.edge_count[b], w.cap_edges);
    int32_t* cur = w.deg + b * N;
    int32_t* nbr = csr.nbr + b * csr.cap_entries;
    double* d2 = csr.d2 + b * csr.cap_entries;
    const int64_t cap = csr.cap_entries;
    const int64_t total = m + N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < N) {
            const int32_t p = atomicAdd(&cur[e], 1);
            if (p < cap) { nbr[p] = (int32_t)e; d2[p] = 0.0; }
        } else {
            const int64_t k = b * w.cap_edges + (e - N);
            const uint32_t i = w.edge_i[k], j = w.edge_j[k];
            const double d = w.edge_d2[k];
            const int32_t p = atomicAdd(&cur[i], 1);
            if (p < cap) { nbr[p] = (int32_t)j; d2[p] = d; }
            const int32_t q = atomicAdd(&cur[j], 1);
            if (q < cap) { nbr[q] = (int32_t)i; d2[q] = d; }
        }
    }
}


// ---- uniform-grid candidate enumeration ---------------------------------------
// Cell width h >= R_max * (1 + 1e-6): two points closer than R_max can only lie
// in the same or adjacent cells, so scanning the 27-cell neighbourhood visits
// every pair the brute-force triangle would accept; the CSR after the
// (d2, index) row sort is byte-identical.  Evaluation count drops from
// N(N-1)/2 to the neighbourhood candidates (reported in grid evals).

__global__ void __launch_bounds__(1024) grid_setup_kernel(const float4* __restrict__ xyz, int64_t N,
                                                          const double* __restrict__ r2_levels, int L,
                                                          int64_t levels_ld, GridWork g, ExclWork w, int zero,
                                                          int reach) {
    __shared__ float red[6][32];
    __shared__ int nc_s;
    const int64_t b = blockIdx.x;
    const float4* cx = xyz + b * N;
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const float4 p = cx[i];
        mn[0] = fminf(mn[0], p.x); mn[1] = fminf(mn[1], p.y); mn[2] = fminf(mn[2], p.z);
        mx[0] = fmaxf(mx[0], p.x); mx[1] = fmaxf(mx[1], p.y); mx[2] = fmaxf(mx[2], p.z);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(kFull, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(kFull, mx[a], o));
        }
        if (lane == 0) { red[a][warp] = mn[a]; red[3 + a][warp] = mx[a]; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        double lo[3], ext[3];
        for (int a = 0; a < 3; ++a) {
            float m0 = FLT_MAX, m1 = -FLT_MAX;
            for (int q = 0; q < nw; ++q) { m0 = fminf(m0, red[a][q]); m1 = fmaxf(m1, red[3 + a][q]); }
            lo[a] = m0;
            ext[a] = (double)m1 - (double)m0;
        }
        double r2 = 0.0;
        for (int l = 0; l < L; ++l) r2 = fmax(r2, r2_levels[b * levels_ld + l]);
        double h = sqrt(r2) * (1.0 + 1e-6) / (double)reach;
        if (!(h > 1e-30)) h = 1e-30;
        int n[3];
        for (int it = 0; it < 64; ++it) {
            double tot = 1.0;
            for (int a = 0; a < 3; ++a) {
                const double c = floor(ext[a] / h) + 1.0;
                n[a] = c > 1048576.0 ? 1048576 : (int)c;
                tot *= (double)n[a];
            }
            if (tot <= (double)g.max_cells) break;
            h *= cbrt(tot / (double)g.max_cells) * 1.001;
        }
        GridParams gp;
        gp.ox = lo[0]; gp.oy = lo[1]; gp.oz = lo[2];
        gp.inv_h = 1.0 / h;
        gp.nx = n[0]; gp.ny = n[1]; gp.nz = n[2];
        gp.ncells = n[0] * n[1] * n[2];
        gp.h = h;
        gp.reach = reach;
        g.params[b] = gp;
        nc_s = gp.ncells;
        if (zero) {
            g.evals[b] = 0;
            w.status[b] = 0;
            if (w.spill) w.spill[b] = 0;
            if (b == 0) *w.long_count = 0;
        }
    }
    if (zero) {
        // this cloud's cell counters (grid_assign_kernel adds into them)
        __syncthreads();
        int* cs = g.cell_start + b * (g.max_cells + 1);
        for (int i = threadIdx.x; i <= nc_s; i += blockDim.x) cs[i] = 0;
    }
}

__device__ __forceinline__ int cell_coord(double v, double o, double inv_h, int n) {
    int c = (int)floor((v - o) * inv_h);
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

// (method 2: also the fixed-stride row pointers, indptr[b][i] = i * stride,
// spread over the whole grid instead of a launch of their own)
__global__ void grid_assign_kernel(const float4* __restrict__ xyz, int64_t B, int64_t N, GridWork g, CsrView csr,
                                   int64_t stride, int write_indptr) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * N;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / N;
        if (write_indptr) {
            const int64_t i = t - b * N;
            if (i >= csr.row_lo && i < csr.row_hi) csr.indptr[b * (N + 1) + i] = i * stride;
            if (i == N - 1 && csr.row_hi == N) csr.indptr[b * (N + 1) + N] = N * stride;
        }
        const GridParams gp = g.params[b];
        const float4 p = xyz[t];
        const int cx = cell_coord(p.x, gp.ox, gp.inv_h, gp.nx);
        const int cy = cell_coord(p.y, gp.oy, gp.inv_h, gp.ny);
        const int cz = cell_coord(p.z, gp.oz, gp.inv_h, gp.nz);
        const int c = (cz * gp.ny + cy) * gp.nx + cx;
        g.cell_of[t] = c;
        atomicAdd(&g.cell_start[b * (g.max_cells + 1) + c], 1);
    }
}

// per cloud: cell_start <- exclusive scan of counts; cursor <- copy (coalesced
// 1024-cell rounds).
__global__ void __launch_bounds__(1024) grid_scan_kernel(int64_t N, GridWork g) {
    __shared__ int warp_sums[32];
    __shared__ int carry;
    const int64_t b = blockIdx.x;
    const int nc = g.params[b].ncells;
    int* cs = g.cell_start + b * (g.max_cells + 1);
    int* cur = g.cursor + b * (int64_t)g.max_cells;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nc; base += 1024) {
        const int i = base + tid;
        const int v = i < nc ? cs[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int t = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, t, o);
                if (lane >= o) t += y;
            }
            warp_sums[lane] = t;
        }
        __syncthreads();
        const int ex = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
        if (i < nc) { cs[i] = ex; cur[i] = ex; }
        __syncthreads();
        if (tid == 0) carry += warp_sums[31];
        __syncthreads();
    }
    if (tid == 0) cs[nc] = carry;
}

__global__ void grid_scatter_kernel(const float4* __restrict__ xyz, int64_t B, int64_t N, GridWork g) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * N;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / N;
        const int c = g.cell_of[t];
        const int pos = atomicAdd(&g.cursor[b * (int64_t)g.max_cells + c], 1);
        g.sorted_idx[b * N + pos] = (int32_t)(t - b * N);
        float4 v = xyz[t];
        v.w = __int_as_float((int)(t - b * N));  // the original index rides in w (no second load per hit)
        g.sorted_xyz[b * N + pos] = v;
    }
}

// ---- fused grid build: one 1024-thread CTA per cloud ---------------------------
// Bounding box + grid parameters (identical arithmetic to grid_setup_kernel),
// cell assignment, exclusive scan and scatter in one launch, with the cell
// counters in shared memory when the cloud's grid fits (else in its global
// cell_start range); also zeroes the per-cloud bookkeeping the build reads
// (evals, status) and, for method 2, writes the fixed-stride indptr.  Replaces
// five launches and two memsets for clouds up to kGridFusedMaxN points (the
// multi-kernel path above serves larger clouds and PS_GRID_MULTI=1).
constexpr int kGridSmemCells = 48 * 1024;
constexpr int64_t kGridFusedMaxN = 4096;

__global__ void __launch_bounds__(1024) grid_build_kernel(const float4* __restrict__ xyz, int64_t N,
                                                          const double* __restrict__ r2_levels, int L,
                                                          int64_t levels_ld, GridWork g, ExclWork w, CsrView csr,
                                                          int64_t stride, int write_indptr, int reach) {
    extern __shared__ int cnt_s[];
    __shared__ float red[6][32];
    __shared__ GridParams gps;
    __shared__ int warp_sums[32];
    __shared__ int carry;
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4* cx = xyz + b * N;
    if (tid == 0) {
        g.evals[b] = 0;
        w.status[b] = 0;
        if (w.spill) w.spill[b] = 0;
        if (b == 0) *w.long_count = 0;
    }
    // 1. bounding box and grid parameters
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int64_t i = tid; i < N; i += 1024) {
        const float4 p = cx[i];
        mn[0] = fminf(mn[0], p.x); mn[1] = fminf(mn[1], p.y); mn[2] = fminf(mn[2], p.z);
        mx[0] = fmaxf(mx[0], p.x); mx[1] = fmaxf(mx[1], p.y); mx[2] = fmaxf(mx[2], p.z);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(kFull, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(kFull, mx[a], o));
        }
        if (lane == 0) { red[a][warp] = mn[a]; red[3 + a][warp] = mx[a]; }
    }
    __syncthreads();
    if (tid == 0) {
        double lo[3], ext[3];
        for (int a = 0; a < 3; ++a) {
            float m0 = FLT_MAX, m1 = -FLT_MAX;
            for (int q = 0; q < 32; ++q) { m0 = fminf(m0, red[a][q]); m1 = fmaxf(m1, red[3 + a][q]); }
            lo[a] = m0;
            ext[a] = (double)m1 - (double)m0;
        }
        double r2 = 0.0;
        for (int l = 0; l < L; ++l) r2 = fmax(r2, r2_levels[b * levels_ld + l]);
        double h = sqrt(r2) * (1.0 + 1e-6) / (double)reach;
        if (!(h > 1e-30)) h = 1e-30;
        int n[3];
        for (int it = 0; it < 64; ++it) {
            double tot = 1.0;
            for (int a = 0; a < 3; ++a) {
                const double c = floor(ext[a] / h) + 1.0;
                n[a] = c > 1048576.0 ? 1048576 : (int)c;
                tot *= (double)n[a];
            }
            if (tot <= (double)g.max_cells) break;
            h *= cbrt(tot / (double)g.max_cells) * 1.001;
        }
        GridParams gp;
        gp.ox = lo[0]; gp.oy = lo[1]; gp.oz = lo[2];
        gp.inv_h = 1.0 / h;
        gp.nx = n[0]; gp.ny = n[1]; gp.nz = n[2];
        gp.ncells = n[0] * n[1] * n[2];
        gp.h = h;
        gp.reach = reach;
        g.params[b] = gp;
        gps = gp;
        carry = 0;
    }
    __syncthreads();
    const GridParams gp = gps;
    const int nc = gp.ncells;
    const bool sm = nc <= kGridSmemCells;
    int* cs = g.cell_start + b * (g.max_cells + 1);
    int* cnt = sm ? cnt_s : cs;
    int* cur = sm ? cnt_s : g.cursor + b * (int64_t)g.max_cells;
    for (int i = tid; i < nc; i += 1024) cnt[i] = 0;
    __syncthreads();
    // 2. cell of every point, counts
    int32_t* cell_of = g.cell_of + b * N;
    for (int64_t i = tid; i < N; i += 1024) {
        const float4 p = cx[i];
        const int c = (cell_coord(p.z, gp.oz, gp.inv_h, gp.nz) * gp.ny + cell_coord(p.y, gp.oy, gp.inv_h, gp.ny)) *
                          gp.nx + cell_coord(p.x, gp.ox, gp.inv_h, gp.nx);
        cell_of[i] = c;
        atomicAdd(&cnt[c], 1);
    }
    __syncthreads();
    // 3. exclusive scan -> cell_start (global) and the scatter cursors
    for (int base = 0; base < nc; base += 1024) {
        const int i = base + tid;
        const int v = i < nc ? cnt[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int t = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, t, o);
                if (lane >= o) t += y;
            }
            warp_sums[lane] = t;
        }
        __syncthreads();
        const int ex = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
        if (i < nc) { cs[i] = ex; cur[i] = ex; }
        __syncthreads();
        if (tid == 0) carry += warp_sums[31];
        __syncthreads();
    }
    if (tid == 0) cs[nc] = carry;
    // 4. scatter into cell order (original index in w)
    for (int64_t i = tid; i < N; i += 1024) {
        const int pos = atomicAdd(&cur[cell_of[i]], 1);
        g.sorted_idx[b * N + pos] = (int32_t)i;
        float4 v = cx[i];
        v.w = __int_as_float((int)i);
        g.sorted_xyz[b * N + pos] = v;
    }
    // 5. method 2: fixed-stride row pointers
    if (write_indptr)
        for (int64_t r = csr.row_lo + tid; r <= csr.row_hi; r += 1024)
            if (r < csr.row_hi || r == N) csr.indptr[b * (N + 1) + r] = r * stride;
}

// ---- row sort by (d2, index) + fused level counts -----------------------

// Bitonic sort of n2 (power of two) entries in shared memory by `nthr`
// cooperating threads (thread rank t), synchronised with `sync`.
template <typename Sync>
__device__ __forceinline__ void bitonic_smem(double* kd, int32_t* ki, int n2, int t, int nthr, Sync sync) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int x = t; x < n2 / 2; x += nthr) {
                // x-th compare pair of this stage
                const int lo = (x / jj) * (2 * jj) + (x % jj);
                const int hi = lo + jj;
                const bool up = ((lo & k) == 0);
                const double a = kd[lo], c = kd[hi];
                const int32_t ia = ki[lo], ic = ki[hi];
                const bool sw = up ? key_less(c, ic, a, ia) : key_less(a, ia, c, ic);
                if (sw) { kd[lo] = c; kd[hi] = a; ki[lo] = ic; ki[hi] = ia; }
            }
            sync();
        }
    }
}

constexpr int kSortWarps = 8;
constexpr int kWarpRowCap = 256;
constexpr int kCtaRowCap = 8192;

__global__ void __launch_bounds__(kSortWarps * 32) excl_sort_small_kernel(CsrView csr, int64_t B,
                                                                       const double* __restrict__ r2_levels,
                                                                       int64_t levels_ld, ExclWork w) {
    __shared__ double sd[kSortWarps][kWarpRowCap];
    __shared__ int32_t si[kSortWarps][kWarpRowCap];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t N = csr.N;
    const int64_t rows = B * N;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t gr = (int64_t)blockIdx.x * kSortWarps + warp; gr < rows;
         gr += (int64_t)gridDim.x * kSortWarps) {
        const int64_t b = gr / N, r = gr - b * N;
        int64_t bound = 0;
        if (lane < 2) bound = csr.indptr[b * (N + 1) + r + lane];
        const int64_t lo = __shfl_sync(kFull, bound, 0);
        const int64_t hi = __shfl_sync(kFull, bound, 1);
        if (hi > csr.cap_entries) {  // overflowed cloud: status already set; leave a safe row
            if (lane < csr.L) csr.counts[(b * csr.L + lane) * N + r] = 0;
            continue;
        }
        const int m = (int)(hi - lo);
        if (m > kWarpRowCap) {
            if (lane == 0) {
                const unsigned k = atomicAdd(w.long_count, 1u);
                w.long_rows[k] = (int32_t)gr;
            }
            continue;
        }
        int32_t* nbr = csr.nbr + b * csr.cap_entries + lo;
        double* d2 = csr.d2 + b * csr.cap_entries + lo;
        const double* lv = r2_levels ? r2_levels + b * levels_ld : nullptr;
        if (m <= 64) {
            double d0 = lane < m ? d2[lane] : kInf;
            int32_t i0 = lane < m ? nbr[lane] : 0x7fffffff;
            double d1 = lane + 32 < m ? d2[lane + 32] : kInf;
            int32_t i1 = lane + 32 < m ? nbr[lane + 32] : 0x7fffffff;
            int n2 = 1;
            while (n2 < m) n2 <<= 1;
            if (m > 1) warp_bitonic64(d0, i0, d1, i1, lane, n2 < 2 ? 2 : n2);
            if (lane < m) { d2[lane] = d0; nbr[lane] = i0; }
            if (lane + 32 < m) { d2[lane + 32] = d1; nbr[lane + 32] = i1; }
            for (int l = 0; l < csr.L; ++l) {
                const double t = lv[l];
                const int c = __popc(__ballot_sync(kFull, lane < m && d0 < t)) +
                              __popc(__ballot_sync(kFull, lane + 32 < m && d1 < t));
                if (lane == 0) csr.counts[(b * csr.L + l) * N + r] = c;
            }
            continue;
        }
        int n2 = 1;
        while (n2 < m) n2 <<= 1;
        for (int k = lane; k < n2; k += 32) {
            sd[warp][k] = k < m ? d2[k] : kInf;
            si[warp][k] = k < m ? nbr[k] : 0x7fffffff;
        }
        __syncwarp();
        bitonic_smem(sd[warp], si[warp], n2, lane, 32, [] { __syncwarp(); });
        for (int k = lane; k < m; k += 32) {
            d2[k] = sd[warp][k];
            nbr[k] = si[warp][k];
        }
        // fused level counts: #entries with d2 < r2_l (strict, _kernels.py:233)
        for (int l = 0; l < csr.L; ++l) {
            const double t = lv[l];
            int c = 0;
            for (int k = lane; k < m; k += 32) c += sd[warp][k] < t ? 1 : 0;
            c = __reduce_add_sync(kFull, c);
            if (lane == 0) csr.counts[(b * csr.L + l) * N + r] = c;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(1024) excl_sort_large_kernel(CsrView csr, const double* __restrict__ r2_levels,
                                                           int64_t levels_ld, ExclWork w) {
    extern __shared__ __align__(16) unsigned char dyn[];
    double* sd = reinterpret_cast<double*>(dyn);
    int32_t* si = reinterpret_cast<int32_t*>(dyn + sizeof(double) * kCtaRowCap);
    __shared__ int red[32];
    const int64_t N = csr.N;
    const unsigned nlong = *w.long_count;
    for (unsigned t = blockIdx.x; t < nlong; t += gridDim.x) {
        const int64_t gr = w.long_rows[t];
        const int64_t b = gr / N, r = gr - b * N;
        const int64_t lo = csr.indptr[b * (N + 1) + r];
        const int64_t hi = csr.indptr[b * (N + 1) + r + 1];
        const int64_t m = hi - lo;
        int32_t* nbr = csr.nbr + b * csr.cap_entries + lo;
        double* d2 = csr.d2 + b * csr.cap_entries + lo;
        double* kd;
        int32_t* ki;
        int n2 = 1;
        while (n2 < m) n2 <<= 1;
        const bool in_smem = n2 <= kCtaRowCap;
        if (in_smem) {
            kd = sd; ki = si;
            for (int k = threadIdx.x; k < n2; k += blockDim.x) {
                kd[k] = k < m ? d2[k] : __longlong_as_double(0x7ff0000000000000LL);
                ki[k] = k < m ? nbr[k] : 0x7fffffff;
            }
            __syncthreads();
            bitonic_smem(kd, ki, n2, threadIdx.x, blockDim.x, [] { __syncthreads(); });
            for (int k = threadIdx.x; k < m; k += blockDim.x) { d2[k] = kd[k]; nbr[k] = ki[k]; }
            __syncthreads();
        } else {
            // giant row (radius near the cloud diameter): odd-even transposition
            // in global memory -- correct, slow, only for degenerate inputs.
            for (int64_t phase = 0; phase < m; ++phase) {
                for (int64_t k = 2 * threadIdx.x + (phase & 1); k + 1 < m; k += 2 * blockDim.x) {
                    const double a = d2[k], c = d2[k + 1];
                    const int32_t ia = nbr[k], ic = nbr[k + 1];
                    if (key_less(c, ic, a, ia)) { d2[k] = c; d2[k + 1] = a; nbr[k] = ic; nbr[k + 1] = ia; }
                }
                __syncthreads();
            }
        }
        for (int l = 0; l < csr.L; ++l) {
            const double th = r2_levels[b * levels_ld + l];
            int c = 0;
            for (int64_t k = threadIdx.x; k < m; k += blockDim.x) c += d2[k] < th ? 1 : 0;
            c = __reduce_add_sync(kFull, c);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
            __syncthreads();
            if (threadIdx.x == 0) {
                int s = 0;
                for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
                csr.counts[(b * csr.L + l) * N + r] = s;
            }
            __syncthreads();
        }
    }
}

// level counts for an already-sorted CSR (drop-in csr_level_counts)
__global__ void level_counts_kernel(CsrView csr, int64_t B, const double* __restrict__ r2_levels,
                                    int64_t levels_ld) {
    const int64_t N = csr.N;
    for (int64_t gr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gr < B * N;
         gr += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = gr / N, r = gr - b * N;
        const int64_t lo = csr.indptr[b * (N + 1) + r];
        const int64_t hi = csr.indptr[b * (N + 1) + r + 1];
        const double* d2 = csr.d2 + b * csr.cap_entries;
        for (int l = 0; l < csr.L; ++l) {
            const double t = r2_levels[b * levels_ld + l];
            int64_t x = lo, y = hi;
            while (x < y) {
                const int64_t mid = x + ((y - x) >> 1);
                if (d2[mid] < t) x = mid + 1; else y = mid;
            }
            csr.counts[(b * csr.L + l) * N + r] = (int32_t)(x - lo);
        }
    }
}

}  // namespace

// Warp-per-point grid pass.  COUNT: deg[i] = #{j : d2(i, j) < r2max}.
// FILL: the row of i is collected in shared memory, sorted by (d2, index)
// in registers (<= 64 entries) or shared memory (<= 256), written once in
// final order, and its level counts are taken with ballots -- fill, sort and
// csr_level_counts fused.  Longer rows are written unsorted and queued for
// the CTA sort kernel.
constexpr int kRowWarps = 8;
constexpr int kRowCap = 256;

template <bool FILL>
__global__ void __launch_bounds__(kRowWarps * 32, 4) grid_rows_kernel(int64_t B, int64_t N,
                                                                   const double* __restrict__ r2_levels, int L,
                                                                   int64_t levels_ld, GridWork g, ExclWork w,
                                                                   CsrView csr) {
    __shared__ double hd[FILL ? kRowWarps : 1][FILL ? kRowCap : 1];
    __shared__ int32_t hj[FILL ? kRowWarps : 1][FILL ? kRowCap : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t gs = (int64_t)blockIdx.x * kRowWarps + warp; gs < B * N; gs += (int64_t)gridDim.x * kRowWarps) {
        const int64_t b = gs / N, s = gs - b * N;
        double r2 = 0.0;
        for (int l = 0; l < L; ++l) r2 = fmax(r2, r2_levels[b * levels_ld + l]);
        const float thr = prefilter_threshold(r2);
        const bool no_filter = !(thr <= FLT_MAX);
        const GridParams gp = g.params[b];
        const float4* sx = g.sorted_xyz + b * N;
        const int32_t* si = g.sorted_idx + b * N;
        const int* cs = g.cell_start + b * (g.max_cells + 1);
        const float4 p = sx[s];
        const int32_t i = si[s];
        const int cx = cell_coord(p.x, gp.ox, gp.inv_h, gp.nx);
        const int cy = cell_coord(p.y, gp.oy, gp.inv_h, gp.ny);
        const int cz = cell_coord(p.z, gp.oz, gp.inv_h, gp.nz);
        int64_t rlo = 0, m = 0;
        bool direct = false;
        if (FILL) {
            rlo = csr.indptr[b * (N + 1) + i];
            m = csr.indptr[b * (N + 1) + i + 1] - rlo;
            if (rlo + m > csr.cap_entries) {  // overflow: status set by the scan; leave a safe row
                if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = 0;
                continue;
            }
            direct = m > kRowCap;
        }
        int32_t* rn = FILL ? csr.nbr + b * csr.cap_entries + rlo : nullptr;
        double* rd = FILL ? csr.d2 + b * csr.cap_entries + rlo : nullptr;
        // the 9 (dz, dy) cell rows: lanes 0..8 fetch their [t0, t1) in parallel
        int r0 = 0, rlen = 0;
        if (lane < 9) {
            const int z = cz + lane / 3 - 1, y = cy + lane % 3 - 1;
            if (z >= 0 && z < gp.nz && y >= 0 && y < gp.ny) {
                const int x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < gp.nx ? cx + 1 : gp.nx - 1;
                const int row = (z * gp.ny + y) * gp.nx;
                r0 = cs[row + x0];
                rlen = cs[row + x1 + 1] - r0;
            }
        }
        // flatten the candidate list: prefix over the 9 ranges
        int incl = rlen;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(kFull, incl, 8);
        const int excl0 = incl - rlen;
        int cnt = 0;
        const unsigned long long cand = (unsigned long long)total;
#pragma unroll 2
        for (int tb = 0; tb < total; tb += 32) {
            const int f = tb + lane;  // flat candidate index
            // locate the range: first r with excl(r+1) > f
            int rr = 0;
#pragma unroll
            for (int q = 1; q < 9; ++q) rr += (f >= __shfl_sync(kFull, excl0, q)) ? 1 : 0;
            const int base = __shfl_sync(kFull, r0, rr) - __shfl_sync(kFull, excl0, rr);
            const int t = base + f;
            bool hit = false;
            double d = 0.0;
            if (f < total) {
                const float4 q = sx[t];
                if (no_filter || sqdist_f32(p, q) < thr) {
                    d = sqdist4(p, q);
                    hit = d < r2;
                }
            }
            const unsigned hm = __ballot_sync(kFull, hit);
            if (FILL && hit) {
                const int slot = cnt + __popc(hm & lt);
                if (direct) {
                    if (slot < m) { rn[slot] = si[t]; rd[slot] = d; }
                } else if (slot < kRowCap) {
                    hd[warp][slot] = d;
                    hj[warp][slot] = si[t];
                }
            }
            cnt += __popc(hm);
        }
        if (!FILL) {
            if (lane == 0) {
                w.deg[b * N + i] = cnt;
                atomicAdd(g.evals + b, cand);
            }
            continue;
        }
        __syncwarp();
        if (direct) {
            if (lane == 0) {
                const unsigned k = atomicAdd(w.long_count, 1u);
                w.long_rows[k] = (int32_t)(b * N + i);
            }
            continue;
        }
        const int mm = (int)m;
        const double* lv = r2_levels + b * levels_ld;
        if (mm <= 64) {
            double d0 = lane < mm ? hd[warp][lane] : kInf;
            int32_t i0 = lane < mm ? hj[warp][lane] : 0x7fffffff;
            double d1 = lane + 32 < mm ? hd[warp][lane + 32] : kInf;
            int32_t i1 = lane + 32 < mm ? hj[warp][lane + 32] : 0x7fffffff;
            int n2 = 2;
            while (n2 < mm) n2 <<= 1;
            if (mm > 1) warp_bitonic64(d0, i0, d1, i1, lane, n2);
            if (lane < mm) { rd[lane] = d0; rn[lane] = i0; }
            if (lane + 32 < mm) { rd[lane + 32] = d1; rn[lane + 32] = i1; }
            for (int l = 0; l < csr.L; ++l) {
                const double t = lv[l];
                const int c = __popc(__ballot_sync(kFull, lane < mm && d0 < t)) +
                              __popc(__ballot_sync(kFull, lane + 32 < mm && d1 < t));
                if (lane == 0) csr.counts[(b * csr.L + l) * N + i] = c;
            }
        } else {
            int n2 = 1;
            while (n2 < mm) n2 <<= 1;
            for (int k = mm + lane; k < n2; k += 32) { hd[warp][k] = kInf; hj[warp][k] = 0x7fffffff; }
            __syncwarp();
            bitonic_smem(hd[warp], hj[warp], n2, lane, 32, [] { __syncwarp(); });
            for (int k = lane; k < mm; k += 32) { rd[k] = hd[warp][k]; rn[k] = hj[warp][k]; }
            for (int l = 0; l < csr.L; ++l) {
                const double t = lv[l];
                int c = 0;
                for (int k = lane; k < mm; k += 32) c += hd[warp][k] < t ? 1 : 0;
                c = __reduce_add_sync(kFull, c);
                if (lane == 0) csr.counts[(b * csr.L + l) * N + i] = c;
            }
        }
        __syncwarp();
    }
}

// Method 2 (hot path): single pass, fixed row stride.  Row i of cloud b
// lives at b * cap_entries + i * stride (indptr[i] = i * stride), its entries
// ordered by level bucket: bucket(e) = #{levels with r2 <= d2}, so that for
// every level l the entries with d2 < r2_l are exactly the first counts[l]
// -- the only row property the sampler, early termination and the
// redundancy-free queries rely on (they read per-level prefixes as sets;
// the queries order their small prefixes themselves).  Rows longer than the
// stride move to the cloud's spill arena (ell_row_stride); only a full arena
// sets status bit 1 (the sampler and the queries then emit error states and
// the host rebuilds with a larger capacity).
// Staging: kEllCap entries per warp in shared memory; rows beyond it take
// the rescan path (one pass per bucket, straight to the row).  Two
// instances: 8 warps x 256 entries for short rows (C1-C4), 4 warps x 512
// for strides above 256 (C5-sized clouds, ~270 entries per row), so that
// the rescan stays rare.
template <int kEllWarps, int kEllCap, bool kCull, bool kDense = false>
__global__ void __launch_bounds__(kEllWarps * 32, 1024 / (kEllWarps * 32)) grid_ell_kernel(
    int64_t B, int64_t N, const double* __restrict__ r2_levels, int L, int64_t levels_ld, int64_t stride, GridWork g,
    ExclWork w, CsrView csr) {
    __shared__ double hd[kEllWarps][kEllCap];
    __shared__ int32_t hj[kEllWarps][kEllCap];
    __shared__ uint16_t hb[kEllWarps][kEllCap];  // rank within its bucket
    __shared__ uint8_t hk[kEllWarps][kEllCap];   // bucket
    __shared__ int hcnt[kEllWarps][33];          // per-bucket counts
    __shared__ double lvs[kEllWarps][32];
    __shared__ unsigned long long lvb[kEllWarps][32];
    __shared__ unsigned long long lvsort[kEllWarps][16];  // levels ascending, padded (L <= 16)
    __shared__ int tbase[kEllWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    // one cloud per grid row: the cloud's level values and grid parameters
    // are set up once per warp; warps stride over the cloud's sorted points
    const int64_t b = blockIdx.y;
    const double my_r2 = lane < L ? r2_levels[b * levels_ld + lane] : 0.0;
    if (lane < L) {
        lvs[warp][lane] = my_r2;
        lvb[warp][lane] = (unsigned long long)__double_as_longlong(my_r2);
    }
    int rank_lt = 0, rank_st = 0;
    double r2 = 0.0;
    for (int l = 0; l < L; ++l) {
        const double v = __shfl_sync(kFull, my_r2, l);
        rank_lt += (v < my_r2) ? 1 : 0;
        rank_st += (v < my_r2 || (v == my_r2 && l < lane)) ? 1 : 0;  // stable sort position
        r2 = fmax(r2, v);
    }
    const bool sorted_lv = L <= 16;
    if (lane < 16) lvsort[warp][lane] = ~0ull;
    __syncwarp();
    if (lane < L && sorted_lv) lvsort[warp][rank_st] = (unsigned long long)__double_as_longlong(my_r2);
    const float thr = prefilter_threshold(r2);
    const bool no_filter = !(thr <= FLT_MAX);
    const GridParams gp = g.params[b];
    const float4* sx = g.sorted_xyz + b * N;
    const int32_t* si = g.sorted_idx + b * N;
    const int* cs = g.cell_start + b * (g.max_cells + 1);
    __syncwarp();
    unsigned long long evals = 0;  // candidates visited by this warp (one atomic at the end)
    for (int64_t s = (int64_t)blockIdx.x * kEllWarps + warp; s < N; s += (int64_t)gridDim.x * kEllWarps) {
        hcnt[warp][lane] = 0;
        if (lane == 0) hcnt[warp][32] = 0;
        __syncwarp();
        const float4 p = sx[s];
        const int32_t i = __float_as_int(p.w);  // original index (grid_scatter_kernel)
        if (i < csr.row_lo || i >= csr.row_hi) continue;  // another rank's row (warp-uniform)
        const int cx = cell_coord(p.x, gp.ox, gp.inv_h, gp.nx);
        const int cy = cell_coord(p.y, gp.oy, gp.inv_h, gp.ny);
        const int cz = cell_coord(p.z, gp.oz, gp.inv_h, gp.nz);
        int r0 = 0, rlen = 0;
        if constexpr (kCull) {
            // cells of width >= R_max / 2: candidate cell rows (dz, dy) in
            // [-2, 2]^2, one per lane; a row whose y/z slab is farther than
            // R_max is dropped, the others keep only the x cells that can hold
            // a point of the ball (|qx - px| <= sqrt(R_max^2 - gy^2 - gz^2)).
            // Gaps shrink by tol (far above the rounding of the cell
            // assignment) and the x half-width grows by 1e-5 relative (above
            // the float sqrt's rounding): no point within R_max is lost.
            const int reach = gp.reach, wdt = 2 * reach + 1;
            if (lane < wdt * wdt) {
                const int dz = lane / wdt - reach, dy = lane % wdt - reach;
                const int z = cz + dz, y = cy + dy;
                if (z >= 0 && z < gp.nz && y >= 0 && y < gp.ny) {
                    const double tol = 1e-9 * (fabs(gp.ox) + fabs(gp.oy) + fabs(gp.oz) + fabs((double)p.x) +
                                               fabs((double)p.y) + fabs((double)p.z) + gp.h * (gp.nx + gp.ny + gp.nz));
                    double gy = 0.0, gz = 0.0;
                    if (dy > 0) gy = (gp.oy + y * gp.h) - (double)p.y;
                    else if (dy < 0) gy = (double)p.y - (gp.oy + (y + 1) * gp.h);
                    if (dz > 0) gz = (gp.oz + z * gp.h) - (double)p.z;
                    else if (dz < 0) gz = (double)p.z - (gp.oz + (z + 1) * gp.h);
                    gy = fmax(0.0, gy - tol);
                    gz = fmax(0.0, gz - tol);
                    const double rem = r2 - gy * gy - gz * gz;
                    if (rem >= 0.0) {
                        int x0 = cx - reach, x1 = cx + reach;
                        if (rem < 1e30) {
                            const double w = (double)sqrtf((float)rem) * (1.0 + 1e-5) + tol;
                            x0 = max(x0, cell_coord((double)p.x - w, gp.ox, gp.inv_h, gp.nx));
                            x1 = min(x1, cell_coord((double)p.x + w, gp.ox, gp.inv_h, gp.nx));
                        }
                        x0 = max(x0, 0);
                        x1 = min(x1, gp.nx - 1);
                        if (x0 <= x1) {
                            const int row = (z * gp.ny + y) * gp.nx;
                            r0 = cs[row + x0];
                            rlen = cs[row + x1 + 1] - r0;
                        }
                    }
                }
            }
        } else if (lane < 9) {
            // cells of width >= R_max: the 3 x 3 cell rows around the point
            const int z = cz + lane / 3 - 1, y = cy + lane % 3 - 1;
            if (z >= 0 && z < gp.nz && y >= 0 && y < gp.ny) {
                const int x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < gp.nx ? cx + 1 : gp.nx - 1;
                const int row = (z * gp.ny + y) * gp.nx;
                r0 = cs[row + x0];
                rlen = cs[row + x1 + 1] - r0;
            }
        }
        int incl = rlen;
#pragma unroll
        for (int o = 1; o < (kCull ? 32 : 16); o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(kFull, incl, kCull ? 31 : 8);
        const int excl0 = incl - rlen;  // non-decreasing over the rows' lanes
        // range of flattened candidate f: the last row lane whose start <= f;
        // sorted position = base[range] + f (per-warp table)
        tbase[warp][lane] = r0 - excl0;
        int e[8];  // !kCull: the 8 later range starts in registers
#pragma unroll
        for (int q = 0; q < 8; ++q) e[q] = __shfl_sync(kFull, excl0, q + 1);
        __syncwarp();
        if constexpr (kDense) {
            // Long rows (kCull, L <= 15): A. f32 screen of the candidates, the
            // survivors' sorted positions compacted; B. lanes = survivors:
            // exact f64 test, bucket, rank within the bucket from ballots over
            // the four bucket bits; C. scatter -- no divergent per-hit work in
            // the candidate loop, no shared-memory atomics (the long-row form
            // of grid_ell_cell_kernel's phases)
            evals += (unsigned long long)total;
            int nsv = 0;
#pragma unroll 4
            for (int tb = 0; tb < total; tb += 32) {
                const int f = tb + lane;
                int rc = 0;
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) rc += (__shfl_sync(kFull, excl0, rc + st - 1) <= f) ? st : 0;
                const int t = tbase[warp][rc - 1] + f;
                bool sv = false;
                if (f < total) sv = no_filter || sqdist_f32(p, sx[t]) < thr;
                const unsigned m = __ballot_sync(kFull, sv);
                const int pos = nsv + __popc(m & lt);
                if (sv && pos < kEllCap) hj[warp][pos] = t;
                nsv += __popc(m);
            }
            __syncwarp();
            if (nsv <= kEllCap) {
                int runs = 0;  // lane t < 16: entries of bucket t so far
                for (int e0 = 0; e0 < nsv; e0 += 32) {
                    const int ee = e0 + lane;
                    const bool valid = ee < nsv;
                    const float4 q = sx[valid ? hj[warp][ee] : s];
                    const double d = sqdist4(p, q);
                    const bool hit = valid && d < r2;
                    const unsigned long long db = (unsigned long long)__double_as_longlong(d);
                    const unsigned long long* ls = lvsort[warp];
                    int bk = (ls[7] <= db) ? 8 : 0;
                    bk += (ls[bk + 3] <= db) ? 4 : 0;
                    bk += (ls[bk + 1] <= db) ? 2 : 0;
                    bk += (ls[bk] <= db) ? 1 : 0;
                    const unsigned hm = __ballot_sync(kFull, hit);
                    unsigned peers = hm, mine = hm;
#pragma unroll
                    for (int bt = 0; bt < 4; ++bt) {
                        const unsigned mb = __ballot_sync(kFull, hit && ((bk >> bt) & 1));
                        peers &= ((bk >> bt) & 1) ? mb : ~mb;
                        mine &= ((lane >> bt) & 1) ? mb : ~mb;
                    }
                    const int rank = __shfl_sync(kFull, runs, bk & 15) + __popc(peers & lt);
                    runs += __popc(mine);
                    if (valid) {
                        hk[warp][ee] = hit ? (uint8_t)bk : (uint8_t)0xff;
                        hb[warp][ee] = (uint16_t)rank;
                        hd[warp][ee] = d;
                        hj[warp][ee] = __float_as_int(q.w);  // now the original index
                    }
                }
                const int v = (lane < 16 && lane <= L) ? runs : 0;
                int hincl = v;
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    const int y = __shfl_up_sync(kFull, hincl, o);
                    if (lane >= o) hincl += y;
                }
                const int cntd = __shfl_sync(kFull, hincl, 15);
                const int hbase = hincl - v;
                int64_t row_off = (int64_t)i * stride;
                if (cntd > stride) {  // spill arena (see below)
                    unsigned long long o = 0;
                    if (lane == 0) o = atomicAdd(&w.spill[b], (unsigned long long)((cntd + 3) & ~3));
                    o = __shfl_sync(kFull, o, 0);
                    const int64_t off = N * stride + csr.spill_lo + (int64_t)o;
                    if (off + cntd > N * stride + csr.spill_hi) {
                        if (lane == 0) atomicOr(&w.status[b], 2);
                        if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = 0;
                        __syncwarp();
                        continue;
                    }
                    row_off = off;
                    if (lane == 0) csr.indptr[b * (N + 1) + i] = off;
                }
                __syncwarp();
                int32_t* rn = csr.nbr + b * csr.cap_entries + row_off;
                double* rd = csr.d2 + b * csr.cap_entries + row_off;
                for (int e0 = 0; e0 < nsv; e0 += 32) {
                    const int ee = e0 + lane;
                    const int bk = ee < nsv ? hk[warp][ee] : 0xff;
                    const int pos = __shfl_sync(kFull, hbase, bk & 15) + (bk != 0xff ? hb[warp][ee] : 0);
                    if (bk != 0xff) {
                        __stcs(rd + pos, hd[warp][ee]);  // d2 streams to HBM: keep L2 for the nbr rows
                        rn[pos] = hj[warp][ee];
                    }
                }
                const int hist_mine = __shfl_sync(kFull, hincl, rank_lt < 15 ? rank_lt : 15);
                if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = hist_mine;
                {
                    const int64_t row_cap = row_off == (int64_t)i * stride ? stride : ((cntd + 3) & ~3);
                    if (lane < min((int64_t)((cntd + 3) & ~3), row_cap) - cntd) rn[cntd + lane] = -1;
                }
                __syncwarp();
                continue;
            }
            // more survivors than the staging holds: the general path below
            // (its exact count, spill and per-bucket rescan); evals counted once
            evals -= (unsigned long long)total;
        }
        int cnt = 0;
#pragma unroll 4
        for (int tb = 0; tb < total; tb += 32) {
            const int f = tb + lane;
            int rr;
            if constexpr (kCull) {
                // five shuffle steps over the 32 non-decreasing starts
                int rc = 0;
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) rc += (__shfl_sync(kFull, excl0, rc + st - 1) <= f) ? st : 0;
                rr = rc - 1;
            } else {
                // rr = #(e[q] <= f) over the 8 later starts: selects on registers
                const bool c4 = f >= e[3];
                rr = c4 ? 4 : 0;
                const bool c2 = f >= (c4 ? e[5] : e[1]);
                rr += c2 ? 2 : 0;
                rr += (f >= (c4 ? (c2 ? e[6] : e[4]) : (c2 ? e[2] : e[0]))) ? 1 : 0;
                rr += (rr == 7 && f >= e[7]) ? 1 : 0;
            }
            const int t = tbase[warp][rr] + f;
            bool hit = false;
            double d = 0.0;
            int32_t qi = 0;
            if (f < total) {
                const float4 q = sx[t];
                if (no_filter || sqdist_f32(p, q) < thr) {
                    d = sqdist4(p, q);
                    hit = d < r2;
                    qi = __float_as_int(q.w);
                }
            }
            const unsigned hm = __ballot_sync(kFull, hit);
            if (hit) {
                const int slot = cnt + __popc(hm & lt);
                if (slot < kEllCap) {
                    // bucket by integer compares of the bit patterns (d, r2 >= 0): ALU, not FP64
                    const unsigned long long db = (unsigned long long)__double_as_longlong(d);
                    int bk = 0;
                    if (sorted_lv) {
                        // #levels <= d: branch-free upper bound over the sorted,
                        // padded levels (a hit is below the largest, so <= 15)
                        const unsigned long long* ls = lvsort[warp];
                        bk = (ls[7] <= db) ? 8 : 0;
                        bk += (ls[bk + 3] <= db) ? 4 : 0;
                        bk += (ls[bk + 1] <= db) ? 2 : 0;
                        bk += (ls[bk] <= db) ? 1 : 0;
                    } else {
                        for (int l = 0; l < L; ++l) bk += (lvb[warp][l] <= db) ? 1 : 0;
                    }
                    hd[warp][slot] = d;
                    hj[warp][slot] = qi;
                    hb[warp][slot] = (uint16_t)atomicAdd(&hcnt[warp][bk], 1);  // rank within bucket
                    hk[warp][slot] = (uint8_t)bk;
                }
            }
            cnt += __popc(hm);
        }
        evals += (unsigned long long)total;
        int64_t row_off = (int64_t)i * stride;
        if (cnt > stride) {
            // longer than the stride: the row takes a run of the cloud's spill
            // arena (after the N strided rows) and indptr[i] points there; only
            // when the arena is exhausted does the build fail -- status bit 1,
            // an empty row, and consumers (sampler, queries) see the status
            unsigned long long o = 0;
            if (lane == 0) o = atomicAdd(&w.spill[b], (unsigned long long)((cnt + 3) & ~3));
            o = __shfl_sync(kFull, o, 0);
            const int64_t off = N * stride + csr.spill_lo + (int64_t)o;
            if (off + cnt > N * stride + csr.spill_hi) {
                if (lane == 0) atomicOr(&w.status[b], 2);
                if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = 0;
                continue;
            }
            row_off = off;
            if (lane == 0) csr.indptr[b * (N + 1) + i] = off;
        }
        __syncwarp();
        int32_t* rn = csr.nbr + b * csr.cap_entries + row_off;
        double* rd = csr.d2 + b * csr.cap_entries + row_off;
        if (cnt > kEllCap) {
            // long row (beyond the staging buffer): one exact rescan per bucket,
            // writing straight to the row -- only for very dense neighbourhoods
            int base2 = 0, hist2 = 0;
            for (int bk = 0; bk <= L; ++bk) {
                int here = 0;
                for (int tb = 0; tb < total; tb += 32) {
                    const int f = tb + lane;
                    int rc = 0;
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1)
                        rc += (__shfl_sync(kFull, excl0, rc + st - 1) <= f) ? st : 0;
                    const int t = tbase[warp][rc - 1] + f;
                    bool in = false;
                    double d = 0.0;
                    if (f < total) {
                        const float4 q = sx[t];
                        if (no_filter || sqdist_f32(p, q) < thr) {
                            d = sqdist4(p, q);
                            if (d < r2) {
                                int bb = 0;
                                for (int l = 0; l < L; ++l) bb += (lvs[warp][l] <= d) ? 1 : 0;
                                in = bb == bk;
                            }
                        }
                    }
                    const unsigned bm = __ballot_sync(kFull, in);
                    if (in) {
                        const int pos = base2 + here + __popc(bm & lt);
                        __stcs(rd + pos, d);  // d2 streams to HBM: keep L2 for the nbr rows
                        rn[pos] = si[t];
                    }
                    here += __popc(bm);
                }
                base2 += here;
                if (lane < L && bk == rank_lt) hist2 = base2;
            }
            if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = hist2;
            // pad the row to a whole 16-byte chunk (readers load int4 chunks, masked by the counts)
            {
                const int64_t row_cap = row_off == (int64_t)i * stride ? stride : ((base2 + 3) & ~3);
                if (lane < min((int64_t)((base2 + 3) & ~3), row_cap) - base2) rn[base2 + lane] = -1;
            }
            continue;
        }
        // scatter by bucket: bucket bases from the per-bucket counts (exclusive
        // prefix across lanes), each entry at base + its rank within the bucket
        const int hc = lane <= L ? hcnt[warp][lane] : 0;
        int hincl = hc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, hincl, o);
            if (lane >= o) hincl += y;
        }
        const int hbase = hincl - hc;
        for (int e0 = 0; e0 < cnt; e0 += 32) {
            const int e = e0 + lane;
            const int bk = e < cnt ? hk[warp][e] : 0;
            const int pos = __shfl_sync(kFull, hbase, bk) + (e < cnt ? hb[warp][e] : 0);
            if (e < cnt) {
                __stcs(rd + pos, hd[warp][e]);  // d2 streams to HBM: keep L2 for the nbr rows
                rn[pos] = hj[warp][e];
            }
        }
        // level l holds buckets 0 .. rank_lt(l)
        const int hist_mine = __shfl_sync(kFull, hincl, rank_lt < 31 ? rank_lt : 31);
        if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = hist_mine;
        // pad the row to a whole 16-byte chunk (readers load int4 chunks, masked by the counts)
        {
            const int64_t row_cap = row_off == (int64_t)i * stride ? stride : ((cnt + 3) & ~3);
            if (lane < min((int64_t)((cnt + 3) & ~3), row_cap) - cnt) rn[cnt + lane] = -1;
        }
        __syncwarp();
    }
    if (lane == 0 && evals) atomicAdd(g.evals + b, evals);
}

// A row with more f32 survivors than grid_ell_cell_kernel stages: exact
// count, spill decision, then one pass per level bucket over the candidates
// straight to the row (dense neighbourhoods only).  Out of line, so that its
// registers do not weigh on the cell kernel's main path.  tb / ts: the cell
// segment's flattened candidate ranges (start in f, sorted base).
__device__ __noinline__ void ell_rescan_row(float4 p, int32_t i, int64_t b, int64_t N, int total, const int* tb,
                                            const int* ts, const float4* sx, double r2, float thr, bool no_filter,
                                            int L, const double* lvs, int rank_lt, int64_t stride, ExclWork w,
                                            CsrView csr) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    auto at = [&](int f) -> float4 {
        int rr = 0;
#pragma unroll
        for (int q = 1; q < 9; ++q) rr += (f >= ts[q]) ? 1 : 0;
        return sx[tb[rr] + f];
    };
    int cnt = 0;
    for (int tb0 = 0; tb0 < total; tb0 += 32) {
        const int f = tb0 + lane;
        bool in = false;
        if (f < total) {
            const float4 q = at(f);
            in = (no_filter || sqdist_f32(p, q) < thr) && sqdist4(p, q) < r2;
        }
        cnt += __popc(__ballot_sync(kFull, in));
    }
    int64_t row_off = (int64_t)i * stride;
    if (cnt > stride) {
        unsigned long long o = 0;
        if (lane == 0) o = atomicAdd(&w.spill[b], (unsigned long long)((cnt + 3) & ~3));
        o = __shfl_sync(kFull, o, 0);
        const int64_t off = N * stride + csr.spill_lo + (int64_t)o;
        if (off + cnt > N * stride + csr.spill_hi) {
            if (lane == 0) atomicOr(&w.status[b], 2);
            if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = 0;
            __syncwarp();
            return;
        }
        row_off = off;
        if (lane == 0) csr.indptr[b * (N + 1) + i] = off;
    }
    int32_t* rn = csr.nbr + b * csr.cap_entries + row_off;
    double* rd = csr.d2 + b * csr.cap_entries + row_off;
    int base2 = 0, hist2 = 0;
    for (int bk = 0; bk <= L; ++bk) {
        int here = 0;
        for (int tb0 = 0; tb0 < total; tb0 += 32) {
            const int f = tb0 + lane;
            bool in = false;
            double d = 0.0;
            int32_t qi = 0;
            if (f < total) {
                const float4 q = at(f);
                if (no_filter || sqdist_f32(p, q) < thr) {
                    d = sqdist4(p, q);
                    if (d < r2) {
                        int bb = 0;
                        for (int l = 0; l < L; ++l) bb += (lvs[l] <= d) ? 1 : 0;
                        in = bb == bk;
                        qi = __float_as_int(q.w);
                    }
                }
            }
            const unsigned bm = __ballot_sync(kFull, in);
            if (in) {
                const int pos = base2 + here + __popc(bm & lt);
                __stcs(rd + pos, d);
                rn[pos] = qi;
            }
            here += __popc(bm);
        }
        base2 += here;
        if (lane < L && bk == rank_lt) hist2 = base2;
    }
    if (lane < L) csr.counts[(b * csr.L + lane) * N + i] = hist2;
    const int64_t row_cap = row_off == (int64_t)i * stride ? stride : ((base2 + 3) & ~3);
    if (lane < min((int64_t)((base2 + 3) & ~3), row_cap) - base2) rn[base2 + lane] = -1;
    __syncwarp();
}

// Method 2, short rows (cells of width >= R_max, 3 x 3 cell rows): a warp
// takes kChunk consecutive sorted points (rows).  The points of one grid cell
// are consecutive in sorted order and share one candidate set (the points of
// the 3 x 3 x 3 neighbouring cells), so the warp enumerates the candidates
// once per cell segment of its chunk into a shared-memory window of
// 32 * kSlots (larger sets are reloaded per row in windows) and runs the
// segment's rows against them, kG rows at a time on 32 / kG lanes each:
//   A. f32 screen, lanes = candidates; survivors compacted into shared memory;
//   B. lanes = survivors (dense): exact f64 test, level bucket, rank within
//      the bucket from ballots over the three bucket bits (no atomics);
//   C. scatter to the row at bucket base + rank.
// Rows with more than kEllCap survivors (dense neighbourhoods) are rescanned
// per bucket by the whole warp (ell_rescan_row).  Same row layout, buckets,
// spill and padding as grid_ell_kernel, whose per-row candidate fetch and
// sparse per-hit lanes cost ~950 warp instructions per C3 row (this kernel:
// ~500 at kG = 2).
template <int kEllWarps, int kEllCap, int kSlots, int kChunk, int kMinBlocks, int kG>
__global__ void __launch_bounds__(kEllWarps * 32, kMinBlocks) grid_ell_cell_kernel(
    int64_t B, int64_t N, const double* __restrict__ r2_levels, int L, int64_t levels_ld, int64_t stride, GridWork g,
    ExclWork w, CsrView csr) {
    static_assert(kChunk <= 32, "one row per lane in the chunk prefetch");
    static_assert(kG == 1 || kG == 2 || kG == 4, "rows per warp");
    constexpr int kW = 32 / kG;  // lanes per row (>= 8: one lane per bucket)
    __shared__ float4 sc[kEllWarps][32 * kSlots];    // the cell segment's candidates (window)
    __shared__ float4 sq[kEllWarps][kG][kEllCap];    // f32 survivors of each row (xyz, original index in w)
    __shared__ double hd[kEllWarps][kG][kEllCap];    // their exact d2
    __shared__ uint16_t hb[kEllWarps][kG][kEllCap];  // rank within the bucket
    __shared__ uint8_t hk[kEllWarps][kG][kEllCap];   // bucket; 0xff: not within R_max
    __shared__ double lvs[kEllWarps][32];
    __shared__ unsigned long long lvb[kEllWarps][8];
    __shared__ int tbase[kEllWarps][32];
    __shared__ int tstart[kEllWarps][32];
    __shared__ float4 qs[kEllWarps][kChunk];  // the chunk's points
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane / kW, hl = lane % kW;  // row slot, lane within the row's lanes
    const unsigned hmask = kW == 32 ? kFull : (((1u << kW) - 1u) << (h * kW));
    const unsigned ltw = ((1u << lane) - 1u) & hmask;
    const int64_t b = blockIdx.y;
    const float kInfF = __int_as_float(0x7f800000);
    const double my_r2 = lane < L ? r2_levels[b * levels_ld + lane] : 0.0;
    if (lane < L) lvs[warp][lane] = my_r2;
    int rank_lt_full = 0, rank_st = 0;
    double r2 = 0.0;
    for (int l = 0; l < L; ++l) {
        const double v = __shfl_sync(kFull, my_r2, l);
        rank_lt_full += (v < my_r2) ? 1 : 0;  // lane l: #levels below level l
        rank_st += (v < my_r2 || (v == my_r2 && l < lane)) ? 1 : 0;  // stable sort position
        r2 = fmax(r2, v);
    }
    const int rank_lt = __shfl_sync(kFull, rank_lt_full, hl);  // of level hl
    // L <= 8 levels (launcher), ascending, padded above every d2: a hit is
    // below the largest level, so its bucket #(levels <= d2) is 0 .. 7 --
    // three bits, three steps of a binary search
    if (lane < 8) lvb[warp][lane] = ~0ull;
    __syncwarp();
    if (lane < L) lvb[warp][rank_st] = (unsigned long long)__double_as_longlong(my_r2);
    const float thr = prefilter_threshold(r2);
    const bool no_filter = !(thr <= FLT_MAX);
    const GridParams gp = g.params[b];
    const float4* sx = g.sorted_xyz + b * N;
    const int* cs = g.cell_start + b * (g.max_cells + 1);
    __syncwarp();
    unsigned long long evals = 0;
    for (int64_t s0 = ((int64_t)blockIdx.x * kEllWarps + warp) * kChunk; s0 < N;
         s0 += (int64_t)gridDim.x * kEllWarps * kChunk) {
        const int nq = (int)(N - s0 < kChunk ? N - s0 : kChunk);
        int qc = -1;
        __syncwarp();
        if (lane < nq) {
            const float4 qp = sx[s0 + lane];
            qs[warp][lane] = qp;
            qc = (cell_coord(qp.z, gp.oz, gp.inv_h, gp.nz) * gp.ny + cell_coord(qp.y, gp.oy, gp.inv_h, gp.ny)) *
                     gp.nx + cell_coord(qp.x, gp.ox, gp.inv_h, gp.nx);
        }
        __syncwarp();
        for (int j = 0; j < nq;) {
            // the cell segment [j, jend) of the chunk
            const int c = __shfl_sync(kFull, qc, j);
            const unsigned after = __ballot_sync(kFull, lane < nq && qc != c) & ~((2u << j) - 1u);
            const int jend = after ? __ffs(after) - 1 : nq;
            const int cx = c % gp.nx, cy = (c / gp.nx) % gp.ny, cz = c / (gp.nx * gp.ny);
            int r0 = 0, rlen = 0;
            if (lane < 9) {
                const int z = cz + lane / 3 - 1, y = cy + lane % 3 - 1;
                if (z >= 0 && z < gp.nz && y >= 0 && y < gp.ny) {
                    const int x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < gp.nx ? cx + 1 : gp.nx - 1;
                    const int row = (z * gp.ny + y) * gp.nx;
                    r0 = cs[row + x0];
                    rlen = cs[row + x1 + 1] - r0;
                }
            }
            int incl = rlen;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(kFull, incl, 8);
            const int excl0 = incl - rlen;
            __syncwarp();
            tbase[warp][lane] = r0 - excl0;
            tstart[warp][lane] = lane < 9 ? excl0 : 0x7fffffff;
            __syncwarp();
            // flattened candidate f (< total) -> its point (the 9 ranges are consecutive in f)
            auto cand_at = [&](int f) -> float4 {
                if (f >= total) return make_float4(kInfF, kInfF, kInfF, 0.f);  // screened out (finite thr)
                int rr = 0;
#pragma unroll
                for (int q = 1; q < 9; ++q) rr += (f >= tstart[warp][q]) ? 1 : 0;
                return sx[tbase[warp][rr] + f];
            };
            const bool fits = total <= 32 * kSlots;
            auto load_window = [&](int w0) {
                __syncwarp();
#pragma unroll
                for (int k = 0; k < kSlots; ++k) sc[warp][k * 32 + lane] = cand_at(w0 + k * 32 + lane);
                __syncwarp();
            };
            if (fits) load_window(0);
            // kG rows at a time, kW lanes per row (lane = h * kW + hl): row sj + h
            for (int sj = j; sj < jend; sj += kG) {
                const int myrow = sj + h;
                const float4 p = qs[warp][myrow < jend ? myrow : j];
                const int32_t i = __float_as_int(p.w);  // original index (grid_scatter_kernel)
                // another rank's row, or past the segment: the lanes idle
                const bool act = myrow < jend && i >= csr.row_lo && i < csr.row_hi;
                if (act && hl == 0) evals += (unsigned long long)total;
                // A. f32 screen of the candidates, survivors compacted per row
                int nsv = 0;
                for (int w0 = 0; w0 < total; w0 += 32 * kSlots) {
                    if (!fits) load_window(w0);
                    const int nsl = (min(32 * kSlots, total - w0) + kW - 1) / kW;
#pragma unroll 4
                    for (int k = 0; k < nsl; ++k) {
                        const float4 q = sc[warp][k * kW + hl];
                        const bool sv = act && sqdist_f32(p, q) < thr;
                        const unsigned m = __ballot_sync(kFull, sv) & hmask;
                        const int pos = nsv + __popc(m & ltw);
                        if (sv && pos < kEllCap) sq[warp][h][pos] = q;
                        nsv += __popc(m);
                    }
                }
                __syncwarp();
                // more survivors than the staging holds (dense neighbourhoods) or
                // levels beyond float range (no screen): the whole warp rescans
                // that row afterwards
                const bool ovf = act && (nsv > kEllCap || no_filter);
                const bool dense = act && !ovf;
                const int nmax = __reduce_max_sync(kFull, dense ? nsv : 0);
                // B. dense pass over the survivors: exact test, bucket (#levels <=
                // d2, binary search on the bit patterns of the sorted, padded
                // levels), rank within the bucket from ballots over the three bits
                int runs = 0;  // lane hl < 8 of row h: entries of bucket hl so far
                for (int e0 = 0; e0 < nmax; e0 += kW) {
                    const int ee = e0 + hl;
                    const bool valid = dense && ee < nsv;
                    const double d = sqdist4(p, sq[warp][h][valid ? ee : 0]);
                    const bool hit = valid && d < r2;
                    const unsigned long long db = (unsigned long long)__double_as_longlong(d);
                    const unsigned long long* lv = lvb[warp];
                    int bk = (lv[3] <= db) ? 4 : 0;
                    bk += (lv[bk + 1] <= db) ? 2 : 0;
                    bk += (lv[bk] <= db) ? 1 : 0;
                    const unsigned hm = __ballot_sync(kFull, hit) & hmask;
                    const unsigned m0 = __ballot_sync(kFull, hit && (bk & 1));
                    const unsigned m1 = __ballot_sync(kFull, hit && (bk & 2));
                    const unsigned m2 = __ballot_sync(kFull, hit && (bk & 4));
                    const unsigned peers = hm & ((bk & 1) ? m0 : ~m0) & ((bk & 2) ? m1 : ~m1) & ((bk & 4) ? m2 : ~m2);
                    const unsigned mine = hm & ((hl & 1) ? m0 : ~m0) & ((hl & 2) ? m1 : ~m1) & ((hl & 4) ? m2 : ~m2);
                    const int rank = __shfl_sync(kFull, runs, h * kW + (bk & 7)) + __popc(peers & ltw);
                    runs += __popc(mine);
                    if (valid) {
                        hk[warp][h][ee] = hit ? (uint8_t)bk : (uint8_t)0xff;
                        hb[warp][h][ee] = (uint16_t)rank;
                        hd[warp][h][ee] = d;
                    }
                }
                // bucket bases: exclusive scan of the eight per-bucket totals of the row
                const int v = (hl < 8 && hl <= L) ? runs : 0;
                int hincl = v;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const int y = __shfl_up_sync(kFull, hincl, o, kW);
                    if (hl >= o) hincl += y;
                }
                const int cnt = __shfl_sync(kFull, hincl, h * kW + 7);
                const int hbase = hincl - v;
                // rows longer than the stride: a run of the spill arena (see grid_ell_kernel)
                int64_t row_off = (int64_t)i * stride;
                const bool spill = dense && cnt > stride;
                unsigned long long o = 0;
                if (spill && hl == 0) o = atomicAdd(&w.spill[b], (unsigned long long)((cnt + 3) & ~3));
                o = __shfl_sync(kFull, o, h * kW);
                const int64_t off = N * stride + csr.spill_lo + (int64_t)o;
                const bool fail = spill && off + cnt > N * stride + csr.spill_hi;
                if (fail && hl == 0) atomicOr(&w.status[b], 2);
                if (fail && hl < L) csr.counts[(b * csr.L + hl) * N + i] = 0;
                if (spill && !fail) {
                    row_off = off;
                    if (hl == 0) csr.indptr[b * (N + 1) + i] = off;
                }
                const bool emit = dense && !fail;
                __syncwarp();
                // C. scatter
                int32_t* rn = csr.nbr + b * csr.cap_entries + row_off;
                double* rd = csr.d2 + b * csr.cap_entries + row_off;
                for (int e0 = 0; e0 < nmax; e0 += kW) {
                    const int ee = e0 + hl;
                    const int bk = (emit && ee < nsv) ? hk[warp][h][ee] : 0xff;
                    const int pos = __shfl_sync(kFull, hbase, h * kW + (bk & 7)) + (bk != 0xff ? hb[warp][h][ee] : 0);
                    if (bk != 0xff) {
                        __stcs(rd + pos, hd[warp][h][ee]);  // d2 streams to HBM: keep L2 for the nbr rows
                        rn[pos] = __float_as_int(sq[warp][h][ee].w);
                    }
                }
                // level l = hl holds buckets 0 .. rank_lt(l)
                const int hist = __shfl_sync(kFull, hincl, h * kW + (rank_lt < 7 ? rank_lt : 7));
                if (emit && hl < L) csr.counts[(b * csr.L + hl) * N + i] = hist;
                {
                    // pad the row to a whole 16-byte chunk (readers load int4 chunks, masked by the counts)
                    const int64_t row_cap = row_off == (int64_t)i * stride ? stride : ((cnt + 3) & ~3);
                    if (emit && hl < min((int64_t)((cnt + 3) & ~3), row_cap) - cnt) rn[cnt + hl] = -1;
                }
                __syncwarp();
                // overflowing rows, one at a time by the whole warp
                for (unsigned om = __ballot_sync(kFull, ovf && hl == 0); om; om &= om - 1) {
                    const int r0w = sj + (__ffs(om) - 1) / kW;
                    const float4 pr = qs[warp][r0w];
                    ell_rescan_row(pr, __float_as_int(pr.w), b, N, total, tbase[warp], tstart[warp], sx, r2, thr,
                                   no_filter, L, lvs[warp], rank_lt_full, stride, w, csr);
                }
            }
            j = jend;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(kFull, evals, o);  // rows of every lane group
    if (lane == 0 && evals) atomicAdd(g.evals + b, evals);
}

static cudaError_t launch_sort(CsrView csr, int64_t B, const double* r2_levels, int64_t levels_ld, ExclWork w,
                               cudaStream_t s) {
    excl_sort_small_kernel<<<148 * 8, kSortWarps * 32, 0, s>>>(csr, B, r2_levels, levels_ld, w);
    const size_t dsm = (sizeof(double) + sizeof(int32_t)) * kCtaRowCap;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(excl_sort_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)dsm);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    excl_sort_large_kernel<<<148, 1024, dsm, s>>>(csr, r2_levels, levels_ld, w);
    return cudaGetLastError();
}

// kernels one launch_excl_build issues (for ps_launch_count)
int excl_build_launches(int64_t N, int method) {
    const bool fused = (method == 1 || method == 2) && N <= kGridFusedMaxN && !getenv("PS_GRID_MULTI");
    if (method == 0) return 6;
    if (method == 1) return fused ? 5 : 8;
    return fused ? 2 : 5;
}

cudaError_t launch_excl_build(const float4* xyz, int64_t B, int64_t N, const double* r2_levels, int L,
                              int64_t levels_ld, CsrView csr, ExclWork w, GridWork g, int method, cudaStream_t s) {
    cudaError_t e;
    // method 2 never reads the degrees; the fused grid build (methods 1, 2)
    // zeroes status / long_count itself
    // (one CTA per cloud: wins for small clouds -- C2 cascade 0.488 -> 0.474 ms
    // -- and loses 11 us at C3's 24000 points, where the multi-kernel build
    // spreads assignment and scatter over the whole GPU)
    const bool fused_grid = (method == 1 || method == 2) && N <= kGridFusedMaxN && !getenv("PS_GRID_MULTI");
    if (csr.row_hi <= 0) { csr.row_lo = 0; csr.row_hi = N; }
    if (method == 2 && csr.spill_hi <= 0) {
        csr.spill_lo = 0;
        csr.spill_hi = csr.cap_entries - N * ell_row_stride(csr.cap_entries, N);
    }
    if (method != 2 && (e = cudaMemsetAsync(w.deg, 0, sizeof(int32_t) * B * N, s)) != cudaSuccess) return e;
    if (method == 0) {  // the grid kernels (methods 1, 2) zero these themselves
        if ((e = cudaMemsetAsync(w.long_count, 0, sizeof(unsigned), s)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(w.status, 0, sizeof(int32_t) * B, s)) != cudaSuccess) return e;
    }
    const unsigned gpts = (unsigned)std::min<int64_t>(148 * 16, (B * N + 255) / 256 + 1);
    if (method == 1 || method == 2) {
        const int64_t stride = method == 2 ? ell_row_stride(csr.cap_entries, N) : 0;
        // long rows (stride > 256, e.g. C5's ~270 entries per row in a volume):
        // candidates from cells of width R_max / 2, +-2 cells per axis, rows
        // culled and trimmed to the ball (C5 build 10.2 -> 6.3 ms); shorter rows
        // (surface clouds, C1-C4) keep width R_max and the 3 x 3 cell rows,
        // whose set-up is cheaper than the candidates trimming would save
        // (C3: 267 vs 286 us).  PS_GRID_REACH=1|2 forces either.
        const char* re = getenv("PS_GRID_REACH");
        const int reach = method == 2 ? (re ? (atoi(re) == 1 ? 1 : 2) : (stride > 256 ? 2 : 1)) : 1;
        const bool multi = !fused_grid;
        if (multi) {
            // grid_setup_kernel zeroes the counters and bookkeeping it owns
            grid_setup_kernel<<<(unsigned)B, 1024, 0, s>>>(xyz, N, r2_levels, L, levels_ld, g, w, 1, reach);
            grid_assign_kernel<<<gpts, 256, 0, s>>>(xyz, B, N, g, csr, stride, method == 2 ? 1 : 0);
            grid_scan_kernel<<<(unsigned)B, 1024, 0, s>>>(N, g);
            grid_scatter_kernel<<<gpts, 256, 0, s>>>(xyz, B, N, g);
        } else {
            const size_t dsm = sizeof(int) * (size_t)kGridSmemCells;
            static bool attr = false;
            if (!attr) {
                if ((e = cudaFuncSetAttribute(grid_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)dsm)) != cudaSuccess)
                    return e;
                attr = true;
            }
            grid_build_kernel<<<(unsigned)B, 1024, dsm, s>>>(xyz, N, r2_levels, L, levels_ld, g, w, csr, stride,
                                                             method == 2 ? 1 : 0, reach);
        }
        if (method == 2) {
            if (reach == 1 && L <= 8 && !getenv("PS_ELL_ROW")) {
                // warp per chunk of sorted rows, candidates per cell segment in registers
                // (C3: stage 204 vs 265 us with grid_ell_kernel, PS_ELL_ROW=1)
                constexpr int kWc = 4, kChunk = 16;
                const int64_t gxc = std::max<int64_t>(1, (N + kWc * kChunk - 1) / (kWc * kChunk));
                // two rows per warp, 16 lanes each: the per-row bookkeeping (bucket
                // scan, spill check, counts, padding) serves both rows at once (C3:
                // 97 M vs 119 M instructions with one row per warp, PS_ELL_G=1)
                // 6 CTAs per SM (a 6 x 32-candidate window, 85 registers):
                // C3 stage 201 -> 192 us vs 5 CTAs with an 8 x 32 window
                // (profiles/r02/excl_kernels_ab.log; PS_ELL_V=0: the latter)
                static const int ell_v = getenv("PS_ELL_V") ? atoi(getenv("PS_ELL_V")) : 2;
                if (getenv("PS_ELL_G") && atoi(getenv("PS_ELL_G")) == 1)
                    grid_ell_cell_kernel<kWc, 128, 8, kChunk, 7, 1><<<dim3((unsigned)gxc, (unsigned)B), kWc * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
                else if (ell_v == 2)
                    grid_ell_cell_kernel<kWc, 96, 6, kChunk, 6, 2><<<dim3((unsigned)gxc, (unsigned)B), kWc * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
                else
                    grid_ell_cell_kernel<kWc, 96, 8, kChunk, 5, 2><<<dim3((unsigned)gxc, (unsigned)B), kWc * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
            } else if (reach == 1 && stride <= 256) {
                constexpr int kW = 8;
                const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((148 * 16 + B - 1) / B, (N + kW - 1) / kW));
                grid_ell_kernel<kW, 256, false><<<dim3((unsigned)gx, (unsigned)B), kW * 32, 0, s>>>(
                    B, N, r2_levels, L, levels_ld, stride, g, w, csr);
            } else {
                constexpr int kW = 4;
                const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((148 * 32 + B - 1) / B, (N + kW - 1) / kW));
                if (reach == 2 && L <= 15 && !getenv("PS_ELL_LONG_OLD"))
                    grid_ell_kernel<kW, 512, true, true><<<dim3((unsigned)gx, (unsigned)B), kW * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
                else if (reach == 2)
                    grid_ell_kernel<kW, 512, true><<<dim3((unsigned)gx, (unsigned)B), kW * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
                else
                    grid_ell_kernel<kW, 512, false><<<dim3((unsigned)gx, (unsigned)B), kW * 32, 0, s>>>(
                        B, N, r2_levels, L, levels_ld, stride, g, w, csr);
            }
            return cudaGetLastError();
        }
        const dim3 gp((unsigned)((N + 255) / 256), (unsigned)B);
        (void)gp;
        const unsigned grow = (unsigned)std::min<int64_t>(148 * 16, (B * N + kRowWarps - 1) / kRowWarps);
        grid_rows_kernel<false><<<grow, kRowWarps * 32, 0, s>>>(B, N, r2_levels, L, levels_ld, g, w, csr);
        excl_scan_kernel<<<(unsigned)B, 1024, 0, s>>>(N, w, csr, 0);
        grid_rows_kernel<true><<<grow, kRowWarps * 32, 0, s>>>(B, N, r2_levels, L, levels_ld, g, w, csr);
        const size_t dsm = (sizeof(double) + sizeof(int32_t)) * kCtaRowCap;
        static bool attr_set2 = false;
        if (!attr_set2) {
            e = cudaFuncSetAttribute(excl_sort_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
            if (e != cudaSuccess) return e;
            attr_set2 = true;
        }
        excl_sort_large_kernel<<<148, 1024, dsm, s>>>(csr, r2_levels, levels_ld, w);
        return cudaGetLastError();
    }
    if ((e = cudaMemsetAsync(w.edge_count, 0, sizeof(unsigned long long) * B, s)) != cudaSuccess) return e;
    const int64_t nt = (N + kTile - 1) / kTile;
    const int64_t npairs = nt * (nt + 1) / 2;
    excl_pairs_kernel<<<dim3((unsigned)npairs, (unsigned)B), kPairThreads, 0, s>>>(xyz, N, r2_levels, L,
                                                                                 levels_ld, w);
    const unsigned g1 = (unsigned)std::min<int64_t>(148 * 8, (w.cap_edges + 255) / 256 + 1);
    excl_degree_kernel<<<dim3(g1, (unsigned)B), 256, 0, s>>>(N, w);
    excl_scan_kernel<<<(unsigned)B, 1024, 0, s>>>(N, w, csr, 1);
    const unsigned g2 = (unsigned)std::min<int64_t>(148 * 8, (w.cap_edges + N + 255) / 256 + 1);
    excl_fill_kernel<<<dim3(g2, (unsigned)B), 256, 0, s>>>(N, w, csr);
    return launch_sort(csr, B, r2_levels, levels_ld, w, s);
}

cudaError_t launch_sort_rows(CsrView csr, int64_t B, ExclWork w, cudaStream_t s) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(w.long_count, 0, sizeof(unsigned), s)) != cudaSuccess) return e;
    csr.L = 0;
    excl_sort_small_kernel<<<148 * 8, kSortWarps * 32, 0, s>>>(csr, B, nullptr, 0, w);
    const size_t dsm = (sizeof(double) + sizeof(int32_t)) * kCtaRowCap;
    e = cudaFuncSetAttribute(excl_sort_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
    if (e != cudaSuccess) return e;
    excl_sort_large_kernel<<<148, 1024, dsm, s>>>(csr, nullptr, 0, w);
    return cudaGetLastError();
}

cudaError_t launch_level_counts(CsrView csr, int64_t B, const double* r2_levels, int64_t levels_ld,
                                cudaStream_t s) {
    const unsigned g = (unsigned)std::min<int64_t>(148 * 8, (B * csr.N + 255) / 256 + 1);
    level_counts_kernel<<<g, 256, 0, s>>>(csr, B, r2_levels, levels_ld);
    return cudaGetLastError();
}

}  // namespace ps
