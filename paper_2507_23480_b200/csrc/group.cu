// group.cu -- K4 grouping (ball query / kNN, naive and redundancy-free) and
// K6 minimum sample spacing.
//
// Semantics follow SPEC.md:483-521 / 563-571 as pinned in oracle/oracle.py:
// strict "d2 < r2" radius test, neighbours ordered by (d2, index), nearest
// first cap at k, distances reported as IEEE sqrt(d2) in float64, padding
// index -1 / distance NaN.
//
//   K4a bq_rf      reads the first min(count_R[c], k) entries of the
//                  centroid's distance-sorted exclusion row -- zero new
//                  distance evaluations.
//   K4b knn_rf     level-1 row entries of the query that are sampled, in row
//                  order; exact brute-force fallback when fewer than k
//                  (SPEC.md:513-521).
//   K4c bq_naive   warp per centroid streams the cloud (L2-resident float4),
//                  float32 pre-filter + exact float64 test, warp-parallel
//                  sorted insertion into a per-warp top-k list.
//   K4d knn_naive  thread per query, pool tiles in shared memory, top-k kept
//                  in registers.
//   K6 spacing     thread per sample, nearest other sample (float64).

#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "group.h"

namespace ps {

namespace {

PS_DEV bool kless(double da, int32_t ia, double db, int32_t ib) {
    return da < db || (da == db && ia < ib);
}

PS_DEV double nan_d() { return __longlong_as_double(0x7ff8000000000000LL); }

// ---- K4a -----------------------------------------------------------------
// Warp per centroid.  The level-r entries are a row prefix of length c (a set:
// the hot-path rows are level-bucketed, the reference-layout rows sorted);
// the first min(c, k) in (d2, index) order are produced here -- in registers
// for c <= 64, by a streaming warp top-k insertion otherwise.
constexpr int kBqWarps = 8;
constexpr int kBqMaxK = 128;

// sorted top-K list (per warp, shared memory): insert (dn, jn) if it ranks < K
PS_DEV void topk_warp_insert(double* ld, int32_t* li, int& len, int K, double dn, int32_t jn, int lane) {
    int below = 0;
    for (int s = lane; s < len; s += 32) below += key_less(ld[s], li[s], dn, jn) ? 1 : 0;
    const int pos = __reduce_add_sync(kFull, below);
    if (pos >= K) return;
    const int newlen = len < K ? len + 1 : K;
    double cd[kBqMaxK / 32];
    int32_t ci[kBqMaxK / 32];
#pragma unroll
    for (int v = 0; v < kBqMaxK / 32; ++v) {
        const int s = lane + 32 * v;
        if (s > pos && s < newlen) { cd[v] = ld[s - 1]; ci[v] = li[s - 1]; }
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < kBqMaxK / 32; ++v) {
        const int s = lane + 32 * v;
        if (s > pos && s < newlen) { ld[s] = cd[v]; li[s] = ci[v]; }
    }
    if (lane == 0) { ld[pos] = dn; li[pos] = jn; }
    __syncwarp();
    len = newlen;
}

// one centroid g by the whole warp (any row length)
PS_DEV void bq_rf_one(const BqArgs& a, int64_t g, double* ld, int32_t* li, int lane) {
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const int K = a.k;
    const int64_t b = g / a.n, t = g - b * a.n;
    const int64_t c = a.centroids[b * a.cent_ld + t];
    int32_t* oi = a.idx_out + g * K;
    double* od = a.dist_out + g * K;
    if (c < 0 || c >= a.N || (a.status && a.status[b] != 0)) {
        // no valid row (invalid centroid, or the cloud's build failed): error state
        for (int s = lane; s < K; s += 32) { oi[s] = -1; od[s] = nan_d(); }
        if (lane == 0) a.cnt_out[g] = -1;
        return;
    }
    const int32_t cnt0 = a.counts[(b * a.L + a.level) * a.N + c];
    const int64_t base = b * a.cap_entries + a.indptr[b * (a.N + 1) + c];
    const int m = cnt0 < K ? cnt0 : K;
    // Only the k nearest are reported, and every level is a row prefix: the
    // shortest level prefix holding >= k of the query level's entries holds
    // the k nearest (the k-th nearest lies below that level's radius) -- rank
    // that prefix instead of the whole query level (C5: ~270 -> ~40 entries).
    int32_t cnt = cnt0;
    if (cnt0 > K) {
        uint32_t cl = 0xffffffffu;
        if (lane < a.L) {
            const int32_t v = a.counts[(b * a.L + lane) * a.N + c];
            if (v >= K && v <= cnt0) cl = (uint32_t)v;
        }
        cl = __reduce_min_sync(kFull, cl);
        if (cl < (uint32_t)cnt0) cnt = (int32_t)cl;
    }
    if (cnt <= 64) {
        double d0 = lane < cnt ? a.d2[base + lane] : kInf;
        int32_t i0 = lane < cnt ? a.nbr[base + lane] : 0x7fffffff;
        double d1 = lane + 32 < cnt ? a.d2[base + lane + 32] : kInf;
        int32_t i1 = lane + 32 < cnt ? a.nbr[base + lane + 32] : 0x7fffffff;
        int n2 = 2;
        while (n2 < cnt) n2 <<= 1;
        if (cnt > 1) warp_bitonic64(d0, i0, d1, i1, lane, n2);
        for (int s = lane; s < K; s += 32) {
            const double d = s < 32 ? d0 : d1;  // valid for s < 64 only
            const int32_t ix = s < 32 ? i0 : i1;
            if (s < m) { oi[s] = ix; od[s] = sqrt(d); }
            else { oi[s] = -1; od[s] = nan_d(); }
        }
    } else {
        int len = 0;
        for (int64_t u0 = 0; u0 < cnt; u0 += 32) {
            const int64_t u = u0 + lane;
            const double dv = u < cnt ? a.d2[base + u] : kInf;
            const int32_t jv = u < cnt ? a.nbr[base + u] : 0x7fffffff;
            const int nval = (int)((cnt - u0) < 32 ? (cnt - u0) : 32);
            for (int q = 0; q < nval; ++q)
                topk_warp_insert(ld, li, len, K, __shfl_sync(kFull, dv, q), __shfl_sync(kFull, jv, q), lane);
        }
        for (int s = lane; s < K; s += 32) {
            if (s < len) { oi[s] = li[s]; od[s] = sqrt(ld[s]); }
            else { oi[s] = -1; od[s] = nan_d(); }
        }
        __syncwarp();
    }
    if (lane == 0) a.cnt_out[g] = m;
}

// warp per centroid (PS_BQ_RF_WARP=1)
__global__ void __launch_bounds__(kBqWarps * 32) bq_rf_kernel(BqArgs a) {
    __shared__ double ld[kBqWarps][kBqMaxK];
    __shared__ int32_t li[kBqWarps][kBqMaxK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * kBqWarps;
    for (int64_t g = blockIdx.x * (int64_t)kBqWarps + warp; g < a.B * a.n; g += nw)
        bq_rf_one(a, g, ld[warp], li[warp], lane);
}

// Two centroids per warp, 16 lanes each (hot path): a level-r prefix of at
// most 16 entries (99.97 % of the C3 centroids at r = 0.1) is sorted by a
// 16-lane bitonic network in registers and written with the padding by the
// same 16 lanes; longer prefixes are answered afterwards by the whole warp
// (bq_rf_one).  Halves the per-centroid address set-up, loads and output
// bookkeeping of the warp-per-centroid kernel.
__global__ void __launch_bounds__(kBqWarps * 32) bq_rf2_kernel(BqArgs a) {
    __shared__ double ld[kBqWarps][kBqMaxK];
    __shared__ int32_t li[kBqWarps][kBqMaxK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, hl = lane & 15;
    const int64_t nw = (int64_t)gridDim.x * kBqWarps;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const int K = a.k;
    const int64_t G = a.B * a.n;
    for (int64_t g0 = (blockIdx.x * (int64_t)kBqWarps + warp) * 2; g0 < G; g0 += nw * 2) {
        const int64_t g = g0 + h;
        bool fast = false;
        int32_t cnt = 0;
        int64_t base = 0;
        if (g < G) {
            const int64_t b = g / a.n, t = g - b * a.n;
            const int64_t c = a.centroids[b * a.cent_ld + t];
            if (c >= 0 && c < a.N && !(a.status && a.status[b] != 0)) {
                cnt = a.counts[(b * a.L + a.level) * a.N + c];
                base = b * a.cap_entries + a.indptr[b * (a.N + 1) + c];
                fast = cnt <= 16;
            }
        }
        double d = fast && hl < cnt ? a.d2[base + hl] : kInf;
        int32_t ix = fast && hl < cnt ? a.nbr[base + hl] : 0x7fffffff;
        // bitonic sort of the 16 lanes by (d2, index), ascending
#pragma unroll
        for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const double od = __shfl_xor_sync(kFull, d, j, 16);
                const int32_t oi = __shfl_xor_sync(kFull, ix, j, 16);
                const bool take_min = ((hl & k) == 0) == ((hl & j) == 0);
                const bool o_less = key_less(od, oi, d, ix);
                if (take_min ? o_less : !o_less && !(od == d && oi == ix)) { d = od; ix = oi; }
            }
        }
        if (fast) {
            const int m = cnt < K ? cnt : K;
            int32_t* oi = a.idx_out + g * K;
            double* od = a.dist_out + g * K;
            for (int s = hl; s < K; s += 16) {
                if (s < m) { oi[s] = ix; od[s] = sqrt(d); }  // s < m <= 16: lane s holds rank s
                else { oi[s] = -1; od[s] = nan_d(); }
            }
            if (hl == 0) a.cnt_out[g] = m;
        }
        // error rows and long prefixes: the whole warp, one centroid at a time
        for (unsigned sl = __ballot_sync(kFull, !fast && g < G && hl == 0); sl; sl &= sl - 1)
            bq_rf_one(a, g0 + (__ffs(sl) - 1) / 16, ld[warp], li[warp], lane);
    }
}

// ---- K4c -----------------------------------------------------------------

__global__ void __launch_bounds__(kBqWarps * 32) bq_naive_kernel(BqArgs a) {
    __shared__ double ld[kBqWarps][kBqMaxK];
    __shared__ int32_t li[kBqWarps][kBqMaxK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * kBqWarps;
    const float thr = prefilter_threshold(a.r2);
    const bool no_filter = !(thr <= FLT_MAX);
    const int K = a.k;
    for (int64_t g = blockIdx.x * (int64_t)kBqWarps + warp; g < a.B * a.n; g += nw) {
        const int64_t b = g / a.n, t = g - b * a.n;
        const float4* xyz = a.xyz + b * a.N;
        const int64_t c = a.centroids[b * a.cent_ld + t];
        const float4 pc = xyz[c];
        int len = 0;
        for (int64_t j0 = 0; j0 < a.N; j0 += 32) {
            const int64_t j = j0 + lane;
            bool hit = false;
            double d = 0.0;
            if (j < a.N) {
                const float4 pj = xyz[j];
                if (no_filter || sqdist_f32(pc, pj) < thr) {
                    d = sqdist4(pc, pj);
                    hit = d < a.r2;
                }
            }
            uint32_t hits = __ballot_sync(kFull, hit);
            while (hits) {
                const int src = __ffs(hits) - 1;
                hits &= hits - 1;
                const double dn = __shfl_sync(kFull, d, src);
                const int32_t jn = (int32_t)(j0 + src);
                // position = #entries with (d2, idx) < new; existing indices are smaller
                int below = 0;
                for (int s = lane; s < len; s += 32) below += (ld[warp][s] <= dn) ? 1 : 0;
                const int pos = __reduce_add_sync(kFull, below);
                if (pos >= K) continue;
                const int newlen = len < K ? len + 1 : K;
                // shift [pos, newlen-1) up by one
                double carry_d[kBqMaxK / 32];
                int32_t carry_i[kBqMaxK / 32];
#pragma unroll
                for (int v = 0; v < kBqMaxK / 32; ++v) {
                    const int s = lane + 32 * v;
                    if (s > pos && s < newlen) { carry_d[v] = ld[warp][s - 1]; carry_i[v] = li[warp][s - 1]; }
                }
                __syncwarp();
#pragma unroll
                for (int v = 0; v < kBqMaxK / 32; ++v) {
                    const int s = lane + 32 * v;
                    if (s > pos && s < newlen) { ld[warp][s] = carry_d[v]; li[warp][s] = carry_i[v]; }
                }
                if (lane == 0) { ld[warp][pos] = dn; li[warp][pos] = jn; }
                __syncwarp();
                len = newlen;
            }
        }
        int32_t* oi = a.idx_out + g * K;
        double* od = a.dist_out + g * K;
        for (int s = lane; s < K; s += 32) {
            if (s < len) { oi[s] = li[warp][s]; od[s] = sqrt(ld[warp][s]); }
            else { oi[s] = -1; od[s] = nan_d(); }
        }
        if (lane == 0) a.cnt_out[g] = len;
        __syncwarp();
    }
}

// ---- K4d / K4b fallback: top-k in registers ---------------------------------
constexpr int kKnnMaxK = 16;

struct TopK {
    double d[kKnnMaxK];
    int32_t i[kKnnMaxK];
};

PS_DEV void topk_init(TopK& tk) {
#pragma unroll
    for (int s = 0; s < kKnnMaxK; ++s) { tk.d[s] = __longlong_as_double(0x7ff0000000000000LL); tk.i[s] = 0x7fffffff; }
}

PS_DEV void topk_insert(TopK& tk, int k, double d, int32_t j) {
    if (!kless(d, j, tk.d[k - 1], tk.i[k - 1])) return;
#pragma unroll
    for (int s = kKnnMaxK - 1; s > 0; --s) {
        if (s < k) {
            const bool shift = kless(d, j, tk.d[s - 1], tk.i[s - 1]);
            const bool here = !shift && kless(d, j, tk.d[s], tk.i[s]);
            if (shift) { tk.d[s] = tk.d[s - 1]; tk.i[s] = tk.i[s - 1]; }
            else if (here) { tk.d[s] = d; tk.i[s] = j; }
        }
    }
    if (kless(d, j, tk.d[0], tk.i[0])) { tk.d[0] = d; tk.i[0] = j; }
}

constexpr int kKnnThreads = 256;
constexpr int kKnnTile = 1024;

__global__ void __launch_bounds__(kKnnThreads) knn_naive_kernel(KnnArgs a) {
    __shared__ float4 tp[kKnnTile];
    __shared__ int32_t ti[kKnnTile];
    const int64_t b = blockIdx.y;
    const float4* xyz = a.xyz + b * a.N;
    const int64_t q = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    const bool active = q < a.nq;
    const int64_t qp = active ? (a.queries ? a.queries[b * a.q_ld + q] : q) : 0;
    const float4 pq = xyz[qp];
    TopK tk;
    topk_init(tk);
    const int k = a.k;
    for (int64_t p0 = 0; p0 < a.npool; p0 += kKnnTile) {
        __syncthreads();
        for (int s = threadIdx.x; s < kKnnTile; s += kKnnThreads) {
            const int64_t p = p0 + s;
            if (p < a.npool) {
                const int64_t j = a.pool[b * a.pool_ld + p];
                ti[s] = (int32_t)j;
                tp[s] = xyz[j];
            }
        }
        __syncthreads();
        const int m = (int)((a.npool - p0) < kKnnTile ? (a.npool - p0) : kKnnTile);
        if (active)
            for (int s = 0; s < m; ++s) topk_insert(tk, k, sqdist4(pq, tp[s]), ti[s]);
    }
    if (!active) return;
    const int64_t g = b * a.nq + q;
    const int take = (int)(a.npool < k ? a.npool : k);
#pragma unroll
    for (int s = 0; s < kKnnMaxK; ++s) {
        if (s < k) {
            a.idx_out[g * k + s] = s < take ? tk.i[s] : -1;
            a.dist_out[g * k + s] = s < take ? sqrt(tk.d[s]) : nan_d();
        }
    }
    a.cnt_out[g] = take;
}

__global__ void __launch_bounds__(kKnnThreads) knn_rf_kernel(KnnArgs a) {
    const int64_t b = blockIdx.y;
    const int64_t q = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    if (q >= a.nq) return;
    const int64_t qp = a.queries ? a.queries[b * a.q_ld + q] : q;
    const int k = a.k;
    const int64_t g = b * a.nq + q;
    if (qp < 0 || qp >= a.N || (a.status && a.status[b] != 0)) {
        for (int s = 0; s < k; ++s) { a.idx_out[g * k + s] = -1; a.dist_out[g * k + s] = nan_d(); }
        a.cnt_out[g] = -1;
        return;
    }
    const int64_t base = b * a.cap_entries + a.indptr[b * (a.N + 1) + qp];
    const int32_t c = a.lvl1_counts[b * a.counts_stride + qp];
    const uint8_t* smp = a.sampled + b * a.N;
    // the k nearest sampled points of the level-1 prefix (a set), by (d2, index)
    TopK tk;
    topk_init(tk);
    int found = 0;
    for (int32_t u = 0; u < c; ++u) {
        const int32_t j = a.nbr[base + u];
        if (smp[j]) {
            topk_insert(tk, k, a.d2[base + u], j);
            ++found;
        }
    }
    if (found < k) {
        // fallback: exact brute force over the whole pool
        atomicAdd(a.fallback_count + b, 1);
        const float4* xyz = a.xyz + b * a.N;
        const float4 pq = xyz[qp];
        topk_init(tk);
        for (int64_t p = 0; p < a.npool; ++p) {
            const int64_t j = a.pool[b * a.pool_ld + p];
            topk_insert(tk, k, sqdist4(pq, xyz[j]), (int32_t)j);
        }
        found = (int)(a.npool < k ? a.npool : k);
    }
    const int take = found < k ? found : k;
#pragma unroll
    for (int s = 0; s < kKnnMaxK; ++s) {
        if (s < k) {
            a.idx_out[g * k + s] = s < take ? tk.i[s] : -1;
            a.dist_out[g * k + s] = s < take ? sqrt(tk.d[s]) : nan_d();
        }
    }
    a.cnt_out[g] = take;
}

// ---- K6 ------------------------------------------------------------------
__global__ void __launch_bounds__(kKnnThreads) min_spacing_kernel(SpacingArgs a) {
    __shared__ float4 tp[kKnnTile];
    const int64_t b = blockIdx.y;
    const float4* xyz = a.xyz + b * a.N;
    const int64_t s = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    const bool active = s < a.n;
    const float4 ps_ = xyz[active ? a.samples[b * a.ld + s] : a.samples[b * a.ld]];
    double best = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t p0 = 0; p0 < a.n; p0 += kKnnTile) {
        __syncthreads();
        for (int t = threadIdx.x; t < kKnnTile; t += kKnnThreads)
            if (p0 + t < a.n) tp[t] = xyz[a.samples[b * a.ld + p0 + t]];
        __syncthreads();
        const int m = (int)((a.n - p0) < kKnnTile ? (a.n - p0) : kKnnTile);
        if (active)
            for (int t = 0; t < m; ++t) {
                if (p0 + t == s) continue;
                const double d = sqdist4(ps_, tp[t]);
                if (d < best) best = d;
            }
    }
    if (active) a.out_d2[b * a.n + s] = best;
}

}  // namespace

cudaError_t launch_bq_rf(const BqArgs& a, cudaStream_t s) {
    if (a.k < 1 || a.k > kBqMaxK) return cudaErrorInvalidValue;  // per-warp top-k lists hold kBqMaxK
    if (getenv("PS_BQ_RF_WARP")) {
        const unsigned g = (unsigned)std::min<int64_t>(148 * 16, (a.B * a.n + 7) / 8 + 1);
        bq_rf_kernel<<<g, 256, 0, s>>>(a);
    } else {
        const unsigned g = (unsigned)std::min<int64_t>(148 * 16, (a.B * a.n + 15) / 16 + 1);
        bq_rf2_kernel<<<g, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_bq_naive(const BqArgs& a, cudaStream_t s) {
    if (a.k > kBqMaxK) return cudaErrorInvalidValue;
    const unsigned g = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.n + kBqWarps - 1) / kBqWarps + 1);
    bq_naive_kernel<<<g, kBqWarps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_knn_naive(const KnnArgs& a, cudaStream_t s) {
    if (a.k > kKnnMaxK || a.k < 1) return cudaErrorInvalidValue;
    dim3 g((unsigned)((a.nq + kKnnThreads - 1) / kKnnThreads), (unsigned)a.B);
    knn_naive_kernel<<<g, kKnnThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_knn_rf(const KnnArgs& a, cudaStream_t s) {
    if (a.k > kKnnMaxK || a.k < 1) return cudaErrorInvalidValue;
    dim3 g((unsigned)((a.nq + kKnnThreads - 1) / kKnnThreads), (unsigned)a.B);
    knn_rf_kernel<<<g, kKnnThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_min_spacing(const SpacingArgs& a, cudaStream_t s) {
    dim3 g((unsigned)((a.n + kKnnThreads - 1) / kKnnThreads), (unsigned)a.B);
    min_spacing_kernel<<<g, kKnnThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ps
