// sampler.cu -- K2 (curve estimate -> thresholds), K3c (predicted-distance
// bitmap sampler) and K3d (early-termination min-distance seeding).
//
// K2 restates the SPEC.md curve/segmentation stage (
// pinned in oracle/oracle.py): a = sequential-sum mean of v_i * i**e over the
// measured prefix, tail a / i**e with a running minimum from the last
// measured value, radii R_s = est[min(floor(n s / nseg), n-1)] with a running
// minimum, R <= 0 -> 5e-324, r2 = max(R*R, 5e-324).  Divisions are IEEE
// (__ddiv_rn) and min is exact, so the parallel evaluation is bit-identical
// to the sequential oracle.
//
// K3c (the sampler, _kernels.py:241-353) lives in sampler_v4.cu.
//
// K3d replaces _kernels.earlyterm_scan (_kernels.py:356-367).

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ps_internal.h"
#include "sampler.h"

namespace ps {

namespace {

constexpr double kTiny = 4.9406564584124654e-324;


// ---------------------------------------------------------------------------
// K2: thresholds

// pinned linear resampling (curve.resample_curve, oracle.resample_pinned)
PS_DEV double resample_at(const double* v, int64_t S, int64_t T, int64_t t) {
    if (T == 1) return v[0];
    const double u = __ddiv_rn(__dmul_rn((double)t, (double)(S - 1)), (double)(T - 1));
    const int64_t i0 = (int64_t)floor(u);
    if (i0 >= S - 1) return v[S - 1];
    const double frac = __dsub_rn(u, (double)i0);
    return __dadd_rn(v[i0], __dmul_rn(frac, __dsub_rn(v[i0 + 1], v[i0])));
}

// one MLP neuron: input-order dot product from 0.0, bias last, optional relu
PS_DEV double mlp_neuron(const double* __restrict__ W, const double* __restrict__ bias, const double* x, int nin,
                         int j, bool relu) {
    double acc = 0.0;
    const double* row = W + (int64_t)j * nin;
    for (int i = 0; i < nin; ++i) acc = __dadd_rn(acc, __dmul_rn(row[i], x[i]));
    acc = __dadd_rn(acc, bias[j]);
    return relu ? (acc > 0.0 ? acc : 0.0) : acc;
}

// order-preserving key of any non-NaN double (for atomicMin)
PS_DEV unsigned long long dkey(double d) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
PS_DEV double dunkey(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

__global__ void __launch_bounds__(1024) thresholds_kernel(ThreshArgs a) {
    __shared__ unsigned long long seg_min[kMaxSeg];
    __shared__ double s_a;
    const int64_t b = blockIdx.x;
    const double* v = a.prefix_curve + b * a.curve_ld;  // measured prefix (k0 values)
    const int64_t k0 = a.k0, n = a.n;
    const int nseg = a.nseg;
    if (threadIdx.x < kMaxSeg) seg_min[threadIdx.x] = 0x7ff0000000000000ull;  // +inf bits
    if (a.mode == 0) {
        // products v_i * i**e in parallel (exact per element), then one
        // thread adds them in index order -- the oracle's sequential sum
        __shared__ double prod[1024];
        double s = 0.0;
        for (int64_t c0 = 1; c0 < k0; c0 += 1024) {
            const int64_t i = c0 + threadIdx.x;
            if (i < k0) prod[threadIdx.x] = __dmul_rn(v[i], a.pow_tab[i]);
            __syncthreads();
            if (threadIdx.x == 0) {
                const int m = (int)((k0 - c0) < 1024 ? (k0 - c0) : 1024);
                for (int j = 0; j < m; ++j) s = __dadd_rn(s, prod[j]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) s_a = __ddiv_rn(s, (double)(k0 - 1));
    }
    __syncthreads();
    double est_d[kMaxSeg];
    if (a.mode == 0) {
        const double amp = s_a;
        // min over tail positions i in [k0, d_s] for every s (prefix-min by
        // segment): each thread takes a contiguous run of positions, keeps a
        // running min per segment and publishes it once per segment it
        // touches (a few shared atomics per thread instead of one per
        // position; min is order-free, so the result is unchanged)
        const int64_t per = (n - k0 + blockDim.x - 1) / blockDim.x;
        const int64_t i0 = k0 + (int64_t)threadIdx.x * per;
        const int64_t i1 = i0 + per < n ? i0 + per : n;
        int s = 0;
        while (s < nseg && a.d[s] < i0) ++s;
        unsigned long long run = 0x7ff0000000000000ull;
        for (int64_t i = i0; i < i1 && s < nseg; ++i) {
            if (a.d[s] < i) {
                atomicMin(&seg_min[s], run);
                run = 0x7ff0000000000000ull;
                while (s < nseg && a.d[s] < i) ++s;
                if (s >= nseg) break;
            }
            const unsigned long long t = (unsigned long long)__double_as_longlong(__ddiv_rn(amp, a.pow_tab[i]));
            run = t < run ? t : run;
        }
        if (s < nseg && i0 < i1) atomicMin(&seg_min[s], run);
        __syncthreads();
        if (threadIdx.x == 0) {
            double run = v[k0 - 1];
            // running min over the tail in order of position; segments partition it
            for (int s = 0; s < nseg; ++s) {
                if (a.d[s] < k0) {
                    est_d[s] = v[a.d[s]];
                } else {
                    const double m = __longlong_as_double((long long)seg_min[s]);
                    if (m < run) run = m;
                    est_d[s] = run;
                }
            }
        }
    } else if (a.mode == 2) {
        // MLP estimator: prefix 1..k0-1 -> 32 values / v[k0-1]
        // -> 32-128-128-64 relu MLP -> * v[k0-1] -> resampled to the n-k0 tail
        // positions -> running minimum from v[k0-1] (pinned in curve.py / oracle)
        __shared__ double xs[32], h1[128], h2[128], ys[64];
        const double* W1 = a.mlp;
        const double* b1 = W1 + 128 * 32;
        const double* W2 = b1 + 128;
        const double* b2 = W2 + 128 * 128;
        const double* W3 = b2 + 128;
        const double* b3 = W3 + 64 * 128;
        const int64_t S = k0 - 1;
        const double scale = v[k0 - 1];
        const bool ok = scale > 0.0 && S >= 2;  // else the tail is 0 (degenerate, R -> tiny)
        if (threadIdx.x < 32) xs[threadIdx.x] = ok ? __ddiv_rn(resample_at(v + 1, S, 32, threadIdx.x), scale) : 0.0;
        __syncthreads();
        if (threadIdx.x < 128) h1[threadIdx.x] = mlp_neuron(W1, b1, xs, 32, threadIdx.x, true);
        __syncthreads();
        if (threadIdx.x < 128) h2[threadIdx.x] = mlp_neuron(W2, b2, h1, 128, threadIdx.x, true);
        __syncthreads();
        if (threadIdx.x < 64) ys[threadIdx.x] = ok ? __dmul_rn(mlp_neuron(W3, b3, h2, 128, threadIdx.x, false), scale)
                                                   : 0.0;
        if (threadIdx.x < kMaxSeg) seg_min[threadIdx.x] = dkey(__longlong_as_double(0x7ff0000000000000LL));
        __syncthreads();
        for (int64_t i = k0 + threadIdx.x; i < n; i += blockDim.x) {
            const double t = resample_at(ys, 64, n - k0, i - k0);
            int s = 0;
            while (s < nseg && a.d[s] < i) ++s;
            if (s < nseg) atomicMin(&seg_min[s], dkey(t));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double run = v[k0 - 1];
            for (int s = 0; s < nseg; ++s) {
                if (a.d[s] < k0) {
                    est_d[s] = v[a.d[s]];
                } else {
                    const double m = dunkey(seg_min[s]);
                    if (m < run) run = m;
                    est_d[s] = run;
                }
            }
        }
    } else {
        if (threadIdx.x == 0) {
            const double* c = a.given_curve + b * a.given_ld;
            for (int s = 0; s < nseg; ++s) est_d[s] = a.d[s] < k0 ? v[a.d[s]] : c[a.d[s]];
        }
    }
    if (threadIdx.x == 0) {
        double run = __longlong_as_double(0x7ff0000000000000LL);
        double* R = a.R_out + b * nseg;
        double* lv = a.r2_levels + b * a.levels_ld;
        for (int s = 0; s < nseg; ++s) {
            if (est_d[s] < run) run = est_d[s];
            R[s] = run;
            const double rc = run > 0.0 ? run : kTiny;
            const double r2 = __dmul_rn(rc, rc);
            lv[s] = r2 > kTiny ? r2 : kTiny;
        }
        for (int e = 0; e < a.n_extra; ++e) lv[nseg + e] = a.extra_r2[e];
    }
}

// ---------------------------------------------------------------------------
// K3d: early termination

__global__ void et_prepare_kernel(EtArgs a) {
    const int64_t total = a.B * a.N;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / a.N;
        if (a.reached[b] >= a.n_total) continue;
        a.taken[g] = 0;
        const int64_t i = g - b * a.N;
        if (a.md_hi == 0 || (i >= a.md_lo && i < a.md_hi)) a.md[g] = __longlong_as_double(0x7ff0000000000000LL);
    }
}

__global__ void et_mark_kernel(EtArgs a) {
    const int64_t total = a.B * a.n_total;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / a.n_total, t = g - b * a.n_total;
        const int64_t r = a.reached[b];
        if (r >= a.n_total || t >= r) continue;
        a.taken[b * a.N + a.out_idx[b * a.ld_out + t]] = 1;
    }
}

// Push form of the early-termination seeding: every sampled point q walks its
// own level-1 row prefix and lowers md[j] to d2(q, j) for each entry j.  By
// the symmetry of the rows (j in row_1(q) <=> q in row_1(j), same d2), this is
// exactly earlyterm_scan's min over taken row entries of every point, but reads
// only the sampled points' rows (reached of N).  md >= 0, so the min is an
// unsigned atomicMin on the bit patterns (order-independent, exact).
// Lane groups of 8 per row.
__global__ void et_push_kernel(EtArgs a) {
    const int gl = threadIdx.x & 7;
    const int64_t total = a.B * a.n_total;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 3;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; g < total; g += ng) {
        const int64_t b = g / a.n_total, t = g - b * a.n_total;
        if (a.reached[b] >= a.n_total || t >= a.reached[b]) continue;
        const int64_t q = a.out_idx[b * a.ld_out + t];
        if (gl == 0) a.taken[b * a.N + q] = 1;  // et_mark's job, fused (push never reads taken)
        const int64_t base = a.indptr[b * (a.N + 1) + q];
        const int32_t c = a.lvl1_counts[b * a.counts_stride + q];
        const int32_t* nbr = a.nbr + b * a.cap_entries + base;
        const double* d2 = a.d2 + b * a.cap_entries + base;
        unsigned long long* md = reinterpret_cast<unsigned long long*>(a.md + b * a.N);
        // four entries per lane in flight: the loads of a batch are issued
        // before its reductions (the row reads are the latency)
        for (int32_t u0 = gl; u0 < c; u0 += 32) {
            int32_t j[4];
            double d[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t u = u0 + 8 * k;
                j[k] = u < c ? __ldg(nbr + u) : -1;
                d[k] = u < c ? __ldg(d2 + u) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (j[k] >= 0) atomicMin(md + j[k], (unsigned long long)__double_as_longlong(d[k]));
        }
    }
}

}  // namespace

// md[i] = min(md[i], min over the first lvl1[i] row entries j with taken[j] of d2)
// Warp per row: coalesced entry loads, exact min (order-independent).
__global__ void et_scan_kernel(EtScanArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t span = a.hi - a.lo;
    const int64_t total = a.B * span;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < total; g += nw) {
        const int64_t b = g / span;
        if (a.reached && a.reached[b] >= a.n_total) continue;
        const int64_t i = a.lo + (g - b * span);
        const int64_t base = a.indptr[b * (a.N + 1) + i];
        const int32_t c = a.lvl1_counts[b * a.counts_stride + i];
        const int32_t* nbr = a.nbr + b * a.cap_entries + base;
        const double* d2 = a.d2 + b * a.cap_entries + base;
        const uint8_t* tk = a.taken + b * a.N;
        double best = __longlong_as_double(0x7ff0000000000000LL);
        for (int32_t u = lane; u < c; u += 32) {
            const int32_t j = nbr[u];
            if (tk[j]) {
                const double d = d2[u];
                if (d < best) best = d;
            }
        }
        // warp min of non-negative doubles via their bit patterns
        const unsigned long long bits = (unsigned long long)__double_as_longlong(best);
        const uint32_t hi = (uint32_t)(bits >> 32);
        const uint32_t mhi = __reduce_min_sync(kFull, hi);
        const uint32_t mlo = __reduce_min_sync(kFull, hi == mhi ? (uint32_t)bits : 0xffffffffu);
        if (lane == 0) {
            const double wmin = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
            double* mp = a.md + b * a.N + i;
            if (wmin < *mp) *mp = wmin;
        }
    }
}

cudaError_t launch_thresholds(const ThreshArgs& a, int64_t B, cudaStream_t s) {
    thresholds_kernel<<<(unsigned)B, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

// kernels one launch_et issues (for ps_launch_count): reset + push (which also
// marks the sampled points), or reset + mark + pull scan
int et_launches() { return getenv("PS_ET_PULL") ? 3 : 2; }

cudaError_t launch_et(const EtArgs& a, cudaStream_t s) {
    const unsigned g1 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.N + 255) / 256 + 1);
    et_prepare_kernel<<<g1, 256, 0, s>>>(a);
    const unsigned g2 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.n_total + 255) / 256 + 1);
    if (!getenv("PS_ET_PULL")) {
        const unsigned g3 = (unsigned)std::min<int64_t>(148 * 16, (a.B * a.n_total + 31) / 32 + 1);
        et_push_kernel<<<g3, 256, 0, s>>>(a);
        return cudaGetLastError();
    }
    et_mark_kernel<<<g2, 256, 0, s>>>(a);
    EtScanArgs sa;
    sa.indptr = a.indptr; sa.nbr = a.nbr; sa.d2 = a.d2; sa.cap_entries = a.cap_entries;
    sa.lvl1_counts = a.lvl1_counts; sa.counts_stride = a.counts_stride;
    sa.taken = a.taken; sa.md = a.md; sa.reached = a.reached; sa.n_total = a.n_total;
    sa.B = a.B; sa.N = a.N; sa.lo = 0; sa.hi = a.N;
    const unsigned g3 = (unsigned)std::min<int64_t>(148 * 16, (a.B * a.N + 7) / 8 + 1);
    et_scan_kernel<<<g3, 256, 0, s>>>(sa);
    return cudaGetLastError();
}

// One rank of a point split: taken from the whole sample prefix, md reset
// and pulled for the rank's points [lo, hi) only -- the rows it holds.
cudaError_t launch_et_shard(const EtArgs& a_in, int64_t lo, int64_t hi, cudaStream_t s) {
    EtArgs a = a_in;
    a.md_lo = lo;  // md of the other ranks' points is theirs (virtual ranks share the buffer)
    a.md_hi = hi;
    const unsigned g1 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.N + 255) / 256 + 1);
    et_prepare_kernel<<<g1, 256, 0, s>>>(a);
    const unsigned g2 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.n_total + 255) / 256 + 1);
    et_mark_kernel<<<g2, 256, 0, s>>>(a);
    EtScanArgs sa;
    sa.indptr = a.indptr; sa.nbr = a.nbr; sa.d2 = a.d2; sa.cap_entries = a.cap_entries;
    sa.lvl1_counts = a.lvl1_counts; sa.counts_stride = a.counts_stride;
    sa.taken = a.taken; sa.md = a.md; sa.reached = a.reached; sa.n_total = a.n_total;
    sa.B = a.B; sa.N = a.N; sa.lo = lo; sa.hi = hi;
    const unsigned g3 = (unsigned)std::min<int64_t>(148 * 16, (a.B * (hi - lo) + 7) / 8 + 1);
    et_scan_kernel<<<g3, 256, 0, s>>>(sa);
    return cudaGetLastError();
}

cudaError_t launch_et_scan(const EtScanArgs& a, cudaStream_t s) {
    const unsigned g = (unsigned)std::min<int64_t>(148 * 16, (a.B * (a.hi - a.lo) + 7) / 8 + 1);
    et_scan_kernel<<<g, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ps
