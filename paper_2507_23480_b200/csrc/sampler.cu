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
// K3c replaces _kernels.sample_predicted (_kernels.py:241-353).  The
// reference's random pick is a swap-remove from the segment pool with
// position z_k mod (L - k), z_k = splitmix64(state + (k+1) * GOLDEN): the
// candidate order of a segment does not depend on the bitmaps, and a
// candidate is accepted iff no earlier accepted candidate of the segment lies
// in its level-s exclusion row (rows are symmetric).  One CTA per cloud
// therefore processes each segment in chunks of 1024 draws:
//   * positions for the chunk in parallel (u64 splitmix + modulo);
//   * the swap chain itself (one thread, shared memory);
//   * greedy maximal independent set over the chunk in parallel rounds
//     (a candidate is IN when every earlier neighbour in the chunk is OUT,
//     OUT when an earlier neighbour is IN) -- identical to the serial greedy;
//   * truncation at the segment boundary (draws consumed = last used
//     accept + 1, which fixes the RNG state), parallel bitmap clears.
// Bit-packed bitmaps, pool and rank tables live in shared memory when they
// fit (N <= ~30k) and in an L2-resident global workspace otherwise.
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

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr double kTiny = 4.9406564584124654e-324;

PS_DEV uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// K2: thresholds

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
        // min over tail positions i in [k0, d_s] for every s (prefix-min by segment)
        for (int64_t i = k0 + threadIdx.x; i < n; i += blockDim.x) {
            const double t = __ddiv_rn(amp, a.pow_tab[i]);
            int s = 0;
            while (s < nseg && a.d[s] < i) ++s;
            if (s < nseg) atomicMin(&seg_min[s], (unsigned long long)__double_as_longlong(t));
        }
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
// K3c: sampler

constexpr int kSampThreads = 1024;
constexpr uint8_t kUndecided = 0, kIn = 1, kOut = 2;
constexpr uint16_t kNoRank = 0xffffu;
constexpr uint16_t kAcceptedMark = 0xfffeu;  // accepted earlier in the current segment

struct SampCtl {
    int64_t i;
    int64_t seg_i0;     // out[] position where the current segment visit started
    int seg;
    int entered;
    int exhausted;
    int done;
    uint64_t state;
    int64_t pool_len;
    int undecided;
    int accepted;
};

// block-wide exclusive scan of one int per thread; returns (exclusive, total)
PS_DEV int block_excl_scan(int v, int* warp_tot, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s;
    }
    __syncthreads();
    const int excl = (warp ? warp_tot[warp - 1] : 0) + x - v;
    *total = warp_tot[31];
    __syncthreads();
    return excl;
}

constexpr int kMaxPred = 8;
constexpr uint8_t kPredOverflow = 0xff;

struct SampView {
    uint32_t* bm;      // [nseg][W] availability bits per segment
    int32_t* pool;     // [N] segment pool (swap-remove array)
    uint16_t* rank;    // [N] draw rank within the current chunk (0xffff = none)
};


PS_DEV void build_pool(const SampView& v, int seg, int64_t W, SampCtl* ctl, int* warp_tot) {
    const uint32_t* row = v.bm + (int64_t)seg * W;
    int64_t carry = 0;
    for (int64_t base = 0; base < W; base += blockDim.x) {
        const int64_t w = base + threadIdx.x;
        const uint32_t word = w < W ? row[w] : 0u;
        int tot;
        const int ex = block_excl_scan(__popc(word), warp_tot, &tot);
        int64_t p = carry + ex;
        uint32_t x = word;
        while (x) {
            const int bit = __ffs(x) - 1;
            x &= x - 1;
            v.pool[p++] = (int32_t)(w * 32 + bit);
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        ctl->pool_len = carry;
        ctl->seg_i0 = ctl->i;
    }
    __syncthreads();
}

// Clear point p (and its level-l row prefix) in the bitmaps of levels
// [l0, nseg).  `nl` cooperating lanes (sub-lane sl).  Level counts are loaded
// in parallel and the row prefix is read once for the widest level (radii
// are non-increasing in s, so count(l0) >= count(l) for l > l0).  `base` is
// the row offset (indptr[p]) when the caller prefetched it, else -1.
PS_DEV void clear_point_levels(const SampView& v, const SampArgs& a, int64_t b, int64_t W, int32_t p, int l0,
                               int sl, int nl, int64_t base = -1) {
    const int64_t N = a.N;
    const int nseg = a.nseg;
    if (base < 0) base = a.indptr[b * (N + 1) + p];
    const int32_t* nbr = a.nbr + b * a.cap_entries + base;
    const uint32_t pbit = ~(1u << (p & 31));
    for (int lb = l0; lb < nseg; lb += 8) {
        int c[8];
#pragma unroll
        for (int l = 0; l < 8; ++l)
            c[l] = (lb + l < nseg) ? a.counts[(b * a.L + a.seg_level_rows[lb + l]) * N + p] : 0;
        const int cmax = c[0];
#pragma unroll 2
        for (int u = sl; u < cmax; u += nl) {
            const int32_t q = __ldg(nbr + u);
            const uint32_t bit = ~(1u << (q & 31));
            uint32_t* w = v.bm + (int64_t)lb * W + (q >> 5);
#pragma unroll
            for (int l = 0; l < 8; ++l)
                if (u < c[l]) atomicAnd(w + (int64_t)l * W, bit);
        }
        if (sl == 0)
            for (int l = lb; l < nseg; ++l) atomicAnd(&v.bm[(int64_t)l * W + (p >> 5)], pbit);
    }
}

// ---- producer / consumer split -------------------------------------------
// Warp 0 produces the candidate order (positions + swap-remove chain) for the
// next chunk while warps 1..31 decide the current one, so the serial chain is
// off the critical path.  Hand-off through two chunk buffers, volatile
// counters in shared memory, and named barrier 1 among the 992 consumers.
constexpr int kConsThreads = kSampThreads - 32;

PS_DEV void cons_bar() { asm volatile("bar.sync 1, 992;" ::: "memory"); }

PS_DEV int vload(const int* p) { return *(volatile const int*)p; }
PS_DEV void vstore(int* p, int v) { *(volatile int*)p = v; }

// exclusive scan of one int per consumer thread (ct in [0, 992))
PS_DEV int cons_excl_scan(int v, int* warp_tot, int* total) {
    const int lane = threadIdx.x & 31, cw = (threadIdx.x >> 5) - 1;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[cw] = x;
    cons_bar();
    if (cw == 0) {
        int s = lane < 31 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s;
    }
    cons_bar();
    const int ex = (cw ? warp_tot[cw - 1] : 0) + x - v;
    *total = warp_tot[30];
    cons_bar();
    return ex;
}

// Candidate order for draws k .. k+K-1 (pool length before draw t is L - t):
// position z_t mod (L - t) with z_t = splitmix64(state0 + (t+1) GOLDEN)
// (precomputed in parallel by the consumers, draw_position), then the
// swap-remove of _kernels.py:325-330.  Groups of up to 32 consecutive
// draws run in parallel up to the first draw whose read locations an earlier
// draw of the group writes (same position, or its last slot); positions of
// the unexecuted draws carry over to the next group.
PS_DEV uint32_t draw_position(uint64_t state0, int64_t L, int64_t t) {
    const uint64_t z = mix64(state0 + (uint64_t)(t + 1) * kGolden);
    return (uint32_t)(z % (uint64_t)(L - t));
}

PS_DEV void produce_chunk(int32_t* pool, int32_t* cand, const uint32_t* pos, int64_t L, int64_t k, int K,
                          int lane, bool pick_lowest) {
    if (pick_lowest) {
        for (int t = lane; t < K; t += 32) cand[t] = pool[k + t];
        __syncwarp();
        return;
    }
    const unsigned lt = (1u << lane) - 1u;
    int g = 0;
    int have = 0;  // lanes [0, have) hold valid positions for draws g .. g+have-1
    uint32_t p = 0;
    while (g < K) {
        if (lane >= have && g + lane < K) p = pos[g + lane];
        const bool act = g + lane < K;
        const uint32_t key = act ? p : (0x80000000u | (uint32_t)lane);
        const int64_t last0 = L - 1 - (k + g);
        const int64_t last = last0 - lane;
        const unsigned same = __match_any_sync(kFull, key);
        bool conflict = act && (same & lt) != 0;
        unsigned mark = 0;
        if (act) {
            const int64_t j = last0 - (int64_t)p;
            if (j > lane && j < 32) mark = 1u << (int)j;
        }
        mark = __reduce_or_sync(kFull, mark);
        conflict = conflict || ((mark >> lane) & 1u);
        const unsigned cmask = __ballot_sync(kFull, conflict);
        const int run = cmask ? (__ffs(cmask) - 1) : 32;
        const int nrun = min(run, K - g);
        int32_t vp = 0, vl = 0;
        if (lane < nrun) {
            vp = pool[p];
            vl = pool[last];
        }
        __syncwarp();
        if (lane < nrun) {
            pool[p] = vl;
            cand[g + lane] = vp;
        }
        __syncwarp();
        p = __shfl_down_sync(kFull, p, nrun & 31);
        have = 32 - nrun;
        g += nrun;
    }
}

// End of a segment visit: the points accepted in it (out[seg_i0, i)) clear
// their rows in the bitmaps of every later segment, in one parallel batch,
// and leave the rank table.  (Bitmap `seg` itself is never read again.)
PS_DEV void end_visit(const SampView& v, const SampArgs& a, int64_t b, int64_t W, int seg, const int64_t* out,
                      int64_t i0, int64_t i1, int32_t* stage) {
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (seg + 1 < a.nseg) {
        const int sub = lane >> 3, sl = lane & 7;
        for (int64_t x0 = i0; x0 < i1; x0 += 2 * kConsThreads) {
            const int64_t xn = (i1 - x0) < 2 * kConsThreads ? (i1 - x0) : 2 * kConsThreads;
            // stage (point, row base) pairs: one latency for the whole batch
            for (int64_t x = threadIdx.x; x < xn; x += blockDim.x) {
                const int32_t p = (int32_t)out[x0 + x];
                stage[2 * x] = p;
                stage[2 * x + 1] = (int32_t)a.indptr[b * (a.N + 1) + p];
            }
            __syncthreads();
            for (int64_t x = (int64_t)warp * 4 + sub; x < xn; x += (int64_t)nwarps * 4)
                clear_point_levels(v, a, b, W, stage[2 * x], seg + 1, sl, 8, stage[2 * x + 1]);
            __syncthreads();
        }
    }
    for (int64_t x = i0 + threadIdx.x; x < i1; x += blockDim.x) v.rank[out[x]] = kNoRank;
    __syncthreads();
}

__global__ void __launch_bounds__(kSampThreads, 1) sampler_kernel(SampArgs a) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ SampCtl ctl;
    __shared__ int warp_tot[32];
    __shared__ int32_t cbuf[2][kConsThreads];
    __shared__ uint32_t posbuf[2][kConsThreads];
    __shared__ uint16_t preds[kConsThreads][kMaxPred];
    __shared__ uint8_t st[kConsThreads];
    __shared__ uint8_t npred[kConsThreads];
    __shared__ int prod_count, cons_count, stop_flag, visit_exhausted;
    const int64_t b = blockIdx.x;
    const int64_t N = a.N;
    const int64_t W = (N + 31) >> 5;
    const int nseg = a.nseg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int ct = tid - 32;  // consumer thread index (warps 1..31)

    // big tables: shared memory when they fit, else this cloud's global slice
    unsigned char* ws = a.use_smem ? dyn : (a.gws + b * a.gws_stride);
    SampView v;
    {
        size_t off = 0;
        v.bm = reinterpret_cast<uint32_t*>(ws + off); off += sizeof(uint32_t) * nseg * W;
        off = (off + 15) & ~size_t(15);
        v.pool = reinterpret_cast<int32_t*>(ws + off); off += sizeof(int32_t) * N;
        v.rank = reinterpret_cast<uint16_t*>(ws + off);
    }
    int64_t* out = a.out_idx + b * a.ld_out;
    const int64_t k0 = a.k0, n_total = a.n_total;
    // development timing (PS_SAMPLER_TIMING): cycles per phase, cloud 0, first consumer
    const bool tdbg = a.dbg && b == 0 && tid == 32;
    __shared__ long long tacc[10];
    if (tdbg)
        for (int k2 = 0; k2 < 10; ++k2) tacc[k2] = 0;
    long long tlast = tdbg ? clock64() : 0;
#define PS_TMARK(k)                                  \
    do {                                             \
        if (tdbg) {                                  \
            const long long _n = clock64();          \
            tacc[k] += _n - tlast;                   \
            tlast = _n;                              \
        }                                            \
    } while (0)

    // ---- init: all bits set (valid points), rank table empty --------------
    for (int64_t w = tid; w < (int64_t)nseg * W; w += blockDim.x) {
        const int64_t ww = w % W;
        const int64_t nb = N - ww * 32;
        v.bm[w] = nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u));
    }
    for (int64_t j = tid; j < N; j += blockDim.x) v.rank[j] = kNoRank;
    if (tid == 0) {
        ctl.state = a.state_io[b];
        ctl.done = 0;
        ctl.exhausted = 0;
        ctl.entered = 0;
    }
    __syncthreads();
    // pre-clear every prefix point's rows at all levels (_kernels.py:273-276)
    {
        const int sub = lane >> 3, sl = lane & 7;
        for (int64_t t = (int64_t)warp * 4 + sub; t < k0; t += (int64_t)nwarps * 4)
            clear_point_levels(v, a, b, W, (int32_t)out[t], 0, sl, 8);
    }
    for (int64_t t = k0 + tid; t < n_total; t += blockDim.x) out[t] = -1;
    __syncthreads();

    if (tid == 0) {
        int seg = 0;
        while (seg < nseg && k0 >= a.boundaries[seg]) ++seg;
        ctl.i = k0;
        ctl.seg = seg;
        if (seg >= nseg) {
            ctl.done = 1;
            ctl.exhausted = 1;
        } else {
            ctl.entered = 1;
        }
    }
    __syncthreads();
    if (!ctl.done) build_pool(v, ctl.seg, W, &ctl, warp_tot);
    PS_TMARK(0);

    // ---- main loop: one iteration per segment visit ----------------------
    while (!ctl.done) {
        if (ctl.i >= n_total) break;
        if (ctl.i >= a.boundaries[ctl.seg]) {
            __syncthreads();
            if (tid == 0) {
                int seg = ctl.seg;
                while (ctl.i >= a.boundaries[seg]) ++seg;
                ctl.seg = seg;
                ctl.entered += 1;
            }
            __syncthreads();
            build_pool(v, ctl.seg, W, &ctl, warp_tot);
        }
        PS_TMARK(1);
        const int seg = ctl.seg;
        const int64_t L = ctl.pool_len;
        const uint64_t state0 = ctl.state;
        const int lvl = a.seg_level_rows[seg];
        const int32_t* cnt_row = a.counts + (b * a.L + lvl) * N;
        const int64_t* indptr = a.indptr + b * (N + 1);
        const int32_t* nbr_all = a.nbr + b * a.cap_entries;
        if (tid == 0) {
            prod_count = 0;
            cons_count = 0;
            stop_flag = 0;
            visit_exhausted = 0;
        }
        if (!a.pick_lowest)
            for (int t = tid; t < 2 * kConsThreads; t += blockDim.x)
                if (t < L) posbuf[t / kConsThreads][t % kConsThreads] = draw_position(state0, L, t);
        __syncthreads();

        if (warp == 0) {
            // ---------------- producer ----------------
            for (int c = 0;; ++c) {
                const int64_t kc = (int64_t)c * kConsThreads;
                if (kc >= L) break;
                // buffer c&1 is free once chunk c-2 was released
                while (vload(&cons_count) < c - 1 && !vload(&stop_flag)) __nanosleep(32);
                if (vload(&stop_flag)) break;
                const int K = (int)((L - kc) < kConsThreads ? (L - kc) : kConsThreads);
                produce_chunk(v.pool, cbuf[c & 1], posbuf[c & 1], L, kc, K, lane, a.pick_lowest != 0);
                __threadfence_block();
                if (lane == 0) vstore(&prod_count, c + 1);
            }
        } else {
            // ---------------- consumers ----------------
            for (int c = 0;; ++c) {
                const int64_t kc = (int64_t)c * kConsThreads;
                if (kc >= L) {
                    // pool exhausted: the picked < 0 path of _kernels.py:335-347
                    if (ct == 0) { vstore(&visit_exhausted, 1); vstore(&stop_flag, 1); }
                    break;
                }
                const int K = (int)((L - kc) < kConsThreads ? (L - kc) : kConsThreads);
                if (ct == 0)
                    while (vload(&prod_count) <= c) __nanosleep(20);
                cons_bar();
                __threadfence_block();
                PS_TMARK(3);
                const int32_t* cand = cbuf[c & 1];
                const int32_t cme = ct < K ? cand[ct] : 0;
                if (ct < K) {
                    st[ct] = kUndecided;
                    v.rank[cme] = (uint16_t)ct;
                }
                if (ct == 0) ctl.undecided = 0;
                cons_bar();
                // every consumer holds its candidate in a register now: refill the
                // position buffer with chunk c+2 and release both buffers of chunk c
                if (!a.pick_lowest) {
                    const int64_t t2 = kc + 2 * kConsThreads + ct;
                    if (t2 < L) posbuf[c & 1][ct] = draw_position(state0, L, t2);
                    __threadfence_block();
                    cons_bar();
                }
                if (ct == 0) vstore(&cons_count, c + 1);
                PS_TMARK(4);
                // greedy MIS, round 0: one pass over the level-seg row
                int und = 0;
                if (ct < K) {
                    const int t = ct;
                    const int32_t m = cnt_row[cme];
                    const int32_t* row = nbr_all + indptr[cme];
                    // aligned 16-byte loads over [row, row + m): 16 entries per batch
                    const uintptr_t ua = reinterpret_cast<uintptr_t>(row);
                    const int4* ap = reinterpret_cast<const int4*>(ua & ~uintptr_t(15));
                    const int skip = (int)((ua & 15) >> 2);
                    int np = 0;
                    bool out_ = false, blocked = false;
                    for (int e0 = -skip; e0 < m; e0 += 16) {
                        int4 qv[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            qv[j] = (e0 + 4 * j < m) ? __ldg(ap + (e0 + skip) / 4 + j) : make_int4(cme, cme, cme, cme);
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int e = e0 + j;
                            const int4 w4 = qv[j >> 2];
                            const int32_t qq = (j & 3) == 0 ? w4.x : (j & 3) == 1 ? w4.y : (j & 3) == 2 ? w4.z : w4.w;
                            const int32_t qj = (e >= 0 && e < m) ? qq : cme;
                            const uint32_t rq = v.rank[qj];
                            if (rq == kAcceptedMark) {
                                out_ = true;
                            } else if (rq < (uint32_t)t) {
                                // OUT is final and never matters; IN rejects; UNDECIDED is remembered
                                const uint8_t sq = st[rq];
                                if (sq == kIn) {
                                    out_ = true;
                                } else if (sq == kUndecided) {
                                    if (np < kMaxPred) preds[t][np] = (uint16_t)rq;
                                    ++np;
                                    blocked = true;
                                }
                            }
                        }
                    }
                    npred[t] = np > kMaxPred ? kPredOverflow : (uint8_t)np;
                    if (out_) st[t] = kOut;
                    else if (!blocked) st[t] = kIn;
                    else und = 1;
                }
                und = __reduce_add_sync(kFull, und);
                if (lane == 0 && und) atomicAdd(&ctl.undecided, und);
                cons_bar();
                PS_TMARK(5);
                // later rounds over the short predecessor lists
                while (ctl.undecided != 0) {
                    cons_bar();
                    if (ct == 0) ctl.undecided = 0;
                    cons_bar();
                    int u2 = 0;
                    if (ct < K && st[ct] == kUndecided) {
                        const int t = ct;
                        bool out_ = false, blocked = false;
                        const uint8_t np = npred[t];
                        if (np != kPredOverflow) {
                            for (int j = 0; j < np; ++j) {
                                const uint8_t sq = st[preds[t][j]];
                                if (sq == kIn) { out_ = true; break; }
                                if (sq == kUndecided) blocked = true;
                            }
                        } else {
                            const int32_t m = cnt_row[cme];
                            const int32_t* row = nbr_all + indptr[cme];
                            for (int32_t u = 0; u < m; ++u) {
                                const uint32_t rq = v.rank[row[u]];
                                if (rq == kAcceptedMark) { out_ = true; break; }
                                if (rq < (uint32_t)t) {
                                    const uint8_t sq = st[rq];
                                    if (sq == kIn) { out_ = true; break; }
                                    if (sq == kUndecided) blocked = true;
                                }
                            }
                        }
                        if (out_) st[t] = kOut;
                        else if (!blocked) st[t] = kIn;
                        else u2 = 1;
                    }
                    u2 = __reduce_add_sync(kFull, u2);
                    if (lane == 0 && u2) atomicAdd(&ctl.undecided, u2);
                    cons_bar();
                }
                PS_TMARK(6);
                // ordered compaction of accepted candidates
                const int64_t i0 = ctl.i;
                const int64_t need = a.boundaries[seg] - i0;
                const int flag = (ct < K && st[ct] == kIn) ? 1 : 0;
                int tot;
                const int ex = cons_excl_scan(flag, warp_tot, &tot);
                const int64_t take = (int64_t)tot < need ? (int64_t)tot : need;
                const bool ends = (take == need);
                if (flag && ex < take) {
                    out[i0 + ex] = cme;
                    if (ex == take - 1 && ends) ctl.accepted = ct;  // draw of the last used accept
                }
                if (ct < K) v.rank[cme] = kNoRank;
                cons_bar();
                if (!ends)
                    for (int64_t x = ct; x < take; x += kConsThreads) v.rank[out[i0 + x]] = kAcceptedMark;
                if (ct == 0) {
                    ctl.i = i0 + take;
                    if (ends && !a.pick_lowest) ctl.state = state0 + (uint64_t)(kc + ctl.accepted + 1) * kGolden;
                    if (ends) vstore(&stop_flag, 1);
                }
                cons_bar();
                PS_TMARK(7);
                if (tdbg) tacc[9] += 1;
                if (ends) break;
            }
        }
        __syncthreads();
        end_visit(v, a, b, W, seg, out, ctl.seg_i0, ctl.i, reinterpret_cast<int32_t*>(preds));
        PS_TMARK(8);
        if (tid == 0 && visit_exhausted) {
            if (!a.pick_lowest) ctl.state = state0 + (uint64_t)L * kGolden;
            ctl.seg += 1;
            if (ctl.seg >= nseg) {
                ctl.exhausted = 1;
                ctl.done = 1;
            } else {
                ctl.entered += 1;
            }
        }
        __syncthreads();
        if (!ctl.done && visit_exhausted) build_pool(v, ctl.seg, W, &ctl, warp_tot);
    }
    __syncthreads();
    if (tdbg)
        for (int k2 = 0; k2 < 10; ++k2) a.dbg[k2] = tacc[k2];
#undef PS_TMARK
    if (tid == 0) {
        a.reached[b] = ctl.i;
        a.exhausted[b] = ctl.exhausted;
        a.entered[b] = ctl.entered;
        a.state_io[b] = ctl.state;
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
        a.md[g] = __longlong_as_double(0x7ff0000000000000LL);
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

size_t sampler_ws_bytes(int64_t N, int nseg) {
    const int64_t W = (N + 31) >> 5;
    size_t off = sizeof(uint32_t) * nseg * W;
    off = (off + 15) & ~size_t(15);
    off += sizeof(int32_t) * N + sizeof(uint16_t) * N;
    return (off + 255) & ~size_t(255);
}

cudaError_t launch_thresholds(const ThreshArgs& a, int64_t B, cudaStream_t s) {
    thresholds_kernel<<<(unsigned)B, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sampler(SampArgs a, int64_t B, cudaStream_t s) {
    a.dbg = nullptr;
    static long long* dbg = nullptr;
    const bool timing = getenv("PS_SAMPLER_TIMING") != nullptr;
    if (timing) {
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 16);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 16, s);
        a.dbg = dbg;
    }
    const size_t need = sampler_ws_bytes(a.N, a.nseg);
    size_t dsm = 0;
    if (a.use_smem) {
        dsm = need;
        cudaError_t e = cudaFuncSetAttribute(sampler_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
        if (e != cudaSuccess) return e;
    }
    sampler_kernel<<<(unsigned)B, kSampThreads, dsm, s>>>(a);
    if (timing) {
        long long h[16];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "[sampler timing] cycles: init+preclear %lld pool %lld - wait_producer %lld rank %lld "
                "mis0 %lld mis_rounds %lld compact %lld end_visit %lld chunks %lld\n", h[0], h[1], h[3], h[4],
                h[5], h[6], h[7], h[8], h[9]);
    }
    return cudaGetLastError();
}

cudaError_t launch_et(const EtArgs& a, cudaStream_t s) {
    const unsigned g1 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.N + 255) / 256 + 1);
    et_prepare_kernel<<<g1, 256, 0, s>>>(a);
    const unsigned g2 = (unsigned)std::min<int64_t>(148 * 8, (a.B * a.n_total + 255) / 256 + 1);
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

cudaError_t launch_et_scan(const EtScanArgs& a, cudaStream_t s) {
    const unsigned g = (unsigned)std::min<int64_t>(148 * 16, (a.B * (a.hi - a.lo) + 7) / 8 + 1);
    et_scan_kernel<<<g, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ps
