// sampler_v4.cu -- K3c: the predicted-distance bitmap sampler
// (_kernels.py:241-353, sample_predicted) as ONE persistent kernel: a
// thread-block cluster of C CTAs per cloud walks all segment visits, with
// cluster barriers between the phases of a visit and the cloud's working
// arrays in global memory (L2-resident, a few MB for a batch).
//
// Reformulation (bit-exact with the reference):
//   * bitmap of segment s at its entry == "no sampled point within the
//     level-s radius": rebuilt per visit by clearing the level-s row prefix
//     of every sampled point (prefix + accepted) -- the reference's
//     _clear_entries of all earlier picks, in one pass of ~N stores;
//   * the pool is the available points in index order (_kernels.py:293-298);
//   * the candidate order of the whole visit is the swap-remove sequence of
//     _kernels.py:322-333 with positions z_t mod (L - t),
//     z_t = splitmix64(state + (t+1) G); it does not depend on acceptance, so
//     all L draws are resolved at once: per-position writer lists
//     (atomicExch), the latest earlier writer of a draw's position and of its
//     tail slot, then the moved-value chains;
//   * acceptance in draw order == greedy maximal independent set of the
//     level-s graph on the pool in that order: parallel rounds (IN when every
//     earlier neighbour is OUT, OUT when one is IN) until all are decided;
//   * truncation: the first `boundary - i` accepts in draw order are taken;
//     draws consumed = position of the last one + 1, or L when the pool runs
//     dry (RNG state = state0 + draws * G);
//   * segment / entered / exhausted bookkeeping of _kernels.py:303-351,
//     evaluated identically by every thread.

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ps_internal.h"
#include "sampler.h"

namespace ps {

namespace {

constexpr uint64_t kGolden4 = 0x9E3779B97F4A7C15ull;
constexpr int kT4 = 512;
constexpr int kW4 = kT4 / 32;
constexpr int kAdj4 = 64;
constexpr uint8_t kAdjOvf = 0xff;
constexpr int kPred4 = 32;
constexpr uint8_t kPredOvf = 0xff;
constexpr uint8_t kUnd4 = 0, kIn4 = 1, kOut4 = 2;
constexpr int kScr = 64;  // int32 scratch per cloud
constexpr int kMaxC4 = 16;
// Grid mode (one or a few huge clouds, C4 / C5): the CTAs of a cloud are a
// slice of one cooperative grid of up to kMaxCG CTAs instead of a cluster;
// their barrier is a global arrive counter + generation word and the
// per-round decided counts go through global slots.
constexpr int kMaxCG = 160;
// scratch slots: cluster mode in kScr ints, grid mode in kScrG ints
template <bool kGrid>
struct Scr {
    enum : int {
        cnt0 = 0,                               // per-CTA available counts (pool)
        cnt1 = kGrid ? kMaxCG : 16,             // per-CTA accepted counts (truncation)
        decided = kGrid ? 2 * kMaxCG : 32,
        last = decided + 1,
        dec = decided + 2,                      // grid: [2][kMaxCG] cumulative decided counts
        bar = dec + 2 * kMaxCG,                 // grid: barrier {count, generation}
        size = kGrid ? bar + 2 : kScr
    };
};
constexpr int kScrG = Scr<true>::size;

struct V4Work {
    uint8_t* avail;    // [B][N]
    int32_t* pool;     // [B][N]
    uint32_t* pos;     // [B][N]
    int32_t* head;     // [B][N]
    int32_t* nxt;      // [B][N]
    int32_t* prv;      // [B][N]
    int32_t* lw;       // [B][N]
    int32_t* cand;     // [B][N]
    int32_t* rank;     // [B][N]
    int32_t* adj;      // [B][N][kAdj4]
    uint8_t* adjcnt;   // [B][N]
    uint8_t* st;       // [B][N]
    int32_t* preds;    // [B][N][kPred4]
    uint8_t* npred;    // [B][N]
    int32_t* scr;      // [B][kScr]
    int32_t* gscr;     // [B][kScrG] (grid mode)
};

PS_DEV uint64_t mix64_4(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

PS_DEV uint8_t ld_st(const uint8_t* p) {
    uint16_t v;
    asm volatile("ld.relaxed.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return (uint8_t)v;
}
PS_DEV void st_st(uint8_t* p, uint8_t v) {
    asm volatile("st.relaxed.gpu.global.u8 [%0], %1;" ::"l"(p), "h"((uint16_t)v) : "memory");
}

constexpr int kRB = 8;  // row entries loaded per batch (independent loads in flight)

// Load up to kRB row entries [u0, u0 + kRB) of a row with c entries; missing
// entries are -1.
PS_DEV void row_batch(const int32_t* row, int32_t u0, int32_t c, int32_t (&q)[kRB]) {
#pragma unroll
    for (int k = 0; k < kRB; ++k) q[k] = (u0 + k < c) ? __ldg(row + u0 + k) : -1;
}

// Lane groups of kG lanes scan one row each: lane gl of the group covers
// entries [u0 + 4 gl, u0 + 4 gl + 4) (one 16-byte load when the row is
// 16-byte aligned -- the ELL layout -- else four scalar loads); a warp thus
// touches 32/kG rows per step instead of 32 scattered lines per load.
constexpr int kG = 4;
constexpr int kGStep = 4 * kG;
PS_DEV int4 grp_load4(const int32_t* row, int32_t u, int32_t c, bool aligned) {
    int4 v = make_int4(-1, -1, -1, -1);
    if (u < c) {
        if (aligned) {
            v = __ldg(reinterpret_cast<const int4*>(row + u));
        } else {
            v.x = __ldg(row + u);
            if (u + 1 < c) v.y = __ldg(row + u + 1);
            if (u + 2 < c) v.z = __ldg(row + u + 2);
            if (u + 3 < c) v.w = __ldg(row + u + 3);
        }
        if (u + 1 >= c) v.y = -1;
        if (u + 2 >= c) v.z = -1;
        if (u + 3 >= c) v.w = -1;
    }
    return v;
}

// exclusive block scan (kT4 threads); *total = block sum
PS_DEV int bscan(int v, int* wt, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int s = lane < kW4 ? wt[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        wt[lane] = s;
    }
    __syncthreads();
    const int ex = (warp ? wt[warp - 1] : 0) + x - v;
    *total = wt[31];
    __syncthreads();
    return ex;
}

PS_DEV int bsum(int v, int* wt) {
    int tot;
    bscan(v, wt, &tot);
    return tot;
}

PS_DEV uint4 ld_cluster_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// relaxed cluster-scope state accesses (the MIS dataflow polls them)
PS_DEV uint8_t ld_shared_u8_rlx(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.relaxed.cluster.shared::cta.u8 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
    return (uint8_t)v;
}
PS_DEV void st_cluster_u8_rlx(uint32_t addr, uint8_t v) {
    asm volatile("st.relaxed.cluster.shared::cluster.u8 [%0], %1;" ::"r"(addr), "h"((uint16_t)v) : "memory");
}
PS_DEV void st_shared_u8_rlx(uint32_t addr, uint8_t v) {
    asm volatile("st.relaxed.cluster.shared::cta.u8 [%0], %1;" ::"r"(addr), "h"((uint16_t)v) : "memory");
}
PS_DEV void red_cluster_max(uint32_t addr, uint32_t v) {
    asm volatile("red.shared::cluster.max.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
PS_DEV void st_cluster_s32(uint32_t addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// cluster barrier, or the block barrier when a cloud has a single CTA
PS_DEV void sync_all(int C) {
    if (C == 1) __syncthreads();
    else cluster_sync_all();
}

// Grid mode: barrier of the C co-resident CTAs of one cloud (cooperative
// launch) -- arrive on a global counter, the last arrival resets it and
// bumps the generation.  The gpu-scope fence before the arrival publishes
// the CTA's writes (cumulative over the preceding block barrier); the
// acquire load of the generation orders the reads after it.
PS_DEV void group_sync(int32_t* barw, int C) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* cnt = reinterpret_cast<unsigned*>(barw);
        unsigned* gen = reinterpret_cast<unsigned*>(barw + 1);
        unsigned g0;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
        __threadfence();
        if (atomicAdd(cnt, 1u) == (unsigned)C - 1u) {
            *reinterpret_cast<volatile unsigned*>(cnt) = 0u;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1u) : "memory");
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
            } while (g == g0);
        }
    }
    __syncthreads();
}

// prefix (over CTAs c < r) and total of per-CTA values v[0..C) in global
// scratch, with one block scan (grid mode: C up to kMaxCG)
PS_DEV void group_prefix(const int32_t* v, int C, int r, int* wt, int* s_tmp, int* off, int* tot) {
    const int tid = threadIdx.x;
    const int x = tid < C ? *reinterpret_cast<const volatile int32_t*>(v + tid) : 0;
    int t;
    const int ex = bscan(x, wt, &t);
    if (tid == r) *s_tmp = ex;
    __syncthreads();
    *off = *s_tmp;
    *tot = t;
    __syncthreads();
}

// kSm: the availability byte map and the rank table live in every CTA's
// shared memory (N bytes + 4N bytes); the map is built by owner CTAs
// (contiguous 16-byte-aligned index ranges, cleared through DSMEM stores)
// and gathered by every CTA.  Otherwise both are global arrays.
template <bool kSm, bool kGrid>
__global__ void __launch_bounds__(kT4, 1) samp4_kernel(SampArgs a, V4Work w) {
    static_assert(!(kSm && kGrid), "grid mode keeps the per-cloud arrays in global memory");
    using SL = Scr<kGrid>;
    __shared__ int wt[32];
    // P1 push, flattened rows (kSm, nseg <= 8): per warp, its 8 rows' entry
    // offsets, nbr index deltas and coverage bounds
    __shared__ int pr_off[kSm ? kW4 : 1][8];
    __shared__ int64_t pr_delta[kSm ? kW4 : 1][8];
    __shared__ __align__(16) int32_t pr_csm[kSm ? kW4 : 1][8][8];
    __shared__ int s_dec[2][kMaxC4];
    __shared__ int s_tmp;
    extern __shared__ __align__(16) uint8_t dsm4[];
    const int tid = threadIdx.x;
    const int C = kGrid ? a.grid_c : (int)cluster_nctarank();
    const int r = kGrid ? (int)(blockIdx.x % (unsigned)a.grid_c) : (int)cluster_ctarank();
    const int64_t b = kGrid ? (int64_t)(blockIdx.x / (unsigned)a.grid_c) : cluster_id_x();
    const int gt = r * kT4 + tid, GT = C * kT4;
    const int64_t N = a.N;
    const int nseg = a.nseg;

    const int64_t Npad = (N + 15) & ~(int64_t)15;
    uint8_t* avail = kSm ? dsm4 : w.avail + b * N;
    int32_t* pool = w.pool + b * N;
    uint32_t* pos = w.pos + b * N;
    int32_t* head = w.head + b * N;
    int32_t* nxt = w.nxt + b * N;
    int32_t* prv = w.prv + b * N;
    int32_t* lw = w.lw + b * N;
    int32_t* cand = w.cand + b * N;
    if (kSm && a.tiny) {
        // one CTA per cloud: every access to these arrays is CTA-local, so
        // they live in shared memory after the kSm layout (L2 round trips ->
        // shared-memory latency for the draw resolution and the pool)
        const int64_t Np = (N + 15) & ~(int64_t)15;
        const int64_t sp0 = ((N + 15) & ~(int64_t)15);
        const int64_t base0 = Np + 4 * Np + 4 * (((N + 31) / 32 + 3) & ~(int64_t)3) + 20 * sp0 + Np;
        int32_t* t0 = reinterpret_cast<int32_t*>(dsm4 + ((base0 + 15) & ~(int64_t)15));
        pool = t0;
        pos = reinterpret_cast<uint32_t*>(t0 + Np);
        head = t0 + 2 * Np;
        nxt = t0 + 3 * Np;
        prv = t0 + 4 * Np;
        lw = t0 + 5 * Np;
        cand = t0 + 6 * Np;
    }
    int32_t* rank = kSm ? reinterpret_cast<int32_t*>(dsm4 + Npad) : w.rank + b * N;
    uint32_t* tkb = reinterpret_cast<uint32_t*>(dsm4 + Npad + 4 * Npad);  // kSm: taken bitmap
    const int64_t Wtk = (N + 31) / 32;
    // kSm: witness row positions of my index range (a taken point at that
    // position of the row; INT_MAX = none), persistent over the visits
    int32_t* wpos = reinterpret_cast<int32_t*>(tkb + ((Wtk + 3) & ~(int64_t)3));
    const int64_t span_sm = ((N + C - 1) / C + 15) & ~(int64_t)15;
    // kSm, per draw of my range [tlo, thi) (written by the resolution pass, read
    // by the MIS pass of the same thread): candidate, its level count, its row
    // offset -- the MIS pass then starts with the row loads, not with three
    // dependent global loads
    int32_t* d_cand = wpos + span_sm;
    int32_t* d_cnt = d_cand + span_sm;
    int32_t* d_row = d_cnt + span_sm;  // (16 bytes per point reserved: d_row + one spare int32)
    // kSm: MIS states of ALL draws, replicated in every CTA of the cluster: the
    // owner of a draw stores its decision into every copy, readers (first pass,
    // dataflow polls) load their local copy
    uint8_t* st_s = reinterpret_cast<uint8_t*>(d_row + 2 * span_sm);
    const bool stash = kSm && a.cap_entries < (int64_t(1) << 31);
    int64_t i_tk = 0;  // sampled points already pushed
    int prev_seg = 0;  // segment of the previous visit (its accepts are pushed next)
    if (kSm) {
        for (int64_t x = tid; x < Wtk; x += kT4) tkb[x] = 0u;
        const int64_t span0 = ((N + C - 1) / C + 15) & ~(int64_t)15;
        for (int64_t x = tid; x < span0; x += kT4) wpos[x] = 0;  // blv: coverage level
        __syncthreads();
    }
    int32_t* adj = w.adj + b * N * kAdj4;
    uint8_t* adjcnt = w.adjcnt + b * N;
    uint8_t* stt = w.st + b * N;
    int32_t* preds = w.preds + b * N * kPred4;
    uint8_t* npred = w.npred + b * N;
    int32_t* scr = kGrid ? w.gscr + b * kScrG : w.scr + b * kScr;
    auto sync_grp = [&]() {
        if constexpr (kGrid) group_sync(scr + SL::bar, C);
        else sync_all(C);
    };
    if (kSm && a.tiny) {
        const int64_t Np = (N + 15) & ~(int64_t)15;
        const int64_t base0 = Np + 4 * Np + 4 * (((N + 31) / 32 + 3) & ~(int64_t)3) + 20 * Np + Np;
        scr = reinterpret_cast<int32_t*>(dsm4 + ((base0 + 15) & ~(int64_t)15)) + 7 * Np;
    }
    int64_t* out = a.out_idx + b * a.ld_out;
    const int64_t* indptr = a.indptr + b * (N + 1);
    const int32_t* nbr = a.nbr + b * a.cap_entries;

    // ---- bookkeeping, evaluated identically by every thread ------------------------
    int64_t i = a.k0;
    uint64_t rng = a.state_io[b];
    int seg = 0;
    while (seg < nseg && a.k0 >= a.boundaries[seg]) ++seg;
    int done = 0, exhausted = 0, entered = 0;
    // a cloud whose exclusion build failed (spill arena exhausted) has
    // incomplete rows: emit the error state instead of sampling from them
    // (out = -1 past the prefix, reached = n_total so early termination has
    // nothing to do, entered = -1); uniform over the cluster
    const bool failed = a.excl_status && a.excl_status[b] != 0;
    if (failed) {
        done = 1;
        i = a.n_total;
        entered = -1;
    } else if (seg >= nseg) {
        done = 1;
        exhausted = 1;
    } else {
        entered = 1;
    }
    for (int64_t t = a.k0 + gt; t < a.n_total; t += GT) out[t] = -1;
    const bool tdbg = a.dbg && b == 0 && gt == 0;
    long long tl = tdbg ? clock64() : 0;
    __shared__ long long s_acc[24];
    if (tdbg)
        for (int k = 0; k < 24; ++k) s_acc[k] = 0;
#define VT4(k)                                             \
    do {                                                   \
        if (tdbg) {                                        \
            const long long n_ = clock64();                \
            s_acc[k] += n_ - tl;                           \
            tl = n_;                                       \
        }                                                  \
    } while (0)

    while (!done) {
        const int lvl = a.seg_level_rows[seg];
        const int32_t* cnt_lvl = a.counts + (b * a.L + lvl) * N;

        // ---- P1: availability = not within the level radius of a sampled point -------
        // owner ranges: 16-byte aligned so a 16-byte chunk has one owner
        const int64_t span = ((N + C - 1) / C + 15) & ~(int64_t)15;
        const int64_t jlo = min(N, (int64_t)r * span), jhi = min(N, jlo + span);
        for (int64_t j = gt; j < N; j += GT) {
            if (!kSm) avail[j] = 1;
            head[j] = -1;
        }
        if (gt == 0) scr[SL::decided] = 0;
        if (kSm) {
            VT4(16);
            VT4(17);
            // push: every point sampled since the last visit (the FPS prefix at the
            // first visit, else the previous visit's accepts) walks its row prefix
            // at the level of the segment it was sampled in; entry j at row
            // position u lies within the radius of every segment s' with
            // u < counts[s'][q] -- a prefix of segments since the radii do not
            // increase -- so blv[j] = max(blv[j], #such s') in j's owner CTA
            // (DSMEM red.max).  j is unavailable in segment s iff blv[j] > s.
            const int lane = tid & 31, warp = tid >> 5, grp = lane / kG, gl = lane % kG;
            const int s_from = i_tk == 0 ? 0 : prev_seg;
            const uint32_t blv_base = smem_u32(wpos);
            const uint32_t span32 = (uint32_t)span;
            const uint32_t inv_span = 0xffffffffu / span32 + 1u;
            auto owner_of = [&](uint32_t j) {
                uint32_t ow = __umulhi(j, inv_span);
                if (ow * span32 > j) --ow;
                else if ((ow + 1u) * span32 <= j) ++ow;
                return ow;
            };
            const int64_t nnew = i - i_tk;
            // kS >= nseg segment slots: csm[s2] = INT_MAX before s_from (past
            // segments always count), the level count for s_from <= s2 < nseg,
            // 0 beyond -- cov = #(s2 : u < csm[s2]) with no per-entry range tests
            // (the slowest group's long rows bound this phase)
            auto push = [&](auto kS_tag) {
                constexpr int kS = decltype(kS_tag)::value;
                for (int64_t kb = (int64_t)r * (kT4 / kG) + warp * (32 / kG); kb < nnew;
                     kb += (int64_t)C * (kT4 / kG)) {
                    const int64_t k = kb + grp;
                    const bool valid = k < nnew;
                    int32_t q = 0, c = 0;
                    int32_t csm[kS];
#pragma unroll
                    for (int s2 = 0; s2 < kS; ++s2) csm[s2] = s2 < s_from ? 0x7fffffff : 0;
                    const int32_t* row = nbr;
                    if (valid) {
                        q = (int32_t)out[i_tk + k];
#pragma unroll
                        for (int s2 = 0; s2 < kS; ++s2)
                            if (s2 >= s_from && s2 < nseg)
                                csm[s2] = a.counts[(b * a.L + a.seg_level_rows[s2]) * N + q];
                        c = a.counts[(b * a.L + a.seg_level_rows[s_from]) * N + q];
                        row = nbr + indptr[q];
                        if (gl == 0) {
                            const uint32_t ow = owner_of((uint32_t)q);
                            red_cluster_max(mapa(blv_base + 4u * ((uint32_t)q - ow * span32), ow), (uint32_t)nseg);
                        }
                    }
                    const bool al = (reinterpret_cast<uintptr_t>(row) & 15u) == 0;
                    constexpr int kPush = 4 * kGStep;
                    for (int32_t u0 = 0;; u0 += kPush) {
                        const bool act = valid && u0 < c;
                        if (!__any_sync(kFull, act)) break;
                        if (!act) continue;
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const int32_t u = u0 + q4 * kGStep + 4 * gl;
                            const int4 v = grp_load4(row, u, c, al);
                            const int32_t jv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int32_t j = jv[e];
                                if (j < 0) continue;
                                uint32_t cov = 0;
#pragma unroll
                                for (int s2 = 0; s2 < kS; ++s2) cov += (u + e < csm[s2]) ? 1u : 0u;
                                const uint32_t ow = owner_of((uint32_t)j);
                                red_cluster_max(mapa(blv_base + 4u * ((uint32_t)j - ow * span32), ow), cov);
                            }
                        }
                    }
                }
            };
            // nseg <= 8: the warp's 8 rows are flattened -- entry f of their
            // concatenation goes to lane f % 32 -- so a warp costs sum(c) / 32
            // entries per lane instead of max(c) / 4 (the grouped walk above
            // issues every slot while any row of the warp is still running)
            auto push_flat = [&]() {
                const int64_t step = (int64_t)C * (kT4 / kG);
                for (int64_t kb = (int64_t)r * (kT4 / kG) + warp * 8; kb < nnew; kb += step) {
                    const int64_t k = kb + lane;
                    const bool valid = lane < 8 && k < nnew;
                    int32_t c = 0;
                    int64_t rowp = 0;
                    if (valid) {
                        const int32_t q = (int32_t)out[i_tk + k];
                        int32_t cm[8];
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2)
                            cm[s2] = s2 < s_from ? 0x7fffffff
                                                 : (s2 < nseg ? a.counts[(b * a.L + a.seg_level_rows[s2]) * N + q] : 0);
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2)
                            if (s2 == s_from) c = cm[s2];
                        rowp = indptr[q];
                        *reinterpret_cast<int4*>(&pr_csm[warp][lane][0]) = make_int4(cm[0], cm[1], cm[2], cm[3]);
                        *reinterpret_cast<int4*>(&pr_csm[warp][lane][4]) = make_int4(cm[4], cm[5], cm[6], cm[7]);
                        const uint32_t ow = owner_of((uint32_t)q);
                        red_cluster_max(mapa(blv_base + 4u * ((uint32_t)q - ow * span32), ow), (uint32_t)nseg);
                    }
                    int incl = c;
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
                        const int y = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int total = __shfl_sync(kFull, incl, 7);
                    const int excl = incl - c;
                    if (lane < 8) {
                        pr_off[warp][lane] = excl;
                        pr_delta[warp][lane] = rowp - excl;  // entry f of row kr: nbr[f + delta]
                    }
                    // row starts 1..7 in every lane: kr = #(starts <= f)
                    int o7[7];
#pragma unroll
                    for (int x = 0; x < 7; ++x) o7[x] = __shfl_sync(kFull, excl, x + 1);
                    __syncwarp();
                    for (int f0 = 0; f0 < total; f0 += 128) {
                        int32_t jv[4], uv[4], kv[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int f = f0 + 32 * e + lane;
                            int kr = 0;
#pragma unroll
                            for (int x = 0; x < 7; ++x) kr += f >= o7[x] ? 1 : 0;
                            kv[e] = kr;
                            uv[e] = f - pr_off[warp][kr];
                            jv[e] = f < total ? __ldg(nbr + (f + pr_delta[warp][kr])) : -1;
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int32_t j = jv[e];
                            if (j < 0) continue;
                            const int4 m0 = *reinterpret_cast<const int4*>(&pr_csm[warp][kv[e]][0]);
                            const int4 m1 = *reinterpret_cast<const int4*>(&pr_csm[warp][kv[e]][4]);
                            const int32_t u = uv[e];
                            const uint32_t cov = (u < m0.x) + (u < m0.y) + (u < m0.z) + (u < m0.w) + (u < m1.x) +
                                                 (u < m1.y) + (u < m1.z) + (u < m1.w);
                            const uint32_t ow = owner_of((uint32_t)j);
                            red_cluster_max(mapa(blv_base + 4u * ((uint32_t)j - ow * span32), ow), cov);
                        }
                    }
                    __syncwarp();
                }
            };
            if (nseg <= 8 && !a.push_grouped) push_flat();
            else if (nseg <= 8) push(std::integral_constant<int, 8>{});
            else push(std::integral_constant<int, kMaxSeg>{});
            i_tk = i;
        }
        sync_grp();
        VT4(13);
        if (!kSm) {
            for (int64_t x = gt; x < i; x += GT) {
                const int32_t q = (int32_t)out[x];
                const int32_t c = cnt_lvl[q];
                const int32_t* row = nbr + indptr[q];
                for (int32_t u0 = 0; u0 < c; u0 += 2 * kRB) {
                    int32_t qq[kRB], q2[kRB];
                    row_batch(row, u0, c, qq);
                    row_batch(row, u0 + kRB, c, q2);
#pragma unroll
                    for (int k = 0; k < kRB; ++k)
                        if (qq[k] >= 0) avail[qq[k]] = 0;
#pragma unroll
                    for (int k = 0; k < kRB; ++k)
                        if (q2[k] >= 0) avail[q2[k]] = 0;
                }
                avail[q] = 0;
            }
            sync_grp();
        }
        if (kSm) {
            for (int64_t j = jlo + tid; j < jhi; j += kT4) avail[j] = (uint32_t)wpos[j - jlo] <= (uint32_t)seg ? 1 : 0;
            sync_grp();
            const uint32_t avail_base = smem_u32(avail);
            // gather the other owners' ranges into my copy of the map
            for (int64_t c16 = tid; c16 < Npad / 16; c16 += kT4) {
                const int64_t j = c16 * 16;
                const uint32_t owner = (uint32_t)(j / span);
                if ((int)owner == r) continue;
                const uint4 v = ld_cluster_v4(mapa(avail_base + (uint32_t)j, owner));
                *reinterpret_cast<uint4*>(avail + j) = v;
            }
            __syncthreads();
        }
        VT4(0);

        // ---- P2: pool (available points in index order) + compressed adjacency -------
        // ---- P2: pool (available points in index order) + compressed adjacency -------
        int mycnt = 0;
        if (kSm) {
            for (int64_t j = jlo + tid; j < jhi; j += kT4) mycnt += avail[j];
        } else {
            // two points per thread in flight (j, j + kT4): their L2 round trips
            // (availability, counts, row entries, neighbours' availability) overlap
            for (int64_t j = jlo + tid; j < jhi; j += 2 * kT4) {
                const int64_t j2 = j + kT4;
                const bool a1 = avail[j] != 0;
                const bool a2 = j2 < jhi && avail[j2] != 0;
                mycnt += (a1 ? 1 : 0) + (a2 ? 1 : 0);
                const int32_t c1 = a1 ? cnt_lvl[j] : 0, c2 = a2 ? cnt_lvl[j2] : 0;
                const int32_t* row1 = nbr + (a1 ? indptr[j] : 0);
                const int32_t* row2 = nbr + (a2 ? indptr[j2] : 0);
                int32_t* ao1 = adj + j * kAdj4;
                int32_t* ao2 = adj + j2 * kAdj4;
                int n1 = 0, n2 = 0;
                const int32_t cm = c1 > c2 ? c1 : c2;
                for (int32_t u0 = 0; u0 < cm; u0 += kRB) {
                    int32_t q1[kRB], q2[kRB];
                    row_batch(row1, u0, c1, q1);
                    row_batch(row2, u0, c2, q2);
                    uint8_t v1[kRB], v2[kRB];
#pragma unroll
                    for (int k = 0; k < kRB; ++k) {
                        v1[k] = (q1[k] >= 0 && q1[k] != (int32_t)j) ? avail[q1[k]] : 0;
                        v2[k] = (q2[k] >= 0 && q2[k] != (int32_t)j2) ? avail[q2[k]] : 0;
                    }
#pragma unroll
                    for (int k = 0; k < kRB; ++k) {
                        if (v1[k]) {
                            if (n1 < kAdj4) ao1[n1] = q1[k];
                            ++n1;
                        }
                        if (v2[k]) {
                            if (n2 < kAdj4) ao2[n2] = q2[k];
                            ++n2;
                        }
                    }
                }
                // pad the lists to whole 16-byte chunks (the MIS pass reads them as int4)
                for (int k = n1; k < ((n1 + 3) & ~3) && k < kAdj4; ++k) ao1[k] = 0;
                for (int k = n2; k < ((n2 + 3) & ~3) && k < kAdj4; ++k) ao2[k] = 0;
                if (a1) adjcnt[j] = n1 > kAdj4 ? kAdjOvf : (uint8_t)n1;
                if (a2) adjcnt[j2] = n2 > kAdj4 ? kAdjOvf : (uint8_t)n2;
            }
        }
        mycnt = bsum(mycnt, wt);
        if (tid == 0) scr[SL::cnt0 + r] = mycnt;
        sync_grp();
        VT4(1);
        int off = 0, L = 0;
        if constexpr (kGrid) {
            group_prefix(scr + SL::cnt0, C, r, wt, &s_tmp, &off, &L);
        } else {
            for (int c2 = 0; c2 < C; ++c2) {
                const int v = scr[SL::cnt0 + c2];
                off += c2 < r ? v : 0;
                L += v;
            }
        }
        {
            // one block scan: each thread takes a contiguous run of my range
            // (runs in thread order keep the pool in index order)
            const int64_t len = jhi - jlo;
            const int E = (int)((len + kT4 - 1) / kT4);
            const int64_t j0 = jlo + (int64_t)tid * E;
            int cl = 0;
            for (int e = 0; e < E; ++e) {
                const int64_t j = j0 + e;
                cl += (j < jhi && avail[j]) ? 1 : 0;
            }
            int tot;
            int pos = off + bscan(cl, wt, &tot);
            for (int e = 0; e < E; ++e) {
                const int64_t j = j0 + e;
                if (j < jhi && avail[j]) pool[pos++] = (int32_t)j;
            }
            off += tot;
        }
        sync_grp();
        VT4(2);
        if (tdbg) { s_acc[10] += 1; s_acc[11] += L; }

        // MIS states / truncation / the draws' stash: CTA r owns the draws [tlo, thi)
        const int tspan = (L + C - 1) / C;
        const int tlo = min(L, r * tspan), thi = min(L, tlo + tspan);
        auto stash_draw = [&](int t, int32_t c) {
            if (stash) {
                d_cand[t - tlo] = c;
                d_cnt[t - tlo] = cnt_lvl[c];
                d_row[t - tlo] = (int32_t)indptr[c];
            }
        };
        // ---- P3: candidate order of all L draws ----------------------------------------
        if (a.pick_lowest) {
            for (int t = tlo + tid; t < thi; t += kT4) {
                const int32_t c = pool[t];
                cand[t] = c;
                if (!kSm) rank[c] = t;
                stash_draw(t, c);
            }
        } else {
            for (int t = gt; t < L; t += GT) {
                const uint64_t z = mix64_4(rng + (uint64_t)(t + 1) * kGolden4);
                const uint32_t p = (uint32_t)(z % (uint64_t)(L - t));
                pos[t] = p;
                nxt[t] = atomicExch(&head[p], t);
            }
            sync_grp();
            VT4(3);
            for (int t = gt; t < L; t += GT) {
                // latest earlier writer of my position, and of my tail slot L-1-t
                int best = -1;
                for (int x = head[pos[t]]; x >= 0; x = nxt[x])
                    if (x < t && x > best) best = x;
                prv[t] = best;
                int bl = -1;
                for (int x = head[L - 1 - t]; x >= 0; x = nxt[x])
                    if (x < t && x > bl) bl = x;
                lw[t] = bl;
            }
            sync_grp();
            VT4(4);
            for (int t = tlo + tid; t < thi; t += kT4) {
                // value at pos[t] before draw t: untouched -> pool; else the value
                // moved in by its latest writer x, i.e. the value of slot L-1-x at
                // draw x, found by following the tail-slot writers back
                const int x = prv[t];
                int32_t c;
                if (x < 0) {
                    c = pool[pos[t]];
                } else {
                    int y = x;
                    for (int z = lw[y]; z >= 0; z = lw[y]) y = z;
                    c = pool[L - 1 - y];
                }
                cand[t] = c;
                if (!kSm) rank[c] = t;
                stash_draw(t, c);
            }
        }
        if (kSm) {
            for (int t = tid; t < L; t += kT4) st_s[t] = kUnd4;
        } else {
            for (int t = tlo + tid; t < thi; t += kT4) stt[t] = kUnd4;
        }
        sync_grp();
        if (kSm) {
            for (int t = tid; t < L; t += kT4) rank[cand[t]] = t;
            __syncthreads();
        }

        VT4(5);
        // ---- P4: greedy MIS in draw order, parallel rounds ------------------------------
        // state of draw q: my range -> local shared memory, a peer's -> DSMEM
        // (kSm); global otherwise.  Reads may be stale within a round (IN/OUT
        // are final, a stale UND only delays); the cluster barrier publishes.
        const uint32_t st_base = kSm ? smem_u32(st_s) : 0u;
        const uint32_t tspan32 = (uint32_t)max(tspan, 1);
        const uint32_t inv_tspan = 0xffffffffu / tspan32 + 1u;
        (void)inv_tspan;
        auto st_get = [&](int q) -> uint8_t {
            if (!kSm) return ld_st(stt + q);
            return ld_shared_u8_rlx(st_base + (uint32_t)q);  // the local copy
        };
        auto st_set = [&](int t, uint8_t v) {
            if (!kSm) {
                st_st(stt + t, v);
            } else if (C == 1) {
                st_shared_u8_rlx(st_base + (uint32_t)t, v);
            } else {
                for (int ow = 0; ow < C; ++ow) st_cluster_u8_rlx(mapa(st_base + (uint32_t)t, (uint32_t)ow), v);
            }
        };
        // decided count: every CTA's cumulative count pushed into every CTA's
        // shared slot (double-buffered by round parity), summed after the barrier
        const uint32_t dec_base = smem_u32(&s_dec[0][0]);
        int my_dec = 0, round = 0;
        auto publish = [&](int add) {
            add = bsum(add, wt);
            my_dec += add;
            if constexpr (kGrid) {
                // cumulative count into this round parity's global slot; a slot is
                // rewritten two rounds later, after every CTA read it
                if (tid == 0) scr[SL::dec + (round & 1) * kMaxCG + r] = my_dec;
                sync_grp();
                int o2, tot;
                group_prefix(scr + SL::dec + (round & 1) * kMaxCG, C, r, wt, &s_tmp, &o2, &tot);
                ++round;
                return tot;
            } else {
                if (tid < C)
                    st_cluster_s32(mapa(dec_base + (uint32_t)(((round & 1) * kMaxC4 + r) * 4), (uint32_t)tid), my_dec);
                sync_grp();
                int tot = 0;
                for (int q = 0; q < C; ++q) tot += s_dec[round & 1][q];
                ++round;
                return tot;
            }
        };
        int decided = 0;
        for (int t = tlo + tid; t < thi; t += kT4) {
            const int32_t c = stash ? d_cand[t - tlo] : cand[t];
            // kSm: no adjacency lists -- the candidate scans its own row prefix
            // (availability and ranks in shared memory, states through DSMEM)
            const uint8_t nc = kSm ? kAdjOvf : adjcnt[c];
            bool outf = false, blocked = false;
            int np = 0;
            if (nc != kAdjOvf) {
                // per 16 neighbours: three batches of independent loads (neighbours,
                // their ranks, their states)
                const int4* ap = reinterpret_cast<const int4*>(adj + (int64_t)c * kAdj4);
                for (int h = 0; h < nc; h += 16) {
                    int32_t q[16];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int4 v = h + 4 * k < nc ? ap[h / 4 + k] : make_int4(0, 0, 0, 0);
                        q[4 * k] = v.x; q[4 * k + 1] = v.y; q[4 * k + 2] = v.z; q[4 * k + 3] = v.w;
                    }
                    int rq[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) rq[u] = h + u < nc ? rank[q[u]] : 0x7fffffff;
                    uint8_t sq[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) sq[u] = rq[u] < t ? st_get(rq[u]) : kOut4;
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        if (sq[u] == kIn4) outf = true;
                        if (rq[u] < t && sq[u] == kUnd4) {
                            if (np < kPred4) preds[(int64_t)t * kPred4 + np] = rq[u];
                            ++np;
                            blocked = true;
                        }
                    }
                }
            } else {
                if (!kSm && a.dbg && b == 0) atomicAdd((unsigned long long*)&a.dbg[14], 1ull);
                const int32_t m = stash ? d_cnt[t - tlo] : cnt_lvl[c];
                const int32_t* row = nbr + (stash ? (int64_t)d_row[t - tlo] : indptr[c]);
                const bool al = (reinterpret_cast<uintptr_t>(row) & 15u) == 0;
                constexpr int kRow = 16;
                for (int32_t u0 = 0; u0 < m && !outf; u0 += kRow) {
                    int32_t qq[kRow];
#pragma unroll
                    for (int k4 = 0; k4 < kRow / 4; ++k4) {
                        const int4 v = grp_load4(row, u0 + 4 * k4, m, al);
                        qq[4 * k4] = v.x; qq[4 * k4 + 1] = v.y; qq[4 * k4 + 2] = v.z; qq[4 * k4 + 3] = v.w;
                    }
                    uint8_t av[kRow];
#pragma unroll
                    for (int k = 0; k < kRow; ++k) av[k] = (qq[k] >= 0 && qq[k] != c) ? avail[qq[k]] : 0;
                    int rq[kRow];
#pragma unroll
                    for (int k = 0; k < kRow; ++k) rq[k] = av[k] ? rank[qq[k]] : 0x7fffffff;
                    uint8_t sq[kRow];
#pragma unroll
                    for (int k = 0; k < kRow; ++k) sq[k] = rq[k] < t ? st_get(rq[k]) : kOut4;
#pragma unroll
                    for (int k = 0; k < kRow; ++k) {
                        if (sq[k] == kIn4) outf = true;
                        if (rq[k] < t && sq[k] == kUnd4) {
                            if (np < kPred4) preds[(int64_t)t * kPred4 + np] = rq[k];
                            ++np;
                            blocked = true;
                        }
                    }
                }
            }
            if (outf) {
                st_set(t, kOut4);
                ++decided;
            } else if (!blocked) {
                st_set(t, kIn4);
                ++decided;
            } else {
                npred[t] = np > kPred4 ? kPredOvf : (uint8_t)np;
            }
        }
        VT4(19);
        if (!a.rounds) {
            // Dataflow: every thread settles its undecided draws in draw order,
            // polling the states of their undecided earlier neighbours until
            // one is IN (-> OUT) or all are OUT (-> IN) -- no barrier between
            // "rounds".  Progress: the smallest undecided draw has only decided
            // predecessors, and its owner thread is at it (each thread walks its
            // draws in increasing order); the CTAs of a cloud are co-resident.
            for (int t = tlo + tid; t < thi; t += kT4) {
                if (st_get(t) != kUnd4) continue;
                for (int spin = 0;; ++spin) {
                    bool outf = false, blocked = false;
                    const uint8_t np = npred[t];
                    if (np != kPredOvf) {
                        for (int k0p = 0; k0p < np && !outf; k0p += 16) {
                            int pr[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k) pr[k] = k0p + k < np ? preds[(int64_t)t * kPred4 + k0p + k] : -1;
                            uint8_t sq[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k) sq[k] = pr[k] >= 0 ? st_get(pr[k]) : kOut4;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                outf = outf || sq[k] == kIn4;
                                blocked = blocked || sq[k] == kUnd4;
                            }
                        }
                    } else {
                        if (a.dbg && b == 0) atomicAdd((unsigned long long*)&a.dbg[15], 1ull);
                        // more than kPred4 undecided predecessors: rescan the neighbours
                        const int32_t c = cand[t];
                        const uint8_t nc = kSm ? kAdjOvf : adjcnt[c];
                        const int32_t m = nc != kAdjOvf ? (int32_t)nc : cnt_lvl[c];
                        const int32_t* row = nc != kAdjOvf ? adj + (int64_t)c * kAdj4 : nbr + indptr[c];
                        for (int32_t u0 = 0; u0 < m && !outf; u0 += kRB) {
                            int32_t qq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) qq[k] = (u0 + k < m) ? row[u0 + k] : -1;
                            uint8_t av[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k)
                                av[k] = (qq[k] >= 0 && qq[k] != c) ? (nc != kAdjOvf ? 1 : avail[qq[k]]) : 0;
                            int rq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) rq[k] = av[k] ? rank[qq[k]] : 0x7fffffff;
                            uint8_t sq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) sq[k] = rq[k] < t ? st_get(rq[k]) : kOut4;
#pragma unroll
                            for (int k = 0; k < kRB; ++k) {
                                outf = outf || sq[k] == kIn4;
                                blocked = blocked || sq[k] == kUnd4;
                            }
                        }
                    }
                    if (outf) { st_set(t, kOut4); break; }
                    if (!blocked) { st_set(t, kIn4); break; }
                    if (a.poll_ns) __nanosleep(spin < 8 ? 32 : (unsigned)a.poll_ns);
                }
            }
            VT4(6);
        } else {
            int total_dec = publish(decided);
            VT4(6);
            while (total_dec < L) {
                if (tdbg) s_acc[12] += 1;
                int dd = 0;
                for (int t = tlo + tid; t < thi; t += kT4) {
                    if (st_get(t) != kUnd4) continue;
                    bool outf = false, blocked = false;
                    const uint8_t np = npred[t];
                    if (np != kPredOvf) {
                        for (int k0p = 0; k0p < np && !outf; k0p += 16) {
                            int pr[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k) pr[k] = k0p + k < np ? preds[(int64_t)t * kPred4 + k0p + k] : -1;
                            uint8_t sq[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k) sq[k] = pr[k] >= 0 ? st_get(pr[k]) : kOut4;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                outf = outf || sq[k] == kIn4;
                                blocked = blocked || sq[k] == kUnd4;
                            }
                        }
                    } else {
                        if (a.dbg && b == 0) atomicAdd((unsigned long long*)&a.dbg[15], 1ull);
                        // more than kPred4 undecided predecessors: rescan the neighbours
                        const int32_t c = cand[t];
                        const uint8_t nc = kSm ? kAdjOvf : adjcnt[c];
                        const int32_t m = nc != kAdjOvf ? (int32_t)nc : cnt_lvl[c];
                        const int32_t* row = nc != kAdjOvf ? adj + (int64_t)c * kAdj4 : nbr + indptr[c];
                        for (int32_t u0 = 0; u0 < m && !outf; u0 += kRB) {
                            int32_t qq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) qq[k] = (u0 + k < m) ? row[u0 + k] : -1;
                            uint8_t av[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k)
                                av[k] = (qq[k] >= 0 && qq[k] != c) ? (nc != kAdjOvf ? 1 : avail[qq[k]]) : 0;
                            int rq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) rq[k] = av[k] ? rank[qq[k]] : 0x7fffffff;
                            uint8_t sq[kRB];
#pragma unroll
                            for (int k = 0; k < kRB; ++k) sq[k] = rq[k] < t ? st_get(rq[k]) : kOut4;
#pragma unroll
                            for (int k = 0; k < kRB; ++k) {
                                outf = outf || sq[k] == kIn4;
                                blocked = blocked || sq[k] == kUnd4;
                            }
                        }
                    }
                    if (outf) {
                        st_set(t, kOut4);
                        ++dd;
                    } else if (!blocked) {
                        st_set(t, kIn4);
                        ++dd;
                    }
                }
                VT4(20);
                total_dec = publish(dd);
            }
        }
        VT4(7);
        // ---- P5: truncation at the segment boundary --------------------------------------
        const int64_t need = a.boundaries[seg] - i;
        int nin = 0;
        for (int t = tlo + tid; t < thi; t += kT4) nin += st_get(t) == kIn4 ? 1 : 0;
        nin = bsum(nin, wt);
        if (tid == 0) scr[SL::cnt1 + r] = nin;
        sync_grp();
        int aoff = 0, A = 0;
        if constexpr (kGrid) {
            group_prefix(scr + SL::cnt1, C, r, wt, &s_tmp, &aoff, &A);
        } else {
            for (int c2 = 0; c2 < C; ++c2) {
                const int v = scr[SL::cnt1 + c2];
                aoff += c2 < r ? v : 0;
                A += v;
            }
        }
        const int64_t take = (int64_t)A < need ? (int64_t)A : need;
        const bool ends = take == need;
        for (int base = tlo; base < thi; base += kT4) {
            const int t = base + tid;
            const int f = (t < thi && st_get(t) == kIn4) ? 1 : 0;
            int tot;
            const int ex = bscan(f, wt, &tot);
            const int64_t k = aoff + ex;
            if (f && k < take) {
                out[i + k] = cand[t];
                if (ends && k == take - 1) scr[SL::last] = t;
            }
            aoff += tot;
        }
        sync_grp();
        VT4(8);
        const int last = ends ? scr[SL::last] : -1;
        prev_seg = seg;
        i += take;
        if (ends) {
            if (!a.pick_lowest) rng = rng + (uint64_t)(last + 1) * kGolden4;
            if (i >= a.n_total) {
                done = 1;
            } else {
                while (i >= a.boundaries[seg]) ++seg;
                entered += 1;
            }
        } else {
            if (!a.pick_lowest) rng = rng + (uint64_t)L * kGolden4;
            seg += 1;
            if (seg >= nseg) {
                exhausted = 1;
                done = 1;
            } else {
                entered += 1;
                if (i >= a.boundaries[seg]) {
                    while (i >= a.boundaries[seg]) ++seg;
                    entered += 1;
                }
            }
        }
        // every thread evaluated the same bookkeeping; the next visit's P1 is
        // ordered after this visit's reads of scr by its cluster barrier
    }
#undef VT4
    if (tdbg)
        for (int k = 0; k < 24; ++k) a.dbg[k] += s_acc[k];
    if (r == 0 && tid == 0) {
        a.reached[b] = i;
        a.exhausted[b] = exhausted;
        a.entered[b] = entered;
        a.state_io[b] = rng;
    }
}

size_t align256_4(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t sampler_v4_ws_bytes(int64_t B, int64_t N) {
    size_t s = 0;
    s += align256_4(sizeof(uint8_t) * B * N);            // avail
    s += align256_4(sizeof(int32_t) * B * N) * 8;        // pool pos head nxt prv lw cand rank
    s += align256_4(sizeof(int32_t) * B * N * kAdj4);    // adj
    s += align256_4(sizeof(uint8_t) * B * N) * 3;        // adjcnt st npred
    s += align256_4(sizeof(int32_t) * B * N * kPred4);   // preds
    s += align256_4(sizeof(int32_t) * B * kScr);         // scr
    s += align256_4(sizeof(int32_t) * B * kScrG);        // gscr
    return s;
}

// CTAs per cloud: ~3000 points per CTA, at most 8, and at most one wave of
// 148 SMs for the batch when that still leaves >= 1 CTA per cloud
static int v4_cluster(int64_t N, int64_t B) {
    const char* e = getenv("PS_SAMPLER_CLUSTER");
    int c = e ? atoi(e) : (int)((N + 2999) / 3000);
    c = c < 1 ? 1 : (c > 8 ? 8 : c);
    if (!e)
        while (c > 1 && B * c > 148) --c;
    return c;
}

cudaError_t launch_sampler_v4(SampArgs a, int64_t B, cudaStream_t s) {
    V4Work w = {};
    const int64_t N = a.N;
    unsigned char* p = a.gws;
    w.avail = p; p += align256_4(sizeof(uint8_t) * B * N);
    w.pool = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.pos = reinterpret_cast<uint32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.head = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.nxt = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.prv = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.lw = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.cand = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.rank = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N);
    w.adj = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N * kAdj4);
    w.adjcnt = p; p += align256_4(sizeof(uint8_t) * B * N);
    w.st = p; p += align256_4(sizeof(uint8_t) * B * N);
    w.npred = p; p += align256_4(sizeof(uint8_t) * B * N);
    w.preds = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * N * kPred4);
    w.scr = reinterpret_cast<int32_t*>(p); p += align256_4(sizeof(int32_t) * B * kScr);
    w.gscr = reinterpret_cast<int32_t*>(p);
    a.B = B;
    a.grid_c = 0;
    const int C = v4_cluster(N, B);
    cudaError_t e = cudaSuccess;
    const int64_t Npad = (N + 15) & ~(int64_t)15;
    const int64_t span0 = ((N + C - 1) / C + 15) & ~(int64_t)15;
    const size_t dsm = (size_t)(Npad + 4 * Npad + 4 * (((N + 31) / 32 + 3) & ~(int64_t)3) + 20 * span0 + Npad);
    const bool sm = dsm <= 220 * 1024 && !getenv("PS_SAMPLER_GLOBAL");
    // one CTA per cloud and room for 7 int32 arrays of N + the scratch: tiny layout
    const size_t dsm_tiny = ((dsm + 15) & ~(size_t)15) + 7 * 4 * (size_t)Npad + 4 * kScr;
    a.tiny = (sm && C == 1 && dsm_tiny <= 220 * 1024 && !getenv("PS_SAMPLER_NOTINY")) ? 1 : 0;
    a.rounds = getenv("PS_SAMPLER_ROUNDS") ? 1 : 0;
    a.poll_ns = getenv("PS_SAMPLER_POLL") ? atoi(getenv("PS_SAMPLER_POLL")) : 128;
    a.push_grouped = getenv("PS_SAMPLER_PUSH_GROUPED") ? 1 : 0;  // A/B knob (flattened rows by default)
    const size_t dsm_used = a.tiny ? dsm_tiny : dsm;
    if (!sm && !getenv("PS_SAMPLER_NOGRID")) {
        // grid mode: few clouds too large for shared memory -- spread each over
        // (SMs / B) co-resident CTAs instead of one cluster of <= 8
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, samp4_kernel<false, true>, kT4, 0);
        const int64_t per = (int64_t)nsm * (occ > 0 ? occ : 1) / B;
        const char* ge = getenv("PS_SAMPLER_GRID_CTAS");
        int64_t cg = ge ? atoi(ge) : std::min<int64_t>(per, std::min<int64_t>(kMaxCG, (N + 2047) / 2048));
        cg = std::min<int64_t>(cg, std::min<int64_t>(per, kMaxCG));
        if (cg > 2 * C) a.grid_c = (int)cg;
    }
    if (a.grid_c > 0) {
        cudaError_t e2 = cudaMemsetAsync(w.gscr, 0, sizeof(int32_t) * B * kScrG, s);  // barrier words
        if (e2 != cudaSuccess) return e2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(B * a.grid_c), 1, 1);
        cfg.blockDim = dim3(kT4, 1, 1);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the group barrier spins
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        a.dbg = nullptr;
        return cudaLaunchKernelEx(&cfg, samp4_kernel<false, true>, a, w);
    }
    auto kern = sm ? samp4_kernel<true, false> : samp4_kernel<false, false>;
    if (sm) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm_used);
        if (e != cudaSuccess) return e;
    }
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * C), 1, 1);
    cfg.blockDim = dim3(kT4, 1, 1);
    cfg.dynamicSmemBytes = sm ? dsm_used : 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    a.dbg = nullptr;
    if (getenv("PS_SAMPLER_TIMING")) {  // development aid (synchronises)
        static long long* dbg = nullptr;
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 32);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 32, s);
        a.dbg = dbg;
        e = cudaLaunchKernelEx(&cfg, kern, a, w);
        {
            long long h2[32];
            cudaMemcpyAsync(h2, dbg, sizeof(h2), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "[sampler v4] P1 %lld (taken bits %lld, stage %lld, pull %lld) | mis0 own %lld + publish %lld | "
                    "rounds own %lld + publish %lld | overflows adj %lld pred %lld\n",
                    h2[13] + h2[16] + h2[17] + h2[18], h2[16], h2[17], h2[18], h2[19], h2[6], h2[20], h2[7],
                    h2[14], h2[15]);
        }
        long long h[16];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "[sampler v4 C=%d] cycles: avail %lld pool+adj %lld compact %lld positions %lld walks %lld "
                "resolve %lld mis0 %lld rounds %lld trunc %lld | visits %lld sum L %lld rounds %lld\n", C, h[0], h[1],
                h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[10], h[11], h[12]);
        return e;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, w);
}

size_t sampler_global_ws_bytes(int64_t B, int64_t N, bool) { return sampler_v4_ws_bytes(B, N); }

cudaError_t launch_sampler(SampArgs a, int64_t B, cudaStream_t s) { return launch_sampler_v4(a, B, s); }

}  // namespace ps
