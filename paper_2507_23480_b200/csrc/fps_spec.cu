// fps_spec.cu -- K1: exact farthest-point sampling with speculation, one
// thread-block cluster per cloud (B200 / sm_100a).
//
// Same result as _kernels.fps_loop (/root/reference/pkg/src/pointsample/
// _kernels.py:35-74) -- indices, curve and the md/taken state, bit for bit
// -- but one cluster exchange yields ~5 (FastPoint prefix) to ~13 (full
// run) samples instead of one.
//
// Why it is exact.  At an exchange every CTA publishes its argmax (the
// "header") and every point whose md >= tau (the "candidates"; tau is one
// threshold all CTAs agree on).  The first pick is the max over the headers:
// the reference's argmax.  Every non-candidate point has md < tau and md only
// decreases, so while the best candidate -- its md lowered exactly, float64
// in the reference's operation order, by every sample taken since the
// exchange -- is still >= tau, it is the argmax the reference would pick
// next (lowest index on ties).  tau only decides how many picks one exchange
// certifies, never which point is picked, so a poor tau costs speed only.
//
// Layout: C CTAs of T threads per cloud.  Each CTA counting-sorts its index
// range by a 16^3 Morton cell so that worker warp w (0..kW-2) owns 32P
// spatially compact points in registers (float32 xyz, float64 md, taken
// bits); a sample farther from a warp's box than every skip threshold of the
// warp is skipped by the whole warp.  The last warp (the lead) owns none and
// runs, per exchange:
//   C. CTA argmax over the warp records + the CTA's candidates (<= kR-1),
//      pushed to every CTA with st.async; each sender announces its byte
//      count on the peer's mbarrier (remote arrive.expect_tx);
//   D. headers in lanes < C, candidates compacted one per lane;
//   E. picks: the first over headers + candidates, then the best candidate
//      while >= tau, each lowering the others by its exact float64 distance
//      to them (the reference's update, same operation order).  Each pick is
//      published to the CTA (release store); the worker warps fold it into
//      their md as soon as it appears, overlapping the lead's serial chain.
//   tau for the next exchange: kTarget samples ahead along the recent curve
//   slope (the curve is non-increasing), gain-corrected by the count seen.
// The duplicate fallback of _kernels.py:65-70 (max <= 0 or winner already
// taken -> lowest untaken index) runs as a cluster-wide exchange when the
// first pick needs it; a later pick that would need it ends the run.
// Development knobs: PS_SPEC_TARGET=<samples> overrides kTarget (< 0: no
// speculation); PS_FPS_NOSPEC=1 selects fps.cu; make TIMING=1 +
// PS_FPS_TIMING=1 prints per-phase cycles (tools/fps_spec_timing.py).
// Measured (profiles/r01/fps_spec.log): 0.50 us/iteration for a full
// 6000-of-24000 FPS on the C3 batch vs 1.13 for the one-sample kernel
// (fps.cu), 0.94 vs 1.37 over the 600-iteration FastPoint prefix.

#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "fps_util.cuh"
#include "ps_internal.h"

namespace ps {

namespace {

// lexicographic (key desc, idx asc): true if (ka, ia) ranks above (kb, ib)
PS_DEV bool ranks_above(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

constexpr int kR = 10;            // records per CTA per exchange: its max + kR-1 threshold candidates
constexpr int kRunMax = 31;       // samples per exchange (one lane each)
constexpr double kTarget = 22.0;  // threshold candidates aimed for per exchange
constexpr uint64_t kTauOff = ~0ull;  // threshold disabled (above every md bit pattern)
// point slots of a CTA (sort arrays): P per worker thread, rounded to 8
constexpr int spec_slots(int P, int T, bool lead_pts) { return ((P * (lead_pts ? T : T - 32)) + 7) / 8 * 8; }
constexpr int64_t kSortMinIters = 64;  // runs shorter than this keep the index order
// Workers refresh their warp record while waiting for the next pick (instead
// of after the run's end, on the lead's critical path) from P = 10 points per
// thread: C3 5-CTA clusters prefix 688 -> 672 us, full run 3608 -> 3461 us;
// at P = 5 the extra issue next to the lead costs more (517 -> 522 us).
// Either way the record is rewritten only when a fold touched the warp.
#ifndef PS_EAGER_REC
#define PS_EAGER_REC 1
#endif
constexpr bool kEagerRec = PS_EAGER_REC;
constexpr float kInfF = __builtin_huge_valf();

template <int P, int T, bool kLeadPts>
__global__ void __launch_bounds__(T, 1) fps_spec_kernel(FpsArgs a) {
    static_assert(P > 0 && P <= 16, "register-resident clouds only");
    constexpr int kW = T / 32;
    // The lead warp runs the exchange and the speculation and owns no points;
    // the other warps own the points and fold each published pick.  (The
    // warp arbiter does not favour the lead over busy co-resident warps --
    // a pick takes 5x longer next to three FFMA-bound warps, tools/micro/
    // pick_micro.cu -- but idling its SMSP's three other warps cost more
    // fold throughput than it saved: profiles/r01/fps_spec.log.)
    constexpr int kLead = kW - 1;
    // kLeadPts: the lead warp owns points too (clouds that need all T threads)
    constexpr int TW = kLeadPts ? T : T - 32;  // point-owning (worker) threads
    __shared__ Rec wrec[kW];
    __shared__ Rec cand[kR - 1];
    __shared__ Rec slots[2][kMaxCluster * kR];
    __shared__ Rec fb_slots[kMaxCluster];
    __shared__ Rec fbw_s;
    __shared__ float4 run_s[32];
    __shared__ uint8_t map_s[kMaxCluster * kR];
    __shared__ double hist_s[32];
    __shared__ unsigned long long tau_s;
    __shared__ int cnt_s;
    __shared__ uint32_t pub_s;
    __shared__ uint32_t bin_s[4096];    // spatial sort: cell counts / offsets
    // sorted position -> local index / local index -> sorted position
    // (dynamic shared memory: 4 bytes per point slot of the CTA)
    extern __shared__ __align__(16) uint16_t dyn_s[];
    constexpr int kS = spec_slots(P, T, kLeadPts);
    uint16_t* const ord_s = dyn_s;
    uint16_t* const pos_s = dyn_s + kS;
    __shared__ float red_s[kW][6], bb_s[6];
    __shared__ uint32_t wsum_s[kW];
    __shared__ __align__(8) uint64_t bars[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool worker = kLeadPts || warp != kLead;
    const uint32_t C = cluster_nctarank();
    const uint32_t r = cluster_ctarank();
    const int64_t b = cluster_id_x();
    const int64_t N = a.N;
    const int64_t S = a.points_per_cta;
    const int64_t lo = (int64_t)r * S;
    const int64_t hi = min(N, lo + S);
    const float4* __restrict__ xyz = a.xyz + b * N;
    double* __restrict__ md = a.md + b * N;
    uint8_t* __restrict__ taken = a.taken + b * N;
    int64_t* __restrict__ out = a.out_idx + b * a.ld_out;
    double* __restrict__ curve = a.curve + b * a.ld_out;

    const int64_t k_start = a.k_start_dev ? a.k_start_dev[b] : a.k_start;
    const int64_t k_stop = a.k_stop;
    const int64_t seed = a.seed_dev ? a.seed_dev[b] : a.seed;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const bool writer = r == 0 && warp == kLead && lane == 0;

    // ---- spatial order -----------------------------------------------------
    // Counting sort of this CTA's points by the Morton code of a 16^3 grid over
    // their bounding box: worker warp w owns sorted positions [w*32P, (w+1)*32P),
    // a compact region, so a pick far from a warp's box skips the whole warp
    // (fold_one).  The order inside a cell follows shared-memory atomics and may
    // differ between runs; no result depends on it (every choice is by
    // (md, original index)).
    static_assert(kS >= P * TW, "sort capacity");
    const int ncta = hi > lo ? (int)(hi - lo) : 0;
    if (k_stop - k_start < kSortMinIters) {
        // short runs (early-termination tails) do not repay the sort
        for (int i = tid; i < ncta; i += T) { ord_s[i] = (uint16_t)i; pos_s[i] = (uint16_t)i; }
        __syncthreads();
    } else {
        float mn[3] = {kInfF, kInfF, kInfF}, mx[3] = {-kInfF, -kInfF, -kInfF};
        for (int i = tid; i < ncta; i += T) {
            const float4 v = xyz[lo + i];
            mn[0] = fminf(mn[0], v.x); mn[1] = fminf(mn[1], v.y); mn[2] = fminf(mn[2], v.z);
            mx[0] = fmaxf(mx[0], v.x); mx[1] = fmaxf(mx[1], v.y); mx[2] = fmaxf(mx[2], v.z);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                mn[d] = fminf(mn[d], __shfl_xor_sync(kFull, mn[d], o));
                mx[d] = fmaxf(mx[d], __shfl_xor_sync(kFull, mx[d], o));
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) { red_s[warp][d] = mn[d]; red_s[warp][3 + d] = mx[d]; }
        }
        for (int i = tid; i < 4096; i += T) bin_s[i] = 0u;
        __syncthreads();
        if (tid < 6) {
            float r = red_s[0][tid];
            for (int w = 1; w < kW; ++w) r = tid < 3 ? fminf(r, red_s[w][tid]) : fmaxf(r, red_s[w][tid]);
            bb_s[tid] = r;
        }
        __syncthreads();
        float org[3], sc[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            org[d] = bb_s[d];
            const float ext = bb_s[3 + d] - bb_s[d];
            sc[d] = ext > 0.f ? 16.0f / ext : 0.f;
        }
        auto cell_of = [&](float4 v) {
            auto q4 = [&](float x, int d) {
                const int c = (int)((x - org[d]) * sc[d]);
                return (uint32_t)(c < 0 ? 0 : (c > 15 ? 15 : c));
            };
            auto spread = [](uint32_t b) { return (b & 1u) | ((b & 2u) << 2) | ((b & 4u) << 4) | ((b & 8u) << 6); };
            return spread(q4(v.x, 0)) | (spread(q4(v.y, 1)) << 1) | (spread(q4(v.z, 2)) << 2);
        };
        for (int i = tid; i < ncta; i += T) {
            const uint32_t c = cell_of(xyz[lo + i]);
            pos_s[i] = (uint16_t)c;
            atomicAdd(&bin_s[c], 1u);
        }
        __syncthreads();
        // exclusive scan of the 4096 bins: kPer consecutive bins per thread
        constexpr int kPer = 4096 / T;
        uint32_t loc = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) loc += bin_s[tid * kPer + k];
        uint32_t inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wsum_s[warp] = inc;
        __syncthreads();
        uint32_t wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += wsum_s[w];
        uint32_t run = wbase + inc - loc;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t c = bin_s[tid * kPer + k];
            bin_s[tid * kPer + k] = run;
            run += c;
        }
        __syncthreads();
        for (int i = tid; i < ncta; i += T) {
            const uint32_t sp = atomicAdd(&bin_s[pos_s[i]], 1u);
            ord_s[sp] = (uint16_t)i;
            pos_s[i] = (uint16_t)sp;
        }
        __syncthreads();
    }
    // 32-bit shared addresses of the hot arrays (see sts_*/lds_* in common.cuh)
    const uint32_t a_ord = smem_u32(ord_s), a_pos = smem_u32(pos_s), a_wrec = smem_u32(wrec),
                   a_cand = smem_u32(cand), a_map = smem_u32(map_s), a_run = smem_u32(run_s),
                   a_hist = smem_u32(hist_s), a_cnt = smem_u32(&cnt_s);
    // original index of my slot q
    auto oid = [&](int q) -> uint32_t { return (uint32_t)lo + lds_u16(a_ord + 2u * (warp * 32 * P + q * 32 + lane)); };

    // ---- state into registers ---------------------------------------------
    float fx[P], fy[P], fz[P], thr[P];
    // md: registers, or (P >= 10) shared memory after the sort arrays -- the
    // float32 screen needs only thr, so md is touched on the exact path,
    // once per exchange for the thread maximum / candidates, and at the ends
    constexpr bool kMs = P >= 10;
    double m_reg[kMs ? 1 : P] = {};
    double* const m_sm = reinterpret_cast<double*>(dyn_s + 2 * kS) + (kMs ? tid : 0);
    auto mget = [&](int q) -> double {
        if constexpr (kMs) return m_sm[q * TW];
        else return m_reg[q];
    };
    auto mset = [&](int q, double v) {
        if constexpr (kMs) m_sm[q * TW] = v;
        else m_reg[q] = v;
    };
    uint32_t tk = 0, valid = 0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int sp = warp * 32 * P + q * 32 + lane;
        fx[q] = fy[q] = fz[q] = 0.f;
        double mq = 0.0;
        if (worker && sp < ncta) {
            const int64_t j = lo + ord_s[sp];
            valid |= 1u << q;
            const float4 v = xyz[j];
            fx[q] = v.x; fy[q] = v.y; fz[q] = v.z;
            if (a.fresh) {
                mq = kInf;
                tk |= (j == seed ? 1u : 0u) << q;
            } else {
                mq = md[j];
                tk |= (taken[j] ? 1u : 0u) << q;
            }
        }
        if (!kMs || worker) mset(q, mq);  // (kMs: the lead owns no md slot)
        thr[q] = ((valid >> q) & 1u) ? skip_threshold(mq) : -1.0f;
    }
    // the warp's bounding box and the largest skip threshold of its points
    float wb[6] = {kInfF, kInfF, kInfF, -kInfF, -kInfF, -kInfF};
#pragma unroll
    for (int q = 0; q < P; ++q) {
        if ((valid >> q) & 1u) {
            wb[0] = fminf(wb[0], fx[q]); wb[1] = fminf(wb[1], fy[q]); wb[2] = fminf(wb[2], fz[q]);
            wb[3] = fmaxf(wb[3], fx[q]); wb[4] = fmaxf(wb[4], fy[q]); wb[5] = fmaxf(wb[5], fz[q]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            wb[d] = fminf(wb[d], __shfl_xor_sync(kFull, wb[d], o));
            wb[3 + d] = fmaxf(wb[3 + d], __shfl_xor_sync(kFull, wb[3 + d], o));
        }
    }
    auto warp_thr_max = [&]() {
        float t = -1.0f;
#pragma unroll
        for (int q = 0; q < P; ++q)
            if ((valid >> q) & 1u) t = fmaxf(t, thr[q]);
        const uint32_t k = __reduce_max_sync(kFull, t < 0.f ? 0u : __float_as_uint(t));  // t >= 0: bits order
        return k == 0u ? -1.0f : __uint_as_float(k);
    };
    float wthr = warp_thr_max();
    if (a.fresh && writer) {
        out[0] = seed;
        curve[0] = kInf;
    }
    if (tid == 0) {
        cnt_s = 0;
        pub_s = 0u;
        mbar_init(&bars[0], C);  // one arrival per sending CTA
        mbar_init(&bars[1], C);
        fence_mbar_init_cluster();
    }
    cluster_sync_all();

    int64_t it = k_start;
    // lead warp: ring of the last 32 squared curve values, for the threshold
    int hc = 0;
    float gain = 1.0f;
    bool tau_boot = false;  // lead: the threshold in use came from the CTA maxima
    if (warp == kLead && !a.fresh && k_start < k_stop) {
        // the most recent finite curve values only: positions filled by the
        // sampler carry +inf and say nothing about the current md
        const int avail = k_start - 1 >= 32 ? 32 : (k_start - 1 > 0 ? (int)(k_start - 1) : 0);
        const double c = lane < avail ? curve[k_start - 1 - lane] : kInf;  // previous epilogue stored sqrt
        const uint32_t fin = __ballot_sync(kFull, lane < avail && c < kInf);
        const int nh = __ffs(~fin) - 1 < 0 ? 32 : __ffs(~fin) - 1;  // unbroken finite run from the end
        if (lane < nh) hist_s[(nh - 1 - lane) & 31] = c * c;
        hc = nh;
    }
    uint64_t tau = kTauOff;

    // cached thread-local max (recomputed when its own point moved)
    bool dirty = true;
    double bv = -1.0;
    int bq = 0;
    float bx = 0.f, by = 0.f, bz = 0.f;

    // mark sample sidx taken if it is mine; fold it into md unless it is the
    // last sample of this call (the reference folds that one at the next call)
    // TIMING build: worker warp 0 of cloud 0 / CTA 0 -- cycles from seeing a
    // run's end to its barrier arrival, picks still unfolded at that point,
    // cycles of phase B, folds run / skipped by the whole-warp test
    const bool wdbg = kTiming && a.dbg && b == 0 && r == 0 && warp == 0 && lane == 0;
    long long w_tdone = 0, wacc[5] = {0, 0, 0, 0, 0};
    bool stale = true;  // the warp's record may not reflect its points (a fold ran since it was written)
    auto fold_one = [&](float sx32, float sy32, float sz32, uint32_t sidx, bool do_fold) {
        const int64_t li = (int64_t)sidx - lo;
        if (li >= 0 && li < ncta) {
            const int sp = (int)lds_u16(a_pos + 2u * (uint32_t)li);
            if (worker && sp / (32 * P) == warp) {  // warp-uniform: the taken bit may be in the record
                if ((sp & 31) == lane) tk |= 1u << ((sp % (32 * P)) >> 5);
                stale = true;
            }
        }
        if (!do_fold) return;
        // whole-warp skip: a rounded-down lower bound of the squared distance
        // from the sample to the warp's box above every skip threshold of the
        // warp proves, as the per-point screen does, that no md can change
        {
            const float ex = fmaxf(fmaxf(__fsub_rd(wb[0], sx32), __fsub_rd(sx32, wb[3])), 0.f);
            const float ey = fmaxf(fmaxf(__fsub_rd(wb[1], sy32), __fsub_rd(sy32, wb[4])), 0.f);
            const float ez = fmaxf(fmaxf(__fsub_rd(wb[2], sz32), __fsub_rd(sz32, wb[5])), 0.f);
            const float dbox = __fadd_rd(__fadd_rd(__fmul_rd(ex, ex), __fmul_rd(ey, ey)), __fmul_rd(ez, ez));
            if (kTiming && wdbg) ++wacc[4];
            if (dbox > wthr) return;
            if (kTiming && wdbg) ++wacc[3];
            stale = true;
        }
        uint32_t need = 0;
        constexpr int kD = P >= 10 ? 1 : P;  // P >= 10: recompute instead of keeping P distances live
        float d32s[kD];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float dx = fx[q] - sx32, dy = fy[q] - sy32, dz = fz[q] - sz32;
            const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            if constexpr (P < 10) d32s[q] = d32;
            need |= (!(d32 > thr[q]) ? 1u : 0u) << q;
        }
        if (__any_sync(kFull, need != 0)) {
            const double sx = sx32, sy = sy32, sz = sz32;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                if (__any_sync(kFull, (need >> q) & 1u)) {
                    const double d = sqdist(sx, sy, sz, (double)fx[q], (double)fy[q], (double)fz[q]);
                    if (((need >> q) & 1u) && dbits(d) < dbits(mget(q))) {
                        float d32;
                        if constexpr (P < 10) {
                            d32 = d32s[q];
                        } else {  // the screen's float32 distance, same operations
                            const float dx = fx[q] - sx32, dy = fy[q] - sy32, dz = fz[q] - sz32;
                            d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                        }
                        mset(q, d);
                        thr[q] = skip_threshold_d32(d, d32);
                        dirty = dirty || (q == bq);
                    }
                }
            }
        }
    };

    if (k_start < k_stop) {
        const int64_t last = a.fresh ? seed : out[k_start - 1];  // refolded, as _kernels.py
        const float4 lv = xyz[last];
        fold_one(lv.x, lv.y, lv.z, (uint32_t)last, true);
    }

    const unsigned poll_ns = a.poll_ns > 0 ? (unsigned)a.poll_ns : 32u;
    uint32_t ex = 0;
    const bool tdbg = kTiming && a.dbg && b == 0 && r == 0 && warp == kLead && lane == 0;
    long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tsp = 0;
    // The lead-only warp (!kLeadPts) runs its own copy of the loop: the
    // workers' register-resident points are dead there, so the two roles
    // share the register budget instead of adding up (room for more
    // points per thread).  Both loops meet the same CTA barriers, at
    // different instructions (warp-uniform roles; a bar.sync completes on
    // thread arrivals).  compute-sanitizer synccheck reports that as
    // divergence; the forms it accepts -- named bar.arrive / bar.sync pairs,
    // the non-.aligned barrier.sync, an mbarrier, one shared loop -- all
    // measured 20-30 % slower at P = 10 (profiles/r02/fps_barrier_ab.log).
    auto lead_step = [&](uint32_t tag, uint32_t par, uint32_t phase, long long& t0, long long& t1) -> uint32_t {
        uint32_t pw = 0;
            // C. CTA record set: header (the CTA max, candidate count) and
            // up to kR-1 threshold candidates, pushed to every CTA; each
            // sender announces its byte count on the peer's mbarrier.
            const uint4 wr = lane < kW ? lds_v4(a_wrec + 32u * lane) : make_uint4(0u, 0u, kNone, 0u);
            const int cl = warp_argmax_lane(((uint64_t)wr.y << 32) | wr.x, wr.z);
            Rec cr;
            {
                const uint32_t ra = a_wrec + 32u * (uint32_t)(cl < 0 ? 0 : cl);
                const uint4 c0 = lds_v4(ra), c1 = lds_v4(ra + 16u);
                cr.klo = c0.x; cr.khi = c0.y; cr.idx = c0.z; cr.taken = c0.w;
                cr.x = __uint_as_float(c1.x); cr.y = __uint_as_float(c1.y); cr.z = __uint_as_float(c1.z); cr.pad = 0;
            }
            const uint32_t cr_idx = cl < 0 ? kNone : cr.idx;
            const int n = (int)lds_u32(a_cnt);
            __syncwarp();
            if (lane == 0) sts_u32(a_cnt, 0u);
            const int nsend = n < kR - 1 ? n : kR - 1;
            if (tdbg) { t1 = clock64(); tacc[3] += t1 - t0; t0 = t1; }
            if (C == 1) {
                if (lane < 2 * (1 + nsend)) {
                    const int k = lane >> 1, half = lane & 1;
                    uint4 w;
                    if (k == 0)
                        w = half ? make_uint4(__float_as_uint(cr.x), __float_as_uint(cr.y), __float_as_uint(cr.z), (uint32_t)n)
                                 : make_uint4(cr.klo, cr.khi, cr_idx, cr.taken);
                    else
                        w = lds_v4(a_cand + 32u * (k - 1) + 16u * half);
                    reinterpret_cast<uint4*>(&slots[par][k])[half] = w;
                }
                __syncwarp();
            } else {
                if (lane < (int)C) {
                    const uint32_t rbar = mapa(smem_u32(&bars[par]), (uint32_t)lane);
                    const uint32_t rbase = mapa(smem_u32(&slots[par][r * kR]), (uint32_t)lane);
                    mbar_remote_arrive_expect_tx(rbar, (uint32_t)(1 + nsend) * (uint32_t)sizeof(Rec));
                    st_async_v4(rbase, rbar, cr.klo, cr.khi, cr_idx, cr.taken);
                    st_async_v4(rbase + 16, rbar, __float_as_uint(cr.x), __float_as_uint(cr.y), __float_as_uint(cr.z),
                                (uint32_t)n);
                    for (int k = 0; k < nsend; ++k) {
                        const uint4 w0 = lds_v4(a_cand + 32u * k);
                        const uint4 w1 = lds_v4(a_cand + 32u * k + 16u);
                        st_async_v4(rbase + 32u * (k + 1), rbar, w0.x, w0.y, w0.z, w0.w);
                        st_async_v4(rbase + 32u * (k + 1) + 16, rbar, w1.x, w1.y, w1.z, w1.w);
                    }
                }
            }
            if (tdbg) { t1 = clock64(); tacc[4] += t1 - t0; t0 = t1; }
            if (C > 1) mbar_wait_cta(&bars[par], phase);
            if (tdbg) { t1 = clock64(); tacc[5] += t1 - t0; t0 = t1; }

            // D. headers in lanes < C; candidates compacted one per lane
            const uint32_t a_sl = smem_u32(slots[par]);
            uint64_t hk = 0;
            uint32_t hidx = kNone, ht = 0;
            float hx = 0.f, hy = 0.f, hz = 0.f;
            int hcnt = 0;
            if (lane < (int)C) {
                const uint4 h0 = lds_v4(a_sl + 32u * (lane * kR));
                const uint4 h1 = lds_v4(a_sl + 32u * (lane * kR) + 16u);
                hk = ((uint64_t)h0.y << 32) | h0.x;
                hidx = h0.z; ht = h0.w;
                hx = __uint_as_float(h1.x); hy = __uint_as_float(h1.y); hz = __uint_as_float(h1.z);
                hcnt = (int)h1.w;
            }
            bool overflow = __any_sync(kFull, hcnt > kR - 1);
            const int hn = hcnt < kR - 1 ? hcnt : kR - 1;  // prefix sum from one ballot per bit of kR - 1
            static_assert(kR - 1 < 16, "four ballots");
            const uint32_t lt = (1u << lane) - 1u;
            const uint32_t b0 = __ballot_sync(kFull, hn & 1), b1 = __ballot_sync(kFull, hn & 2),
                           b2 = __ballot_sync(kFull, hn & 4), b3 = kR - 1 > 7 ? __ballot_sync(kFull, hn & 8) : 0u;
            const int base = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt) + 8 * __popc(b3 & lt);
            const int ncand_all = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2) + 8 * __popc(b3);
            for (int k = 0; k < hn; ++k)
                if (base + k < 32) sts_u8(a_map + base + k, (uint32_t)(lane * kR + 1 + k));
            overflow = overflow || ncand_all > 32;
            const int ncand = ncand_all < 32 ? ncand_all : 32;
            __syncwarp();
            double cm = 0.0;
            uint32_t ci = kNone, ct = 0;
            float cx = 0.f, cy = 0.f, cz = 0.f;
            if (lane < ncand) {
                const int j = (int)lds_u8(a_map + lane);
                const uint4 c0 = lds_v4(a_sl + 32u * j);
                const uint4 c1 = lds_v4(a_sl + 32u * j + 16u);
                cm = bitsd(((uint64_t)c0.y << 32) | c0.x);
                ci = c0.z; ct = c0.w;
                cx = __uint_as_float(c1.x); cy = __uint_as_float(c1.y); cz = __uint_as_float(c1.z);
            }
            // a taken candidate (resumed state only) would need the fallback: no speculation
            overflow = overflow || __any_sync(kFull, lane < ncand && ct);
            bool alive = lane < ncand;
            // float32 screen bound of my candidate's md (as the fold's): a pick
            // whose float32 distance exceeds it cannot lower md
            float cthr = alive ? skip_threshold(cm) : -1.0f;
            // lower my candidate by the pick at (sx, sy, sz): float32 screen,
            // the exact float64 update only where the screen cannot exclude it
            auto lower_by = [&](float sx, float sy, float sz) {
                const float dx = cx - sx, dy = cy - sy, dz = cz - sz;
                const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                const bool need = alive && !(d32 > cthr);
                if (__any_sync(kFull, need)) {
                    const double d = sqdist((double)sx, (double)sy, (double)sz, (double)cx, (double)cy, (double)cz);
                    if (need && dbits(d) < dbits(cm)) {
                        cm = d;
                        cthr = skip_threshold_d32(d, d32);
                    }
                }
            };
            if (tdbg) { t1 = clock64(); tacc[0] += t1 - t0; t0 = t1; }
            __syncwarp();
            if (tdbg) { t1 = clock64(); tacc[6] += t1 - t0; t0 = t1; }

            // E. speculation.  First pick: the global max over the CTA maxima
            // (and candidates); later picks: candidates only, while they stay
            // above the threshold every other point is below.
            int rnl = 0, fb = 0;
            int64_t itl = it;
            if (itl < k_stop) {
                const bool hv = hidx != kNone;
                const bool use_c = alive && (!hv || ranks_above(dbits(cm), ci, hk, hidx));
                const uint64_t k0 = use_c ? dbits(cm) : hk;
                const uint32_t i0 = use_c ? ci : (hv ? hidx : kNone);
                const int wl = warp_argmax_lane(k0, i0);
                if (wl >= 0) {
                    const uint64_t wk = __shfl_sync(kFull, k0, wl);
                    const uint32_t wi = __shfl_sync(kFull, i0, wl);
                    const uint32_t wt = __shfl_sync(kFull, use_c ? ct : ht, wl);
                    const float sx = __shfl_sync(kFull, use_c ? cx : hx, wl);
                    const float sy = __shfl_sync(kFull, use_c ? cy : hy, wl);
                    const float sz = __shfl_sync(kFull, use_c ? cz : hz, wl);
                    const double wm = bitsd(wk);
                    if (!(wm > 0.0) || wt) {
                        fb = 1;
                        if (lane == 0) {
                            Rec w{};
                            w.klo = (uint32_t)wk; w.khi = (uint32_t)(wk >> 32); w.idx = wi;
                            w.x = sx; w.y = sy; w.z = sz;
                            fbw_s = w;
                        }
                    } else {
                        if (lane == 0) {
                            sts_v4(a_run, make_uint4(__float_as_uint(sx), __float_as_uint(sy), __float_as_uint(sz), wi));
                            sts_f64(a_hist + 8u * (hc & 31), wm);
                            st_release_cta(&pub_s, tag | 1u);
                        }
                        ++itl;
                        rnl = 1;
                        alive = alive && ci != wi && !overflow;
                        lower_by(sx, sy, sz);
                    }
                }
            }
            if (tdbg) { t1 = clock64(); tacc[7] += t1 - t0; t0 = t1; }
            // later picks: the best candidate while it clears the threshold
            while (rnl > 0 && itl < k_stop && rnl < kRunMax) {
                alive = alive && dbits(cm) >= tau;
                const int wl = warp_argmax_lane(alive ? dbits(cm) : 0ull, alive ? ci : kNone);
                if (wl < 0) break;
                const bool win = lane == wl;
                const float sx = __shfl_sync(kFull, cx, wl);
                const float sy = __shfl_sync(kFull, cy, wl);
                const float sz = __shfl_sync(kFull, cz, wl);
                if (win) {
                    sts_v4(a_run + 16u * rnl, make_uint4(__float_as_uint(cx), __float_as_uint(cy), __float_as_uint(cz), ci));
                    sts_f64(a_hist + 8u * ((hc + rnl) & 31), cm);
                    st_release_cta(&pub_s, tag | (uint32_t)(rnl + 1));
                }
                alive = alive && !win;
                lower_by(sx, sy, sz);  // the reference's update of every other candidate
                ++itl;
                ++rnl;
            }
            const int hbase = hc;
            hc += rnl;
            __syncwarp();
            const int ctot = ncand_all;
            if (tdbg) { t1 = clock64(); tacc[8] += t1 - t0; t0 = t1; tsp += rnl; }

            // next threshold: the curve is non-increasing; aim kTarget samples
            // ahead along its recent slope, gain corrected by the observed count
            const double target = a.spec_target != 0.0 ? a.spec_target : kTarget;  // PS_SPEC_TARGET
            if (tau != kTauOff && !tau_boot) {  // a bootstrap threshold says nothing about the gain
                if (overflow || ctot > (int)(2 * target)) gain *= 0.7f;
                else if (ctot < (int)(target / 2)) gain *= 1.3f;
                gain = fminf(fmaxf(gain, 0.05f), 20.0f);
            }
            uint64_t tnew = kTauOff;
            tau_boot = hc < 3 && target > 0.0;
            if (tau_boot) {
                // no curve history yet: the third-largest CTA maximum of this
                // exchange (a few candidates per exchange until the slope exists)
                uint64_t hk2 = hidx != kNone ? hk : 0ull;
                uint32_t hi2 = hidx;
#pragma unroll
                for (int rep3 = 0; rep3 < 3; ++rep3) {
                    const int wl = warp_argmax_lane(hk2, hi2);
                    if (wl < 0) { hk2 = 0ull; break; }
                    const uint64_t top = __shfl_sync(kFull, hk2, wl);
                    if (rep3 == 2) { tnew = top > 0ull ? top : kTauOff; break; }
                    if (lane == wl) { hk2 = 0ull; hi2 = kNone; }
                }
            }
            if (hc >= 3 && target > 0.0) {
                const int L = hc - 1 < 16 ? hc - 1 : 16;
                const double m0 = lds_f64(a_hist + 8u * ((hc - 1) & 31));
                const double mL = lds_f64(a_hist + 8u * ((hc - 1 - L) & 31));
                const double stepv = fmax((mL - m0) * (double)__frcp_rn((float)L), m0 * 2.44140625e-4);
                const double tv = m0 - (double)gain * target * stepv;
                if (tv > 0.0 && tv < kInf) tnew = dbits(tv);
            }
            if (lane == 0) tau_s = tnew;
            pw = tag | (uint32_t)rnl | 0x100u | ((uint32_t)fb << 9);
            __syncwarp();
            if (lane == 0) st_release_cta(&pub_s, pw);
            if (tdbg) { t1 = clock64(); tacc[9] += t1 - t0; t0 = t1; }
            // the run's out / curve entries, one store batch (after the
            // release stores, so no publish waits on global stores)
            if (r == 0 && lane < rnl) {
                out[it + lane] = (int64_t)lds_u32(a_run + 16u * lane + 12u);
                curve[it + lane] = lds_f64(a_hist + 8u * ((hbase + lane) & 31));
            }
            if (kLeadPts) {  // the lead's own points
                for (int k = 0; k < rnl; ++k) {
                    const uint4 rv = lds_v4(a_run + 16u * k);
                    fold_one(__uint_as_float(rv.x), __uint_as_float(rv.y), __uint_as_float(rv.z), rv.w,
                             it + k < k_stop - 1);
                }
            }
        return pw;
    };
    // the warp's record (thread maxima -> warp argmax -> wrec) and its skip
    // bound: in phase B, or earlier while a worker waits for the next pick
    // (only after this exchange's first pick: the lead has read wrec by then)
    auto refresh_record = [&]() {
        wthr = warp_thr_max();
        if (__any_sync(kFull, dirty)) {
            double tv0;
            int ti0;
            if constexpr (P >= 10) {
                // many points per thread: a running maximum (three live
                // registers instead of the tree's 3P)
                tv0 = -1.0;
                ti0 = 0;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const double v = ((valid >> q) & 1u) ? mget(q) : -1.0;
                    bool take = v > tv0;
                    if (v == tv0 && v >= 0.0) take = oid(q) < oid(ti0);  // lowest index
                    if (take) { tv0 = v; ti0 = q; }
                }
            } else {
                double tv[P];
                int ti[P];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    tv[q] = ((valid >> q) & 1u) ? mget(q) : -1.0;
                    ti[q] = q;
                }
#pragma unroll
                for (int st = 1; st < P; st <<= 1) {
#pragma unroll
                    for (int q = 0; q + st < P; q += 2 * st) {
                        bool take = tv[q + st] > tv[q];
                        if (tv[q + st] == tv[q] && tv[q] >= 0.0) take = oid(ti[q + st]) < oid(ti[q]);  // lowest index
                        if (take) { tv[q] = tv[q + st]; ti[q] = ti[q + st]; }
                    }
                }
                tv0 = tv[0];
                ti0 = ti[0];
            }
            if (dirty) {
                bv = tv0;
                bq = ti0;
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (q == bq) { bx = fx[q]; by = fy[q]; bz = fz[q]; }
            }
            dirty = false;
        }
        const uint64_t bkey = bv >= 0.0 ? dbits(bv) : 0ull;
        const uint32_t bidx = bv >= 0.0 ? oid(bq) : kNone;
        const int wl = warp_argmax_lane(bkey, bidx);
        if (wl < 0) {
            if (lane == 0) sts_v4(a_wrec + 32u * warp, make_uint4(0u, 0u, kNone, 0u));
        } else if (lane == wl) {
            sts_v4(a_wrec + 32u * warp, make_uint4((uint32_t)bkey, (uint32_t)(bkey >> 32), bidx, (tk >> bq) & 1u));
            sts_v4(a_wrec + 32u * warp + 16u,
                   make_uint4(__float_as_uint(bx), __float_as_uint(by), __float_as_uint(bz), 0u));
        }
        stale = false;
    };
    auto worker_step = [&](uint32_t tag) -> uint32_t {
        uint32_t pw = 0;
        // fold each pick as soon as the lead warp publishes it
        int k = 0;
        while (true) {
            pw = ld_acquire_cta(&pub_s);
            const int n = (pw & 0xffff0000u) == tag ? (int)(pw & 0xffu) : 0;
            if (kTiming && wdbg && (pw & 0xffff0000u) == tag && (pw & 0x100u) && w_tdone == 0) {
                w_tdone = clock64();
                wacc[1] += n - k;
            }
            if (n <= k && !((pw & 0xffff0000u) == tag && (pw & 0x100u))) {
                // nothing new: refresh the warp's record if a fold changed
                // it (off the critical path), else back off so the lead
                // warp's shared-memory traffic is not queued behind the polls
                if (kEagerRec && P >= 10 && stale && k > 0) {
                    refresh_record();
                    continue;
                }
                __nanosleep(poll_ns);
                continue;
            }
            for (; k < n; ++k) {
                const uint4 rv = lds_v4(a_run + 16u * k);
                fold_one(__uint_as_float(rv.x), __uint_as_float(rv.y), __uint_as_float(rv.z), rv.w,
                         it + k < k_stop - 1);
            }
            if ((pw & 0xffff0000u) == tag && (pw & 0x100u)) break;
        }
        return pw;
    };
    if (!kLeadPts && warp == kLead) {
        while (it < k_stop) {
            const uint32_t par = ex & 1u, phase = (ex >> 1) & 1u;
            ++ex;
            long long t0 = 0, t1 = 0;
            if (tdbg) t0 = clock64();
            // B: no points -- an empty warp record
            if (lane == 0) sts_v4(a_wrec + 32u * warp, make_uint4(0u, 0u, kNone, 0u));
            if (tdbg) { t1 = clock64(); tacc[1] += t1 - t0; t0 = t1; }
            __syncthreads();
            if (tdbg) { t1 = clock64(); tacc[2] += t1 - t0; t0 = t1; }
            const uint32_t tag = (ex & 0xffffu) << 16;
            uint32_t pw = lead_step(tag, par, phase, t0, t1);
            pw = __shfl_sync(kFull, pw, 0);
            const int rn = (int)(pw & 0xffu);
            it += rn;
            tau = tau_s;

            if (pw & 0x200u) {
                // duplicate fallback, lead side (see the workers' loop)
                __syncthreads();  // wrec reuse
                if (lane == 0) { Rec z{}; z.idx = kNone; wrec[warp] = z; }
                __syncthreads();
                cluster_sync_all();
                const Rec fw = warp_min_idx_recs(fb_slots, (int)C, lane);
                Rec w = fbw_s;  // no untaken point left: the argmax stands
                if (fw.idx != kNone) w = fw;
                cluster_sync_all();  // fb_slots / wrec free again
                if (writer) {
                    out[it] = (int64_t)w.idx;
                    curve[it] = bitsd(rec_key(w));
                }
                if (lane == 0) hist_s[hc & 31] = bitsd(rec_key(w));
                ++hc;
                ++it;
            }
        }
    } else {
        while (it < k_stop) {
            const uint32_t par = ex & 1u, phase = (ex >> 1) & 1u;
            ++ex;
            long long t0 = 0, t1 = 0;
            if (tdbg) t0 = clock64();

            long long wb0 = 0;
            if (kTiming && wdbg) wb0 = clock64();
            // B. thread max (cached), threshold candidates, warp argmax; the
            // warp's skip bound for the next exchange's folds (thr only falls)
            if (stale) refresh_record();  // else the record written while polling stands
            {
                uint32_t cm = 0;
    #pragma unroll
                for (int q = 0; q < P; ++q) cm |= ((((valid >> q) & 1u) && dbits(mget(q)) >= tau) ? 1u : 0u) << q;
                if (__any_sync(kFull, cm != 0)) {
    #pragma unroll
                    for (int q = 0; q < P; ++q) {
                        if ((cm >> q) & 1u) {
                            const int slot = atomicAdd(&cnt_s, 1);
                            if (slot < kR - 1) {
                                const uint64_t kq = dbits(mget(q));
                                const uint32_t ca = a_cand + 32u * (uint32_t)slot;
                                sts_v4(ca, make_uint4((uint32_t)kq, (uint32_t)(kq >> 32), oid(q), (tk >> q) & 1u));
                                sts_v4(ca + 16u, make_uint4(__float_as_uint(fx[q]), __float_as_uint(fy[q]),
                                                             __float_as_uint(fz[q]), 0u));
                            }
                        }
                    }
                }
            }
            if (tdbg) { t1 = clock64(); tacc[1] += t1 - t0; t0 = t1; }
            if (kTiming && wdbg) {
                const long long wn = clock64();
                wacc[2] += wn - wb0;
                if (w_tdone) wacc[0] += wn - w_tdone;
                w_tdone = 0;
            }
            __syncthreads();
            if (tdbg) { t1 = clock64(); tacc[2] += t1 - t0; t0 = t1; }
            const uint32_t tag = (ex & 0xffffu) << 16;
            uint32_t pw = (kLeadPts && warp == kLead) ? lead_step(tag, par, phase, t0, t1) : worker_step(tag);
            pw = __shfl_sync(kFull, pw, 0);
            const int rn = (int)(pw & 0xffu);
            it += rn;
            tau = tau_s;

            if (pw & 0x200u) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken index
                uint32_t fidx = kNone;
                Rec fr{};
    #pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (((valid >> q) & 1u) && !((tk >> q) & 1u) && oid(q) < fidx) {
                        fidx = oid(q);
                        const uint64_t kk = dbits(mget(q));
                        fr.klo = (uint32_t)kk; fr.khi = (uint32_t)(kk >> 32);
                        fr.x = fx[q]; fr.y = fy[q]; fr.z = fz[q];
                    }
                }
                fr.idx = fidx;
                const uint32_t wmin = __reduce_min_sync(kFull, fidx);
                __syncthreads();  // wrec reuse
                if (fidx == wmin && fidx != kNone) wrec[warp] = fr;
                else if (lane == 0 && wmin == kNone) { Rec z{}; z.idx = kNone; wrec[warp] = z; }
                __syncthreads();
                if (warp == 0) {
                    const Rec cr = warp_min_idx_recs(wrec, kW, lane);
                    if (lane < (int)C) {
                        const uint32_t dst = mapa(smem_u32(&fb_slots[r]), lane);
                        st_cluster_u64(dst, ((uint64_t)cr.khi << 32) | cr.klo);
                        st_cluster_u64(dst + 8, ((uint64_t)cr.taken << 32) | cr.idx);
                        st_cluster_u64(dst + 16, ((uint64_t)__float_as_uint(cr.y) << 32) | __float_as_uint(cr.x));
                        st_cluster_u64(dst + 24, (uint64_t)__float_as_uint(cr.z));
                    }
                }
                cluster_sync_all();
                const Rec fw = warp_min_idx_recs(fb_slots, (int)C, lane);
                Rec w = fbw_s;  // no untaken point left: the argmax stands
                if (fw.idx != kNone) w = fw;
                cluster_sync_all();  // fb_slots / wrec free again
                if (writer) {
                    out[it] = (int64_t)w.idx;
                    curve[it] = bitsd(rec_key(w));
                }
                if (warp == kLead) {
                    if (lane == 0) hist_s[hc & 31] = bitsd(rec_key(w));
                    ++hc;
                }
                fold_one(w.x, w.y, w.z, w.idx, it < k_stop - 1);
                stale = true;  // wrec now holds the fallback records
                ++it;
            }
        }
        if (kTiming && wdbg)
            for (int i = 0; i < 5; ++i) a.dbg[12 + i] = wacc[i];
        // ---- write back md / taken; curve = sqrt(best) (_kernels.py:72) ---------
    #pragma unroll
        for (int q = 0; q < P; ++q) {
            if ((valid >> q) & 1u) {
                const int64_t j = oid(q);
                md[j] = mget(q);
                taken[j] = (tk >> q) & 1u;
            }
        }
    }

    if (tdbg) {
        a.dbg[0] = ex;
        a.dbg[1] = tsp;
        for (int i = 0; i < 10; ++i) a.dbg[2 + i] = tacc[i];
    }

    if (r == 0 && k_start < k_stop) {
        __syncthreads();
        for (int64_t i = k_start + tid; i < k_stop; i += T) curve[i] = sqrt(curve[i]);
    }
    cluster_sync_all();
}

template <int P, int T, bool kLeadPts>
cudaError_t launch_spec(const FpsArgs& a, int64_t B, int C, cudaStream_t s) {
    auto kern = fps_spec_kernel<P, T, kLeadPts>;
    cudaError_t e = cudaSuccess;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    // sort arrays (4 B per slot) + md in shared memory for P >= 10 (8 B per slot)
    const size_t dyn = (P >= 10 ? 12 : 4) * (size_t)spec_slots(P, T, kLeadPts);
    static bool dyn_set = false;
    if (!dyn_set) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
        dyn_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * C), 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

// Same cluster plan as the one-sample kernel (fps_choose_cluster); clouds
// that do not fit the cluster's registers (P == 0) are not handled here.
cudaError_t launch_fps_spec(FpsArgs a, int64_t B, cudaStream_t s) {
    int C = 1, P = 0, T = 256;
    fps_choose_cluster(a.N, B, &C, &P, &T);
    if (getenv("PS_SPEC_C")) { C = atoi(getenv("PS_SPEC_C")); P = 1; }  // development override (A/B)
    if (P == 0) return cudaErrorNotSupported;
    // clouds of one or two CTAs: the one-sample kernel has no cluster
    // exchange to amortise and is faster (profiles/r01/fps_spec.log: 0.65-0.86
    // vs 0.9-1.7 us per iteration up to N = 2048; from C = 4 speculation wins
    // up to 2.2x); PS_FPS_SPEC=1 forces speculation
    if (C <= 2 && !getenv("PS_FPS_SPEC")) return cudaErrorNotSupported;
    // one warp per CTA leads the exchange and owns no points (below)
    const int64_t S = (a.N + C - 1) / C;
    // 512 threads, 15 worker warps, P <= 10 points per thread: up to 4800
    // points per CTA without points on the lead warp.  The lead runs its own
    // loop (its registers and the workers' points do not add up) and from
    // P = 10 md lives in shared memory, so P = 10 fits 128 registers without
    // spills (profiles/r02/fps_pmax.log: C3 throughput width 6 -> 5 CTAs)
    P = 0;
    T = 512;
    // up to 10 points per thread spill-free (md in shared memory from P = 10);
    // 11-13 compile with small spills (development: PS_SPEC_PMAX)
    static const int pmax = getenv("PS_SPEC_PMAX") ? atoi(getenv("PS_SPEC_PMAX")) : 10;
    for (int p : {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13})
        if (!P && (int64_t)p * (T - 32) >= S && p <= pmax) P = p;
    // up to 4096 points per CTA: the lead warp owns points as well
    const bool lead_pts = P == 0 && S <= 8 * 512;
    if (lead_pts) { P = 8; T = 512; }
    if (P == 0) return cudaErrorNotSupported;
    a.points_per_cta = S;
    a.dbg = nullptr;
    a.spec_target = getenv("PS_SPEC_TARGET") ? atof(getenv("PS_SPEC_TARGET")) : 0.0;  // development override
    a.poll_ns = getenv("PS_SPEC_POLL_NS") ? atoi(getenv("PS_SPEC_POLL_NS")) : 0;        // development override
    static long long* dbg = nullptr;
    const bool timing = kTiming && getenv("PS_FPS_TIMING");
    if (timing) {
        // development aid (make TIMING=1): exchanges, samples taken by
        // speculation and per-phase SM cycles of cloud 0 / CTA 0 / lead lane 0
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 17);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 17, s);
        a.dbg = dbg;
    }
    if (getenv("PS_FPS_VERBOSE"))
        fprintf(stderr, "[fps-spec] N=%lld B=%lld C=%d P=%d T=%d lead_pts=%d\n", (long long)a.N, (long long)B, C, P,
                T, (int)lead_pts);
    cudaError_t e = cudaErrorNotSupported;
#define PS_SPEC_CASE(PP, TT) \
    case PP: e = launch_spec<PP, TT, false>(a, B, C, s); break;
    if (lead_pts) return launch_spec<8, 512, true>(a, B, C, s);
    switch (P) {
        PS_SPEC_CASE(1, 512)
        PS_SPEC_CASE(2, 512)
        PS_SPEC_CASE(3, 512)
        PS_SPEC_CASE(4, 512)
        PS_SPEC_CASE(5, 512)
        PS_SPEC_CASE(6, 512)
        PS_SPEC_CASE(7, 512)
        PS_SPEC_CASE(8, 512)
        PS_SPEC_CASE(9, 512)
        PS_SPEC_CASE(10, 512)
        PS_SPEC_CASE(11, 512)
        PS_SPEC_CASE(12, 512)
        PS_SPEC_CASE(13, 512)
        default: break;
    }
#undef PS_SPEC_CASE
    if (timing && e == cudaSuccess) {
        long long h[17];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const double nx = h[0] > 0 ? (double)h[0] : 1.0;
        fprintf(stderr, "[fps-spec timing] C=%d P=%d T=%d N=%lld iters=%lld exchanges=%lld taken/ex=%.2f "
                "cycles/ex: compact %.0f max+cand %.0f bar1 %.0f ctamax %.0f send %.0f wait %.0f gather %.0f pick0 %.0f "
                "picks %.0f tau+publish %.0f\n",
                C, P, T, (long long)a.N, (long long)(a.k_stop - a.k_start), h[0], (double)h[1] / nx,
                h[2] / nx, h[3] / nx, h[4] / nx, h[5] / nx, h[6] / nx, h[7] / nx, h[8] / nx, h[9] / nx, h[10] / nx,
                h[11] / nx);
        fprintf(stderr, "[fps-spec timing] worker warp 0 per exchange: end-of-run -> barrier %.0f cycles, unfolded picks "
                "at the end %.2f, phase B %.0f cycles; folds run %.1f of %.1f (whole-warp skip %.0f %%)\n",
                h[12] / nx, h[13] / nx, h[14] / nx, h[15] / nx, h[16] / nx,
                h[16] > 0 ? 100.0 * (1.0 - (double)h[15] / (double)h[16]) : 0.0);
    }
    return e;
}

}  // namespace ps
