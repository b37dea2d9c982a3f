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
// Layout: C CTAs of T threads per cloud.  Warps 0..kW-2 own P points per
// thread in registers (float32 xyz, float64 md, taken bits); the last warp
// (the lead) owns none and runs, per exchange:
//   C. CTA argmax over the warp records + the CTA's candidates (<= kR-1),
//      pushed to every CTA with st.async; each sender announces its byte
//      count on the peer's mbarrier (remote arrive.expect_tx);
//   D. headers in lanes < C, candidates compacted one per lane, and their
//      pairwise float64 distances in shared memory (dm_s);
//   E. picks: the first over headers + candidates, then the best candidate
//      while >= tau, each lowering the others by its dm_s row.  Each pick is
//      published to the CTA (release store); the worker warps fold it into
//      their md as soon as it appears, overlapping the lead's serial chain.
//   tau for the next exchange: kTarget samples ahead along the recent curve
//   slope (the curve is non-increasing), gain-corrected by the count seen.
// The duplicate fallback of _kernels.py:65-70 (max <= 0 or winner already
// taken -> lowest untaken index) runs as a cluster-wide exchange when the
// first pick needs it; a later pick that would need it ends the run.
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

constexpr int kR = 8;             // records per CTA per exchange: its max + kR-1 threshold candidates
constexpr int kRunMax = 31;       // samples per exchange (one lane each)
constexpr double kTarget = 22.0;  // threshold candidates aimed for per exchange
constexpr uint64_t kTauOff = ~0ull;  // threshold disabled (above every md bit pattern)

template <int P, int T>
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
    constexpr int TW = T - 32;  // point-owning (worker) threads
    __shared__ Rec wrec[kW];
    __shared__ Rec cand[kR - 1];
    __shared__ Rec slots[2][kMaxCluster * kR];
    __shared__ Rec fb_slots[kMaxCluster];
    __shared__ Rec fbw_s;
    __shared__ float4 run_s[32];
    __shared__ uint8_t map_s[kMaxCluster * kR];
    __shared__ double hist_s[32];
    __shared__ double dm_s[32 * 32];  // candidate pair distances, row = picked candidate
    __shared__ unsigned long long tau_s;
    __shared__ int cnt_s;
    __shared__ uint32_t pub_s;
    __shared__ __align__(8) uint64_t bars[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool worker = warp != kLead;
    const int wt = tid;  // worker thread index
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

    // ---- state into registers (as fps.cu) ---------------------------------
    float fx[P], fy[P], fz[P], thr[P];
    double m[P];
    uint32_t tk = 0, valid = 0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int64_t j = lo + wt + (int64_t)q * TW;
        fx[q] = fy[q] = fz[q] = 0.f;
        m[q] = 0.0;
        if (worker && j < hi) {
            valid |= 1u << q;
            const float4 v = xyz[j];
            fx[q] = v.x; fy[q] = v.y; fz[q] = v.z;
            if (a.fresh) {
                m[q] = kInf;
                tk |= (j == seed ? 1u : 0u) << q;
            } else {
                m[q] = md[j];
                tk |= (taken[j] ? 1u : 0u) << q;
            }
        }
        thr[q] = ((valid >> q) & 1u) ? skip_threshold(m[q]) : -1.0f;
    }
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
    if (warp == kLead && !a.fresh && k_start < k_stop) {
        const int nh = k_start - 1 >= 32 ? 32 : (k_start - 1 > 0 ? (int)(k_start - 1) : 0);
        if (lane < nh) {
            const double c = curve[k_start - 1 - lane];  // previous call's epilogue stored sqrt
            hist_s[(nh - 1 - lane) & 31] = c * c;
        }
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
    auto fold_one = [&](float sx32, float sy32, float sz32, uint32_t sidx, bool do_fold) {
        const uint32_t o32 = (uint32_t)((int64_t)sidx - lo - wt);  // wraps below lo
        if (o32 < (uint32_t)(P * TW) && o32 % TW == 0) tk |= 1u << (o32 / TW);
        if (!do_fold) return;
        uint32_t need = 0;
        float d32s[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const float dx = fx[q] - sx32, dy = fy[q] - sy32, dz = fz[q] - sz32;
            const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            d32s[q] = d32;
            need |= (!(d32 > thr[q]) ? 1u : 0u) << q;
        }
        if (__any_sync(kFull, need != 0)) {
            const double sx = sx32, sy = sy32, sz = sz32;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                if (__any_sync(kFull, (need >> q) & 1u)) {
                    const double d = sqdist(sx, sy, sz, (double)fx[q], (double)fy[q], (double)fz[q]);
                    if (((need >> q) & 1u) && dbits(d) < dbits(m[q])) {
                        m[q] = d;
                        thr[q] = skip_threshold_d32(d, d32s[q]);
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

    uint32_t ex = 0;
    const bool tdbg = kTiming && a.dbg && b == 0 && r == 0 && warp == kLead && lane == 0;
    long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tsp = 0;
    while (it < k_stop) {
        const uint32_t par = ex & 1u, phase = (ex >> 1) & 1u;
        ++ex;
        long long t0 = 0, t1 = 0;
        if (tdbg) t0 = clock64();

        // B. thread max (cached), threshold candidates, warp argmax
        if (__any_sync(kFull, dirty)) {
            double tv[P];
            int ti[P];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                tv[q] = ((valid >> q) & 1u) ? m[q] : -1.0;
                ti[q] = q;
            }
#pragma unroll
            for (int st = 1; st < P; st <<= 1) {
#pragma unroll
                for (int q = 0; q + st < P; q += 2 * st)
                    if (tv[q + st] > tv[q]) { tv[q] = tv[q + st]; ti[q] = ti[q + st]; }
            }
            if (dirty) {
                bv = tv[0];
                bq = ti[0];
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (q == bq) { bx = fx[q]; by = fy[q]; bz = fz[q]; }
            }
            dirty = false;
        }
        {
            uint32_t cm = 0;
#pragma unroll
            for (int q = 0; q < P; ++q) cm |= ((((valid >> q) & 1u) && dbits(m[q]) >= tau) ? 1u : 0u) << q;
            if (__any_sync(kFull, cm != 0)) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if ((cm >> q) & 1u) {
                        const int slot = atomicAdd(&cnt_s, 1);
                        if (slot < kR - 1) {
                            const uint64_t kq = dbits(m[q]);
                            uint4* c4 = reinterpret_cast<uint4*>(&cand[slot]);
                            c4[0] = make_uint4((uint32_t)kq, (uint32_t)(kq >> 32),
                                               (uint32_t)(lo + wt + (int64_t)q * TW), (tk >> q) & 1u);
                            c4[1] = make_uint4(__float_as_uint(fx[q]), __float_as_uint(fy[q]), __float_as_uint(fz[q]), 0u);
                        }
                    }
                }
            }
            const uint64_t bkey = bv >= 0.0 ? dbits(bv) : 0ull;
            const uint32_t bidx = bv >= 0.0 ? (uint32_t)(lo + wt + (int64_t)bq * TW) : kNone;
            const int wl = warp_argmax_lane(bkey, bidx);
            if (wl < 0) {
                if (lane == 0) { Rec z{}; z.idx = kNone; wrec[warp] = z; }
            } else if (lane == wl) {
                uint4* w4 = reinterpret_cast<uint4*>(&wrec[warp]);
                w4[0] = make_uint4((uint32_t)bkey, (uint32_t)(bkey >> 32), bidx, (tk >> bq) & 1u);
                w4[1] = make_uint4(__float_as_uint(bx), __float_as_uint(by), __float_as_uint(bz), 0u);
            }
        }
        if (tdbg) { t1 = clock64(); tacc[1] += t1 - t0; t0 = t1; }
        __syncthreads();
        if (tdbg) { t1 = clock64(); tacc[2] += t1 - t0; t0 = t1; }

        // published word: exchange tag << 16 | fallback << 9 | done << 8 | picks
        const uint32_t tag = (ex & 0xffffu) << 16;
        uint32_t pw;
        if (warp == kLead) {
            // C. CTA record set: header (the CTA max, candidate count) and
            // up to kR-1 threshold candidates, pushed to every CTA; each
            // sender announces its byte count on the peer's mbarrier.
            const Rec wr = lane < kW ? wrec[lane] : Rec{0, 0, kNone, 0, 0.f, 0.f, 0.f, 0};
            const int cl = warp_argmax_lane(rec_key(wr), wr.idx);
            const Rec cr = wrec[cl < 0 ? 0 : cl];
            const uint32_t cr_idx = cl < 0 ? kNone : cr.idx;
            const int n = cnt_s;
            __syncwarp();
            if (lane == 0) cnt_s = 0;
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
                        w = reinterpret_cast<const uint4*>(&cand[k - 1])[half];
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
                        const uint4 w0 = reinterpret_cast<const uint4*>(&cand[k])[0];
                        const uint4 w1 = reinterpret_cast<const uint4*>(&cand[k])[1];
                        st_async_v4(rbase + 32u * (k + 1), rbar, w0.x, w0.y, w0.z, w0.w);
                        st_async_v4(rbase + 32u * (k + 1) + 16, rbar, w1.x, w1.y, w1.z, w1.w);
                    }
                }
            }
            if (tdbg) { t1 = clock64(); tacc[4] += t1 - t0; t0 = t1; }
            if (C > 1) mbar_wait_cta(&bars[par], phase);
            if (tdbg) { t1 = clock64(); tacc[5] += t1 - t0; t0 = t1; }

            // D. headers in lanes < C; candidates compacted one per lane
            const Rec* sl = slots[par];
            uint64_t hk = 0;
            uint32_t hidx = kNone, ht = 0;
            float hx = 0.f, hy = 0.f, hz = 0.f;
            int hcnt = 0;
            if (lane < (int)C) {
                const uint4 h0 = reinterpret_cast<const uint4*>(&sl[lane * kR])[0];
                const uint4 h1 = reinterpret_cast<const uint4*>(&sl[lane * kR])[1];
                hk = ((uint64_t)h0.y << 32) | h0.x;
                hidx = h0.z; ht = h0.w;
                hx = __uint_as_float(h1.x); hy = __uint_as_float(h1.y); hz = __uint_as_float(h1.z);
                hcnt = (int)h1.w;
            }
            bool overflow = __any_sync(kFull, hcnt > kR - 1);
            const int hn = hcnt < kR - 1 ? hcnt : kR - 1;  // <= 7: prefix sum from three ballots
            const uint32_t lt = (1u << lane) - 1u;
            const uint32_t b0 = __ballot_sync(kFull, hn & 1), b1 = __ballot_sync(kFull, hn & 2),
                           b2 = __ballot_sync(kFull, hn & 4);
            const int base = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
            const int ncand_all = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
            for (int k = 0; k < hn; ++k)
                if (base + k < 32) map_s[base + k] = (uint8_t)(lane * kR + 1 + k);
            overflow = overflow || ncand_all > 32;
            const int ncand = ncand_all < 32 ? ncand_all : 32;
            __syncwarp();
            double cm = 0.0;
            uint32_t ci = kNone, ct = 0;
            float cx = 0.f, cy = 0.f, cz = 0.f;
            if (lane < ncand) {
                const int j = map_s[lane];
                const uint4 c0 = reinterpret_cast<const uint4*>(&sl[j])[0];
                const uint4 c1 = reinterpret_cast<const uint4*>(&sl[j])[1];
                cm = bitsd(((uint64_t)c0.y << 32) | c0.x);
                ci = c0.z; ct = c0.w;
                cx = __uint_as_float(c1.x); cy = __uint_as_float(c1.y); cz = __uint_as_float(c1.z);
            }
            // a taken candidate (resumed state only) would need the fallback: no speculation
            overflow = overflow || __any_sync(kFull, lane < ncand && ct);
            bool alive = lane < ncand;
            if (tdbg) { t1 = clock64(); tacc[0] += t1 - t0; t0 = t1; }
            // distances between candidates, exactly the float64 update a pick applies
            if (!overflow) {
                const double dcx = cx, dcy = cy, dcz = cz;
                for (int w0 = 0; w0 < ncand; w0 += 8) {  // chunks of 8 independent rows
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float wx = __shfl_sync(kFull, cx, w0 + i);
                        const float wy = __shfl_sync(kFull, cy, w0 + i);
                        const float wz = __shfl_sync(kFull, cz, w0 + i);
                        const double d = sqdist((double)wx, (double)wy, (double)wz, dcx, dcy, dcz);
                        if (alive && w0 + i < ncand) dm_s[(w0 + i) * 32 + lane] = d;
                    }
                }
            }
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
                    const bool wc = __shfl_sync(kFull, use_c ? 1 : 0, wl);
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
                            run_s[0] = make_float4(sx, sy, sz, __uint_as_float(wi));
                            hist_s[hc & 31] = wm;
                            st_release_cta(&pub_s, tag | 1u);
                        }
                        ++itl;
                        rnl = 1;
                        alive = alive && ci != wi && !overflow;
                        if (alive) {
                            const double d = wc ? dm_s[wl * 32 + lane]
                                                : sqdist((double)sx, (double)sy, (double)sz, (double)cx, (double)cy,
                                                         (double)cz);
                            if (dbits(d) < dbits(cm)) cm = d;
                        }
                    }
                }
            }
            if (tdbg) { t1 = clock64(); tacc[7] += t1 - t0; t0 = t1; }
            // Later picks, in rounds: rank the candidates still above the
            // threshold, follow that order with every key updated exactly
            // (dm_s rows, the same float64 values a pick-by-pick loop
            // applies), and accept the order up to the first step at which a
            // later candidate would outrank the pick, or a pick would fall
            // below the threshold.
            // later picks: the best candidate while it clears the threshold;
            // the others' keys are lowered by its dm_s row (the exact float64
            // update the reference applies)
            while (rnl > 0 && itl < k_stop && rnl < kRunMax) {
                alive = alive && dbits(cm) >= tau;
                const int wl = warp_argmax_lane(alive ? dbits(cm) : 0ull, alive ? ci : kNone);
                if (wl < 0) break;
                const bool win = lane == wl;
                const double d = dm_s[wl * 32 + lane];
                if (win) {
                    run_s[rnl] = make_float4(cx, cy, cz, __uint_as_float(ci));
                    hist_s[(hc + rnl) & 31] = cm;
                    st_release_cta(&pub_s, tag | (uint32_t)(rnl + 1));
                }
                alive = alive && !win;
                cm = (alive && dbits(d) < dbits(cm)) ? d : cm;
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
            const double target = kTarget;
            if (tau != kTauOff) {
                if (overflow || ctot > (int)(2 * target)) gain *= 0.7f;
                else if (ctot < (int)(target / 2)) gain *= 1.3f;
                gain = fminf(fmaxf(gain, 0.05f), 20.0f);
            }
            uint64_t tnew = kTauOff;
            if (hc >= 3) {
                const int L = hc - 1 < 16 ? hc - 1 : 16;
                const double m0 = hist_s[(hc - 1) & 31];
                const double mL = hist_s[(hc - 1 - L) & 31];
                const double stepv = fmax((mL - m0) * (double)__frcp_rn((float)L), m0 * 2.44140625e-4);
                const double tv = m0 - (double)gain * target * stepv;
                if (tv > 0.0 && tv < kInf) tnew = dbits(tv);
            }
            if (lane == 0) tau_s = tnew;
            pw = tag | (uint32_t)rnl | 0x100u | ((uint32_t)fb << 9);
            __syncwarp();
            if (lane == 0) st_release_cta(&pub_s, pw);
            if (tdbg) { t1 = clock64(); tacc[8] += t1 - t0; t0 = t1; }
            // the run's out / curve entries, one store batch (after the
            // release stores, so no publish waits on global stores)
            if (r == 0 && lane < rnl) {
                out[it + lane] = (int64_t)__float_as_uint(run_s[lane].w);
                curve[it + lane] = hist_s[(hbase + lane) & 31];
            }
        } else {
            // fold each pick as soon as the lead warp publishes it
            int k = 0;
            while (true) {
                pw = ld_acquire_cta(&pub_s);
                const int n = (pw & 0xffff0000u) == tag ? (int)(pw & 0xffu) : 0;
                if (n <= k && !((pw & 0xffff0000u) == tag && (pw & 0x100u))) {
                    // nothing new: back off so the lead warp's shared-memory
                    // traffic is not queued behind the polls
                    __nanosleep(32);
                    continue;
                }
                for (; k < n; ++k) {
                    const float4 rv = run_s[k];
                    fold_one(rv.x, rv.y, rv.z, __float_as_uint(rv.w), it + k < k_stop - 1);
                }
                if ((pw & 0xffff0000u) == tag && (pw & 0x100u)) break;
            }
        }
        pw = __shfl_sync(kFull, pw, 0);
        const int rn = (int)(pw & 0xffu);
        it += rn;
        tau = tau_s;
        if (tdbg) { t1 = clock64(); tacc[9] += t1 - t0; t0 = t1; }

        if (pw & 0x200u) {
            // duplicate fallback (_kernels.py:65-70): lowest untaken index
            uint32_t fidx = kNone;
            Rec fr{};
#pragma unroll
            for (int q = P - 1; q >= 0; --q) {
                if (((valid >> q) & 1u) && !((tk >> q) & 1u)) {
                    fidx = (uint32_t)(lo + wt + (int64_t)q * TW);
                    const uint64_t kk = dbits(m[q]);
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
            ++it;
        }
    }

    if (tdbg) {
        a.dbg[0] = ex;
        a.dbg[1] = tsp;
        for (int i = 0; i < 10; ++i) a.dbg[2 + i] = tacc[i];
    }

    // ---- write back md / taken; curve = sqrt(best) (_kernels.py:72) ---------
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int64_t j = lo + wt + (int64_t)q * TW;
        if (worker && j < hi) {
            md[j] = m[q];
            taken[j] = (tk >> q) & 1u;
        }
    }
    if (r == 0 && k_start < k_stop) {
        __syncthreads();
        for (int64_t i = k_start + tid; i < k_stop; i += T) curve[i] = sqrt(curve[i]);
    }
    cluster_sync_all();
}

template <int P, int T>
cudaError_t launch_spec(const FpsArgs& a, int64_t B, int C, cudaStream_t s) {
    auto kern = fps_spec_kernel<P, T>;
    cudaError_t e = cudaSuccess;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * C), 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
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
    if (P == 0) return cudaErrorNotSupported;
    // one warp per CTA leads the exchange and owns no points
    const int64_t S = (a.N + C - 1) / C;
    P = 0;
    for (int t : {512, 256}) {
        static const int kP512[] = {1, 2, 3, 4, 5, 6, 7, 8};
        static const int kP256[] = {12, 16};
        const int* ps = t == 512 ? kP512 : kP256;
        const int np = t == 512 ? 8 : 2;
        const int tw = t - 32;
        for (int i = 0; i < np && !P; ++i)
            if ((int64_t)ps[i] * tw >= S) { P = ps[i]; T = t; }
        if (P) break;
    }
    if (P == 0) return cudaErrorNotSupported;
    a.points_per_cta = S;
    a.dbg = nullptr;
    static long long* dbg = nullptr;
    const bool timing = kTiming && getenv("PS_FPS_TIMING");
    if (timing) {
        // development aid (make TIMING=1): exchanges, samples taken by
        // speculation and per-phase SM cycles of cloud 0 / CTA 0 / lead lane 0
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 12);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 12, s);
        a.dbg = dbg;
    }
    if (getenv("PS_FPS_VERBOSE"))
        fprintf(stderr, "[fps-spec] N=%lld B=%lld C=%d P=%d T=%d\n", (long long)a.N, (long long)B, C, P, T);
    cudaError_t e = cudaErrorNotSupported;
#define PS_SPEC_CASE(PP, TT) \
    case PP: e = launch_spec<PP, TT>(a, B, C, s); break;
    switch (P) {
        PS_SPEC_CASE(1, 512)
        PS_SPEC_CASE(2, 512)
        PS_SPEC_CASE(3, 512)
        PS_SPEC_CASE(4, 512)
        PS_SPEC_CASE(5, 512)
        PS_SPEC_CASE(6, 512)
        PS_SPEC_CASE(7, 512)
        PS_SPEC_CASE(8, 512)
        PS_SPEC_CASE(12, 256)
        PS_SPEC_CASE(16, 256)
        default: break;
    }
#undef PS_SPEC_CASE
    if (timing && e == cudaSuccess) {
        long long h[12];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const double nx = h[0] > 0 ? (double)h[0] : 1.0;
        fprintf(stderr, "[fps-spec timing] C=%d P=%d T=%d N=%lld iters=%lld exchanges=%lld taken/ex=%.2f "
                "cycles/ex: compact %.0f max+cand %.0f bar1 %.0f ctamax %.0f send %.0f wait %.0f recv %.0f pick0 %.0f "
                "picks %.0f tau+bar2 %.0f\n",
                C, P, T, (long long)a.N, (long long)(a.k_stop - a.k_start), h[0], (double)h[1] / nx,
                h[2] / nx, h[3] / nx, h[4] / nx, h[5] / nx, h[6] / nx, h[7] / nx, h[8] / nx, h[9] / nx, h[10] / nx,
                h[11] / nx);
    }
    return e;
}

}  // namespace ps
