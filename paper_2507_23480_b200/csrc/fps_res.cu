// fps_res.cu -- K1 v2: exact farthest-point sampling with the cloud resident
// in shared memory, spatially ordered per CTA (B200 / sm_100a).
//
// Replaces _kernels.fps_loop (/root/reference/pkg/src/pointsample/_kernels.py:35-74)
// and its chunked merge fps_update_chunk/first_untaken (:77-100).
//
// One thread-block cluster of C CTAs per cloud (per cloud shard when a cloud
// is split over G ranks, see below).  CTA r of the cluster owns the points
// with original index in [lo, hi) and, at launch, counting-sorts them by a
// 12-bit Morton cell of their own bounding box into shared memory as
// float4 {x, y, z, original index}.  Warp w owns the sorted range
// [w*32P, (w+1)*32P): 32P spatially close points whose bounding box it keeps
// in registers, together with the float64 min-distance md of each of its
// points (registers, P per lane) and its cached argmax record (shared).
//
// Per iteration, with s the last sample:
//   1. warp skip: a rounded-down lower bound of |s - box|^2 above the warp's
//      skip threshold (>= max md of the warp) proves that no md in the warp
//      can decrease -- the warp does nothing and its record stays valid;
//   2. touched warps: float32 screen per point, exact float64 fold
//      ((dx*dx + dy*dy) + dz*dz, no FMA, _kernels.py:55-60) where the screen
//      cannot exclude an update; if an md changed, the thread max and the
//      warp argmax (max md, lowest ORIGINAL index) are recomputed;
//   3. the leader warp waits for the others on a named barrier (they do not
//      wait), reduces the warp records and pushes the CTA record to every
//      CTA of the cluster with st.async + mbarrier complete_tx;
//   4. every warp reduces the C records identically (max md, lowest index);
//   5. with G > 1 ranks, CTA 0 of every rank publishes the cluster record to
//      every rank's global mailbox (peer memory over NVLink, or the same GPU
//      for virtual ranks), each CTA's leader polls the G records of this
//      iteration (sequence-tagged 16-byte halves) and broadcasts the winner.
// The duplicate fallback of _kernels.py:65-70 (max <= 0 or winner taken ->
// lowest untaken index) is a rare second exchange with the same structure.
//
// kSpec (default; PS_RES_NOSPEC=1 selects the loop above): the speculation of
// fps_spec.cu at rank scale -- per exchange every CTA publishes its argmax and
// its points with md >= tau, CTA 0 of each rank forwards the rank's header and
// candidates to every rank's mailbox, and every lead warp picks the same run
// (first pick = max over the headers, later picks = candidates still >= tau,
// lowered by exact float64 distances).  C5 (2^20 -> 65536 over 10 virtual
// ranks on one B200): 5.5 -> 1.07 us per sample.
//
// Bit-exactness: every md is the reference float64 value; the float32 tests
// only skip folds that provably cannot change md (margins in common.cuh /
// skip_threshold); ties resolve to the lowest original index at every level,
// so any partition of the cloud gives the reference's choice.

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

namespace {

constexpr int kT = 512;
constexpr int kW = kT / 32;
constexpr int kMaxC = 16;
constexpr int kBins = 4096;  // 16^3 Morton cells per CTA bounding box
constexpr uint32_t kNone = 0xffffffffu;
constexpr int kMaxP = 24;
#ifndef PS_TIMING
#define PS_TIMING 0
#endif
constexpr bool kTiming = PS_TIMING;  // per-iteration cycle stamps (make TIMING=1)
constexpr uint32_t kForeign = 0x7fffffffu;  // owner field of another rank's point (g field all ones)
constexpr int kRc = 7;            // kSpec: threshold candidates a CTA publishes per exchange
constexpr int kRS = kRc + 1;      // kSpec: records per CTA per exchange (header + candidates)
constexpr uint64_t kTauOffR = ~0ull;

struct __align__(16) Rec {
    uint32_t klo, khi, idx, own;  // own: bit31 taken | rank g << 18 | cta r << 14 | local sorted pos
    float x, y, z;
    uint32_t pad;
};

PS_DEV uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
PS_DEV double bitsd(uint64_t k) { return __longlong_as_double((long long)k); }
PS_DEV uint64_t rec_key(const Rec& r) { return ((uint64_t)r.khi << 32) | r.klo; }
// (key desc, idx asc): true if (ka, ia) ranks above (kb, ib)
PS_DEV bool ranks_above_r(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}
PS_DEV Rec none_rec() {
    Rec z;
    z.klo = z.khi = 0; z.idx = kNone; z.own = 0; z.x = z.y = z.z = 0.f; z.pad = 0;
    return z;
}

// Winner lane of a warp argmax over (key, idx): max key, lowest idx on ties;
// -1 if no lane has idx != kNone.
PS_DEV int argmax_lane(uint64_t key, uint32_t idx) {
    const bool valid = idx != kNone;
    const uint32_t hi = valid ? (uint32_t)(key >> 32) : 0u;
    const uint32_t mhi = __reduce_max_sync(kFull, hi);
    unsigned cand = __ballot_sync(kFull, valid && hi == mhi);
    if (cand == 0) return -1;
    if (__popc(cand) == 1) return __ffs(cand) - 1;
    const bool c1 = (cand >> (threadIdx.x & 31)) & 1u;
    const uint32_t lo = (uint32_t)key;
    const uint32_t mlo = __reduce_max_sync(kFull, c1 ? lo : 0u);
    const bool c2 = c1 && lo == mlo;
    const uint32_t midx = __reduce_min_sync(kFull, c2 ? idx : kNone);
    return __ffs(__ballot_sync(kFull, c2 && idx == midx)) - 1;
}

// conservative float32 skip threshold for "d < md" (see fps.cu): any exact
// float64 distance whose float32 evaluation (or rounded-down lower bound)
// exceeds it is > md.
PS_DEV float skip_thr(double md) {
    if (md == 0.0) return -1.0f;
    if (!(md >= 7.888609052210118e-31)) return __int_as_float(0x7f800000);
    return __fmul_ru(__double2float_ru(md), 1.0f + 3.814697265625e-06f);  // * (1 + 2^-18)
}

// branch-free form of skip_thr for predicated folds (d > 0 finite or 0)
PS_DEV float skip_thr_nb(double md) {
    const float t = __fmul_ru(__double2float_ru(md), 1.0f + 3.814697265625e-06f);
    const float u = md >= 7.888609052210118e-31 ? t : __int_as_float(0x7f800000);
    return md == 0.0 ? -1.0f : u;
}

PS_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
PS_DEV void named_bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

PS_DEV uint32_t morton12(float x, float y, float z, float ox, float oy, float oz, float sx, float sy, float sz) {
    const uint32_t qx = (uint32_t)min(15, max(0, (int)((x - ox) * sx)));
    const uint32_t qy = (uint32_t)min(15, max(0, (int)((y - oy) * sy)));
    const uint32_t qz = (uint32_t)min(15, max(0, (int)((z - oz) * sz)));
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        c |= (((qx >> i) & 1u) << (3 * i)) | (((qy >> i) & 1u) << (3 * i + 1)) | (((qz >> i) & 1u) << (3 * i + 2));
    return c;
}

// ---- global mailboxes (G > 1) ----------------------------------------------------
// Mailbox of a rank: uint4[B][3][G][kRecU4 * kMbRecs]; set 0/1 = exchange
// parity, set 2 = duplicate fallback; a slot holds one record (one-sample
// loop) or a rank's meta record, header and up to 32 candidates (speculative
// loop).  Every 64-bit word of a record carries its 32-bit payload next to the
// 32-bit sequence tag and is written with a relaxed system-scope store
// (possibly from a peer GPU over NVLink): naturally aligned 64-bit accesses
// are single-copy atomic, so a word whose tag matches holds this exchange's
// payload whatever order the words land in -- the reader accepts a record
// when all six tags match.  Waits are bounded (FpsRanks::timeout_ns).

PS_DEV void st_sys_v2(uint4* p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
PS_DEV void ld_sys_v2(const uint4* p, uint64_t& a, uint64_t& b) {
    asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
PS_DEV uint64_t tagw(uint32_t v, uint32_t seq) { return ((uint64_t)seq << 32) | v; }
PS_DEV bool tag_ok(uint64_t w, uint32_t seq) { return (uint32_t)(w >> 32) == seq; }
PS_DEV unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// bounded wait bookkeeping: called every poll that found a stale record
struct MboxWait {
    unsigned long long t0 = 0;
    uint32_t polls = 0;
    PS_DEV void tick(const FpsRanks& rk, uint32_t seq) {
        if ((++polls & 1023u) != 0u) return;
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) { t0 = now; return; }
        if (now - t0 > rk.timeout_ns) {
            if (rk.err) atomicCAS(rk.err, 0u, seq | 0x80000000u);
            printf("ps fps split: mailbox wait for tag %u exceeded %llu ns (peer dead or late)\n", seq,
                   rk.timeout_ns);
            __trap();
        }
    }
};

// idx travels with the taken flag in bit 31 (indices are < 2^30)
PS_DEV void mbox_put(uint4* slot, const Rec& r, uint32_t seq) {
    const uint32_t ix = r.idx == kNone ? kNone : (r.idx | (r.own & 0x80000000u));
    st_sys_v2(slot, tagw(r.klo, seq), tagw(r.khi, seq));
    st_sys_v2(slot + 1, tagw(ix, seq), tagw(__float_as_uint(r.x), seq));
    st_sys_v2(slot + 2, tagw(__float_as_uint(r.y), seq), tagw(__float_as_uint(r.z), seq));
}

PS_DEV Rec mbox_get(const uint4* slot, uint32_t seq, const FpsRanks& rk) {
    uint64_t w[6];
    MboxWait wt;
    while (true) {
        ld_sys_v2(slot, w[0], w[1]);
        ld_sys_v2(slot + 1, w[2], w[3]);
        ld_sys_v2(slot + 2, w[4], w[5]);
        if (tag_ok(w[0], seq) && tag_ok(w[1], seq) && tag_ok(w[2], seq) && tag_ok(w[3], seq) &&
            tag_ok(w[4], seq) && tag_ok(w[5], seq))
            break;
        wt.tick(rk, seq);
    }
    const uint32_t ix = (uint32_t)w[2];
    Rec r;
    r.klo = (uint32_t)w[0]; r.khi = (uint32_t)w[1];
    r.idx = ix == kNone ? kNone : (ix & 0x7fffffffu);
    r.own = ix == kNone ? 0u : ((ix & 0x80000000u) | kForeign);
    r.x = __uint_as_float((uint32_t)w[3]); r.y = __uint_as_float((uint32_t)w[4]); r.z = __uint_as_float((uint32_t)w[5]);
    r.pad = 0;
    return r;
}

// meta record of a speculative exchange: candidate count and overflow flag
PS_DEV void mbox_put_meta(uint4* slot, uint32_t cn, uint32_t ovf, uint32_t seq) {
    st_sys_v2(slot, tagw(cn, seq), tagw(ovf, seq));
}
PS_DEV void mbox_get_meta(const uint4* slot, uint32_t seq, const FpsRanks& rk, uint32_t& cn, uint32_t& ovf) {
    uint64_t a, b;
    MboxWait wt;
    while (true) {
        ld_sys_v2(slot, a, b);
        if (tag_ok(a, seq) && tag_ok(b, seq)) break;
        wt.tick(rk, seq);
    }
    cn = (uint32_t)a;
    ovf = (uint32_t)b;
}

// slot of (cloud b, set, from-rank f) inside a rank's mailbox; record k of it
PS_DEV size_t mb_slot(int64_t b, int set, int G, int f) {
    return (size_t)(((b * 3 + set) * G + f)) * (size_t)(kRecU4 * kMbRecs);
}

// Per-launch tag base for the internal virtual-rank split (graph-replay
// safe): seq[0] = base of this launch, seq[1] = next base; when the 32-bit
// tag space would wrap, the mailboxes are wiped (0xff) first.
__global__ void mbox_epoch_kernel(uint32_t* seq, uint4* buf, size_t n_u4, uint32_t span) {
    __shared__ uint32_t base;
    if (threadIdx.x == 0) {
        const uint32_t nx = seq[1];
        base = ((uint64_t)nx + span + 1 >= 0xffffffffull) ? 0xffffffffu : nx;
    }
    __syncthreads();
    if (base == 0xffffffffu) {
        for (size_t i = threadIdx.x; i < n_u4; i += blockDim.x) buf[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
        __syncthreads();
        if (threadIdx.x == 0) base = 0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        seq[0] = base;
        seq[1] = base + span + 1;
    }
}

template <int P, bool kSpec>
__global__ void __launch_bounds__(kT, 1) fps_res_kernel(FpsArgs a, FpsRanks rk) {
    constexpr int QG = P <= 8 ? P : (P % 8 == 0 ? 8 : 6);  // slots per screen group
    extern __shared__ __align__(16) unsigned char dsm[];
    float4* pts = reinterpret_cast<float4*>(dsm);                // [P * kT] sorted points
    uint32_t* hist = reinterpret_cast<uint32_t*>(pts + P * kT);  // [kBins]
    __shared__ Rec warp_rec[kW];
    __shared__ Rec fb_rec[kW];
    __shared__ Rec slots[2][kMaxC];
    __shared__ Rec fb_slots[kMaxC];
    __shared__ Rec gslot;
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ float red[6][kW];
    __shared__ uint32_t scan_tot[kW];
    __shared__ uint32_t cbound[kMaxC + 1];
    // kSpec exchange state
    __shared__ Rec cslots[kSpec ? 2 : 1][kSpec ? kMaxC * kRS : 1];
    __shared__ Rec ccand_s[kRc];
    __shared__ Rec cl_s[kSpec ? 32 : 1], cl_s2[kSpec ? 32 : 1], uh_s[kSpec ? 32 : 1];
    __shared__ Rec gslot2;
    __shared__ float4 run_s[32];
    __shared__ uint32_t run_own_s[32];
    __shared__ uint8_t run_fold_s[32];
    __shared__ double hist_s[32];
    __shared__ unsigned long long tau_s;
    __shared__ int ccnt_s, rn_s, fb_s;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t C = cluster_nctarank();
    const uint32_t r = cluster_ctarank();
    const int64_t cid = cluster_id_x();
    const int G = rk.G;
    const int64_t b = cid / rk.Gl;
    const int g = rk.g_base + (int)(cid % rk.Gl);
    const int64_t N = a.N;
    const int64_t Ns = (N + G - 1) / G;
    const int64_t shard_lo = min(N, (int64_t)g * Ns);
    const int64_t shard_hi = min(N, shard_lo + Ns);
    const int64_t S = a.points_per_cta;
    const int64_t lo = min(shard_hi, shard_lo + (int64_t)r * S);
    const int64_t hi = min(shard_hi, lo + S);
    const float4* __restrict__ xyz = a.xyz + b * N;
    double* __restrict__ md = a.md + b * N;
    uint8_t* __restrict__ taken = a.taken + b * N;
    int64_t* __restrict__ out = a.out_idx + b * a.ld_out;
    double* __restrict__ curve = a.curve + b * a.ld_out;
    const bool writer = (g == 0 || rk.all_write) && r == 0;
    const uint32_t seq_base = rk.seq_dev ? *reinterpret_cast<const volatile uint32_t*>(rk.seq_dev) : rk.seq_base;

    const int64_t k_start = a.k_start_dev ? a.k_start_dev[b] : a.k_start;
    const int64_t k_stop = a.k_stop;
    const int64_t seed = a.seed_dev ? a.seed_dev[b] : a.seed;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const uint32_t tx_bytes = C * (uint32_t)sizeof(Rec);
    uint4* mb_dst = nullptr;          // lane's destination rank mailbox (G > 1)
    const uint4* mb_mine = nullptr;   // this rank's mailbox
    if (G > 1) {
        mb_dst = lane < G ? rk.mbox[lane] : nullptr;
        mb_mine = rk.mbox[g];
    }

    // ---- 1. points of this CTA, Morton-ordered in shared memory -----------------------
    // spatial partition (rk.spatial): every CTA histograms the whole shard over
    // 4096 Morton cells of the shard's bounding box; cell c goes to CTA
    // min(C-1, start(c) * C / Ns) (start = exclusive prefix count), so CTA
    // ranges are contiguous runs of cells -- compact regions -- decided
    // identically by every CTA.  If a CTA would exceed its P*kT slots, all CTAs
    // fall back to index ranges [lo, hi) sorted locally.
    int cnt = 0;
    {
        const int64_t Nsh = shard_hi - shard_lo;
        for (int attempt = rk.spatial && C > 1 ? 0 : 1; attempt < 2; ++attempt) {
            const bool sp = attempt == 0;
            const int64_t src_lo = sp ? shard_lo : lo, src_hi = sp ? shard_hi : hi;
            float bmn[3] = {INFINITY, INFINITY, INFINITY}, bmx[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int64_t j = src_lo + tid; j < src_hi; j += kT) {
                const float4 v = xyz[j];
                bmn[0] = fminf(bmn[0], v.x); bmn[1] = fminf(bmn[1], v.y); bmn[2] = fminf(bmn[2], v.z);
                bmx[0] = fmaxf(bmx[0], v.x); bmx[1] = fmaxf(bmx[1], v.y); bmx[2] = fmaxf(bmx[2], v.z);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    bmn[k] = fminf(bmn[k], __shfl_xor_sync(kFull, bmn[k], o));
                    bmx[k] = fmaxf(bmx[k], __shfl_xor_sync(kFull, bmx[k], o));
                }
            }
            __syncthreads();  // red / hist reuse across attempts
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 3; ++k) { red[k][warp] = bmn[k]; red[3 + k][warp] = bmx[k]; }
            }
            for (int i = tid; i < kBins; i += kT) hist[i] = 0u;
            __syncthreads();
            float ox, oy, oz, scx, scy, scz;
            {
                float mn[3], mx[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    mn[k] = INFINITY; mx[k] = -INFINITY;
                    for (int w = 0; w < kW; ++w) { mn[k] = fminf(mn[k], red[k][w]); mx[k] = fmaxf(mx[k], red[3 + k][w]); }
                }
                const float ex = fmaxf(mx[0] - mn[0], 1e-30f), ey = fmaxf(mx[1] - mn[1], 1e-30f),
                            ez = fmaxf(mx[2] - mn[2], 1e-30f);
                ox = mn[0]; oy = mn[1]; oz = mn[2];
                scx = 16.f / ex; scy = 16.f / ey; scz = 16.f / ez;
            }
            for (int64_t j = src_lo + tid; j < src_hi; j += kT) {
                const float4 v = xyz[j];
                atomicAdd(&hist[morton12(v.x, v.y, v.z, ox, oy, oz, scx, scy, scz)], 1u);
            }
            __syncthreads();
            {
                // exclusive scan of the 4096 bins: 8 consecutive bins per thread
                constexpr int kPer = kBins / kT;
                uint32_t loc[kPer], sum = 0;
#pragma unroll
                for (int i = 0; i < kPer; ++i) { loc[i] = hist[tid * kPer + i]; sum += loc[i]; }
                uint32_t x = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) scan_tot[warp] = x;
                __syncthreads();
                uint32_t base = 0;
                for (int w = 0; w < warp; ++w) base += scan_tot[w];
                base += x - sum;
#pragma unroll
                for (int i = 0; i < kPer; ++i) { hist[tid * kPer + i] = base; base += loc[i]; }
            }
            __syncthreads();
            uint32_t my_c0 = 0, my_c1 = kBins, my_s0 = 0;
            if (sp) {
                // first cell of every CTA (owner is non-decreasing in the cell index)
                if (tid <= (int)C) {
                    uint32_t l = 0, h2 = kBins;  // first c with owner(c) >= tid
                    while (l < h2) {
                        const uint32_t mid = (l + h2) >> 1;
                        const int64_t ow = min((int64_t)C - 1, (int64_t)hist[mid] * C / max((int64_t)1, Nsh));
                        if (ow >= tid) h2 = mid; else l = mid + 1;
                    }
                    cbound[tid] = tid == 0 ? 0u : (tid == (int)C ? (uint32_t)kBins : l);
                }
                __syncthreads();
                bool fits = true;
                for (uint32_t q = 0; q < C; ++q) {
                    const uint32_t s0 = cbound[q] < kBins ? hist[cbound[q]] : (uint32_t)Nsh;
                    const uint32_t s1 = cbound[q + 1] < kBins ? hist[cbound[q + 1]] : (uint32_t)Nsh;
                    if (s1 - s0 > (uint32_t)(P * kT)) fits = false;
                }
                if (!fits) continue;  // uniform across the cluster: every CTA sees the same histogram
                my_c0 = cbound[r];
                my_c1 = cbound[r + 1];
                my_s0 = my_c0 < kBins ? hist[my_c0] : (uint32_t)Nsh;
                const uint32_t my_s1 = my_c1 < kBins ? hist[my_c1] : (uint32_t)Nsh;
                cnt = (int)(my_s1 - my_s0);
            } else {
                cnt = (int)(hi - lo);
            }
            __syncthreads();
            for (int64_t j = src_lo + tid; j < src_hi; j += kT) {
                const float4 v = xyz[j];
                const uint32_t c = morton12(v.x, v.y, v.z, ox, oy, oz, scx, scy, scz);
                if (c < my_c0 || c >= my_c1) continue;
                const uint32_t pos = atomicAdd(&hist[c], 1u) - my_s0;
                pts[pos] = make_float4(v.x, v.y, v.z, __int_as_float((int)j));
            }
            break;
        }
    }
    for (int j = cnt + tid; j < P * kT; j += kT) pts[j] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    __syncthreads();

    // ---- 2. per-slot state in registers, warp bounding boxes --------------------
    const int wbase = warp * 32 * P;
    double m[P];
    float thr[P];
    uint32_t tk = 0, valid = 0;
    float wb[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const float4 v = pts[wbase + q * 32 + lane];
        const int oi = __float_as_int(v.w);
        m[q] = 0.0;
        thr[q] = -1.0f;
        if (oi >= 0) {
            valid |= 1u << q;
            if (a.fresh) {
                m[q] = kInf;
                tk |= (oi == seed ? 1u : 0u) << q;
            } else {
                m[q] = md[oi];
                tk |= (taken[oi] ? 1u : 0u) << q;
            }
            thr[q] = skip_thr(m[q]);
            wb[0] = fminf(wb[0], v.x); wb[1] = fminf(wb[1], v.y); wb[2] = fminf(wb[2], v.z);
            wb[3] = fmaxf(wb[3], v.x); wb[4] = fmaxf(wb[4], v.y); wb[5] = fmaxf(wb[5], v.z);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wb[k] = fminf(wb[k], __shfl_xor_sync(kFull, wb[k], o));
            wb[3 + k] = fmaxf(wb[3 + k], __shfl_xor_sync(kFull, wb[3 + k], o));
        }
    }
    const bool wvalid = __any_sync(kFull, valid != 0);
    bool force = wvalid;           // recompute the warp record at the next iteration
    float thr_w = wvalid ? __int_as_float(0x7f800000) : -1.0f;
    uint64_t bk = 0;               // cached thread max: md bits, slot, original index (kNone: none)
    int bq = 0;
    uint32_t bo = kNone;
    if (lane == 0) warp_rec[warp] = none_rec();
    if (a.fresh && writer && tid == 0) {
        out[0] = seed;
        curve[0] = kInf;
    }

    if (tid == 0) {
        ccnt_s = 0;
        mbar_init(&bars[0], kSpec ? C : 1);  // kSpec: one arrival per sending CTA
        mbar_init(&bars[1], kSpec ? C : 1);
        fence_mbar_init_cluster();
        if (!kSpec) {
            mbar_arrive_expect_tx(&bars[0], tx_bytes);
            mbar_arrive_expect_tx(&bars[1], tx_bytes);
        }
    }
    cluster_sync_all();

    if constexpr (!kSpec) {
    if (k_start < k_stop) {
        const int64_t last = a.fresh ? seed : out[k_start - 1];
        const float4 lv = xyz[last];
        float sx32 = lv.x, sy32 = lv.y, sz32 = lv.z;

        for (int64_t it = k_start; it < k_stop; ++it) {
            const uint32_t t_abs = (uint32_t)(it - k_start);
            const uint32_t par = t_abs & 1u;
            const uint32_t phase = (t_abs >> 1) & 1u;
            const uint32_t t = t_abs - (uint32_t)a.dbg_t0;
            const bool tdbg = kTiming && a.dbg && b == 0 && r == 0 && tid == kT - 32 && t_abs >= a.dbg_t0 && t < 256 && g == 0;
            long long ts0 = 0;
            if (tdbg) ts0 = clock64();

            // 1. warp skip test: rounded-down |s - box|^2 against the warp threshold
            const float gx = fmaxf(fmaxf(__fsub_rd(wb[0], sx32), __fsub_rd(sx32, wb[3])), 0.f);
            const float gy = fmaxf(fmaxf(__fsub_rd(wb[1], sy32), __fsub_rd(sy32, wb[4])), 0.f);
            const float gz = fmaxf(fmaxf(__fsub_rd(wb[2], sz32), __fsub_rd(sz32, wb[5])), 0.f);
            const float lb = __fadd_rd(__fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)), __fmul_rd(gz, gz));
            if (force || !(lb > thr_w)) {
                const double sx = sx32, sy = sy32, sz = sz32;
                uint32_t chg = 0;
                uint32_t og[QG];  // original indices of the last group (all slots when QG == P)
                // groups of QG slots: all loads and float32 screens first, one
                // vote, then the group's float64 folds as independent,
                // predicated chains (no per-slot branches)
#pragma unroll
                for (int q0 = 0; q0 < P; q0 += QG) {
                    float4 v[QG];
#pragma unroll
                    for (int u = 0; u < QG; ++u) v[u] = pts[wbase + (q0 + u) * 32 + lane];
                    uint32_t need = 0;
#pragma unroll
                    for (int u = 0; u < QG; ++u) {
                        og[u] = __float_as_uint(v[u].w);
                        const float dx = v[u].x - sx32, dy = v[u].y - sy32, dz = v[u].z - sz32;
                        const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                        need |= (!(d32 > thr[q0 + u]) ? 1u : 0u) << u;
                    }
                    if (__any_sync(kFull, need != 0)) {
#pragma unroll
                        for (int u = 0; u < QG; ++u) {
                            const double d = sqdist(sx, sy, sz, (double)v[u].x, (double)v[u].y, (double)v[u].z);
                            const bool upd = ((need >> u) & 1u) && d < m[q0 + u];
                            m[q0 + u] = upd ? d : m[q0 + u];
                            thr[q0 + u] = upd ? skip_thr_nb(d) : thr[q0 + u];
                            chg |= (upd ? 1u : 0u) << (q0 + u);
                        }
                    }
                }
                const bool redo = force || ((chg >> bq) & 1u);  // my cached max slot moved
                if (__any_sync(kFull, chg != 0 || force)) {
                    if (redo) {
                        // thread max over my slots: max md (bit order), lowest original index
                        uint32_t o[P];
#pragma unroll
                        for (int q = 0; q < P; ++q)
                            o[q] = QG == P ? og[q % QG] : __float_as_uint(pts[wbase + q * 32 + lane].w);
                        bk = 0; bq = 0; bo = kNone;
#pragma unroll
                        for (int q = 0; q < P; ++q) {
                            const uint64_t kq = dbits(m[q]);
                            if (((valid >> q) & 1u) && (bo == kNone || kq > bk || (kq == bk && o[q] < bo))) {
                                bk = kq; bq = q; bo = o[q];
                            }
                        }
                    }
                    const int wl = argmax_lane(bk, bo);
                    if (wl < 0) {
                        thr_w = -1.0f;
                        if (lane == 0) warp_rec[warp] = none_rec();
                    } else {
                        const uint64_t wk = __shfl_sync(kFull, bk, wl);
                        thr_w = skip_thr(bitsd(wk));
                        if (lane == wl) {
                            const int lp = wbase + bq * 32 + lane;
                            const float4 v = pts[lp];
                            Rec rr;
                            rr.klo = (uint32_t)bk; rr.khi = (uint32_t)(bk >> 32);
                            rr.idx = bo;
                            rr.own = (((tk >> bq) & 1u) << 31) | ((uint32_t)g << 18) | (r << 14) | (uint32_t)lp;
                            rr.x = v.x; rr.y = v.y; rr.z = v.z; rr.pad = 0;
                            warp_rec[warp] = rr;
                        }
                    }
                    force = false;
                }
            }
            if (tdbg) a.dbg[t * 8 + 0] = clock64() - ts0;

            // 2-4. the leader warp alone: block argmax, push the CTA record to the
            // cluster, wait for the C records, (ranks) exchange through the
            // mailboxes; the winner is broadcast through shared memory on a
            // named barrier on which the other warps block in hardware
            if (warp == kW - 1) {
                named_bar_sync(1, kT);
                if (tdbg) a.dbg[t * 8 + 1] = clock64() - ts0;
                const Rec wr = lane < kW ? warp_rec[lane] : none_rec();
                const int cl = argmax_lane(rec_key(wr), wr.idx);
                if (tdbg) a.dbg[t * 8 + 6] = clock64() - ts0;
                const Rec cr = warp_rec[cl < 0 ? 0 : cl];
                if (tdbg) a.dbg[t * 8 + 7] = (long long)cr.idx * 0 + clock64() - ts0;
                if (lane < (int)C) {
                    const uint32_t dst = mapa(smem_u32(&slots[par][r]), lane);
                    const uint32_t dbar = mapa(smem_u32(&bars[par]), lane);
                    st_async_v4(dst, dbar, cr.klo, cr.khi, cl < 0 ? kNone : cr.idx, cr.own);
                    st_async_v4(dst + 16, dbar, __float_as_uint(cr.x), __float_as_uint(cr.y), __float_as_uint(cr.z),
                                0u);
                }
                if (tdbg) a.dbg[t * 8 + 2] = clock64() - ts0;
                mbar_wait_cluster(&bars[par], phase);
                if (tdbg) a.dbg[t * 8 + 3] = clock64() - ts0;
                const Rec sr = lane < (int)C ? slots[par][lane] : none_rec();
                const int gl = argmax_lane(rec_key(sr), sr.idx);
                const Rec cw = gl < 0 ? none_rec() : slots[par][gl];
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&bars[par], tx_bytes);
                if (G > 1) {
                    const uint32_t seq = seq_base + (uint32_t)it;
                    if (r == 0 && lane < G) mbox_put(mb_dst + mb_slot(b, par, G, g), cw, seq);
                    const Rec pr = lane < G ? mbox_get(mb_mine + mb_slot(b, par, G, lane), seq, rk) : none_rec();
                    const int pl = argmax_lane(rec_key(pr), pr.idx);
                    if (lane == (pl < 0 ? 0 : pl)) {
                        Rec gw = pl < 0 ? none_rec() : pr;
                        if (pl >= 0 && gw.idx == cw.idx) gw.own = cw.own;  // my rank's point: keep its owner
                        gslot = gw;
                    }
                } else if (lane == 0) {
                    gslot = cw;
                }
                if (tdbg) a.dbg[t * 8 + 4] = clock64() - ts0;
                named_bar_arrive(2, kT);
            } else {
                named_bar_arrive(1, kT);
                named_bar_sync(2, kT);
            }
            Rec win = gslot;

            double best = bitsd(rec_key(win));
            const bool win_taken = (win.own >> 31) & 1u;
            if (win.idx == kNone || best <= 0.0 || win_taken) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken original index
                uint32_t fidx = kNone;
                int fq = -1;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (((valid >> q) & 1u) && !((tk >> q) & 1u)) {
                        const uint32_t o = __float_as_uint(pts[wbase + q * 32 + lane].w);
                        if (o < fidx) { fidx = o; fq = q; }
                    }
                }
                const uint32_t wm = __reduce_min_sync(kFull, fidx);
                if (fidx == wm && fidx != kNone) {
                    const int lp = wbase + fq * 32 + lane;
                    const float4 v = pts[lp];
                    double mv = 0.0;
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if (q == fq) mv = m[q];
                    const uint64_t k = dbits(mv);
                    Rec fr;
                    fr.klo = (uint32_t)k; fr.khi = (uint32_t)(k >> 32); fr.idx = fidx;
                    fr.own = ((uint32_t)g << 18) | (r << 14) | (uint32_t)lp;
                    fr.x = v.x; fr.y = v.y; fr.z = v.z; fr.pad = 0;
                    fb_rec[warp] = fr;
                } else if (lane == 0 && wm == kNone) {
                    fb_rec[warp] = none_rec();
                }
                __syncthreads();
                if (warp == 0) {
                    const uint32_t ci = lane < kW ? fb_rec[lane].idx : kNone;
                    const uint32_t cm = __reduce_min_sync(kFull, ci);
                    const unsigned wv = __ballot_sync(kFull, ci == cm && ci != kNone);
                    const Rec cr = wv ? fb_rec[__ffs(wv) - 1] : none_rec();
                    if (lane < (int)C) {
                        const uint32_t dst = mapa(smem_u32(&fb_slots[r]), lane);
                        st_cluster_u64(dst, ((uint64_t)cr.khi << 32) | cr.klo);
                        st_cluster_u64(dst + 8, ((uint64_t)cr.own << 32) | cr.idx);
                        st_cluster_u64(dst + 16, ((uint64_t)__float_as_uint(cr.y) << 32) | __float_as_uint(cr.x));
                        st_cluster_u64(dst + 24, (uint64_t)__float_as_uint(cr.z));
                    }
                }
                cluster_sync_all();
                Rec fw;
                {
                    const uint32_t ci = lane < (int)C ? fb_slots[lane].idx : kNone;
                    const uint32_t cm = __reduce_min_sync(kFull, ci);
                    const unsigned wv = __ballot_sync(kFull, ci == cm && ci != kNone);
                    fw = wv ? fb_slots[__ffs(wv) - 1] : none_rec();
                }
                if (G > 1) {
                    const uint32_t seq = seq_base + (uint32_t)it;
                    __syncthreads();
                    if (warp == kW - 1) {
                        if (r == 0 && lane < G) mbox_put(mb_dst + mb_slot(b, 2, G, g), fw, seq);
                        const Rec pr = lane < G ? mbox_get(mb_mine + mb_slot(b, 2, G, lane), seq, rk) : none_rec();
                        const uint32_t pm = __reduce_min_sync(kFull, pr.idx);
                        const unsigned wv = __ballot_sync(kFull, pr.idx == pm && pr.idx != kNone);
                        if (lane == (wv ? __ffs(wv) - 1 : 0)) {
                            Rec gw = wv ? pr : none_rec();
                            if (wv && gw.idx == fw.idx) gw.own = fw.own;
                            gslot = gw;
                        }
                    }
                    __syncthreads();
                    fw = gslot;
                }
                if (fw.idx != kNone) {
                    win = fw;
                    best = bitsd(rec_key(fw));
                }
                cluster_sync_all();  // fb_slots / fb_rec / gslot free for the next fallback
            }

            // record (curve holds squared values until the epilogue), mark taken
            if (writer && tid == 0) {
                out[it] = (int64_t)win.idx;
                curve[it] = best;
            }
            const uint32_t own = win.own & 0x7fffffffu;
            if (win.idx != kNone && (own >> 18) == (uint32_t)g && ((own >> 14) & 15u) == r) {
                const uint32_t lp = own & 0x3fffu;
                if ((int)(lp / (32 * P)) == warp) {
                    force = true;  // the record's taken flag changes
                    if ((int)(lp & 31u) == lane) tk |= 1u << ((lp >> 5) % P);
                }
            }
            sx32 = win.x; sy32 = win.y; sz32 = win.z;
            if (tdbg) a.dbg[t * 8 + 5] = clock64() - ts0;
        }
    }

    } else {
        // ---- speculative exchange loop (kSpec) -----------------------------------
        // As fps_spec.cu: every CTA publishes its argmax (header) and its points
        // with md >= tau (candidates); with G > 1 ranks, CTA 0 of each rank
        // forwards the rank's header and candidates to every rank's mailbox.
        // Every lead warp of every CTA of every rank then picks identically:
        // the max over the headers, then the best candidate while it stays
        // >= tau (every other point is < tau and md only falls), lowering the
        // other candidates by their exact float64 distance to each pick.  The
        // run is broadcast on a named barrier and folded by every warp.
        const uint32_t tag0 = seq_base;
        int rn = 0;
        int hc = 0;
        float gain = 1.0f;
        bool tau_boot = false;
        uint64_t tau = kTauOffR;
        if (k_start < k_stop && tid == 0) {
            const int64_t last = a.fresh ? seed : out[k_start - 1];  // refolded, as _kernels.py
            const float4 lv = xyz[last];
            run_s[0] = make_float4(lv.x, lv.y, lv.z, __uint_as_float((uint32_t)last));
            run_own_s[0] = kForeign;  // already taken: fold only
            run_fold_s[0] = 1;
        }
        if (k_start < k_stop) rn = 1;
        if (warp == kW - 1 && !a.fresh && k_start < k_stop) {
            const int avail = k_start - 1 >= 32 ? 32 : (k_start - 1 > 0 ? (int)(k_start - 1) : 0);
            const double c = lane < avail ? curve[k_start - 1 - lane] : kInf;
            const uint32_t fin = __ballot_sync(kFull, lane < avail && c < kInf);
            const int nh = __ffs(~fin) - 1 < 0 ? 32 : __ffs(~fin) - 1;
            if (lane < nh) hist_s[(nh - 1 - lane) & 31] = c * c;
            hc = nh;
        }
        __syncthreads();
        int64_t it = k_start;
        uint32_t ex = 0;
        while (it < k_stop) {
            const uint32_t par = ex & 1u, phase = (ex >> 1) & 1u;
            ++ex;
            const uint32_t seq = tag0 + (uint32_t)it;

            // A. fold the run (warp skip per sample), then refresh the warp record
            uint32_t chg = 0;
            for (int k = 0; k < rn; ++k) {
                const float4 sv = run_s[k];
                const uint32_t sown = run_own_s[k];
                const uint32_t own = sown & 0x7fffffffu;
                if (sown != kForeign && (own >> 18) == (uint32_t)g && ((own >> 14) & 15u) == r) {
                    const uint32_t lp = own & 0x3fffu;
                    if ((int)(lp / (32 * P)) == warp) {
                        force = true;  // the record's taken flag changes
                        if ((int)(lp & 31u) == lane) tk |= 1u << ((lp >> 5) % P);
                    }
                }
                if (!run_fold_s[k]) continue;
                const float sx32 = sv.x, sy32 = sv.y, sz32 = sv.z;
                const float gx = fmaxf(fmaxf(__fsub_rd(wb[0], sx32), __fsub_rd(sx32, wb[3])), 0.f);
                const float gy = fmaxf(fmaxf(__fsub_rd(wb[1], sy32), __fsub_rd(sy32, wb[4])), 0.f);
                const float gz = fmaxf(fmaxf(__fsub_rd(wb[2], sz32), __fsub_rd(sz32, wb[5])), 0.f);
                const float lb = __fadd_rd(__fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)), __fmul_rd(gz, gz));
                if (!(lb > thr_w)) {
                    const double sx = sx32, sy = sy32, sz = sz32;
#pragma unroll
                    for (int q0 = 0; q0 < P; q0 += QG) {
                        float4 v[QG];
#pragma unroll
                        for (int u = 0; u < QG; ++u) v[u] = pts[wbase + (q0 + u) * 32 + lane];
                        uint32_t need = 0;
#pragma unroll
                        for (int u = 0; u < QG; ++u) {
                            const float dx = v[u].x - sx32, dy = v[u].y - sy32, dz = v[u].z - sz32;
                            const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                            need |= (!(d32 > thr[q0 + u]) ? 1u : 0u) << u;
                        }
                        if (__any_sync(kFull, need != 0)) {
#pragma unroll
                            for (int u = 0; u < QG; ++u) {
                                const double d = sqdist(sx, sy, sz, (double)v[u].x, (double)v[u].y, (double)v[u].z);
                                const bool upd = ((need >> u) & 1u) && d < m[q0 + u];
                                m[q0 + u] = upd ? d : m[q0 + u];
                                thr[q0 + u] = upd ? skip_thr_nb(d) : thr[q0 + u];
                                chg |= (upd ? 1u : 0u) << (q0 + u);
                            }
                        }
                    }
                }
            }
            const bool redo = force || ((chg >> bq) & 1u);
            if (__any_sync(kFull, chg != 0 || force)) {
                if (redo) {
                    bk = 0; bq = 0; bo = kNone;
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const uint32_t o = __float_as_uint(pts[wbase + q * 32 + lane].w);
                        const uint64_t kq = dbits(m[q]);
                        if (((valid >> q) & 1u) && (bo == kNone || kq > bk || (kq == bk && o < bo))) {
                            bk = kq; bq = q; bo = o;
                        }
                    }
                }
                const int wl = argmax_lane(bk, bo);
                if (wl < 0) {
                    thr_w = -1.0f;
                    if (lane == 0) warp_rec[warp] = none_rec();
                } else {
                    const uint64_t wk = __shfl_sync(kFull, bk, wl);
                    thr_w = skip_thr(bitsd(wk));
                    if (lane == wl) {
                        const int lp = wbase + bq * 32 + lane;
                        const float4 v = pts[lp];
                        Rec rr;
                        rr.klo = (uint32_t)bk; rr.khi = (uint32_t)(bk >> 32);
                        rr.idx = bo;
                        rr.own = (((tk >> bq) & 1u) << 31) | ((uint32_t)g << 18) | (r << 14) | (uint32_t)lp;
                        rr.x = v.x; rr.y = v.y; rr.z = v.z; rr.pad = 0;
                        warp_rec[warp] = rr;
                    }
                }
                force = false;
            }
            // B. candidates: my points with md >= tau
            {
                uint32_t cmask = 0;
#pragma unroll
                for (int q = 0; q < P; ++q) cmask |= ((((valid >> q) & 1u) && dbits(m[q]) >= tau) ? 1u : 0u) << q;
                if (__any_sync(kFull, cmask != 0)) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        if ((cmask >> q) & 1u) {
                            const int slot = atomicAdd(&ccnt_s, 1);
                            if (slot < kRc) {
                                const int lp = wbase + q * 32 + lane;
                                const float4 v = pts[lp];
                                Rec rr;
                                const uint64_t kq = dbits(m[q]);
                                rr.klo = (uint32_t)kq; rr.khi = (uint32_t)(kq >> 32);
                                rr.idx = __float_as_uint(v.w);
                                rr.own = (((tk >> q) & 1u) << 31) | ((uint32_t)g << 18) | (r << 14) | (uint32_t)lp;
                                rr.x = v.x; rr.y = v.y; rr.z = v.z; rr.pad = 0;
                                ccand_s[slot] = rr;
                            }
                        }
                    }
                }
            }

            if (warp == kW - 1) {
                named_bar_sync(1, kT);
                // C. CTA header + candidates to every CTA of the cluster
                const Rec wr = lane < kW ? warp_rec[lane] : none_rec();
                const int cl = argmax_lane(rec_key(wr), wr.idx);
                const Rec cr = cl < 0 ? none_rec() : warp_rec[cl];
                const int n = ccnt_s;
                __syncwarp();
                if (lane == 0) ccnt_s = 0;
                const int nsend = n < kRc ? n : kRc;
                if (C == 1) {
                    if (lane < 1 + nsend) {
                        Rec x = lane == 0 ? cr : ccand_s[lane - 1];
                        if (lane == 0) x.pad = (uint32_t)n;
                        cslots[par][lane] = x;
                    }
                    __syncwarp();
                } else if (lane < (int)C) {
                    const uint32_t rbar = mapa(smem_u32(&bars[par]), (uint32_t)lane);
                    const uint32_t rbase = mapa(smem_u32(&cslots[par][r * kRS]), (uint32_t)lane);
                    mbar_remote_arrive_expect_tx(rbar, (uint32_t)(1 + nsend) * (uint32_t)sizeof(Rec));
                    st_async_v4(rbase, rbar, cr.klo, cr.khi, cr.idx, cr.own);
                    st_async_v4(rbase + 16, rbar, __float_as_uint(cr.x), __float_as_uint(cr.y), __float_as_uint(cr.z),
                                (uint32_t)n);
                    for (int k = 0; k < nsend; ++k) {
                        const Rec x = ccand_s[k];
                        st_async_v4(rbase + 32u * (k + 1), rbar, x.klo, x.khi, x.idx, x.own);
                        st_async_v4(rbase + 32u * (k + 1) + 16, rbar, __float_as_uint(x.x), __float_as_uint(x.y),
                                    __float_as_uint(x.z), 0u);
                    }
                }
                if (C > 1) mbar_wait_cta(&bars[par], phase);

                // D. units: the C CTAs (G == 1) or the G ranks (G > 1).  Unit
                // headers to uh_s, candidates compacted to cl_s.
                // cluster level: headers in lanes < C, counts, candidate prefix
                Rec h = lane < (int)C ? cslots[par][lane * kRS] : none_rec();
                const int hcnt = lane < (int)C ? (int)h.pad : 0;
                bool ovf = __any_sync(kFull, hcnt > kRc);
                const int hn = hcnt < kRc ? hcnt : kRc;
                const uint32_t lt = (1u << lane) - 1u;
                static_assert(kRc < 16, "four ballots");
                const uint32_t b0 = __ballot_sync(kFull, hn & 1), b1 = __ballot_sync(kFull, hn & 2),
                               b2 = __ballot_sync(kFull, hn & 4), b3 = kRc > 7 ? __ballot_sync(kFull, hn & 8) : 0u;
                const int cbase = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt) + 8 * __popc(b3 & lt);
                const int cn_all = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2) + 8 * __popc(b3);
                ovf = ovf || cn_all > 32;
                for (int k = 0; k < hn; ++k)
                    if (cbase + k < 32) cl_s[cbase + k] = cslots[par][lane * kRS + 1 + k];
                const int cn = cn_all < 32 ? cn_all : 32;
                int nunits, ncand;
                if (G == 1) {
                    if (lane < (int)C) uh_s[lane] = h;
                    nunits = (int)C;
                    ncand = cn;
                } else {
                    // my rank: header = max over my CTAs (owner fields kept)
                    const int hl = argmax_lane(rec_key(h), h.idx);
                    const Rec rh = hl < 0 ? none_rec() : cslots[par][hl * kRS];
                    __syncwarp();
                    if (r == 0) {
                        // forward my rank's set: meta, header, candidates
                        uint4* mb = lane < G ? rk.mbox[lane] : nullptr;
                        if (lane < G) {
                            uint4* sl = mb + mb_slot(b, par, G, g);
                            for (int k = 0; k < cn; ++k) mbox_put(sl + kRecU4 * (2 + k), cl_s[k], seq);
                            mbox_put(sl + kRecU4, rh, seq);
                            mbox_put_meta(sl, (uint32_t)cn, ovf ? 1u : 0u, seq);
                        }
                    }
                    // every rank's set: mine from the cluster, others from my mailbox
                    const uint4* mine = mb_mine + mb_slot(b, par, G, 0);
                    Rec uh = none_rec();
                    int ucnt = 0;
                    bool uovf = false;
                    if (lane < G) {
                        if (lane == g) {
                            uh = rh;
                            ucnt = cn;
                            uovf = ovf;
                        } else {
                            const uint4* sl = mine + (size_t)lane * (kRecU4 * kMbRecs);
                            uint32_t mc, mo;
                            mbox_get_meta(sl, seq, rk, mc, mo);
                            ucnt = (int)mc;
                            uovf = mo != 0u;
                            uh = mbox_get(sl + kRecU4, seq, rk);
                        }
                    }
                    ovf = __any_sync(kFull, uovf);
                    if (lane < G) uh_s[lane] = uh;
                    // candidate prefix over the ranks (counts <= 32: five ballots)
                    const uint32_t u0 = __ballot_sync(kFull, ucnt & 1), u1 = __ballot_sync(kFull, ucnt & 2),
                                   u2 = __ballot_sync(kFull, ucnt & 4), u3 = __ballot_sync(kFull, ucnt & 8),
                                   u4 = __ballot_sync(kFull, ucnt & 16), u5 = __ballot_sync(kFull, ucnt & 32);
                    const int ubase = __popc(u0 & lt) + 2 * __popc(u1 & lt) + 4 * __popc(u2 & lt) +
                                      8 * __popc(u3 & lt) + 16 * __popc(u4 & lt) + 32 * __popc(u5 & lt);
                    const int un_all = __popc(u0) + 2 * __popc(u1) + 4 * __popc(u2) + 8 * __popc(u3) +
                                       16 * __popc(u4) + 32 * __popc(u5);
                    ovf = ovf || un_all > 32;
                    __syncwarp();
                    // my rank's candidates move from cl_s to their rank position
                    Rec minec[2];
                    const int mybase = __shfl_sync(kFull, ubase, g);
                    minec[0] = lane < cn ? cl_s[lane] : none_rec();
                    __syncwarp();
                    if (lane < cn && mybase + lane < 32) cl_s2[mybase + lane] = minec[0];
                    if (lane < G && lane != g) {
                        const uint4* sl = mine + (size_t)lane * (kRecU4 * kMbRecs);
                        for (int k = 0; k < ucnt; ++k)
                            if (ubase + k < 32) cl_s2[ubase + k] = mbox_get(sl + kRecU4 * (2 + k), seq, rk);
                    }
                    __syncwarp();
                    const int unn = un_all < 32 ? un_all : 32;
                    if (lane < unn) cl_s[lane] = cl_s2[lane];
                    __syncwarp();
                    nunits = G;
                    ncand = unn;
                }
                __syncwarp();

                // E. picks (identical in every lead warp of every CTA and rank)
                Rec uh2 = lane < nunits ? uh_s[lane] : none_rec();
                Rec cc = lane < ncand ? cl_s[lane] : none_rec();
                double cm = bitsd(rec_key(cc));
                const uint32_t ct = (cc.own >> 31) & 1u;
                ovf = ovf || __any_sync(kFull, lane < ncand && ct);
                bool alive = lane < ncand;
                int rnl = 0, fb = 0;
                int64_t itl = it;
                const bool hv = uh2.idx != kNone;
                {
                    const bool use_c = alive && (!hv || ranks_above_r(dbits(cm), cc.idx, rec_key(uh2), uh2.idx));
                    const uint64_t k0 = use_c ? dbits(cm) : rec_key(uh2);
                    const uint32_t i0 = use_c ? cc.idx : (hv ? uh2.idx : kNone);
                    const int wl = argmax_lane(k0, i0);
                    if (wl >= 0) {
                        const uint64_t wk = __shfl_sync(kFull, k0, wl);
                        const uint32_t wi = __shfl_sync(kFull, i0, wl);
                        const bool wc = __shfl_sync(kFull, use_c ? 1 : 0, wl);
                        const uint32_t wown = __shfl_sync(kFull, use_c ? cc.own : uh2.own, wl);
                        const float sx = __shfl_sync(kFull, use_c ? cc.x : uh2.x, wl);
                        const float sy = __shfl_sync(kFull, use_c ? cc.y : uh2.y, wl);
                        const float sz = __shfl_sync(kFull, use_c ? cc.z : uh2.z, wl);
                        (void)wc;
                        const double wm = bitsd(wk);
                        if (!(wm > 0.0) || ((wown >> 31) & 1u)) {
                            fb = 1;
                            if (lane == 0) {
                                Rec w = none_rec();
                                w.klo = (uint32_t)wk; w.khi = (uint32_t)(wk >> 32); w.idx = wi; w.own = wown;
                                w.x = sx; w.y = sy; w.z = sz;
                                gslot = w;
                            }
                        } else {
                            if (lane == 0) {
                                run_s[0] = make_float4(sx, sy, sz, __uint_as_float(wi));
                                run_own_s[0] = wown;
                                hist_s[hc & 31] = wm;
                            }
                            ++itl;
                            rnl = 1;
                            alive = alive && cc.idx != wi && !ovf;
                            if (alive) {
                                const double d = sqdist((double)sx, (double)sy, (double)sz, (double)cc.x, (double)cc.y,
                                                        (double)cc.z);
                                if (dbits(d) < dbits(cm)) cm = d;
                            }
                        }
                    }
                }
                while (rnl > 0 && itl < k_stop && rnl < 31) {
                    alive = alive && dbits(cm) >= tau;
                    const int wl = argmax_lane(alive ? dbits(cm) : 0ull, alive ? cc.idx : kNone);
                    if (wl < 0) break;
                    const bool win = lane == wl;
                    const float sx = __shfl_sync(kFull, cc.x, wl);
                    const float sy = __shfl_sync(kFull, cc.y, wl);
                    const float sz = __shfl_sync(kFull, cc.z, wl);
                    const double d = sqdist((double)sx, (double)sy, (double)sz, (double)cc.x, (double)cc.y, (double)cc.z);
                    if (win) {
                        run_s[rnl] = make_float4(cc.x, cc.y, cc.z, __uint_as_float(cc.idx));
                        run_own_s[rnl] = cc.own;
                        hist_s[(hc + rnl) & 31] = cm;
                    }
                    alive = alive && !win;
                    cm = (alive && dbits(d) < dbits(cm)) ? d : cm;
                    ++itl;
                    ++rnl;
                }
                const int hbase = hc;
                hc += rnl;
                __syncwarp();
                // next threshold (as fps_spec.cu)
                if (tau != kTauOffR && !tau_boot) {
                    if (ovf || ncand > 44) gain *= 0.7f;
                    else if (ncand < 11) gain *= 1.3f;
                    gain = fminf(fmaxf(gain, 0.05f), 20.0f);
                }
                uint64_t tnew = kTauOffR;
                tau_boot = hc < 3;
                if (tau_boot) {
                    uint64_t hk2 = hv ? rec_key(uh2) : 0ull;
                    uint32_t hi2 = uh2.idx;
#pragma unroll
                    for (int rep3 = 0; rep3 < 3; ++rep3) {
                        const int wl = argmax_lane(hk2, hi2);
                        if (wl < 0) break;
                        const uint64_t top = __shfl_sync(kFull, hk2, wl);
                        if (rep3 == 2) { tnew = top > 0ull ? top : kTauOffR; break; }
                        if (lane == wl) { hk2 = 0ull; hi2 = kNone; }
                    }
                } else {
                    const int L = hc - 1 < 16 ? hc - 1 : 16;
                    const double m0 = hist_s[(hc - 1) & 31];
                    const double mL = hist_s[(hc - 1 - L) & 31];
                    const double stepv = fmax((mL - m0) * (double)__frcp_rn((float)L), m0 * 2.44140625e-4);
                    const double tv = m0 - (double)gain * 22.0 * stepv;
                    if (tv > 0.0 && tv < kInf) tnew = dbits(tv);
                }
                if (writer && lane < rnl) {
                    out[it + lane] = (int64_t)__float_as_uint(run_s[lane].w);
                    curve[it + lane] = hist_s[(hbase + lane) & 31];
                }
                if (lane == 0) {
                    tau_s = tnew;
                    rn_s = rnl;
                    fb_s = fb;
                }
                named_bar_arrive(2, kT);
            } else {
                named_bar_arrive(1, kT);
                named_bar_sync(2, kT);
            }
            __syncwarp();
            rn = rn_s;
            tau = tau_s;
            const int fbf = fb_s;
            // the fold flags of this run: every sample but the call's last
            for (int k = tid; k < rn; k += kT) run_fold_s[k] = (it + k < k_stop - 1) ? 1 : 0;
            it += rn;
            __syncthreads();  // run_fold_s; run_s / rn_s reads before the lead's next writes

            if (fbf) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken original index
                Rec win = gslot;
                double best = bitsd(rec_key(win));
                uint32_t fidx = kNone;
                int fq = -1;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (((valid >> q) & 1u) && !((tk >> q) & 1u)) {
                        const uint32_t o = __float_as_uint(pts[wbase + q * 32 + lane].w);
                        if (o < fidx) { fidx = o; fq = q; }
                    }
                }
                const uint32_t wm = __reduce_min_sync(kFull, fidx);
                if (fidx == wm && fidx != kNone) {
                    const int lp = wbase + fq * 32 + lane;
                    const float4 v = pts[lp];
                    double mv = 0.0;
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if (q == fq) mv = m[q];
                    const uint64_t k = dbits(mv);
                    Rec fr;
                    fr.klo = (uint32_t)k; fr.khi = (uint32_t)(k >> 32); fr.idx = fidx;
                    fr.own = ((uint32_t)g << 18) | (r << 14) | (uint32_t)lp;
                    fr.x = v.x; fr.y = v.y; fr.z = v.z; fr.pad = 0;
                    fb_rec[warp] = fr;
                } else if (lane == 0 && wm == kNone) {
                    fb_rec[warp] = none_rec();
                }
                __syncthreads();
                if (warp == 0) {
                    const uint32_t ci = lane < kW ? fb_rec[lane].idx : kNone;
                    const uint32_t cmn = __reduce_min_sync(kFull, ci);
                    const unsigned wv = __ballot_sync(kFull, ci == cmn && ci != kNone);
                    const Rec cr = wv ? fb_rec[__ffs(wv) - 1] : none_rec();
                    if (lane < (int)C) {
                        const uint32_t dst = mapa(smem_u32(&fb_slots[r]), lane);
                        st_cluster_u64(dst, ((uint64_t)cr.khi << 32) | cr.klo);
                        st_cluster_u64(dst + 8, ((uint64_t)cr.own << 32) | cr.idx);
                        st_cluster_u64(dst + 16, ((uint64_t)__float_as_uint(cr.y) << 32) | __float_as_uint(cr.x));
                        st_cluster_u64(dst + 24, (uint64_t)__float_as_uint(cr.z));
                    }
                }
                cluster_sync_all();
                Rec fw;
                {
                    const uint32_t ci = lane < (int)C ? fb_slots[lane].idx : kNone;
                    const uint32_t cmn = __reduce_min_sync(kFull, ci);
                    const unsigned wv = __ballot_sync(kFull, ci == cmn && ci != kNone);
                    fw = wv ? fb_slots[__ffs(wv) - 1] : none_rec();
                }
                if (G > 1) {
                    __syncthreads();
                    if (warp == kW - 1) {
                        if (r == 0 && lane < G) mbox_put(rk.mbox[lane] + mb_slot(b, 2, G, g), fw, seq);
                        const Rec pr = lane < G ? mbox_get(mb_mine + mb_slot(b, 2, G, lane), seq, rk)
                                                : none_rec();
                        const uint32_t pm = __reduce_min_sync(kFull, pr.idx);
                        const unsigned wv = __ballot_sync(kFull, pr.idx == pm && pr.idx != kNone);
                        if (lane == (wv ? __ffs(wv) - 1 : 0)) {
                            Rec gw = wv ? pr : none_rec();
                            if (wv && gw.idx == fw.idx) gw.own = fw.own;
                            gslot2 = gw;
                        }
                    }
                    __syncthreads();
                    fw = gslot2;
                }
                if (fw.idx != kNone) {
                    win = fw;
                    best = bitsd(rec_key(fw));
                }
                cluster_sync_all();  // fb_slots / fb_rec free for the next fallback
                if (writer && tid == 0) {
                    out[it] = (int64_t)win.idx;
                    curve[it] = best;
                }
                if (warp == kW - 1) {
                    if (lane == 0) hist_s[hc & 31] = best;
                    ++hc;
                }
                __syncthreads();
                if (tid == 0) {
                    run_s[0] = make_float4(win.x, win.y, win.z, __uint_as_float(win.idx));
                    run_own_s[0] = win.own;
                    run_fold_s[0] = it < k_stop - 1 ? 1 : 0;
                }
                rn = 1;
                ++it;
                __syncthreads();
            }
        }
        // the last run is marked above; its samples are folded except the call's last
        if (rn > 0) {
            for (int k = 0; k < rn; ++k) {
                const uint32_t sown = run_own_s[k];
                const uint32_t own = sown & 0x7fffffffu;
                if (sown != kForeign && (own >> 18) == (uint32_t)g && ((own >> 14) & 15u) == r) {
                    const uint32_t lp = own & 0x3fffu;
                    if ((int)(lp / (32 * P)) == warp && (int)(lp & 31u) == lane) tk |= 1u << ((lp >> 5) % P);
                }
                if (!run_fold_s[k]) continue;
                const float4 sv = run_s[k];
                const double sx = sv.x, sy = sv.y, sz = sv.z;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if ((valid >> q) & 1u) {
                        const float4 v = pts[wbase + q * 32 + lane];
                        const double d = sqdist(sx, sy, sz, (double)v.x, (double)v.y, (double)v.z);
                        if (d < m[q]) m[q] = d;
                    }
                }
            }
        }
    }

    // ---- write back md / taken; curve = sqrt(best) (_kernels.py:72) -------------
#pragma unroll
    for (int q = 0; q < P; ++q) {
        if ((valid >> q) & 1u) {
            const int oi = __float_as_int(pts[wbase + q * 32 + lane].w);
            md[oi] = m[q];
            taken[oi] = (tk >> q) & 1u;
        }
    }
    if (writer && k_start < k_stop) {
        __syncthreads();  // thread 0's curve stores are visible block-wide
        for (int64_t it = k_start + tid; it < k_stop; it += kT) curve[it] = sqrt(curve[it]);
    }
    cluster_sync_all();  // no CTA leaves while peers may still target its smem
}

size_t res_smem_bytes(int P) { return (size_t)P * kT * sizeof(float4) + kBins * sizeof(uint32_t); }

template <int P, bool kSpec>
cudaError_t launch_res_p(const FpsArgs& a, const FpsRanks& rk, int64_t nclusters, int C, cudaStream_t s,
                         bool query_only, int* max_clusters) {
    auto kern = fps_res_kernel<P, kSpec>;
    const size_t smem = res_smem_bytes(P);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nclusters * C), 1, 1);
    cfg.blockDim = dim3(kT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (query_only) {
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *max_clusters = n;
        return cudaSuccess;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, rk);
}

template <typename F>
cudaError_t with_res(int P, F f) {
    switch (P) {
        case 1: return f.template run<1>();
        case 2: return f.template run<2>();
        case 4: return f.template run<4>();
        case 6: return f.template run<6>();
        case 8: return f.template run<8>();
        case 12: return f.template run<12>();
        case 16: return f.template run<16>();
        default: return f.template run<24>();
    }
}

struct ResF {
    const FpsArgs* a;
    const FpsRanks* rk;
    int64_t nclusters;
    int C;
    cudaStream_t s;
    bool query;
    int* maxc;
    bool spec = false;
    template <int P>
    cudaError_t run() const {
        return spec ? launch_res_p<P, true>(*a, *rk, nclusters, C, s, query, maxc)
                    : launch_res_p<P, false>(*a, *rk, nclusters, C, s, query, maxc);
    }
};

int res_choose_P(int64_t S) {
    static const int kPs[] = {1, 2, 4, 6, 8, 12, 16, 24};
    for (int p : kPs)
        if ((int64_t)p * kT >= S) return p;
    return 0;
}

int res_max_clusters(int P, int C) {
    static int cache[kMaxC + 1][kMaxP + 1];
    static bool init = false;
    if (!init) {
        for (auto& row : cache)
            for (int& v : row) v = -1;
        init = true;
    }
    if (cache[C][P] >= 0) return cache[C][P];
    FpsArgs a = {};
    FpsRanks rk = {};
    int n = 0;
    with_res(P, ResF{&a, &rk, 64, C, nullptr, true, &n});
    cache[C][P] = n;
    return n;
}

}  // namespace

// Resident plan for clouds of N points split over G ranks (G clusters per
// cloud): cluster width C and points per thread P.  Returns false when no
// width keeps every cluster of the launch co-resident.
bool fps_res_plan(int64_t N, int64_t nclusters, int G, int* C_out, int* P_out) {
    const char* env = getenv("PS_FPS_CLUSTER");
    const char* tgt = getenv("PS_FPS_TARGET");
    const int64_t Ns = (N + G - 1) / G;
    const int64_t target = tgt ? atoll(tgt) : 2048;  // points per CTA
    int want = (int)((Ns + target - 1) / target);
    want = want < 1 ? 1 : (want > kMaxC ? kMaxC : want);
    static const int kCs[] = {16, 14, 12, 10, 8, 7, 6, 5, 4, 3, 2, 1};
    for (int C : kCs) {
        if (env && C != atoi(env)) continue;
        if (!env && C > want) continue;
        const int64_t S = (Ns + C - 1) / C;
        const int P = res_choose_P(S);
        if (P == 0) {
            if (C == kMaxC || env) return false;
            continue;
        }
        if (res_max_clusters(P, C) >= nclusters) {
            *C_out = C;
            *P_out = P;
            return true;
        }
        if (env) return false;
    }
    return false;
}

cudaError_t launch_fps_res(FpsArgs a, const FpsRanks& rk_in, int64_t B, int C, int P, cudaStream_t s) {
    FpsRanks rk = rk_in;
    const char* spe = getenv("PS_FPS_SPATIAL");
    rk.spatial = spe ? atoi(spe) : 1;
    const int64_t Ns = (a.N + rk.G - 1) / rk.G;
    a.points_per_cta = (Ns + C - 1) / C;
    const int64_t nclusters = B * rk.Gl;
    if (kTiming && getenv("PS_FPS_TIMING")) {
        // development aid: per-phase SM cycles of the first 256 iterations
        // (cloud 0, rank 0, CTA 0, thread 0) printed to stderr; synchronises.
        static long long* dbg = nullptr;
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 256 * 12);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 256 * 12, s);
        a.dbg = dbg;
        a.dbg_t0 = getenv("PS_FPS_T0") ? atoll(getenv("PS_FPS_T0")) : 0;
        cudaError_t e = with_res(P, ResF{&a, &rk, nclusters, C, s, false, nullptr});
        if (e != cudaSuccess) return e;
        static long long h[256 * 12];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const int iters = (int)((a.k_stop - a.k_start - a.dbg_t0) < 256 ? (a.k_stop - a.k_start - a.dbg_t0) : 256);
        for (int lo = 8; lo < iters; lo += 64) {
            double acc[8] = {0};
            int cnt = 0;
            for (int t = lo; t < iters && t < lo + 64; ++t, ++cnt)
                for (int k = 0; k < 8; ++k) acc[k] += (double)h[t * 8 + k];
            if (cnt)
                fprintf(stderr, "[fps-res timing] C=%d P=%d G=%d N=%lld iters %d-%d (leader) cycles: fold %.0f "
                        "bar %.0f (argmax %.0f, rec %.0f) send %.0f wait %.0f bcast %.0f total %.0f\n", C, P, rk.G,
                        (long long)a.N, lo, lo + cnt, acc[0] / cnt, acc[1] / cnt, acc[6] / cnt, acc[7] / cnt,
                        acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt);
        }
        return cudaSuccess;
    }
    a.dbg = nullptr;
    ResF f{&a, &rk, nclusters, C, s, false, nullptr};
    f.spec = getenv("PS_RES_NOSPEC") == nullptr;  // speculative exchange loop (default)
    return with_res(P, f);
}

// Clouds too large for one cluster (> 16 CTAs x 24 points per thread): the
// point split over G co-resident virtual ranks on this GPU -- the protocol of
unsigned long long split_timeout_ns() {
    const char* e = getenv("PS_SPLIT_TIMEOUT_MS");
    return e ? (unsigned long long)atoll(e) * 1000000ull : kMboxTimeoutNs;
}

// ps_fps on a cloud too large for one cluster: the point split over G
// virtual ranks with mailboxes owned here, one buffer per (device, stream, B,
// G), so launches that share one are ordered by their stream.  The first use
// allocates; inside a graph capture (no allocation possible) the capture
// borrows the buffer last made for (device, B, G) -- the eager warm-up run
// that precedes a capture -- or, without one, declines (the streaming
// kernel runs instead).

static cudaError_t launch_fps_virtual_split(FpsArgs a, int64_t B, cudaStream_t s) {
    static const int kGs[] = {10, 12, 16, 8, 20, 24, 32};
    int C = 0, P = 0, G = 0;
    for (int gg : kGs) {
        if (fps_res_plan(a.N, B * gg, gg, &C, &P)) { G = gg; break; }
    }
    if (G == 0) return cudaErrorNotSupported;
    struct Box {
        int dev;
        cudaStream_t stream;
        int64_t B;
        int G;
        uint8_t* buf;
        uint4** ptrs;
        size_t per_rank;
        uint32_t* seq;  // device: [0] tag base of the current launch, [1] next base
    };
    static Box boxes[16];
    static int nboxes = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    Box* bx = nullptr;
    for (int i = 0; i < nboxes; ++i)
        if (boxes[i].dev == dev && boxes[i].stream == s && boxes[i].B == B && boxes[i].G == G) bx = &boxes[i];
    const size_t per_rank = (size_t)B * 3 * (size_t)G * kMbRecs * kRecU4 * sizeof(uint4);
    if (!bx) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
            for (int i = nboxes - 1; i >= 0 && !bx; --i)
                if (boxes[i].dev == dev && boxes[i].B == B && boxes[i].G == G) bx = &boxes[i];
            if (!bx) return cudaErrorNotSupported;
        }
    }
    if (!bx) {
        if (nboxes == 16) return cudaErrorNotSupported;  // the streaming kernel serves the rest
        Box nb = {dev, s, B, G, nullptr, nullptr, per_rank, nullptr};
        cudaError_t e = cudaMalloc(&nb.buf, per_rank * G);
        if (e != cudaSuccess) return e;
        e = cudaMalloc(&nb.ptrs, sizeof(uint4*) * G);
        if (e != cudaSuccess) return e;
        e = cudaMalloc(&nb.seq, sizeof(uint32_t) * 2);
        if (e != cudaSuccess) return e;
        uint4* hp[kMaxRanks];
        for (int g = 0; g < G; ++g) hp[g] = reinterpret_cast<uint4*>(nb.buf + per_rank * g);
        e = cudaMemcpy(nb.ptrs, hp, sizeof(uint4*) * G, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return e;
        e = cudaMemset(nb.buf, 0xff, per_rank * G);
        if (e != cudaSuccess) return e;
        e = cudaMemset(nb.seq, 0, sizeof(uint32_t) * 2);
        if (e != cudaSuccess) return e;
        boxes[nboxes] = nb;
        bx = &boxes[nboxes++];
    }
    // the tag base is advanced on the device, in stream order, so that every
    // launch -- also every replay of a captured graph -- gets fresh tags
    mbox_epoch_kernel<<<1, 256, 0, s>>>(bx->seq, reinterpret_cast<uint4*>(bx->buf), bx->per_rank * G / sizeof(uint4),
                                        (uint32_t)a.k_stop);
    FpsRanks rk = {};
    rk.G = G; rk.Gl = G; rk.g_base = 0; rk.all_write = 0;
    rk.seq_base = 0;
    rk.seq_dev = bx->seq;
    rk.timeout_ns = split_timeout_ns();
    rk.mbox = bx->ptrs;
    if (getenv("PS_FPS_VERBOSE"))
        fprintf(stderr, "[fps-split] N=%lld B=%lld G=%d C=%d P=%d (virtual ranks)\n", (long long)a.N,
                (long long)B, G, C, P);
    return launch_fps_res(a, rk, B, C, P, s);
}

cudaError_t launch_fps(FpsArgs a, int64_t B, cudaStream_t s) {
    // The legacy register kernel (fps.cu) has the shorter per-iteration
    // chain while a cluster holds the cloud in registers (<= 16 points per
    // thread); beyond that it streams md/xyz through L2 and the resident
    // kernel's warp skipping wins (measured: profiles/r01/fps_resident.log).
    // PS_FPS_RESIDENT=1 / PS_FPS_LEGACY=1 force either kernel.
    int C = 0, P = 0;
    const bool force_res = getenv("PS_FPS_RESIDENT") != nullptr;
    const bool force_leg = getenv("PS_FPS_LEGACY") != nullptr;
    if (!force_res && !force_leg && !getenv("PS_FPS_NOSMALL") && !getenv("PS_FPS_NOSPEC") && !getenv("PS_FPS_SPEC")) {
        const cudaError_t e = launch_fps_small(a, B, s);  // small clouds: one CTA each, registers
        if (e != cudaErrorNotSupported) return e;
    }
    bool use_res = force_res;
    if (!force_res && !force_leg) {
        int lc = 0, lp = 0, lt = 0;
        fps_choose_cluster(a.N, B, &lc, &lp, &lt);
        use_res = lp == 0;
    }
    if (use_res && fps_res_plan(a.N, B, 1, &C, &P)) {
        if (getenv("PS_FPS_VERBOSE"))
            fprintf(stderr, "[fps-res] N=%lld B=%lld C=%d P=%d\n", (long long)a.N, (long long)B, C, P);
        FpsRanks rk = {};
        rk.G = 1; rk.Gl = 1; rk.g_base = 0;
        return launch_fps_res(a, rk, B, C, P, s);
    }
    if (!getenv("PS_FPS_NOSPEC")) {
        const cudaError_t e = launch_fps_spec(a, B, s);
        if (e != cudaErrorNotSupported) return e;
    }
    if (use_res && !force_leg && !getenv("PS_FPS_NOSPLIT")) {
        const cudaError_t e = launch_fps_virtual_split(a, B, s);
        if (e != cudaErrorNotSupported) return e;
    }
    return launch_fps_legacy(a, B, s);
}

}  // namespace ps
