// fps_util.cuh -- record type and argmax / skip-threshold helpers shared by
// the register-resident FPS kernels (fps.cu: one sample per exchange,
// fps_spec.cu: top-K speculation).
#pragma once

#include "common.cuh"

namespace ps {
namespace {

constexpr int kMaxCluster = 16;
#ifndef PS_TIMING
#define PS_TIMING 0
#endif
constexpr bool kTiming = PS_TIMING;  // per-iteration cycle stamps (make TIMING=1)
constexpr uint32_t kNone = 0xffffffffu;

struct __align__(16) Rec {
    uint32_t klo, khi, idx, taken;
    float x, y, z;
    uint32_t pad;
};

PS_DEV uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
PS_DEV double bitsd(uint64_t k) { return __longlong_as_double((long long)k); }

// Winner lane of a warp argmax over (key, idx): max key, lowest idx on ties.
// Fast path: one REDUX on the high key word; the full comparison only runs
// when several lanes share that word.  Returns -1 if no lane has idx != kNone.
PS_DEV int warp_argmax_lane(uint64_t key, uint32_t idx) {
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

PS_DEV uint64_t rec_key(const Rec& r) { return ((uint64_t)r.khi << 32) | r.klo; }

// Lowest-index record among recs[0..n), broadcast to every lane (fallback).
PS_DEV Rec warp_min_idx_recs(const Rec* recs, int n, int lane) {
    const uint32_t idx = lane < n ? recs[lane].idx : kNone;
    const uint32_t m = __reduce_min_sync(kFull, idx);
    const unsigned w = __ballot_sync(kFull, idx == m && idx != kNone);
    if (!w) { Rec z{}; z.idx = kNone; return z; }
    return recs[__ffs(w) - 1];
}

// conservative float32 skip threshold for "d < md" (see kernel comment)
PS_DEV float skip_threshold(double md) {
    if (md == 0.0) return -1.0f;                     // nothing is closer than 0
    if (!(md >= 7.888609052210118e-31)) return __int_as_float(0x7f800000);  // tiny: always exact
    return __fmul_ru(__double2float_ru(md), 1.0f + 3.814697265625e-06f);    // * (1 + 2^-18)
}

// Same threshold from the float32 distance already computed for the screen:
// d32 >= d (1 - 6 * 2^-24), so f32_ru(d32 * (1 + 2^-17)) >= d (1 + 2^-18) and
// the skip argument above holds; d = 0 -> never fold, tiny/overflowing ->
// always fold exactly.  Avoids a float64->float32 conversion per update.
PS_DEV float skip_threshold_d32(double d, float d32) {
    if (dbits(d) == 0) return -1.0f;
    if (!(d32 >= 7.888609052210118e-31f) || !(d32 < 1e38f)) return __int_as_float(0x7f800000);
    return __fmul_ru(d32, 1.0f + 7.62939453125e-06f);  // * (1 + 2^-17)
}

}  // namespace
}  // namespace ps
