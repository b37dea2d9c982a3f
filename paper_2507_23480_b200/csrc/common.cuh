// common.cuh -- shared device helpers for the sm_100a FastPoint kernels.
//
// Numerics contract: every squared distance that decides an
// index is computed in float64 as ((dx*dx + dy*dy) + dz*dz) with explicitly
// rounded intrinsics, so nvcc can never contract it into DFMA -- the exact
// operation sequence of the reference numba kernels
// (/root/reference/pkg/src/pointsample/_kernels.py:55-58, 149-152).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define PS_DEV __device__ __forceinline__

namespace ps {

constexpr uint32_t kFull = 0xffffffffu;

// f64 squared distance, no contraction (DADD/DMUL only).
PS_DEV double sqdist(double ax, double ay, double az, double bx, double by, double bz) {
    const double dx = __dsub_rn(bx, ax);
    const double dy = __dsub_rn(by, ay);
    const double dz = __dsub_rn(bz, az);
    double s = __dmul_rn(dx, dx);
    s = __dadd_rn(s, __dmul_rn(dy, dy));
    s = __dadd_rn(s, __dmul_rn(dz, dz));
    return s;
}

PS_DEV double sqdist4(float4 a, float4 b) {
    return sqdist((double)a.x, (double)a.y, (double)a.z, (double)b.x, (double)b.y, (double)b.z);
}

// Conservative float32 pre-filter for "d2 < r2": the f32
// evaluation of three rounded squared differences has relative error below
// 6 * 2^-24 when nothing underflows, and absolute error below 2^-125 when
// something does.  thr = f32(r2) * (1 + 2^-16) + 2^-120 therefore never
// rejects a pair whose exact float64 d2 is below r2; every accepted pair is
// re-checked exactly in float64.  Returns +inf-ish thresholds unchanged.
PS_DEV float prefilter_threshold(double r2) {
    float t = __double2float_ru(r2);
    t = __fmul_ru(t, 1.0f + 1.52587890625e-05f);  // 1 + 2^-16
    return __fadd_ru(t, 7.52316384526264e-37f);   // + 2^-120
}

PS_DEV float sqdist_f32(float4 a, float4 b) {
    const float dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// ---- warp argmax over (float64 key >= 0, lowest index on ties) -----------
// key = raw bits of a non-negative double (monotone as u64).
struct ArgMax {
    uint64_t key;
    uint32_t idx;
};

PS_DEV ArgMax warp_argmax(uint64_t key, uint32_t idx) {
    const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
    const uint32_t mhi = __reduce_max_sync(kFull, hi);
    const uint32_t mlo = __reduce_max_sync(kFull, hi == mhi ? lo : 0u);
    const bool win = (hi == mhi) && (lo == mlo);
    const uint32_t midx = __reduce_min_sync(kFull, win ? idx : 0xffffffffu);
    ArgMax r;
    r.key = ((uint64_t)mhi << 32) | mlo;
    r.idx = midx;
    return r;
}

// ---- cluster / DSMEM / mbarrier PTX wrappers (sm_90+) -------------------

PS_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
PS_DEV uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
PS_DEV uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
PS_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
PS_DEV uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// map a local shared::cta address to the same variable in CTA `rank`
PS_DEV uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
PS_DEV void st_cluster_u64(uint32_t addr, uint64_t v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
PS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PS_DEV void fence_mbar_init_cluster() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
PS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// wait for phase `parity` of a local mbarrier; acquire at cluster scope so
// st.async data from peer CTAs is visible afterwards.
PS_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity) : "memory");
}
// Same wait with CTA-scope acquire: enough for bytes delivered into this
// CTA's shared memory by st.async / cp.async.bulk complete_tx (the
// transaction mechanism makes them visible), and ptxas emits no L1
// invalidation (CCTL.IVALL) for it, unlike the cluster-scope acquire.
PS_DEV void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity) : "memory");
}
// 16-byte asynchronous store into a peer CTA's shared memory that signals
// the peer's mbarrier with complete_tx(16).
PS_DEV void st_async_v4(uint32_t remote_addr, uint32_t remote_bar, uint32_t a, uint32_t b,
                        uint32_t c, uint32_t d) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%2, %3, %4, %5}, [%1];"
        ::"r"(remote_addr), "r"(remote_bar), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Remote arrive on a peer CTA's mbarrier that also raises its expected
// transaction bytes: a sender announces a variable-length st.async payload
// (barrier initialised with one arrival per sender).
PS_DEV void mbar_remote_arrive_expect_tx(uint32_t remote_bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;"
                 ::"r"(remote_bar), "r"(bytes) : "memory");
}

// CTA-scope release store / acquire load on shared memory (producer warp
// publishing to consumer warps without a block barrier).
PS_DEV void st_release_cta(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
PS_DEV uint32_t ld_acquire_cta(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// Named barriers (ids 1..15; 0 is __syncthreads): producer arrives without
// waiting, consumers sync; nthreads counts both sides.
PS_DEV void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
PS_DEV void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Shared-memory accesses on 32-bit shared::cta addresses (smem_u32 of a
// __shared__ symbol is a constant): in cluster kernels nvcc otherwise forms
// many shared addresses from the CTA's cluster id (S2R SR_CgaCtaId, a
// variable-latency read) on the critical path.
PS_DEV void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
PS_DEV void sts_u32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
PS_DEV void sts_f64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); }
PS_DEV void sts_v4(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
PS_DEV uint32_t lds_u8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
PS_DEV uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
PS_DEV uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
PS_DEV double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
PS_DEV uint4 lds_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}

// ---- row ordering by (d2, index) ----------------------------------------
// (d2, index) order.  d2 >= 0 (or +inf padding), so its bit pattern orders
// like an unsigned integer: integer compares keep the sort off the FP64 pipe.
__device__ __forceinline__ bool key_less(double da, int32_t ia, double db, int32_t ib) {
    const unsigned long long ua = (unsigned long long)__double_as_longlong(da);
    const unsigned long long ub = (unsigned long long)__double_as_longlong(db);
    return ua < ub || (ua == ub && ia < ib);
}

// Warp bitonic network over 64 keys held two per lane (slot lane, lane+32),
// padded with (+inf, INT_MAX).  All compare-exchanges are register shuffles.
__device__ __forceinline__ void warp_bitonic64(double& d0, int32_t& i0, double& d1, int32_t& i1, int lane,
                                               int n2) {
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
        if (k > n2) break;
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                // partner of slot lane is slot lane+32, same thread
                const bool up = ((lane & k) == 0);  // k == 64: always ascending
                const bool sw = up ? key_less(d1, i1, d0, i0) : key_less(d0, i0, d1, i1);
                if (sw) {
                    const double td = d0; d0 = d1; d1 = td;
                    const int32_t ti = i0; i0 = i1; i1 = ti;
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double& d = h ? d1 : d0;
                    int32_t& ix = h ? i1 : i0;
                    const int s = lane + 32 * h;
                    const double od = __shfl_xor_sync(kFull, d, j);
                    const int32_t oi = __shfl_xor_sync(kFull, ix, j);
                    const bool lower = (s & j) == 0;
                    const bool up = (s & k) == 0;
                    // the lower slot keeps the min when ascending
                    const bool mine_less = key_less(d, ix, od, oi);
                    const bool keep_min = (lower == up);
                    if (keep_min != mine_less) { d = od; ix = oi; }
                }
            }
        }
    }
}

}  // namespace ps
