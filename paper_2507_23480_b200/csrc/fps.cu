// fps.cu -- K1: exact farthest-point sampling, one thread-block cluster per
// cloud (B200 / sm_100a).
//
// Replaces _kernels.fps_loop (/root/reference/pkg/src/pointsample/_kernels.py:35-74)
// and its chunked form fps_update_chunk/first_untaken (:77-100).
//
// Layout: a cloud is float4[N] (x, y, z, pad) in HBM.  The cluster's C CTAs
// split the cloud into C contiguous ranges; every thread keeps P points
// (coordinates widened to float64, and the float64 min-distance md) in
// registers for the whole run, so an iteration touches no memory except the
// exchange records.  Per iteration:
//   1. fold the last sample into md (float64, no FMA), thread-local argmax;
//   2. warp argmax with three REDUX ops (max hi word, max lo word, min index:
//      md >= 0 so its bits order like u64, and the lowest index wins ties);
//   3. block argmax over the 8 warp records in shared memory;
//   4. each CTA pushes its 32-byte record (key, index, taken, xyz) into every
//      peer CTA's shared memory with st.async + mbarrier complete_tx
//      (double-buffered by iteration parity) -- no cluster-wide barrier on
//      the critical path;
//   5. every warp waits on its CTA's mbarrier and reduces the C records
//      identically, so all CTAs agree on the winner without a second round.
// The duplicate fallback of _kernels.py:65-70 (max <= 0 or winner already
// taken -> lowest untaken index) runs as a rare second exchange.
//
// Clouds larger than C*THREADS*16 points use the P == 0 instantiation which
// streams xyz/md through L2 each iteration (same exchange protocol).

#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

namespace {

constexpr int kFpsThreads = 256;
constexpr int kFpsWarps = kFpsThreads / 32;
constexpr int kMaxCluster = 16;
constexpr uint32_t kNone = 0xffffffffu;

struct __align__(16) Rec {
    uint32_t klo, khi, idx, taken;
    float x, y, z;
    uint32_t pad;
};

PS_DEV uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
PS_DEV double bitsd(uint64_t k) { return __longlong_as_double((long long)k); }

// Reduce records rec[0..n) (n <= 32) held by lanes < n; returns winner in all lanes.
PS_DEV Rec warp_reduce_recs(const Rec* recs, int n, int lane) {
    uint64_t key = 0;
    uint32_t idx = kNone;
    Rec mine{};
    if (lane < n) {
        mine = recs[lane];
        key = ((uint64_t)mine.khi << 32) | mine.klo;
        idx = mine.idx;
    }
    const ArgMax am = warp_argmax(key, idx);
    const uint32_t winmask = __ballot_sync(kFull, idx == am.idx && idx != kNone);
    Rec out;
    out.klo = (uint32_t)am.key;
    out.khi = (uint32_t)(am.key >> 32);
    out.idx = am.idx;
    const int src = winmask ? __ffs(winmask) - 1 : 0;
    out.taken = __shfl_sync(kFull, mine.taken, src);
    out.x = __shfl_sync(kFull, mine.x, src);
    out.y = __shfl_sync(kFull, mine.y, src);
    out.z = __shfl_sync(kFull, mine.z, src);
    out.pad = 0;
    return out;
}

// Same, but minimum index (fallback: lowest untaken point).
PS_DEV Rec warp_min_idx_recs(const Rec* recs, int n, int lane) {
    Rec mine{};
    uint32_t idx = kNone;
    if (lane < n) {
        mine = recs[lane];
        idx = mine.idx;
    }
    const uint32_t m = __reduce_min_sync(kFull, idx);
    const uint32_t winmask = __ballot_sync(kFull, idx == m && idx != kNone);
    const int src = winmask ? __ffs(winmask) - 1 : 0;
    Rec out;
    out.klo = __shfl_sync(kFull, mine.klo, src);
    out.khi = __shfl_sync(kFull, mine.khi, src);
    out.idx = m;
    out.taken = __shfl_sync(kFull, mine.taken, src);
    out.x = __shfl_sync(kFull, mine.x, src);
    out.y = __shfl_sync(kFull, mine.y, src);
    out.z = __shfl_sync(kFull, mine.z, src);
    out.pad = 0;
    return out;
}

template <int P>
__global__ void __launch_bounds__(kFpsThreads, 1) fps_cluster_kernel(FpsArgs a) {
    __shared__ Rec warp_rec[kFpsWarps];
    __shared__ Rec slots[2][kMaxCluster];
    __shared__ Rec fb_slots[kMaxCluster];
    __shared__ __align__(8) uint64_t bars[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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

    // ---- state into registers -------------------------------------------
    double px[P > 0 ? P : 1], py[P > 0 ? P : 1], pz[P > 0 ? P : 1], m[P > 0 ? P : 1];
    uint32_t tk = 0;
    if constexpr (P > 0) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int64_t j = lo + tid + (int64_t)q * kFpsThreads;
            if (j < hi) {
                const float4 v = xyz[j];
                px[q] = v.x; py[q] = v.y; pz[q] = v.z;
                if (a.fresh) {
                    m[q] = __longlong_as_double(0x7ff0000000000000LL);
                    tk |= (j == seed ? 1u : 0u) << q;
                } else {
                    m[q] = md[j];
                    tk |= (taken[j] ? 1u : 0u) << q;
                }
            } else {
                px[q] = py[q] = pz[q] = 0.0;
                m[q] = 0.0;
            }
        }
    } else {
        if (a.fresh) {
            for (int64_t j = lo + tid; j < hi; j += kFpsThreads) {
                md[j] = __longlong_as_double(0x7ff0000000000000LL);
                taken[j] = (j == seed) ? 1 : 0;
            }
        }
    }
    if (a.fresh && r == 0 && tid == 0) {
        out[0] = seed;
        curve[0] = __longlong_as_double(0x7ff0000000000000LL);
    }

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init_cluster();
        mbar_arrive_expect_tx(&bars[0], C * (uint32_t)sizeof(Rec));
        mbar_arrive_expect_tx(&bars[1], C * (uint32_t)sizeof(Rec));
    }
    // also orders the fresh-mode md/taken init (P == 0) before the loop
    cluster_sync_all();

    if (k_start < k_stop) {
        // last sample coordinates
        int64_t last = out[k_start - 1];
        float4 lv = xyz[last];
        double sx = lv.x, sy = lv.y, sz = lv.z;

        for (int64_t it = k_start; it < k_stop; ++it) {
            const uint32_t t = (uint32_t)(it - k_start);
            const uint32_t par = t & 1u;
            const uint32_t phase = (t >> 1) & 1u;

            // 1. fold + thread argmax
            uint64_t bkey = 0;
            uint32_t bidx = kNone;
            float bx = 0.f, by = 0.f, bz = 0.f;
            uint32_t btk = 0;
            if constexpr (P > 0) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int64_t j = lo + tid + (int64_t)q * kFpsThreads;
                    if (j < hi) {
                        const double d = sqdist(sx, sy, sz, px[q], py[q], pz[q]);
                        if (d < m[q]) m[q] = d;
                        const uint64_t key = dbits(m[q]);
                        if (bidx == kNone || key > bkey) {
                            bkey = key;
                            bidx = (uint32_t)j;
                            bx = (float)px[q]; by = (float)py[q]; bz = (float)pz[q];
                            btk = (tk >> q) & 1u;
                        }
                    }
                }
            } else {
                for (int64_t j = lo + tid; j < hi; j += kFpsThreads) {
                    const float4 v = xyz[j];
                    const double d = sqdist(sx, sy, sz, (double)v.x, (double)v.y, (double)v.z);
                    double mj = md[j];
                    if (d < mj) { mj = d; md[j] = d; }
                    const uint64_t key = dbits(mj);
                    if (bidx == kNone || key > bkey) {
                        bkey = key; bidx = (uint32_t)j;
                        bx = v.x; by = v.y; bz = v.z;
                    }
                }
                if (bidx != kNone) btk = taken[bidx];
            }

            // 2. warp argmax
            const ArgMax wa = warp_argmax(bkey, bidx);
            if (bidx == wa.idx && bidx != kNone) {
                Rec rr;
                rr.klo = (uint32_t)wa.key; rr.khi = (uint32_t)(wa.key >> 32);
                rr.idx = wa.idx; rr.taken = btk;
                rr.x = bx; rr.y = by; rr.z = bz; rr.pad = 0;
                warp_rec[warp] = rr;
            } else if (lane == 0 && wa.idx == kNone) {
                Rec rr{};
                rr.idx = kNone;
                warp_rec[warp] = rr;
            }
            __syncthreads();

            // 3+4. block argmax, push record to every CTA of the cluster
            if (warp == 0) {
                const Rec cr = warp_reduce_recs(warp_rec, kFpsWarps, lane);
                if (lane < (int)C) {
                    const uint32_t dst = mapa(smem_u32(&slots[par][r]), lane);
                    const uint32_t dbar = mapa(smem_u32(&bars[par]), lane);
                    st_async_v4(dst, dbar, cr.klo, cr.khi, cr.idx, cr.taken);
                    st_async_v4(dst + 16, dbar, __float_as_uint(cr.x), __float_as_uint(cr.y),
                                __float_as_uint(cr.z), 0u);
                }
            }

            // 5. wait for all C records, reduce identically in every warp
            mbar_wait_cluster(&bars[par], phase);
            Rec win = warp_reduce_recs(slots[par], (int)C, lane);
            __syncwarp();
            if (tid == 0) mbar_arrive_expect_tx(&bars[par], C * (uint32_t)sizeof(Rec));

            double best = bitsd(((uint64_t)win.khi << 32) | win.klo);
            if (best <= 0.0 || win.taken) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken index
                uint32_t fidx = kNone;
                Rec fr{};
                if constexpr (P > 0) {
#pragma unroll
                    for (int q = P - 1; q >= 0; --q) {
                        const int64_t j = lo + tid + (int64_t)q * kFpsThreads;
                        if (j < hi && !((tk >> q) & 1u)) {
                            fidx = (uint32_t)j;
                            const uint64_t k = dbits(m[q]);
                            fr.klo = (uint32_t)k; fr.khi = (uint32_t)(k >> 32);
                            fr.x = (float)px[q]; fr.y = (float)py[q]; fr.z = (float)pz[q];
                        }
                    }
                } else {
                    for (int64_t j = lo + tid; j < hi; j += kFpsThreads) {
                        if (!taken[j]) {
                            fidx = (uint32_t)j;
                            const uint64_t k = dbits(md[j]);
                            const float4 v = xyz[j];
                            fr.klo = (uint32_t)k; fr.khi = (uint32_t)(k >> 32);
                            fr.x = v.x; fr.y = v.y; fr.z = v.z;
                            break;
                        }
                    }
                }
                fr.idx = fidx;
                const uint32_t wm = __reduce_min_sync(kFull, fidx);
                __syncthreads();  // warp_rec reuse
                if (fidx == wm && fidx != kNone) warp_rec[warp] = fr;
                else if (lane == 0 && wm == kNone) { Rec z{}; z.idx = kNone; warp_rec[warp] = z; }
                __syncthreads();
                if (warp == 0) {
                    const Rec cr = warp_min_idx_recs(warp_rec, kFpsWarps, lane);
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
                if (fw.idx != kNone) {
                    win = fw;
                    best = bitsd(((uint64_t)fw.khi << 32) | fw.klo);
                }
            }

            // record, mark taken, next sample
            if (r == 0 && tid == 0) {
                out[it] = (int64_t)win.idx;
                curve[it] = sqrt(best);
            }
            const int64_t wj = (int64_t)win.idx;
            if constexpr (P > 0) {
                if (wj >= lo && wj < hi && ((wj - lo) % kFpsThreads) == tid)
                    tk |= 1u << (uint32_t)((wj - lo) / kFpsThreads);
            } else {
                if (wj >= lo && wj < hi && ((wj - lo) % kFpsThreads) == tid) taken[wj] = 1;
            }
            sx = win.x; sy = win.y; sz = win.z;
        }
    }

    // ---- write back md / taken ---------------------------------------------
    if constexpr (P > 0) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int64_t j = lo + tid + (int64_t)q * kFpsThreads;
            if (j < hi) {
                md[j] = m[q];
                taken[j] = (tk >> q) & 1u;
            }
        }
    }
    cluster_sync_all();  // no CTA leaves while peers may still target its smem
}

template <int P>
cudaError_t launch_p(const FpsArgs& a, int64_t B, int C, cudaStream_t s) {
    auto kern = fps_cluster_kernel<P>;
    cudaError_t e = cudaSuccess;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * C), 1, 1);
    cfg.blockDim = dim3(kFpsThreads, 1, 1);
    cfg.dynamicSmemBytes = 0;
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

int fps_choose_cluster(int64_t N, int64_t B, int* C_out, int* P_out) {
    static const int kPs[] = {1, 2, 3, 4, 6, 8, 12, 16};
    const char* env = getenv("PS_FPS_CLUSTER");
    int C = 1;
    if (env) {
        C = atoi(env);
    } else {
        const int64_t target = (int64_t)kFpsThreads * 4;
        int64_t c = (N + target - 1) / target;
        C = (int)(c < 1 ? 1 : (c > kMaxCluster ? kMaxCluster : c));
        // more clusters than fit in one wave: trade cluster width for concurrency
        while (C > 8 && B * C > 128) C /= 2;
    }
    if (C < 1) C = 1;
    if (C > kMaxCluster) C = kMaxCluster;
    const int64_t S = (N + C - 1) / C;
    int P = 0;
    for (int p : kPs) {
        if ((int64_t)p * kFpsThreads >= S) { P = p; break; }
    }
    *C_out = C;
    *P_out = P;  // 0 = streaming
    return 0;
}

cudaError_t launch_fps(FpsArgs a, int64_t B, cudaStream_t s) {
    int C = 1, P = 0;
    fps_choose_cluster(a.N, B, &C, &P);
    a.points_per_cta = (a.N + C - 1) / C;
    switch (P) {
        case 1: return launch_p<1>(a, B, C, s);
        case 2: return launch_p<2>(a, B, C, s);
        case 3: return launch_p<3>(a, B, C, s);
        case 4: return launch_p<4>(a, B, C, s);
        case 6: return launch_p<6>(a, B, C, s);
        case 8: return launch_p<8>(a, B, C, s);
        case 12: return launch_p<12>(a, B, C, s);
        case 16: return launch_p<16>(a, B, C, s);
        default: return launch_p<0>(a, B, C, s);
    }
}

}  // namespace ps
