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
#include "fps_util.cuh"
#include "ps_internal.h"

namespace ps {

namespace {


// Per point: the float32 distance to the new sample decides whether the exact
// float64 fold can change md.  d32 carries relative error < 6 * 2^-24, so
// d32 > f32_up(md) * (1 + 2^-18) proves d_exact > md and the fold is a no-op;
// otherwise the float64 distance ((dx*dx + dy*dy) + dz*dz) is evaluated and
// folded exactly as _kernels.py:55-60.  The float32 test only skips work --
// md, the argmax and every output are the float64 reference values.
template <int P, int T>
__global__ void __launch_bounds__(T, 1) fps_cluster_kernel(FpsArgs a) {
    constexpr int kFpsThreads = T;
    constexpr int kFpsWarps = T / 32;
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
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const uint32_t tx_bytes = C * (uint32_t)sizeof(Rec);

    // ---- state into registers -------------------------------------------
    constexpr int PP = P > 0 ? P : 1;
    float fx[PP], fy[PP], fz[PP], thr[PP];
    double m[PP];
    uint32_t tk = 0, valid = 0;
    double bv = -1.0;  // cached thread-local max md (P > 0), its slot and coordinates
    int bq = 0;
    float bx = 0.f, by = 0.f, bz = 0.f;
    if constexpr (P > 0) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int64_t j = lo + tid + (int64_t)q * kFpsThreads;
            fx[q] = fy[q] = fz[q] = 0.f;
            m[q] = 0.0;
            if (j < hi) {
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
            thr[q] = ((valid >> q) & 1u) ? skip_threshold(m[q]) : -1.0f;  // invalid: never folded
        }
    } else {
        if (a.fresh) {
            for (int64_t j = lo + tid; j < hi; j += kFpsThreads) {
                md[j] = kInf;
                taken[j] = (j == seed) ? 1 : 0;
            }
        }
    }
    if (a.fresh && r == 0 && tid == 0) {
        out[0] = seed;
        curve[0] = kInf;
    }

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init_cluster();
        mbar_arrive_expect_tx(&bars[0], tx_bytes);
        mbar_arrive_expect_tx(&bars[1], tx_bytes);
    }
    // also orders the fresh-mode md/taken init (P == 0) before the loop
    cluster_sync_all();

    if (k_start < k_stop) {
        const int64_t last = a.fresh ? seed : out[k_start - 1];
        const float4 lv = xyz[last];
        float sx32 = lv.x, sy32 = lv.y, sz32 = lv.z;
        bool dirty = true;  // recompute the cached local max
        // exchange addresses of this lane's destination CTA (leader warp, lane < C)
        const uint32_t dl = (uint32_t)lane < C ? (uint32_t)lane : 0u;
        const uint32_t dst0 = mapa(smem_u32(&slots[0][r]), dl), dst1 = mapa(smem_u32(&slots[1][r]), dl);
        const uint32_t dbar0 = mapa(smem_u32(&bars[0]), dl), dbar1 = mapa(smem_u32(&bars[1]), dl);

        for (int64_t it = k_start; it < k_stop; ++it) {
            const uint32_t t_abs = (uint32_t)(it - k_start);
            const uint32_t par = t_abs & 1u;
            const uint32_t phase = (t_abs >> 1) & 1u;
            const uint32_t t = t_abs - (uint32_t)a.dbg_t0;
            const bool tdbg = kTiming && a.dbg && b == 0 && r == 0 && tid == 0 && t_abs >= a.dbg_t0 && t < 256;
            long long ts0 = 0;
            if (tdbg) ts0 = clock64();
            const double sx = sx32, sy = sy32, sz = sz32;

            // 1. fold + thread argmax
            uint64_t bkey = 0;
            uint32_t bidx = kNone;
            Rec mine;
            mine.pad = 0;
            mine.taken = 0;
            mine.x = mine.y = mine.z = 0.f;
            if constexpr (P > 0) {
                // 1a. float32 screen: which of my points can the new sample move?
                uint32_t need = 0;
                float d32s[P];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const float dx = fx[q] - sx32, dy = fy[q] - sy32, dz = fz[q] - sz32;
                    const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                    d32s[q] = d32;
                    need |= (!(d32 > thr[q]) ? 1u : 0u) << q;
                }
                // 1b. exact float64 fold where needed (warp-uniform branches, predicated update)
                if (__any_sync(kFull, need != 0)) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        if (__any_sync(kFull, (need >> q) & 1u)) {
                            const double d = sqdist(sx, sy, sz, (double)fx[q], (double)fy[q], (double)fz[q]);
                            // d, m >= 0: the bit patterns order like the values (ALU compare)
                            if (((need >> q) & 1u) && dbits(d) < dbits(m[q])) {
                                m[q] = d;
                                thr[q] = skip_threshold_d32(d, d32s[q]);
                                dirty = dirty || (q == bq);
                            }
                        }
                    }
                }
                // 1c. the cached local max only changes when its own point moved
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
                if (bv >= 0.0) {
                    bkey = dbits(bv);
                    bidx = (uint32_t)(lo + tid + (int64_t)bq * kFpsThreads);
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
                        mine.x = v.x; mine.y = v.y; mine.z = v.z;
                    }
                }
            }
            if (tdbg) a.dbg[t * 8 + 0] = clock64() - ts0;

            // 2. warp argmax: the winning lane publishes its record
            const int wl = warp_argmax_lane(bkey, bidx);
            if (wl < 0) {
                if (lane == 0) { Rec z{}; z.idx = kNone; warp_rec[warp] = z; }
            } else if (lane == wl) {
                if constexpr (P > 0) {
                    mine.x = bx; mine.y = by; mine.z = bz;
                    mine.taken = (tk >> bq) & 1u;
                } else {
                    mine.taken = taken[bidx];
                }
                mine.klo = (uint32_t)bkey;
                mine.khi = (uint32_t)(bkey >> 32);
                mine.idx = bidx;
                warp_rec[warp] = mine;
            }
            if (tdbg) a.dbg[t * 8 + 1] = clock64() - ts0;
            __syncthreads();
            if (tdbg) a.dbg[t * 8 + 2] = clock64() - ts0;

            Rec win;
            if (C == 1) {
                // single-CTA cloud: the block argmax is the answer, no exchange
                if (warp == kFpsWarps - 1) {
                    const Rec wr = lane < kFpsWarps ? warp_rec[lane] : Rec{0, 0, kNone, 0, 0.f, 0.f, 0.f, 0};
                    const int cl = warp_argmax_lane(rec_key(wr), wr.idx);
                    if (lane == 0) {
                        Rec cr = warp_rec[cl < 0 ? 0 : cl];
                        if (cl < 0) cr.idx = kNone;
                        slots[par][0] = cr;
                    }
                }
                __syncthreads();
                win = slots[par][0];
                if (tdbg) { a.dbg[t * 8 + 3] = clock64() - ts0; a.dbg[t * 8 + 4] = a.dbg[t * 8 + 3]; a.dbg[t * 8 + 5] = a.dbg[t * 8 + 3]; }
            } else {
            // 3+4. block argmax, push the CTA record to every CTA of the cluster
            // (the highest warp id leads: the SMSP arbiter favours high ids)
            if (warp == kFpsWarps - 1) {
                const Rec wr = lane < kFpsWarps ? warp_rec[lane] : Rec{0, 0, kNone, 0, 0.f, 0.f, 0.f, 0};
                const int cl = warp_argmax_lane(rec_key(wr), wr.idx);
                const Rec cr = warp_rec[cl < 0 ? 0 : cl];
                if (lane < (int)C) {
                    const uint32_t dst = par ? dst1 : dst0;
                    const uint32_t dbar = par ? dbar1 : dbar0;
                    st_async_v4(dst, dbar, cr.klo, cr.khi, cl < 0 ? kNone : cr.idx, cr.taken);
                    st_async_v4(dst + 16, dbar, __float_as_uint(cr.x), __float_as_uint(cr.y),
                                __float_as_uint(cr.z), 0u);
                }
            }
            if (tdbg) a.dbg[t * 8 + 3] = clock64() - ts0;

            // 5. wait for all C records, reduce identically in every warp
            mbar_wait_cluster(&bars[par], phase);
            if (tdbg) a.dbg[t * 8 + 4] = clock64() - ts0;
            const Rec sr = lane < (int)C ? slots[par][lane] : Rec{0, 0, kNone, 0, 0.f, 0.f, 0.f, 0};
            const int gl = warp_argmax_lane(rec_key(sr), sr.idx);
            win = slots[par][gl < 0 ? 0 : gl];
            __syncwarp();
            if (tid == 0) mbar_arrive_expect_tx(&bars[par], tx_bytes);
            if (tdbg) a.dbg[t * 8 + 5] = clock64() - ts0;
            }

            double best = bitsd(rec_key(win));
            if (best <= 0.0 || win.taken) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken index
                uint32_t fidx = kNone;
                Rec fr{};
                if constexpr (P > 0) {
#pragma unroll
                    for (int q = P - 1; q >= 0; --q) {
                        if (((valid >> q) & 1u) && !((tk >> q) & 1u)) {
                            fidx = (uint32_t)(lo + tid + (int64_t)q * kFpsThreads);
                            const uint64_t k = dbits(m[q]);
                            fr.klo = (uint32_t)k; fr.khi = (uint32_t)(k >> 32);
                            fr.x = fx[q]; fr.y = fy[q]; fr.z = fz[q];
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
                    best = bitsd(rec_key(fw));
                }
                cluster_sync_all();  // fb_slots / warp_rec free for the next fallback
            }

            // record (curve holds squared values until the epilogue), mark taken
            if (r == 0 && tid == 0) {
                out[it] = (int64_t)win.idx;
                curve[it] = best;
            }
            const int64_t off = (int64_t)win.idx - lo - tid;
            if constexpr (P > 0) {
                const uint32_t o32 = (uint32_t)off;  // wraps for off < 0: fails the range test
                if (o32 < (uint32_t)(P * kFpsThreads) && (o32 & (kFpsThreads - 1)) == 0)
                    tk |= 1u << (o32 / kFpsThreads);
            } else {
                if (off >= 0 && (off % kFpsThreads) == 0 && (int64_t)win.idx < hi) taken[win.idx] = 1;
            }
            sx32 = win.x; sy32 = win.y; sz32 = win.z;
            if (tdbg) a.dbg[t * 8 + 6] = clock64() - ts0;
        }
    }

    // ---- write back md / taken; curve = sqrt(best) (_kernels.py:72) ---------
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
    if (r == 0 && k_start < k_stop) {
        __syncthreads();  // thread 0's curve stores are visible block-wide
        for (int64_t it = k_start + tid; it < k_stop; it += kFpsThreads) curve[it] = sqrt(curve[it]);
    }
    cluster_sync_all();  // no CTA leaves while peers may still target its smem
}

template <int P, int T>
cudaError_t launch_p(const FpsArgs& a, int64_t B, int C, cudaStream_t s) {
    auto kern = fps_cluster_kernel<P, T>;
    cudaError_t e = cudaSuccess;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * C), 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
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

static int fps_threads_env() {
    const char* e = getenv("PS_FPS_THREADS");
    return e ? (atoi(e) == 512 ? 512 : 256) : 0;
}

static int choose_P(int64_t N, int C, int T) {
    static const int kPs[] = {1, 2, 3, 4, 6, 8, 12, 16};
    const int64_t S = (N + C - 1) / C;
    for (int p : kPs)
        if ((int64_t)p * T >= S) return p;
    return 0;  // streaming
}

// dispatch a functor over the (P, T) instantiations
template <typename F>
static auto with_kernel(int P, int T, F f) {
#define PS_FPS_CASE(PP)                                        \
    case PP:                                                   \
        return T == 512 ? f.template run<PP, 512>() : f.template run<PP, 256>();
    switch (P) {
        PS_FPS_CASE(1)
        PS_FPS_CASE(2)
        PS_FPS_CASE(3)
        PS_FPS_CASE(4)
        PS_FPS_CASE(6)
        PS_FPS_CASE(8)
        case 12:  // 512-thread CTAs only up to P = 8 (register budget)
            return f.template run<12, 256>();
        case 16:
            return f.template run<16, 256>();
        default:
            return f.template run<0, 256>();
    }
#undef PS_FPS_CASE
}

template <int P, int T>
static int max_clusters_p(int C) {
    auto kern = fps_cluster_kernel<P, T>;
    if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(C * 64), 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

struct MaxClustersF {
    int C;
    template <int P, int T>
    int run() const { return max_clusters_p<P, T>(C); }
};

struct LaunchF {
    const FpsArgs* a;
    int64_t B;
    int C;
    cudaStream_t s;
    template <int P, int T>
    cudaError_t run() const { return launch_p<P, T>(*a, B, C, s); }
};

// Co-resident clusters of size C for the instantiation serving N (cached;
// depends on the GPU's GPC floor-sweeping, so it is queried, not assumed).
static int max_active_clusters(int64_t N, int C, int T) {
    static int cache[17][9][2];
    static bool init = false;
    if (!init) {
        for (auto& a2 : cache)
            for (auto& row : a2)
                for (int& v : row) v = -1;
        init = true;
    }
    const int P = choose_P(N, C, T);
    const int pi = P == 0 ? 0 : (P <= 4 ? P : (P == 6 ? 5 : (P == 8 ? 6 : (P == 12 ? 7 : 8))));
    const int ti = T == 512 ? 1 : 0;
    if (cache[C][pi][ti] >= 0) return cache[C][pi][ti];
    const int n = with_kernel(P, T, MaxClustersF{C});
    cache[C][pi][ti] = n;
    if (getenv("PS_FPS_VERBOSE")) fprintf(stderr, "[fps] N=%lld C=%d P=%d T=%d max_active_clusters=%d\n",
                                          (long long)N, C, P, T, n);
    return n;
}

// Throughput hint (ps_set_fps_inflight): clouds the caller keeps in flight
// across concurrent streams.  0: latency mode.
static int64_t g_inflight = 0;
int64_t fps_set_inflight(int64_t clouds) {
    const int64_t old = g_inflight;
    g_inflight = clouds > 0 ? clouds : 0;
    return old;
}

// Cluster width C and CTA size T: the widest cluster whose B clusters are
// all co-resident (one wave, every cloud in lock step), preferring 512-thread
// CTAs (more warps hide the fold's latency) while P <= 8 points per thread.
// With a throughput hint of H > B clouds in flight, the width with the most
// clouds finished per unit time instead: min(H, co-resident clusters) /
// latency(C), latency(C) ~ a + b / C per sample with b / a ~ 9 (speculative
// kernel, C3 prefix: 0.49 / 0.56 / 0.60 / 0.64 ms at C = 10 / 8 / 7 / 6,
// profiles/r02/cluster_sweep.log).  Clusters pack into the GPCs: 22 clusters
// of 6 fit where 15 of 9 or 11 of 10 do, so C3 with 5 chains in flight runs
// 6-CTA clusters (64.5 -> 70.2 M samples/s).
int fps_choose_cluster(int64_t N, int64_t B, int* C_out, int* P_out, int* T_out) {
    if (g_inflight > B && !getenv("PS_FPS_CLUSTER")) {
        const int tenv0 = fps_threads_env();
        const int64_t c0 = (N + 1023) / 1024;
        const int want = (int)(c0 < 1 ? 1 : (c0 > kMaxCluster ? kMaxCluster : c0));
        // deep concurrency (>= 2 batches in flight): the other stages share the
        // SMs, so SM-time per cloud, C x latency(C), decides -- lowest at the
        // narrowest width the speculative kernel holds without spills (<= 10
        // points on each of its 480 point-owning threads; C3: 5-CTA clusters,
        // 85.5 -> 89.4 M samples/s, profiles/r02/fps_pmax.log)
        const bool deep = g_inflight >= 2 * B;
        int bestC = 0;
        int64_t bestCov = -1;
        for (int cc = want; cc >= 3; --cc) {
            const int p = choose_P(N, cc, 512);
            if (tenv0 && tenv0 != 512) break;
            const int64_t S = (N + cc - 1) / cc;
            const int ps = (int)((S + 479) / 480);  // speculative kernel's points per thread
            if (p < 1 || (p > 8 && ps > 10)) continue;
            const int64_t act = max_active_clusters(N, cc, 512);
            if (act < B) continue;  // the batch itself must still fit one wave
            const int64_t score = deep ? (int64_t)(kMaxCluster + 1 - cc)
                                       : (act < g_inflight ? act : g_inflight) * cc * 1024 / (cc + 9);
            if (score >= bestCov) { bestCov = score; bestC = cc; }
        }
        if (bestC) {
            *C_out = bestC;
            *T_out = 512;
            *P_out = choose_P(N, bestC, 512);
            return 0;
        }
    }
    const char* env = getenv("PS_FPS_CLUSTER");
    const int tenv = fps_threads_env();
    const int64_t target = (int64_t)256 * 4;
    const int64_t c0 = (N + target - 1) / target;
    const int want = (int)(c0 < 1 ? 1 : (c0 > kMaxCluster ? kMaxCluster : c0));
    int C = 0, T = 0;
    if (env) {
        C = atoi(env);
        if (C < 1) C = 1;
        if (C > kMaxCluster) C = kMaxCluster;
        T = tenv ? tenv : (choose_P(N, C, 512) >= 1 && choose_P(N, C, 512) <= 8 ? 512 : 256);
    } else {
        for (int t : {512, 256}) {
            if (tenv && t != tenv) continue;
            for (int cc : {16, 14, 12, 10, 8, 6, 4, 3, 2, 1}) {
                if (cc > want) continue;
                const int p = choose_P(N, cc, t);
                if (t == 512 && (p == 0 || p > 8)) continue;
                if (p == 0 && cc != kMaxCluster) continue;
                if (max_active_clusters(N, cc, t) >= B) { C = cc; T = t; break; }
            }
            if (C) break;
        }
        if (!C) {  // batch larger than one wave at any width
            C = want > 8 ? 8 : want;
            T = tenv ? tenv : 256;
        }
    }
    *C_out = C;
    *T_out = T;
    *P_out = choose_P(N, C, T);
    return 0;
}

cudaError_t launch_fps_legacy(FpsArgs a, int64_t B, cudaStream_t s) {
    int C = 1, P = 0, T = 256;
    fps_choose_cluster(a.N, B, &C, &P, &T);
    a.points_per_cta = (a.N + C - 1) / C;
    a.dbg = nullptr;
    if (kTiming && getenv("PS_FPS_TIMING")) {
        // development aid: per-phase SM cycles of the first 256 iterations
        // (cloud 0, CTA rank 0, thread 0) printed to stderr; synchronises.
        static long long* dbg = nullptr;
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 256 * 8);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 256 * 8, s);
        a.dbg = dbg;
        a.dbg_t0 = getenv("PS_FPS_T0") ? atoll(getenv("PS_FPS_T0")) : 0;
        cudaError_t e = with_kernel(P, T, LaunchF{&a, B, C, s});
        if (e != cudaSuccess) return e;
        long long h[256 * 8];
        cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const int iters = (int)((a.k_stop - a.k_start - a.dbg_t0) < 256 ? (a.k_stop - a.k_start - a.dbg_t0) : 256);
        double acc[7] = {0};
        int cnt = 0;
        for (int t = 8; t < iters; ++t, ++cnt)
            for (int k = 0; k < 7; ++k) acc[k] += (double)h[t * 8 + k];
        if (cnt)
            fprintf(stderr, "[fps timing] C=%d P=%d T=%d N=%lld iters=%d cycles: compute %.0f warpred %.0f bar %.0f send %.0f wait %.0f final %.0f total %.0f\n",
                    C, P, T, (long long)a.N, cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt,
                    acc[4] / cnt, acc[5] / cnt, acc[6] / cnt);
        return cudaSuccess;
    }
    return with_kernel(P, T, LaunchF{&a, B, C, s});
}

}  // namespace ps
