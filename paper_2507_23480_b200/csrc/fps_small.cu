// fps_small.cu -- K1 for small clouds: one CTA of W warps per cloud, every
// point in a register, one CTA barrier per sample (B200 / sm_100a).
//
// Same result as _kernels.fps_loop (/root/reference/pkg/src/pointsample/
// _kernels.py:35-74) -- indices, curve, md and taken bit for bit.  Thread
// (warp w, lane l) owns points j = (r * W + w) * 32 + l, r < R, with their
// coordinates, float64 md, float32 skip threshold and taken bit in registers.
// Per iteration:
//   1. the last sample's coordinates come from a shared-memory copy of the
//      cloud (one LDS.128);
//   2. float32 screen of all R points (fps_util.cuh skip_threshold*); the
//      exact float64 fold in the reference's operation order runs only for
//      groups of four r some lane of the warp needs (warp-uniform branch,
//      per-lane select), so late iterations skip it almost entirely;
//   3. per-lane argmax (tree over r, lower index wins ties), per-warp argmax
//      (fps_util.cuh warp_argmax_lane), lane 0 posts {md bits, index, taken}
//      to a parity-double-buffered slot;
//   4. one __syncthreads, then every warp reduces the W slots itself -- all
//      warps reach the same pick, no second barrier;
//   5. duplicate fallback of _kernels.py:65-70 (max <= 0 or winner taken ->
//      lowest untaken index), a second slot round only when it triggers.
// The block kernels of fps.cu pay two barriers and a shared-memory argmax per
// sample over one point per thread; here a sample costs one barrier and a
// register sweep, which is what tiny clouds (C2's 512/256/128-point stages)
// are bound by (profiles/r01/fps_spec.log).

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "fps_util.cuh"
#include "ps_internal.h"

namespace ps {

namespace {

constexpr int kSmallMaxN = 4096;

template <int W, int R>
__global__ void __launch_bounds__(W * 32) fps_small_kernel(FpsArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ uint4 slot[2][W];        // per-warp best: {key lo, key hi, index, taken}
    __shared__ uint4 fslot[2][W];       // fallback: {md lo, md hi, lowest untaken index, -}
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t b = blockIdx.x;
    const int N = (int)a.N;
    float4* pts = reinterpret_cast<float4*>(dsm);                         // W * 32 * R
    double* best_s = reinterpret_cast<double*>(dsm + 16 * W * 32 * R);    // per iteration
    uint32_t* idx_s = reinterpret_cast<uint32_t*>(dsm + 24 * W * 32 * R);
    const float4* __restrict__ xyz = a.xyz + b * a.N;
    double* __restrict__ md = a.md + b * a.N;
    uint8_t* __restrict__ taken = a.taken + b * a.N;
    int64_t* __restrict__ out = a.out_idx + b * a.ld_out;
    double* __restrict__ curve = a.curve + b * a.ld_out;
    const int64_t k_start = a.k_start_dev ? a.k_start_dev[b] : a.k_start;
    const int64_t k_stop = a.k_stop;
    const int64_t seed = a.seed_dev ? a.seed_dev[b] : a.seed;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);

    float px[R], py[R], pz[R], th[R];
    double m[R];
    uint32_t tk = 0;  // bit r: point r taken (padding counts as taken)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = (r * W + w) * 32 + lane;
        if (j < N) {
            const float4 p = xyz[j];
            pts[j] = p;
            px[r] = p.x; py[r] = p.y; pz[r] = p.z;
            m[r] = a.fresh ? kInf : md[j];
            th[r] = skip_threshold(m[r]);
            if (a.fresh ? (j == seed) : (taken[j] != 0)) tk |= 1u << r;
        } else {
            px[r] = py[r] = pz[r] = 0.f;
            m[r] = 0.0;
            th[r] = -__int_as_float(0x7f800000);  // padding never folds
            tk |= 1u << r;
        }
    }
    if (a.fresh && threadIdx.x == 0) {
        out[0] = seed;
        curve[0] = kInf;
    }
    __syncthreads();

    uint4* const myslot = &slot[0][w];
    const int64_t n_it = k_stop - k_start;
    if (n_it > 0) {
        const int64_t last = a.fresh ? seed : out[k_start - 1];  // refolded, as _kernels.py
        float4 s = pts[last];
        for (int64_t it = 0; it < n_it; ++it) {
            const int par = (int)(it & 1);
            uint32_t need = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float dx = px[r] - s.x, dy = py[r] - s.y, dz = pz[r] - s.z;
                const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                if (!(d32 > th[r])) need |= 1u << r;
            }
            const uint32_t wneed = __reduce_or_sync(kFull, need);
            if (wneed) {
                const double sx = s.x, sy = s.y, sz = s.z;
#pragma unroll
                for (int g = 0; g < R; g += 4) {
                    constexpr int GS = R < 4 ? R : 4;
                    if ((wneed >> g) & ((1u << GS) - 1u)) {
#pragma unroll
                        for (int r = g; r < g + GS; ++r) {
                            const float dx = px[r] - s.x, dy = py[r] - s.y, dz = pz[r] - s.z;
                            const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                            const double d = sqdist(sx, sy, sz, (double)px[r], (double)py[r], (double)pz[r]);
                            // branch-free skip_threshold_d32 (fps_util.cuh)
                            float t = __fmul_ru(d32, 1.0f + 7.62939453125e-06f);
                            t = (!(d32 >= 7.888609052210118e-31f) || !(d32 < 1e38f)) ? __int_as_float(0x7f800000) : t;
                            t = dbits(d) == 0 ? -1.0f : t;
                            const bool upd = ((need >> r) & 1u) && d < m[r];
                            m[r] = upd ? d : m[r];
                            th[r] = upd ? t : th[r];
                        }
                    }
                }
            }
            // per-lane argmax, tree over r (left wins ties: lower index)
            double v[R];
            int ri[R];
#pragma unroll
            for (int r = 0; r < R; ++r) { v[r] = m[r]; ri[r] = r; }
#pragma unroll
            for (int st = 1; st < R; st *= 2)
#pragma unroll
                for (int r = 0; r + st < R; r += 2 * st)
                    if (v[r + st] > v[r]) { v[r] = v[r + st]; ri[r] = ri[r + st]; }
            const uint32_t myj = (uint32_t)((ri[0] * W + w) * 32 + lane);
            const uint64_t myk = dbits(v[0]);
            const uint32_t myt = (tk >> ri[0]) & 1u;
            const int wl = warp_argmax_lane(myk, myj);
            if (lane == wl) myslot[par * W] = make_uint4((uint32_t)myk, (uint32_t)(myk >> 32), myj, myt);
            __syncthreads();
            // every lane reduces the W slots itself (broadcast loads; identical
            // result everywhere, no shuffles)
            uint4 q = slot[par][0];
            uint64_t qk = ((uint64_t)q.y << 32) | q.x;
#pragma unroll
            for (int u = 1; u < W; ++u) {
                const uint4 o = slot[par][u];
                const uint64_t ok = ((uint64_t)o.y << 32) | o.x;
                if (ok > qk || (ok == qk && o.z < q.z)) { q = o; qk = ok; }
            }
            uint32_t widx = q.z;
            double best = bitsd(qk);
            const uint32_t wtaken = q.w;
            if (best <= 0.0 || wtaken) {
                // duplicate fallback (_kernels.py:65-70): lowest untaken index
                const uint32_t fr = ~tk & (R == 32 ? ~0u : ((1u << R) - 1u));
                const uint32_t f = fr ? (uint32_t)(((__ffs(fr) - 1) * W + w) * 32 + lane) : kNone;
                double mf = 0.0;
#pragma unroll
                for (int r = R - 1; r >= 0; --r)
                    if ((fr >> r) & 1u) mf = m[r];
                const uint32_t fm = __reduce_min_sync(kFull, f);
                const int fl = fm == kNone ? 0 : (int)(fm & 31);
                const uint64_t fk = dbits(__shfl_sync(kFull, mf, fl));
                if (lane == 0) fslot[par][w] = make_uint4((uint32_t)fk, (uint32_t)(fk >> 32), fm, 0);
                __syncthreads();
                uint4 fq = make_uint4(0, 0, kNone, 0);
                if (lane < W) fq = fslot[par][lane];
                const uint32_t gm = __reduce_min_sync(kFull, fq.z);
                if (gm != kNone) {
                    const int gl = __ffs(__ballot_sync(kFull, fq.z == gm)) - 1;
                    widx = gm;
                    best = bitsd(__shfl_sync(kFull, ((uint64_t)fq.y << 32) | fq.x, gl));
                }
            }
            if (w == (int)((widx >> 5) % W) && lane == (int)(widx & 31)) tk |= 1u << ((widx >> 5) / W);
            if (threadIdx.x == 0) {
                idx_s[it] = widx;
                best_s[it] = best;
            }
            s = pts[widx];
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n_it; i += W * 32) {
            out[k_start + i] = (int64_t)idx_s[i];
            curve[k_start + i] = sqrt(best_s[i]);  // _kernels.py:72
        }
    }

    // write back md / taken
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = (r * W + w) * 32 + lane;
        if (j < N) {
            md[j] = m[r];
            taken[j] = (tk >> r) & 1u;
        }
    }
}

template <int W, int R>
cudaError_t launch_wr(FpsArgs a, int64_t B, cudaStream_t s) {
    const size_t smem = (size_t)W * 32 * R * (16 + 8 + 4);
    static bool attr = false;
    if (!attr) {
        const cudaError_t e =
            cudaFuncSetAttribute(fps_small_kernel<W, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    fps_small_kernel<W, R><<<(unsigned)B, W * 32, smem, s>>>(a);
    return cudaGetLastError();
}

template <int W>
cudaError_t launch_w(FpsArgs a, int64_t B, cudaStream_t s) {
    const int64_t per = W * 32;
    if (a.N <= per) return launch_wr<W, 1>(a, B, s);
    if (a.N <= 2 * per) return launch_wr<W, 2>(a, B, s);
    if (a.N <= 4 * per) return launch_wr<W, 4>(a, B, s);
    if (a.N <= 8 * per) return launch_wr<W, 8>(a, B, s);
    if (a.N <= 16 * per) return launch_wr<W, 16>(a, B, s);
    return cudaErrorNotSupported;
}

}  // namespace

// Small clouds (N <= kSmallMaxN).  Warps per cloud from the sweep in
// profiles/r01/fps_spec.log (tools/fps_small_sweep.py); PS_FPS_SMALL_W
// overrides.  Above 2048 points the kernel only wins when the batch fills the
// chip; smaller batches go to fps_spec.
cudaError_t launch_fps_small(FpsArgs a, int64_t B, cudaStream_t s) {
    if (a.N > kSmallMaxN || a.k_stop > a.N || B < 1 || B > 0x7fffffff) return cudaErrorNotSupported;
    int W = a.N <= 256 ? 1 : a.N <= 1024 ? (B < 148 ? 4 : 2) : a.N <= 2048 ? 4 : 8;
    if (W == 8 && B < 128) return cudaErrorNotSupported;
    if (getenv("PS_FPS_SMALL_W")) W = atoi(getenv("PS_FPS_SMALL_W"));
    if (getenv("PS_FPS_VERBOSE")) fprintf(stderr, "[fps-small] N=%lld B=%lld W=%d\n", (long long)a.N, (long long)B, W);
    switch (W) {
        case 1: return launch_w<1>(a, B, s);
        case 2: return launch_w<2>(a, B, s);
        case 4: return launch_w<4>(a, B, s);
        case 8: return launch_w<8>(a, B, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace ps
