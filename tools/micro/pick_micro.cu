// The speculation pick loop of fps_spec.cu in isolation: one warp, ncand
// candidates (one per lane), distance rows in shared memory.  Cycles per
// pick with the publish (release store) on and off, alone and with 15
// co-resident warps spinning on a shared word.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2507_23480_b200/csrc -o pick_micro pick_micro.cu
#include <cstdio>
#include <cstdint>
#include "common.cuh"
#include "fps_util.cuh"

using namespace ps;

template <bool kPub>
__global__ void picks(long long* cyc, int ncand, int spin, uint32_t* sink) {
    __shared__ double dm_s[32 * 32];
    __shared__ float4 run_s[32];
    __shared__ double hist_s[32];
    __shared__ uint32_t pub_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) dm_s[i] = 1.0 + ((i * 7919) % 1000) * 1e-3;
    if (threadIdx.x == 0) pub_s = 0;
    __syncthreads();
    if (warp != 15) {
        if (!spin) return;
        uint32_t v = 0;
        float f = threadIdx.x * 1e-3f;
        double dd = 1.0;
        while (true) {
            v = ld_acquire_cta(&pub_s);
            if (v == 0xffffffffu) break;
            if (spin >= 4) {  // issue-saturating FP32 on the lead's SMSP (4) / the other SMSPs (5)
                const bool mine = (warp & 3) == 3;
                if (spin == 4 ? mine : !mine) {
                    float g0 = f, g1 = f + 1, g2 = f + 2, g3 = f + 3;
#pragma unroll
                    for (int i = 0; i < 64; ++i) {
                        g0 = __fmaf_rn(g0, 0.999f, 1e-7f); g1 = __fmaf_rn(g1, 0.999f, 1e-7f);
                        g2 = __fmaf_rn(g2, 0.999f, 1e-7f); g3 = __fmaf_rn(g3, 0.999f, 1e-7f);
                    }
                    f = g0 + g1 + g2 + g3;
                }
            } else if (spin >= 2) {  // fold-like work: screens, votes, some FP64
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    f = __fmaf_rn(f, 0.999f, 1e-7f);
                    const bool need = (__float_as_uint(f) & 0x70) == 0;
                    if (spin == 2 ? __any_sync(0xffffffffu, need) : need) dd = __dadd_rn(dd, (double)f);
                }
            }
        }
        sink[threadIdx.x] = v + (uint32_t)dd;
        return;
    }
    const uint64_t tau = dbits(0.5);
    long long tot = 0;
    int np = 0;
    for (int rep = 0; rep < 200; ++rep) {
        double cm = 2.0 + lane * 0.01 + rep * 1e-6;
        uint32_t ci = lane < ncand ? (uint32_t)(1000 + lane) : kNone;
        bool alive = lane < ncand;
        int rnl = 1;
        __syncwarp();
        const long long t0 = clock64();
        while (rnl < 31) {
            alive = alive && dbits(cm) >= tau;
            const int wl = warp_argmax_lane(alive ? dbits(cm) : 0ull, alive ? ci : kNone);
            if (wl < 0) break;
            const bool win = lane == wl;
            const double d = dm_s[wl * 32 + lane];
            if (win) {
                run_s[rnl] = make_float4(1.f, 2.f, 3.f, __uint_as_float(ci));
                hist_s[rnl & 31] = cm;
                if (kPub) st_release_cta(&pub_s, (uint32_t)(rnl + 1));
            }
            alive = alive && !win;
            cm = (alive && dbits(d) < dbits(cm)) ? d : cm;
            ++rnl;
        }
        const long long t1 = clock64();
        tot += t1 - t0;
        np += rnl - 1;
    }
    if (lane == 0) { cyc[0] = tot; cyc[1] = np; }
    __syncwarp();
    if (lane == 0) st_release_cta(&pub_s, 0xffffffffu);
}

int main() {
    long long* c;
    uint32_t* s;
    cudaMalloc(&c, 16);
    cudaMalloc(&s, 4096);
    for (int spin = 0; spin < 6; ++spin)
        for (int pub = 0; pub < 2; ++pub) {
            long long h[2];
            for (int k = 0; k < 2; ++k) {
                if (pub) picks<true><<<1, 512>>>(c, 12, spin, s);
                else picks<false><<<1, 512>>>(c, 12, spin, s);
            }
            cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
            printf("worker mode %d (0 none,1 spin,2 fold+votes,3 fold,4 FFMA same SMSP,5 FFMA other SMSPs), publish %d: %.1f cycles per pick (%lld picks) %s\n", spin, pub,
                   (double)h[0] / h[1], h[1], cudaGetErrorString(cudaGetLastError()));
            (void)spin;
        }
    return 0;
}
