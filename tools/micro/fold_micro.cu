// Latency of the resident-FPS touched-warp path in isolation (sm_100a):
// P slots per lane, points in shared memory, float32 screen, float64 fold,
// thread max, warp argmax, record store.  One CTA; W warps all touched.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fold_micro fold_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 1000;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double sqd(double ax, double ay, double az, double bx, double by, double bz) {
    const double dx = __dsub_rn(bx, ax), dy = __dsub_rn(by, ay), dz = __dsub_rn(bz, az);
    double s = __dmul_rn(dx, dx);
    s = __dadd_rn(s, __dmul_rn(dy, dy));
    return __dadd_rn(s, __dmul_rn(dz, dz));
}
__device__ __forceinline__ long long clk() {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    return c;
}
__device__ __forceinline__ float thr_nb(double md) {
    const float t = __fmul_ru(__double2float_ru(md), 1.0f + 3.814697265625e-06f);
    const float u = md >= 7.888609052210118e-31 ? t : __int_as_float(0x7f800000);
    return md == 0.0 ? -1.0f : u;
}

// MODE 0: screen only; 1: screen + f64 fold; 2: + thread max; 3: + warp argmax + record
__device__ __forceinline__ uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
// skip threshold from the bit pattern: integer tests instead of DSETP
__device__ __forceinline__ float thr_bits(double md) {
    const uint64_t b = dbits(md);
    const float t = __fmul_ru(__double2float_ru(md), 1.0f + 3.814697265625e-06f);
    const float u = b >= 0x39B0000000000000ull ? t : __int_as_float(0x7f800000);  // 2^-100
    return b == 0 ? -1.0f : u;
}

template <int P, int MODE>
__global__ void k(float4* gp, long long* cyc, unsigned* out) {
    __shared__ float4 pts[MODE == 4 ? 8 : P * 512 - 64];
    __shared__ uint4 rec[16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    extern __shared__ double2 ptd[];
    if (MODE == 4) {
        for (int i = threadIdx.x; i < P * 512; i += blockDim.x) {
            const float4 v = gp[i];
            ptd[2 * i] = make_double2(v.x, v.y);
            ptd[2 * i + 1] = make_double2(v.z, 0.0);
        }
    } else {
        for (int i = threadIdx.x; i < P * 512 - 64; i += blockDim.x) pts[i] = gp[i];
    }
    __syncthreads();
    const int wbase = MODE == 4 ? warp * 32 * P : (warp * 32 * P) % (P * 512 - 64 - 32 * P);
    const float4* fp = MODE == 4 ? gp : pts;
    double m[P];
    float thr[P];
#pragma unroll
    for (int q = 0; q < P; ++q) { m[q] = 1e30; thr[q] = 1e30f; }
    uint64_t bk = 0;
    unsigned bo = 0;
    int bq = 0;
    float sx32 = 0.5f, sy32 = 0.5f, sz32 = 0.5f;
    unsigned acc = 0;
    long long tsum = 0, ph[5] = {0, 0, 0, 0, 0};
    for (int it = 0; it < IT; ++it) {
        const long long t0 = clk();
        float4 v[P];
        unsigned og[P];
#pragma unroll
        for (int u = 0; u < P; ++u) v[u] = fp[wbase + u * 32 + lane];
        unsigned need = 0;
#pragma unroll
        for (int u = 0; u < P; ++u) {
            og[u] = __float_as_uint(v[u].w);
            const float dx = v[u].x - sx32, dy = v[u].y - sy32, dz = v[u].z - sz32;
            const float d32 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
            need |= (!(d32 > thr[u]) ? 1u : 0u) << u;
        }
        const long long ta = clk();
        ph[0] += ta - t0;
        unsigned chg = 0;
        if (MODE == 4 && __any_sync(kFull, need != 0)) {
            const double sx = sx32, sy = sy32, sz = sz32;
#pragma unroll
            for (int u = 0; u < P; ++u) {
                const double2 a = ptd[2 * (wbase + u * 32 + lane)];
                const double2 c = ptd[2 * (wbase + u * 32 + lane) + 1];
                const double d = sqd(sx, sy, sz, a.x, a.y, c.x);
                const bool upd = ((need >> u) & 1u) && dbits(d) < dbits(m[u]);
                m[u] = upd ? d : m[u];
                thr[u] = upd ? thr_bits(d) : thr[u];
                chg |= (upd ? 1u : 0u) << u;
            }
        } else if (MODE >= 1 && MODE != 4 && __any_sync(kFull, need != 0)) {
            const double sx = sx32, sy = sy32, sz = sz32;
#pragma unroll
            for (int u = 0; u < P; ++u) {
                const double d = sqd(sx, sy, sz, (double)v[u].x, (double)v[u].y, (double)v[u].z);
                const bool upd = ((need >> u) & 1u) && d < m[u];
                m[u] = upd ? d : m[u];
                thr[u] = upd ? thr_nb(d) : thr[u];
                chg |= (upd ? 1u : 0u) << u;
            }
        }
        const long long tb = clk();
        ph[1] += tb - ta;
        if (MODE == 4) {
            // branch-free tree over (key, orig): max key, lowest orig
            uint64_t tk_[P];
            unsigned to_[P];
            int tq_[P];
#pragma unroll
            for (int q = 0; q < P; ++q) { tk_[q] = dbits(m[q]); to_[q] = og[q]; tq_[q] = q; }
#pragma unroll
            for (int st = 1; st < P; st <<= 1) {
#pragma unroll
                for (int q = 0; q + st < P; q += 2 * st) {
                    const bool take = tk_[q + st] > tk_[q] || (tk_[q + st] == tk_[q] && to_[q + st] < to_[q]);
                    tk_[q] = take ? tk_[q + st] : tk_[q];
                    to_[q] = take ? to_[q + st] : to_[q];
                    tq_[q] = take ? tq_[q + st] : tq_[q];
                }
            }
            bk = tk_[0]; bo = to_[0]; bq = tq_[0];
        } else if (MODE >= 2) {
            bk = 0; bo = 0xffffffffu; bq = 0;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const uint64_t kq = (uint64_t)__double_as_longlong(m[q]);
                if (bo == 0xffffffffu || kq > bk || (kq == bk && og[q] < bo)) { bk = kq; bq = q; bo = og[q]; }
            }
        }
        const long long tc = clk();
        ph[2] += tc - tb;
        if (MODE >= 3 || MODE == 4) {
            const uint32_t hi = (uint32_t)(bk >> 32);
            const uint32_t mhi = __reduce_max_sync(kFull, hi);
            unsigned cand = __ballot_sync(kFull, hi == mhi);
            int wl = __ffs(cand) - 1;
            if (__popc(cand) > 1) {
                const uint32_t lo = (uint32_t)bk;
                const bool c1 = (cand >> lane) & 1u;
                const uint32_t mlo = __reduce_max_sync(kFull, c1 ? lo : 0u);
                const bool c2 = c1 && lo == mlo;
                const uint32_t midx = __reduce_min_sync(kFull, c2 ? bo : 0xffffffffu);
                wl = __ffs(__ballot_sync(kFull, c2 && bo == midx)) - 1;
            }
            const uint64_t wk = __shfl_sync(kFull, bk, wl);
            thr[0] = fminf(thr[0], thr_nb(__longlong_as_double((long long)wk)) + 1e30f);
            if (lane == wl) {
                const float4 pv = fp[wbase + bq * 32 + lane];
                rec[warp] = make_uint4((uint32_t)bk, (uint32_t)(bk >> 32), bo, __float_as_uint(pv.x));
            }
        }
        __syncwarp();
        const long long t1 = clk();
        ph[3] += t1 - tc;
        tsum += t1 - t0;
        acc += need + chg + bo;
        sx32 += 1e-4f * (float)(it & 7);  // new sample each iteration
        // make every point need a fold again
#pragma unroll
        for (int q = 0; q < P; ++q) thr[q] = 1e30f;
    }
    if (lane == 0) { cyc[warp] = tsum; out[warp] = acc + rec[warp].x; }
    if (threadIdx.x == 0) for (int i = 0; i < 4; ++i) cyc[16 + i] = ph[i];
}

template <int P, int MODE>
void run(int warps) {
    float4* gp;
    long long* c;
    unsigned* o;
    cudaMalloc(&gp, sizeof(float4) * P * 512);
    cudaMalloc(&c, 8 * 32);
    cudaMalloc(&o, 4 * 16);
    float4 h[P * 512];
    for (int i = 0; i < P * 512; ++i) h[i] = make_float4((i % 97) / 97.f, (i % 89) / 89.f, (i % 83) / 83.f, (float)i);
    cudaMemcpy(gp, h, sizeof(h), cudaMemcpyHostToDevice);
    const int dsm = MODE == 4 ? P * 512 * 32 : 0;
    cudaFuncSetAttribute(k<P, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
    k<P, MODE><<<1, 32 * warps, dsm>>>(gp, c, o);
    k<P, MODE><<<1, 32 * warps, dsm>>>(gp, c, o);
    long long hc[32];
    cudaMemcpy(hc, c, 8 * 32, cudaMemcpyDeviceToHost);
    printf("P=%d mode=%d warps=%2d: %7.1f cycles per touched-warp pass (warp 0): screen %.1f fold %.1f tmax %.1f argmax+rec %.1f\n",
           P, MODE, warps, (double)hc[0] / IT, (double)hc[16] / IT, (double)hc[17] / IT, (double)hc[18] / IT, (double)hc[19] / IT);
    cudaFree(gp);
    cudaFree(c);
    cudaFree(o);
}

int main() {
    for (int w : {1, 4, 16}) {
        run<6, 3>(w);
        run<6, 4>(w);
    }
    run<2, 4>(1);
    run<2, 4>(16);
    run<2, 3>(1);
    run<2, 3>(16);
    return 0;
}
