// Latency (1 warp, dependent chain) and per-SM throughput (16 warps,
// independent chains) of the ops on the FPS speculation path (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o op_micro op_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 1024;

template <int OP>
__global__ void chain(long long* cyc, double* sink, int nwarp) {
    if ((int)(threadIdx.x >> 5) >= nwarp) return;
    double d = threadIdx.x * 1e-3 + 1.0;
    float f = threadIdx.x * 1e-3f + 1.0f;
    uint32_t u = threadIdx.x;
    __shared__ double sm[1024];
    sm[threadIdx.x] = d;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < IT; ++i) {
        if (OP == 0) d = __dadd_rn(d, 1e-9);                          // DADD
        if (OP == 1) d = __dmul_rn(d, 0.999999);                      // DMUL
        if (OP == 2) { d = (double)f; f = (float)d + 1e-7f; }         // F2F.F64.F32 + F2F.F32.F64
        if (OP == 3) u = __shfl_sync(0xffffffffu, u, (u + 1) & 31);   // SHFL
        if (OP == 4) u = __reduce_max_sync(0xffffffffu, u) ^ threadIdx.x;  // REDUX
        if (OP == 5) u = __ballot_sync(0xffffffffu, u & 1) ^ threadIdx.x; // VOTE
        if (OP == 6) { d = sm[(int)(d) & 1023]; }                     // LDS.64 dependent
        if (OP == 7) f = __fmaf_rn(f, 0.999f, 1e-7f);                 // FFMA
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
    sink[threadIdx.x] = d + f + u;
}

template <int OP>
void run(const char* name, long long* c, double* s) {
    long long h[32];
    double r[2];
    for (int k = 0; k < 2; ++k) {
        int nw = k == 0 ? 1 : 16;
        chain<OP><<<1, 512>>>(c, s, nw);
        chain<OP><<<1, 512>>>(c, s, nw);
        cudaMemcpy(h, c, sizeof(long long) * 16, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
        r[k] = (double)mx / IT;
    }
    printf("%-28s latency %6.1f cyc/op (1 warp)   16 warps: %6.2f cyc per op-round (%.2f warp-ops/cyc/SM)\n", name,
           r[0], r[1], 16.0 / r[1]);
}

int main() {
    long long* c;
    double* s;
    cudaMalloc(&c, 8 * 32);
    cudaMalloc(&s, 8 * 1024);
    run<0>("DADD", c, s);
    run<1>("DMUL", c, s);
    run<2>("F2F f32->f64->f32 (pair)", c, s);
    run<3>("SHFL.IDX", c, s);
    run<4>("REDUX.MAX + LOP", c, s);
    run<5>("VOTE.ballot + LOP", c, s);
    run<6>("LDS.64 dependent", c, s);
    run<7>("FFMA", c, s);
    return 0;
}
