// Micro-benchmarks for the sm_100a pipes the sampling kernels lean on:
// FP64 add/mul, f32<->f64 conversion, FP32 FMA, integer 64-bit compare.
// Prints cycles per warp-instruction (throughput, full SM) and dependent
// latency (one warp).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define ITER 4096

__global__ void lat_dadd(double* out, long long* cyc, double a) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < ITER; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}
__global__ void lat_dmul(double* out, long long* cyc, double a) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < ITER; ++i) x = __dmul_rn(x, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}
// throughput: 8 independent chains per thread
template <int OP>
__global__ void thr_kernel(double* out, long long* cyc, double a) {
    double x[8];
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { x[k] = a + k; f[k] = (float)a + k; }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITER / 8; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) x[k] = __dadd_rn(x[k], a);
            if (OP == 1) x[k] = __dmul_rn(x[k], a);
            if (OP == 2) x[k] = __dadd_rn(x[k], (double)f[k]);           // F2F f32->f64 + DADD
            if (OP == 3) f[k] = __fmaf_rn(f[k], 1.0001f, 0.5f);
            if (OP == 4) f[k] = f[k] + (float)x[k];                      // F2F f64->f32 + FADD
            if (OP == 5) { unsigned long long u = __double_as_longlong(x[k]); x[k] = (u > 12345ull) ? a : x[k] + 1.0; }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k] + f[k];
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (s == 12345.678) out[1] = s;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    long long h;
    lat_dadd<<<1, 32>>>(out, cyc, 1.0000001); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)h / ITER);
    lat_dmul<<<1, 32>>>(out, cyc, 1.0000001); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.2f cycles\n", (double)h / ITER);
    const char* names[] = {"DADD", "DMUL", "F2F.F64.F32+DADD", "FFMA", "F2F.F32.F64+FADD", "U64cmp+sel+DADD"};
    for (int op = 0; op < 6; ++op) {
        for (int threads : {256, 1024}) {
            void (*k)(double*, long long*, double) = op == 0 ? thr_kernel<0> : op == 1 ? thr_kernel<1> :
                op == 2 ? thr_kernel<2> : op == 3 ? thr_kernel<3> : op == 4 ? thr_kernel<4> : thr_kernel<5>;
            k<<<148, threads>>>(out, cyc, 1.0000001);
            cudaDeviceSynchronize();
            k<<<148, threads>>>(out, cyc, 1.0000001);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            const double warp_ops = (double)(threads / 32) * ITER;  // per SM
            printf("%-18s threads/SM=%4d: %.3f cycles per warp-op per SM (%.1f lanes/clk/SM)\n", names[op], threads,
                   (double)h / warp_ops, 32.0 * warp_ops / (double)h);
        }
    }
    return 0;
}
